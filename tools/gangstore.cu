// gangstore.cu -- B200 HBM write throughput of the walk kernel's store pattern
// against alternatives, stores only, in the walk's launch shape
// (148 x 4 CTAs of 4 warps, 16 warps/SM).  Two 16 GiB tables ("RSS", "BIC").
//   gang64  : the walk's pattern: per step each lane (worker w, part h) stores NE
//             doubles per table; entry e of part h goes to a random 256 B region,
//             warp wib writes bytes [64 wib, 64 wib + 64) of it (its 8 workers);
//             the 4 warps of a CTA complete the region; bar.sync per step (or not)
//   full256 : per step the CTA's 4 NE regions per table are written by whole warps,
//             256 B per store instruction (a staged layout)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gangstore tools/gangstore.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t h)
{
    h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
    return h;
}

template <int NE>
__global__ void gang64(double* a, double* b, uint32_t nreg, int steps, int sync, int spin)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, w = lane & 7, h = lane >> 3;
    const uint32_t gang = blockIdx.x;
    double acc = lane;
    for (int t = 0; t < steps; ++t) {
        for (int s = 0; s < spin; ++s) acc = fma(acc, 0.999, 1e-3);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const uint32_t rg = mix(gang * 1000003u + (uint32_t)t * 977u + (uint32_t)(e * 4 + h)) & (nreg - 1);
            const size_t ix = (size_t)rg * 32 + wib * 8 + w;
            __stcs(a + ix, acc);
            __stcs(b + ix, acc + 1.0);
        }
        if (sync) asm volatile("bar.sync 1, 128;" ::: "memory");
    }
}

template <int NE>
__global__ void full256(double* a, double* b, uint32_t nreg, int steps, int sync, int spin)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t gang = blockIdx.x;
    double acc = lane;
    for (int t = 0; t < steps; ++t) {
        for (int s = 0; s < spin; ++s) acc = fma(acc, 0.999, 1e-3);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const uint32_t rg = mix(gang * 1000003u + (uint32_t)t * 977u + (uint32_t)(e * 4 + wib)) & (nreg - 1);
            const size_t ix = (size_t)rg * 32 + lane;
            __stcs(a + ix, acc);
            __stcs(b + ix, acc + 1.0);
        }
        if (sync) asm volatile("bar.sync 1, 128;" ::: "memory");
    }
}

int main()
{
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t bytes = (size_t)16 << 30;
    double *A, *B;
    CK(cudaMalloc(&A, bytes));
    CK(cudaMalloc(&B, bytes));
    CK(cudaMemset(A, 0, bytes));
    CK(cudaMemset(B, 0, bytes));
    const uint32_t nreg = (uint32_t)(bytes / 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 4;
    constexpr int NE = 5;
    const int steps = (int)((double)bytes / (grid * 128.0 * NE * 8)) ;   // ~ one table's worth
    for (int kind = 0; kind < 2; ++kind)
        for (int sync = 0; sync < 2; ++sync)
            for (int spin : {0, 64, 128}) {
                auto f = kind == 0 ? gang64<NE> : full256<NE>;
                f<<<grid, 128>>>(A, B, nreg, 50, sync, spin);
                CK(cudaDeviceSynchronize());
                cudaEventRecord(e0);
                f<<<grid, 128>>>(A, B, nreg, steps, sync, spin);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double by = (double)grid * 128 * NE * 16.0 * steps;
                printf("%-8s sync %d spin %3d: %8.3f ms  %7.1f GB/s\n", kind ? "full256" : "gang64", sync, spin, ms,
                       by / ms / 1e6);
            }
    return 0;
}
