// tmembench.cu -- B200 (sm_100a) TMEM as per-thread state storage: latency of
// tcgen05.ld/st + wait and the throughput of ld/st loops at several warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmembench tools/tmembench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void tm_alloc(uint32_t* dst_smem, int ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tm_dealloc(uint32_t a, int ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(a), "r"(ncols));
}
__device__ __forceinline__ void ld8(uint32_t a, uint32_t* r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
}
__device__ __forceinline__ void st8(uint32_t a, const uint32_t* r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode 0: ld8 + wait::ld chain; mode 1: st8 + wait::st + ld8 + wait::ld chain (same columns);
// mode 2: LDS.128 x2 chain (reference)
__global__ void lat_kernel(int mode, int iters, long long* out, double* sink)
{
    __shared__ uint32_t taddr;
    __shared__ double2 sm[1024];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (wib == 0) tm_alloc(&taddr, 512);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr + ((uint32_t)(wib * 32) << 16);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1.0, 0.0);
    __syncthreads();
    uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    st8(base, r);
    wait_st();
    uint32_t col = 0;
    double acc = 0;
    long long t0 = 0, t1 = 0;
    if (wib == 0) {
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode == 0) {
                ld8(base + col, r);
                wait_ld();
                col = (r[0] & 7) * 8;   // dependent address (r = 0 -> col 0)
            } else if (mode == 1) {
                r[0] += 0;
                st8(base + col, r);
                wait_st();
                ld8(base + col, r);
                wait_ld();
                col = (r[0] & 7) * 8;
            } else {
                double2 v = sm[(col + lane) & 1023];
                acc += v.y;
                col = (unsigned)v.y;   // 0
            }
        }
        t1 = clock64();
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = acc + r[1];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (wib == 0) tm_dealloc(taddr, 512);
}

// throughput: each CTA (4 warps) allocates ncols; each thread walks rows of its
// columns: per iteration ld x8 (two 16-B pairs) at a moving column, some DFMAs,
// st x8 back (wait::st only when `wst`)
__global__ void tput_kernel(int ncols, int iters, int wst, double* sink)
{
    __shared__ uint32_t taddr;
    const int wib = threadIdx.x >> 5;
    if (wib == 0) tm_alloc(&taddr, ncols);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr + ((uint32_t)((wib & 3) * 32) << 16);
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = 0;
    for (int c = 0; c < ncols; c += 8) st8(base + c, r);
    wait_st();
    double acc = threadIdx.x;
    int pos = 0, dir = 1;
    const int nslots = ncols / 8;
    for (int it = 0; it < iters; ++it) {
        ld8(base + pos * 8, r);
        wait_ld();
        double a = __hiloint2double(r[1], r[0]), b = __hiloint2double(r[3], r[2]);
        double c2 = __hiloint2double(r[5], r[4]), d = __hiloint2double(r[7], r[6]);
        a = fma(a, 0.999, b);
        c2 = fma(c2, 0.999, d);
        acc += a + c2;
        r[0] = __double2loint(a); r[1] = __double2hiint(a);
        r[4] = __double2loint(c2); r[5] = __double2hiint(c2);
        st8(base + pos * 8, r);
        if (wst) wait_st();
        pos += dir;
        if (pos == nslots - 1 || pos == 0) dir = -dir;
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (wib == 0) tm_dealloc(taddr, ncols);
}

int main()
{
    long long* dout;
    double* sink;
    CK(cudaMalloc(&dout, 8));
    CK(cudaMalloc(&sink, 148 * 16 * 128 * 8));
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        lat_kernel<<<1, 128>>>(mode, iters, dout, sink);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        long long c;
        CK(cudaMemcpy(&c, dout, 8, cudaMemcpyDeviceToHost));
        const char* nm[3] = {"ld8+wait_ld", "st8+wait_st+ld8+wait_ld", "lds128 (ref)"};
        printf("latency %-26s %.1f cycles/iter\n", nm[mode], (double)c / iters);
    }
    int sms = 148;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int ctas = 1; ctas <= 4; ctas *= 2)
        for (int wst = 0; wst < 2; ++wst) {
            const int ncols = 512 / ctas;
            const int it2 = 20000;
            tput_kernel<<<sms * ctas, 128>>>(ncols, 100, wst, sink);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            tput_kernel<<<sms * ctas, 128>>>(ncols, it2, wst, sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = (double)sms * ctas * 128 * it2 * 32.0;   // ld bytes (st same)
            printf("tput ctas/SM %d (warps/SM %2d) ncols %3d wait_st %d: %.3f ms, TMEM ld %.1f TB/s (+st same), %.1f B/clk/SM ld, %.1f cyc/iter/warp\n",
                   ctas, ctas * 4, ncols, wst, ms, bytes / ms / 1e9, bytes / (ms * 1e-3) / 1.965e9 / sms,
                   ms * 1e-3 * 1.965e9 / it2);
        }
    return 0;
}
