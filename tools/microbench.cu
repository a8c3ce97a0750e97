// microbench.cu -- B200 measurements that set this project's rooflines and
// latency model (run under gpurun; results summarised in profiles/).
//   1. DFMA dependent-chain latency, MUFU.RSQ64H latency, LDS latency
//   2. FP64 FMA throughput (the FP64 roofline denominator)
//   3. HBM store-only bandwidth: coalesced STG.64, and the traversal's pattern
//      (each group of 4 lanes writes one full aligned 32 B sector at a
//      pseudo-random location), with and without .cs (evict-first)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void lat_dfma(double* out, long long* cyc, double a, double b)
{
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}

__global__ void lat_rsq(double* out, long long* cyc, double a)
{
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 512; ++i) {
        double y;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        x = y + 1.0;
    }
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}

__global__ void lat_lds(int* out, long long* cyc)
{
    __shared__ int chain[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) chain[i] = (i * 97 + 13) & 1023;
    __syncthreads();
    if (threadIdx.x) return;
    int p = 0;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) p = chain[p];
    long long t1 = clock64();
    out[0] = p;
    cyc[0] = t1 - t0;
}

__global__ void thr_dfma(double* out, int iters)
{
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;
}

__global__ void store_coalesced(double* p, size_t n)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) p[i] = (double)i;
}

// each warp store: 8 groups of 4 lanes, group g writes the aligned 32 B sector
// hash(...) -- full sectors at scattered addresses (the traversal's pattern)
template <bool CS>
__global__ void store_sectors(double* p, size_t nsec, int iters)
{
    const int lane = threadIdx.x & 31;
    size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    uint64_t h = warp * 0x9E3779B97F4A7C15ull + (lane >> 2);
    for (int it = 0; it < iters; ++it) {
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        size_t sec = h % nsec;
        double* a = p + sec * 4 + (lane & 3);
        if (CS) __stcs(a, (double)it); else *a = (double)it;
    }
}

// groups of G lanes write G*8 contiguous bytes (aligned) at pseudo-random locations
template <int G>
__global__ void store_chunks(double* p, size_t nchunk, int iters)
{
    const int lane = threadIdx.x & 31;
    size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    uint64_t h = warp * 0x9E3779B97F4A7C15ull + (lane / G);
    for (int it = 0; it < iters; ++it) {
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        size_t ch = h % nchunk;
        p[ch * G + (lane % G)] = (double)it;
    }
}

// warp writes a contiguous 8 KB region as 32 stores of 256 B, region chosen at random,
// many warps interleaved: emulates "complete small regions"
__global__ void store_regions(double* p, size_t nreg, int iters)
{
    const int lane = threadIdx.x & 31;
    size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    uint64_t h = warp * 0x9E3779B97F4A7C15ull;
    for (int it = 0; it < iters; ++it) {
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        double* r = p + (h % nreg) * 1024;
        for (int j = 0; j < 32; ++j) r[j * 32 + lane] = (double)it;
    }
}

int main()
{
    double* d; long long* c; int* di;
    CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&c, 64)); CK(cudaMalloc(&di, 64));
    long long cyc;
    lat_dfma<<<1, 1>>>(d, c, 1.0, 0.5); CK(cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost));
    lat_dfma<<<1, 1>>>(d, c, 1.0, 0.5); CK(cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost));
    printf("dfma_latency_cycles %.2f\n", cyc / 1024.0);
    lat_rsq<<<1, 1>>>(d, c, 2.0); lat_rsq<<<1, 1>>>(d, c, 2.0); CK(cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost));
    printf("rsq64h_plus_dadd_latency_cycles %.2f\n", cyc / 512.0);
    lat_lds<<<1, 32>>>(di, c); lat_lds<<<1, 32>>>(di, c); CK(cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost));
    printf("lds_latency_cycles %.2f\n", cyc / 1024.0);

    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    int iters = 20000;
    thr_dfma<<<sms * 8, 256>>>(d, iters);
    cudaEventRecord(e0); thr_dfma<<<sms * 8, 256>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)sms * 8 * 256;
    printf("fp64_fma_tflops %.2f  (sms %d, max clock %d MHz)\n", flops / ms / 1e9, sms, clk / 1000);

    size_t bytes = (size_t)8 << 30;
    double* big; CK(cudaMalloc(&big, bytes));
    size_t n = bytes / 8;
    store_coalesced<<<sms * 16, 512>>>(big, n);
    cudaEventRecord(e0); store_coalesced<<<sms * 16, 512>>>(big, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("store_coalesced_gbs %.1f\n", bytes / ms / 1e6);
    size_t nsec = bytes / 32;
    int threads = sms * 32 * 256;
    int it2 = (int)(nsec * 4 / threads);
    store_sectors<false><<<sms * 32, 256>>>(big, nsec, it2);
    cudaEventRecord(e0); store_sectors<false><<<sms * 32, 256>>>(big, nsec, it2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("store_scattered_sectors_gbs %.1f\n", (double)it2 * threads * 8 / ms / 1e6);
    store_sectors<true><<<sms * 32, 256>>>(big, nsec, it2);
    cudaEventRecord(e0); store_sectors<true><<<sms * 32, 256>>>(big, nsec, it2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("store_scattered_sectors_cs_gbs %.1f\n", (double)it2 * threads * 8 / ms / 1e6);
    {
        size_t nch = bytes / 128; int it3 = (int)(nch * 16 / threads);
        store_chunks<16><<<sms * 32, 256>>>(big, nch, it3);
        cudaEventRecord(e0); store_chunks<16><<<sms * 32, 256>>>(big, nch, it3); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("store_random_128B_lines_gbs %.1f\n", (double)it3 * threads * 8 / ms / 1e6);
        nch = bytes / 256; it3 = (int)(nch * 32 / threads);
        store_chunks<32><<<sms * 32, 256>>>(big, nch, it3);
        cudaEventRecord(e0); store_chunks<32><<<sms * 32, 256>>>(big, nch, it3); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("store_random_256B_gbs %.1f\n", (double)it3 * threads * 8 / ms / 1e6);
        size_t nreg = bytes / 8192; int it4 = (int)(nreg * 32 / (threads / 32) / 32);
        if (it4 < 1) it4 = 1;
        store_regions<<<sms * 32, 256>>>(big, nreg, it4);
        cudaEventRecord(e0); store_regions<<<sms * 32, 256>>>(big, nreg, it4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("store_random_8KB_regions_gbs %.1f\n", (double)it4 * (threads / 32) * 8192 / ms / 1e6);
    }
    return 0;
}
