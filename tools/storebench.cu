// storebench.cu -- HBM write-pattern sweep on B200 (which output layouts can
// reach the store roofline?).  All patterns write 8 B doubles, full 128 B lines.
//   chunk C   : a warp writes one random aligned C-byte chunk at once
//               (C/256 consecutive 256 B warp stores), then picks another
//   skew C s  : groups of G = C/128 "writer" lanes-of-4-warps emulate a
//               lockstep gang: in iteration it, writer w writes line w of the
//               region chosen at iteration (it - s*w) -- the region's lines
//               arrive spread over s*(G-1) iterations
//   fill C R  : a warp owns R open regions of C bytes and writes one line of
//               each in turn (the current traversal: many partially written
//               regions, each filled slowly)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t h)
{
    h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
    return h;
}

// one warp writes a random aligned chunk of `lines` 128 B lines per iteration
__global__ void chunk(double* p, size_t nchunk, int lines, int iters)
{
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const size_t c = mix((uint32_t)(warp * 1000003u + it)) & (nchunk - 1);
        double* r = p + c * (size_t)lines * 16;
        for (int j = lane; j < lines * 16; j += 32) __stcs(r + j, (double)it);
    }
}

// writer warps grouped by G (= lines per region); each warp writes one 128 B
// line of its group's current region per iteration
__global__ void skew(double* p, size_t nreg, int G, int s, int iters)
{
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t grp = warp / G;
    const int w = (int)(warp % G);
    for (int it = 0; it < iters; ++it) {
        const int64_t t = (int64_t)it - (int64_t)s * w;
        if (t < 0) continue;
        const size_t rg = mix((uint32_t)(grp * 1000003u + (uint32_t)t)) & (nreg - 1);
        double* r = p + rg * (size_t)G * 16 + (size_t)w * 16;
        if (lane < 16) __stcs(r + lane, (double)it);
    }
}

// U x 2 writers per warp (half-warp each, U stores in flight per lane): writer
// v = warp * 2U + 2u + (lane >> 4); group = v / G, w = v % G; in iteration it
// writer w writes line w of region hash(group, it - s*w).  G = 1: random lines.
template <int U>
__global__ void skew2(double* p, uint32_t nreg, int lgG, int s, int iters)
{
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int G = 1 << lgG;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t v = warp * 2 * U + 2 * u + (lane >> 4);
            const uint32_t grp = v >> lgG;
            const int w = v & (G - 1);
            const int t = it - s * w;
            const uint32_t rg = mix(grp * 1000003u + (uint32_t)t) & (nreg - 1);
            double* r = p + ((size_t)rg << (lgG + 4)) + ((size_t)w << 4);
            if (t >= 0) __stcs(r + (lane & 15), (double)it);
        }
    }
}

__global__ void fill(double* p, size_t nreg, int lines, int R, int iters)
{
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const int slot = it & (R - 1);
        const int round = it >> __ffs(R) - 1;
        const int line = round & (lines - 1);
        const int gen = round >> (__ffs(lines) - 1);
        const size_t rg = mix((uint32_t)((warp * 64 + slot) * 1000003u + gen)) & (nreg - 1);
        double* r = p + rg * (size_t)lines * 16 + (size_t)((line * 7) & (lines - 1)) * 16;
        if (lane < 16) __stcs(r + lane, (double)it);
    }
}

int main()
{
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    size_t bytes = (size_t)16 << 30;
    double* big; CK(cudaMalloc(&big, bytes));
    CK(cudaMemset(big, 0, bytes));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    const int blocks = sms * 8, threads = 256;
    const double warps = blocks * threads / 32.0;
    for (int C = 128; C <= 16384; C *= 2) {
        const int lines = C / 128;
        const size_t nch = bytes / C;
        const int iters = (int)(bytes / 2 / C / warps) + 1;
        chunk<<<blocks, threads>>>(big, nch, lines, iters);
        cudaEventRecord(e0); chunk<<<blocks, threads>>>(big, nch, lines, iters); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("chunk %6d B           %7.1f GB/s\n", C, iters * warps * C / ms / 1e6);
    }
    int Gs[] = {16, 32, 64};
    int ss[] = {0, 1, 4, 16, 64};
    for (int G : Gs)
        for (int s : ss) {
            const size_t nreg = bytes / (G * 128);
            const int iters = (int)(bytes / 2 / 128 / warps) + s * G;
            skew<<<blocks, threads>>>(big, nreg, G, s, iters);
            cudaEventRecord(e0); skew<<<blocks, threads>>>(big, nreg, G, s, iters); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            // lines written: per warp iters - s*w (approx: average)
            double lw = 0;
            for (int w = 0; w < G; ++w) lw += (iters - s * w > 0 ? iters - s * w : 0);
            lw = lw / G * warps;
            printf("skew region %5d B (G=%2d) skew %3d it  %7.1f GB/s\n", G * 128, G, s, lw * 128 / ms / 1e6);
        }
    for (int lgG = 0; lgG <= 6; ++lgG)
        for (int s : ss) {
            if (lgG == 0 && s) continue;
            const int G = 1 << lgG;
            const uint32_t nreg = (uint32_t)(bytes / (G * 128));
            const int wr = (int)(warps * 8);
            const int iters = (int)(bytes / 2 / 128 / wr) + s * G;
            skew2<4><<<blocks, threads>>>(big, nreg, lgG, s, iters);
            cudaEventRecord(e0); skew2<4><<<blocks, threads>>>(big, nreg, lgG, s, iters); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            double lw = 0;
            for (int w = 0; w < G; ++w) lw += (iters - s * w > 0 ? iters - s * w : 0);
            lw = lw / G * wr;
            printf("skew2 region %5d B (G=%2d) skew %3d it  %7.1f GB/s  (%.3f ms)\n", G * 128, G, s, lw * 128 / ms / 1e6, ms);
        }
    int Cs[] = {1024, 4096, 16384};
    int Rs[] = {1, 4, 16, 64};
    for (int C : Cs)
        for (int R : Rs) {
            const int lines = C / 128;
            const size_t nreg = bytes / C;
            const int iters = (int)(bytes / 2 / 128 / warps) + 1;
            fill<<<blocks, threads>>>(big, nreg, lines, R, iters);
            cudaEventRecord(e0); fill<<<blocks, threads>>>(big, nreg, lines, R, iters); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            printf("fill region %5d B, %2d open/warp (%.0f MB open)  %7.1f GB/s\n", C, R, warps * R * C / 1e6,
                   iters * warps * 128 / ms / 1e6);
        }
    return 0;
}
