// bps_kernel.cu -- best parent set within every candidate set (SURVEY.md §8(f)
// NEXT 3, the step after the score table in exact structure search):
// for every child v and candidate set C (compressed mask index c of v's block),
//   bps(v, C) = max over S subset of C of score(v, S)
// with the G14 tie-break (larger score, then smaller |S|, then smaller mask).
//
// It is a subset-max transform over the m - 1 bits of the compressed index
// (compression keeps the order and the popcount of the masks, so G14 can compare
// compressed indices): for every bit b, bps[c] = better(bps[c], bps[c ^ 2^b]) for
// the c with bit b set.  HBM-bound: the bits are processed in groups inside
// shared-memory tiles, one read and one write of the (score, mask) table per group:
//   * low group (bits 0..T-1, T <= 12): a tile = 2^T consecutive entries;
//   * higher groups of <= 8 bits: a tile = 2^LO consecutive entries (coalesced rows,
//     LO >= 5 and LO + G >= 12 where the bits allow) x the 2^G settings of the group.
// The last pass writes user-id masks (bit v inserted).
#include <cstdint>
#include <algorithm>
#include "kernels.h"

namespace bnr {

__device__ __forceinline__ bool bps_better(double s1, uint32_t c1, double s2, uint32_t c2)
{
    if (s1 != s2) return s1 > s2;
    const int p1 = __popc(c1), p2 = __popc(c2);
    return p1 != p2 ? p1 < p2 : c1 < c2;
}

__device__ __forceinline__ uint32_t user_mask(uint32_t c, int v)
{
    const uint32_t lm = (1u << v) - 1u;
    return (c & lm) | ((c & ~lm) << 1);
}

// bits 0..T-1: one CTA per (child, tile of 2^T consecutive entries)
__global__ void __launch_bounds__(512) bps_low_kernel(const double* __restrict__ sc_in, int64_t stride, int m, int T,
                                                      double* __restrict__ out_s, uint32_t* __restrict__ out_m,
                                                      int final_pass)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = 1 << T;
    double* const s = (double*)smem;
    uint32_t* const c = (uint32_t*)(smem + (size_t)n * 8);
    const int tiles = 1 << (m - 1 - T);
    const int v = blockIdx.x / tiles;
    const uint32_t base = (uint32_t)(blockIdx.x % tiles) << T;
    const int64_t row = (int64_t)v << (m - 1);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s[i] = sc_in[(row + base + i) * stride];
        c[i] = base + (uint32_t)i;
    }
    __syncthreads();
    for (int b = 0; b < T; ++b) {
        const int bit = 1 << b;
        for (int q = threadIdx.x; q < n / 2; q += blockDim.x) {
            const int i = ((q >> b) << (b + 1)) | (q & (bit - 1)) | bit;   // the q-th index with bit b set
            const int j = i ^ bit;
            const double sj = s[j];
            const uint32_t cj = c[j];
            if (bps_better(sj, cj, s[i], c[i])) {
                s[i] = sj;
                c[i] = cj;
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        out_s[row + base + i] = s[i];
        out_m[row + base + i] = final_pass ? user_mask(c[i], v) : c[i];
    }
}

// bits b0..b0+G-1: one CTA per (child, setting of the bits outside the tile); tile =
// 2^LO consecutive entries (bits 0..LO-1, LO <= b0, coalesced rows) x the 2^G settings
// of the group's bits
__global__ void __launch_bounds__(512) bps_group_kernel(int m, int b0, int G, int LO, double* __restrict__ s_io,
                                                        uint32_t* __restrict__ m_io, int final_pass)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = 1 << (LO + G);
    double* const s = (double*)smem;
    uint32_t* const c = (uint32_t*)(smem + (size_t)n * 8);
    const int nb = m - 1;                                    // compressed index bits
    const int rest_bits = nb - LO - G;                       // bits LO..b0-1 and b0+G..nb-1
    const int v = blockIdx.x >> rest_bits;
    const uint32_t r = blockIdx.x & ((1u << rest_bits) - 1u);
    const int lowr = b0 - LO;
    const uint32_t fixed = ((r & ((1u << lowr) - 1u)) << LO) | ((r >> lowr) << (b0 + G));
    const uint32_t lom = (1u << LO) - 1u;
    const int64_t row = (int64_t)v << nb;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const uint32_t idx = fixed | ((uint32_t)(e >> LO) << b0) | ((uint32_t)e & lom);
        s[e] = s_io[row + idx];
        c[e] = m_io[row + idx];
    }
    __syncthreads();
    for (int b = 0; b < G; ++b) {
        const int tb = LO + b, bit = 1 << tb;                // group bit b within the tile index
        for (int q = threadIdx.x; q < n / 2; q += blockDim.x) {
            const int i = ((q >> tb) << (tb + 1)) | (q & (bit - 1)) | bit;
            const int j = i ^ bit;
            const double sj = s[j];
            const uint32_t cj = c[j];
            if (bps_better(sj, cj, s[i], c[i])) {
                s[i] = sj;
                c[i] = cj;
            }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const uint32_t idx = fixed | ((uint32_t)(e >> LO) << b0) | ((uint32_t)e & lom);
        s_io[row + idx] = s[e];
        m_io[row + idx] = final_pass ? user_mask(c[e], v) : c[e];
    }
}

cudaError_t launch_bps(const double* scores, int64_t stride, int m, double* out_s, uint32_t* out_m, cudaStream_t st)
{
    if (m < 2 || m > 30) return cudaErrorInvalidValue;
    const int nb = m - 1;
    const int T = std::min(nb, 12);
    const bool low_final = T == nb;
    {
        const size_t smem = ((size_t)1 << T) * 12;
        cudaError_t e = cudaFuncSetAttribute(bps_low_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const int grid = m << (nb - T);
        bps_low_kernel<<<grid, 512, smem, st>>>(scores, stride, m, T, out_s, out_m, low_final ? 1 : 0);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    for (int b0 = T; b0 < nb;) {
        const int G = std::min(8, nb - b0);
        const int LO = std::min(b0, std::max(5, 12 - G));    // tiles of >= 4096 entries (96 KB at G = 8)
        const bool last = b0 + G == nb;
        const size_t smem = ((size_t)1 << (LO + G)) * 12;
        cudaError_t e = cudaFuncSetAttribute(bps_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const int grid = m << (nb - LO - G);
        bps_group_kernel<<<grid, 512, smem, st>>>(m, b0, G, LO, out_s, out_m, last ? 1 : 0);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        b0 += G;
    }
    return cudaSuccess;
}

}  // namespace bnr
