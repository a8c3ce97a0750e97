// bps_kernel.cu -- best parent set within every candidate set (SURVEY.md §8(f)
// NEXT 3, the step after the score table in exact structure search):
// for every child v and candidate set C (compressed mask index c of v's block),
//   bps(v, C) = max over S subset of C of score(v, S)
// with the G14 tie-break (larger score, then smaller |S|, then smaller mask).
//
// It is a subset-max transform over the m - 1 bits of the compressed index
// (compression keeps the order and the popcount of the masks, so G14 can compare
// compressed indices): for every bit b, bps[c] = better(bps[c], bps[c ^ 2^b]) for
// the c with bit b set.  HBM-bound: the bits are processed in passes, one read and one
// write of the (score, mask) table per pass, the user-id masks written by the last:
//   * m - 1 >= 12: the low 12 bits, then balanced groups of 4..8 bits, in
//     register-tiled tiles of 4096 entries (16 per thread, see below);
//   * small cases (m <= 12, a leftover group of 1..3 bits): shared-memory tiles, one
//     barrier per bit.
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

// ---- register-tiled passes (nb >= 12): each thread keeps 16 entries in registers ----
// A tile's index bits are split three ways in each phase: lane bits (5; coalesced in
// the phases that touch HBM), register bits (4: the entries one thread holds) and
// warp bits.  Only register bits are transformed, in registers; between the phases the
// tile goes through shared memory so that the remaining bits become register bits
// (group tiles: 2 phases, one exchange; the 12-bit low tile: 3 phases, two exchanges,
// swizzled so that no phase's accesses conflict).  No shuffles.
constexpr int kRegE = 16;

struct Ent {
    double s[kRegE];
    uint32_t c[kRegE];
};

// bit j of the register index, for the first `active` register bits
__device__ __forceinline__ void reg_pass(Ent& e, int active)
{
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (j >= active) break;
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            if (!((r >> j) & 1)) continue;
            const int q = r ^ (1 << j);
            if (bps_better(e.s[q], e.c[q], e.s[r], e.c[r])) {
                e.s[r] = e.s[q];
                e.c[r] = e.c[q];
            }
        }
    }
}

__device__ __forceinline__ uint32_t scatter4(int r, int p0, int p1, int p2, int p3)
{
    return ((uint32_t)(r & 1) << p0) | ((uint32_t)((r >> 1) & 1) << p1) | ((uint32_t)((r >> 2) & 1) << p2) |
           ((uint32_t)((r >> 3) & 1) << p3);
}

// shared-memory swizzles of the low tile (bijections on 0..4095): scores (8 B) XOR
// bits 0..3 with bits 4..7, masks (4 B) bits 0..4 with bits 4..8, so that a warp whose
// lanes run over bits 0..4 or over bits 4..8 hits distinct banks
__device__ __forceinline__ uint32_t swz_s(uint32_t t) { return t ^ ((t >> 4) & 15u); }
__device__ __forceinline__ uint32_t swz_c(uint32_t t) { return t ^ ((t >> 4) & 31u); }

// bits 0..11 of the compressed index: tile = 4096 consecutive entries, 256 threads,
// three register phases with two shared-memory exchanges (swizzled):
// phase A: lane = bits 0..4 (coalesced loads), registers = bits 5..8, warps = bits 9..11;
// phase B: registers = bits 0..3, lane = bits 4..8, warps = bits 9..11;
// phase C: registers = bits 9, 10, 11, 4, lane = bits 0..3 and 8, warps = bits 5..7.
__global__ void __launch_bounds__(256, 4) bps_low_reg_kernel(const double* __restrict__ sc_in, int64_t stride, int m,
                                                          double* __restrict__ out_s, uint32_t* __restrict__ out_m,
                                                          int final_pass)
{
    __shared__ double ts[4096];
    __shared__ uint32_t tc[4096];
    const int nb = m - 1;
    const int tiles = 1 << (nb - 12);
    const int v = blockIdx.x / tiles;
    const uint32_t base = (uint32_t)(blockIdx.x % tiles) << 12;
    const int64_t row = (int64_t)v << nb;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Ent e;
    {
        const uint32_t tb = (uint32_t)lane | ((uint32_t)warp << 9);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const uint32_t t = tb | ((uint32_t)r << 5);
            e.s[r] = __ldcs(sc_in + (row + base + t) * stride);
            e.c[r] = base + t;
        }
        reg_pass(e, 4);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const uint32_t t = tb | ((uint32_t)r << 5);
            ts[swz_s(t)] = e.s[r];
            tc[swz_c(t)] = e.c[r];
        }
    }
    __syncthreads();
    {
        // registers = bits 0..3, lane = bits 4..8, warps = bits 9..11 (swizzled: conflict-free)
        const uint32_t tb = ((uint32_t)lane << 4) | ((uint32_t)warp << 9);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            e.s[r] = ts[swz_s(tb | (uint32_t)r)];
            e.c[r] = tc[swz_c(tb | (uint32_t)r)];
        }
        reg_pass(e, 4);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            ts[swz_s(tb | (uint32_t)r)] = e.s[r];
            tc[swz_c(tb | (uint32_t)r)] = e.c[r];
        }
    }
    __syncthreads();
    {
        // registers = bits 9, 10, 11, 4, lane = bits 0..3 and 8 (16-entry runs: full
        // sectors), warps = bits 5..7
        const uint32_t tb = ((uint32_t)lane & 15u) | (((uint32_t)lane >> 4) << 8) | ((uint32_t)warp << 5);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const uint32_t t = tb | scatter4(r, 9, 10, 11, 4);
            e.s[r] = ts[swz_s(t)];
            e.c[r] = tc[swz_c(t)];
        }
        reg_pass(e, 4);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const uint32_t t = tb | scatter4(r, 9, 10, 11, 4);
            __stcs(out_s + row + base + t, e.s[r]);
            __stcs(out_m + row + base + t, final_pass ? user_mask(e.c[r], v) : e.c[r]);
        }
    }
}

// group bits b0..b0+G-1, 4 <= G <= 7: tile = 2^LO consecutive entries x 2^G group
// settings (LO + G = 12), tile index t = (g << LO) | row bits,
// 2^(LO+G-4) threads.  phase A: lane = row bits 0..4, registers = g bits 0..3,
// warps = g bits 4..G-1 then row bits 5..LO-1; phase B: registers = g bits 4..G-1
// (the active ones) then g bits 0..7-G, warps = g bits 8-G..3 then row bits 5..LO-1.
__global__ void __launch_bounds__(256, 4) bps_group_reg_kernel(int m, int b0, int G, int LO, double* __restrict__ s_io,
                                                            uint32_t* __restrict__ m_io, int final_pass)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = 1 << (LO + G);
    double* const ts = (double*)smem;
    uint32_t* const tc = (uint32_t*)(smem + (size_t)n * 8);
    const int nb = m - 1;
    const int rest_bits = nb - LO - G;
    const int v = blockIdx.x >> rest_bits;
    const uint32_t rr = blockIdx.x & ((1u << rest_bits) - 1u);
    const int lowr = b0 - LO;
    const uint32_t fixed = ((rr & ((1u << lowr) - 1u)) << LO) | ((rr >> lowr) << (b0 + G));
    const int64_t row = (int64_t)v << nb;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = G - 4;                                     // group bits among the warp bits
    const uint32_t wlo = warp & ((1u << gw) - 1u), whi = warp >> gw;
    const uint32_t rowbits = lane | (whi << 5);
    const int64_t gs = (int64_t)1 << b0;                      // index step of one group setting
    Ent e;
    // phase A: g = (wlo << 4) | r
    {
        const int64_t i0 = row + fixed + rowbits + ((int64_t)wlo << (b0 + 4));
        const double* ps = s_io + i0;
        const uint32_t* pm = m_io + i0;
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            e.s[r] = __ldcs(ps);
            e.c[r] = __ldcs(pm);
            ps += gs;
            pm += gs;
        }
    }
    reg_pass(e, 4);
    {
        const uint32_t tb = rowbits | (wlo << (LO + 4));
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            ts[tb | ((uint32_t)r << LO)] = e.s[r];
            tc[tb | ((uint32_t)r << LO)] = e.c[r];
        }
    }
    __syncthreads();
    // phase B: register bit j < gw is g bit 4 + j, the others g bit j - gw:
    // g = (wlo << (8 - G)) | (rl << 4) | rh
    const uint32_t tb = rowbits | (wlo << (LO + 8 - G));
#pragma unroll
    for (int r = 0; r < kRegE; ++r) {
        const uint32_t t = tb | (((uint32_t)r & ((1u << gw) - 1u)) << (LO + 4)) | (((uint32_t)r >> gw) << LO);
        e.s[r] = ts[t];
        e.c[r] = tc[t];
    }
    reg_pass(e, gw);
    {
        const int64_t i0 = row + fixed + rowbits + ((int64_t)wlo << (b0 + 8 - G));
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const int64_t i = i0 + ((int64_t)((((uint32_t)r & ((1u << gw) - 1u)) << 4) | ((uint32_t)r >> gw)) << b0);
            __stcs(s_io + i, e.s[r]);
            __stcs(m_io + i, final_pass ? user_mask(e.c[r], v) : e.c[r]);
        }
    }
}

// group of 8 bits b0..b0+7 over tiles of 16 consecutive entries (128 B runs of scores:
// full sectors) x the 256 group settings, 256 threads, 48 KB: tile index t = (g << 4) |
// row bits.  phase A: lane = row bits 0..3 and g bit 7, registers = g bits 0..3, warps =
// g bits 4..6; phase B: lane = row bits 0..3 and g bit 0, registers = g bits 4..7,
// warps = g bits 1..3.  Masks swizzled (t bit 4 ^= t bit 11) so both phases hit 32 banks.
__device__ __forceinline__ uint32_t swz_g8(uint32_t t) { return t ^ ((t >> 7) & 16u); }

__global__ void __launch_bounds__(256, 4) bps_group8_kernel(int m, int b0, double* __restrict__ s_io,
                                                         uint32_t* __restrict__ m_io, int final_pass)
{
    __shared__ double ts[4096];
    __shared__ uint32_t tc[4096];
    const int nb = m - 1;
    const int rest_bits = nb - 12;
    const int v = blockIdx.x >> rest_bits;
    const uint32_t rr = blockIdx.x & ((1u << rest_bits) - 1u);
    const int lowr = b0 - 4;
    const uint32_t fixed = ((rr & ((1u << lowr) - 1u)) << 4) | ((rr >> lowr) << (b0 + 8));
    const int64_t row = (int64_t)v << nb;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t rowbits = lane & 15u, lg = lane >> 4;
    const int64_t gs = (int64_t)1 << b0;
    Ent e;
    {
        // g = (lg << 7) | (warp << 4) | r
        const uint32_t g0 = (lg << 7) | (warp << 4);
        const int64_t i0 = row + fixed + rowbits + ((int64_t)g0 << b0);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            e.s[r] = __ldcs(s_io + i0 + r * gs);
            e.c[r] = __ldcs(m_io + i0 + r * gs);
        }
        reg_pass(e, 4);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const uint32_t t = ((g0 | (uint32_t)r) << 4) | rowbits;
            ts[t] = e.s[r];
            tc[swz_g8(t)] = e.c[r];
        }
    }
    __syncthreads();
    {
        // g = (r << 4) | (warp << 1) | lg
        const uint32_t g0 = (warp << 1) | lg;
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            const uint32_t t = ((g0 | ((uint32_t)r << 4)) << 4) | rowbits;
            e.s[r] = ts[t];
            e.c[r] = tc[swz_g8(t)];
        }
        reg_pass(e, 4);
        const int64_t i0 = row + fixed + rowbits + ((int64_t)g0 << b0);
#pragma unroll
        for (int r = 0; r < kRegE; ++r) {
            __stcs(s_io + i0 + ((int64_t)r << (b0 + 4)), e.s[r]);
            __stcs(m_io + i0 + ((int64_t)r << (b0 + 4)), final_pass ? user_mask(e.c[r], v) : e.c[r]);
        }
    }
}

cudaError_t launch_bps(const double* scores, int64_t stride, int m, double* out_s, uint32_t* out_m, cudaStream_t st)
{
    if (m < 2 || m > 30) return cudaErrorInvalidValue;
    const int nb = m - 1;
    cudaError_t e;
    if (nb < 12) {                                            // one tile per child: shared-memory passes
        const size_t smem = ((size_t)1 << nb) * 12;
        e = cudaFuncSetAttribute(bps_low_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        bps_low_kernel<<<m, 512, smem, st>>>(scores, stride, m, nb, out_s, out_m, 1);
        return cudaGetLastError();
    }
    bps_low_reg_kernel<<<m << (nb - 12), 256, 0, st>>>(scores, stride, m, out_s, out_m, nb == 12 ? 1 : 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int R = nb - 12;                                    // high bits: groups of 4..8 (1..3: one small group)
    const int ng = R == 0 ? 0 : (R < 4 ? 1 : (R + 7) / 8);
    for (int g = 0, b0 = 12; g < ng; ++g) {
        const int G = R / ng + (g < R % ng ? 1 : 0);
        const bool last = g == ng - 1;
        if (G < 4) {
            const int LO = std::min(b0, 12 - G);
            const size_t smem = ((size_t)1 << (LO + G)) * 12;
            e = cudaFuncSetAttribute(bps_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            bps_group_kernel<<<m << (nb - LO - G), 512, smem, st>>>(m, b0, G, LO, out_s, out_m, last ? 1 : 0);
        } else if (G == 8) {
            bps_group8_kernel<<<m << (nb - 12), 256, 0, st>>>(m, b0, out_s, out_m, last ? 1 : 0);
        } else {
            const int LO = 12 - G;
            const size_t smem = ((size_t)1 << (LO + G)) * 12;
            e = cudaFuncSetAttribute(bps_group_reg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            bps_group_reg_kernel<<<m << (nb - LO - G), 1 << (LO + G - 4), smem, st>>>(m, b0, G, LO, out_s, out_m,
                                                                                      last ? 1 : 0);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        b0 += G;
    }
    return cudaSuccess;
}

}  // namespace bnr
