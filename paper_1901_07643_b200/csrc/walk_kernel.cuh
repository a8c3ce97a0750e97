// walk_kernel.cuh -- the hot kernel of the bnreg path:
// Alg.2 workers each walk d + Upsilon(k) (Alg.1 with Eq.10's
// +1) from their seed R, one GRC per step
// (Eq.3-4 with reading G1), harvesting every new family from
// suffix sums of squares (Eq.5, reading G3), computing its
// BIC (a9, reading G5), storing RSS and BIC into the (child, mask)-indexed
// table (a10) and keeping a per-child running best (a11, G14).
//
// B200 mapping:
//   * a warp runs W = 8 workers in lockstep; lane = (worker w = lane % 8,
//     part h = lane / 8).  All workers of a warp follow the same step records,
//     so control flow is warp-uniform.  A step's list of entries is
//     [back slots | free slots after the prefix], dealt round-robin to the 4
//     parts: back slot b always belongs to part b % 4 (entry j = b / 4), free
//     list entry f to part (NB + f) % 4.
//   * the W workers differ in the W lowest user ids (the "warp variables"), the
//     CTA's 4 warps in the next 2 ids (the "gang variables"): for every child
//     and step a CTA's 32 workers own 32 adjacent entries -- 512 B of (RSS, BIC)
//     records, or 256 B of each separate table; a gang barrier before the harvest
//     (every step for the tables, every 16th for the records) keeps the warps'
//     parts of a region close in time (DRAM write combining: tools/gangstore.cu)
//   * walk state E(l, slot) = (R_l, U_{l+1}) of the k free rows l of a column,
//     U_l = sum_{r >= l} R_r^2 (+ the rows below the free block); suffix sums
//     are updated by addition only.  Back slots are statically
//     owned by one lane, so their state lives in TENSOR MEMORY (tcgen05.ld/st,
//     the lane's own TMEM lane: rows i, i+1 of all its back slots are one
//     contiguous column range); the free slots, whose list position moves every
//     step, live in shared memory (worker-interleaved, 128 B per LDS phase).
//     Moving the back state out of shared memory is what lets 16 warps share an
//     SM (shared memory held 8 before).
#pragma once
// (included by walk_pairs.cu and walk_tables.cu, which instantiate the kernel for the
// record layout and the two-table layouts in separate translation units)
#include <cstdint>
#include <cmath>
#include <algorithm>
#include "kernels.h"
#include "device.cuh"
#include "tmem.cuh"

#ifndef BNREG_SYNC_EVERY
#define BNREG_SYNC_EVERY 16  // (RSS, BIC) records: gang barrier every this many steps (a power of two;
                             // measured at cfg5: 1 13.0 ms, 4 12.45, 16 12.3, 64 12.7, none 13.7); the
                             // two-table layout's 64 B pieces need it every step (16: 20.3 vs 15.2 ms)
#endif

namespace bnr {

constexpr int kW = 8;          // lockstep workers per warp
constexpr int kCS = kW * 16;   // bytes between free slots of the shared state

// ---------------------------------------------------------------- shared memory layout
// Per CTA: [log table 512 x 16 B][K(s) 33 doubles] then per warp:
//   state   k * k * W * 16 B   free-slot state E(l, f, w) at ((l*k + f)*W + w)*16
//   rec     SA * 16 B          per slot (shared by the warp's workers): the warp's running
//                              best BIC of the slot's child, the table index of (child,
//                              F without the warp and free variables), lm = (1 << v) - 1
//   bb      SA * 8 B           the running best BIC of the slot's child (rec holds the candidate
//                              threshold min(best, tiny_bic))
//   bm      SA * 4 B           the mask of that running best
//   wbb/wbm 32 * 12 B          the warp's running best per child (kept across items)
struct WalkLayout {
    int state, rec, bb, bm, wbb, wbm, per_warp;
};

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline WalkLayout walk_layout(int k, int SA)
{
    WalkLayout L;
    int o = 0;
    L.state = o;
    o += al16(k * k * kW * 16);
    L.rec = o;
    L.bb = o + SA * 16;
    L.bm = o + SA * 24;
    o += al16(SA * 28);
    L.wbb = o;
    o += 32 * 8;
    L.wbm = o;
    o += 32 * 4;
    L.per_warp = al16(o);
    return L;
}

constexpr int kWalkHead = 16 * kLnEntries + 272;   // log table + K(s) table

inline size_t walk_cta_smem_h(int m, int k, int SA, int g, int lw)
{
    (void)m;
    (void)lw;
    return (size_t)kWalkHead + ((size_t)1 << g) * (size_t)walk_layout(k, SA).per_warp;
}

// TMEM columns a CTA allocates: a warp's back state is k rows x JB slots x 4 columns
inline int walk_tmem_cols_h(int k, int jbmax)
{
    int need = k * jbmax * 4, c = 32;
    while (c < need) c <<= 1;
    return c;
}

// Launch constants: BNREG_LCONST reads them from the kernel parameters (constant bank) in
// the hot loop instead of per-lane registers (A/B of register pressure)
#ifdef BNREG_LCONST
#define LC_mhalf_n P.mhalf_n
#define LC_out_pairs P.out_pairs
#define LC_tiny_bic P.tiny_bic
#define LC_fv0 (P.p + P.g)
#define LC_RS (P.k * kW * 16)
#else
#define LC_mhalf_n L.mhalf_n
#define LC_out_pairs L.out_pairs
#define LC_tiny_bic L.tiny_bic
#define LC_fv0 L.fv0
#define LC_RS L.RS
#endif
#define LC(x) LC_##x

// Per-lane constants of the current item.
struct LaneC {
    unsigned sbase;   // shared address of the free state (row 0, slot 0, worker w)
    unsigned recb;    // shared address of rec[slot 0]
    unsigned recB;    // shared address of the record of back slot h: rec[k + h]
    unsigned bmb;     // shared address of bm[slot 0]
    unsigned bbb;     // shared address of bb[slot 0]
    double tiny_bic;  // a lower bound of the BIC of any RSS <= 1e-300 (G13)
    uint32_t tb;      // TMEM address of (this warp's lane quarter, column 0)
    uint32_t bval;    // bit j: back entry j (slot k + b0 + 4j + h) holds a family of this worker
    int hfree;        // this pass harvests the free entries (split items: only the first pass)
    uint32_t w;       // worker id = its warp-variable bits
    uint32_t Xw;      // the worker's warp and gang variables in F (user-id bits)
    uint32_t Fw;      // the worker's F (user ids)
    int fh0;          // this part's first free-list entry: (h - NB) mod 4
    int live;         // w < 2^p
    int h;
    int RS;           // bytes between free rows l and l+1
    int fv0;          // user id of free slot 0
    double mhalf_n;
    const double* KCw;   // K(|S|) = KCw[i + 1] (K shifted by the worker's d)
    unsigned lnt;        // shared address of the log table
    double* out_rss;
    double* out_bic;
    double* out_pairs;
    long long* gbest;    // per child: the best BIC found by any warp so far (bic_ord), or null
    unsigned* k8;        // BNREG_K8: write counters (+ the violation counter k8[k8_n])
    unsigned long long k8_n;
    unsigned sb0;        // BNREG_K8 bounds checks: the warp's shared state [sb0, sb0 + sbytes)
    unsigned sbytes;
    unsigned tmcols;     // and the TMEM columns it may address
};

// phase C of a step: ln RSS, BIC (a9), the two table stores (a10) and the
// running-best candidates; new bests (rare) are resolved warp-serially (a11, G14)
template <int NE, bool HR, bool HB, bool HP>
__device__ __forceinline__ void harvest(const LaneC& L, const TravParams& P, const double* rs, const unsigned* ra,
                                        const bool* okv, double Kw, uint32_t X, uint32_t S)
{
    const double PINF = __longlong_as_double(0x7ff0000000000000LL);
    const uint32_t X1 = X >> 1;
    uint32_t upd = 0;
    double bics[NE > 0 ? NE : 1];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const double rss = rs[e];
#ifdef BNREG_FAKE_HARVEST   // timing experiment only (wrong BICs): no log
        const double lnr = rss;
#else
        const double lnr = fast_ln9s(rss, L.lnt);
#endif
        const double bic = fma(LC(mhalf_n), lnr, Kw);
        bics[e] = bic;
        const double2 rr = lds2(ra[e]);
        const uint32_t idx = (uint32_t)__double2loint(rr.y);        // table index of (child, F_w)
        const uint32_t lm = (uint32_t)__double2hiint(rr.y);         // (1 << child) - 1
        const uint32_t ix = idx + ((X & lm) | (X1 & ~lm));           // + compress(T | w-bits, child)
        if (HR) stg_cs_if(L.out_rss + ix, rss, okv[e]);
        if (HB) stg_cs_if(L.out_bic + ix, bic, okv[e]);
        if (HP) stg2_cs_if(LC(out_pairs) + 2 * (size_t)ix, rss, bic, okv[e]);
        K8_COUNT(L, okv[e], ix);   // K8 debug builds: every entry written exactly once, in range
        // candidate: BIC >= the slot's threshold min(running best, tiny_bic); a perfect fit
        // (RSS <= 1e-300, G13: BIC = +inf, fixed on the rare path) has BIC >= tiny_bic
        upd |= (okv[e] && bic >= rr.x) ? (1u << e) : 0u;
    }
    unsigned bal = __ballot_sync(FULLMASK, upd != 0);
    while (bal) {
        // rare: a family beats (or ties, G14) the warp's running best of its child; the
        // 8 workers share the record, so lanes with candidates take turns
        const int l = __ffs(bal) - 1;
        bal &= bal - 1;
        if ((int)(threadIdx.x & 31) == l) {
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                if ((upd >> e) & 1u) {
                    const unsigned a = ra[e];
                    const unsigned ma = L.bmb + ((a - L.recb) >> 2);   // bm[slot]
                    const unsigned ba = L.bbb + ((a - L.recb) >> 1);   // bb[slot]
                    double b = bics[e];
                    if (rs[e] <= 1e-300) {
                        // a perfect fit (G13): BIC = +inf, stored over the finite value written above
                        b = PINF;
                        double rr;
                        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(rr) : "r"(a + 8));
                        const uint32_t idx = (uint32_t)__double2loint(rr), lm = (uint32_t)__double2hiint(rr);
                        if (HB) L.out_bic[idx + ((X & lm) | (X1 & ~lm))] = PINF;
                        if (HP) LC(out_pairs)[2 * (size_t)(idx + ((X & lm) | (X1 & ~lm))) + 1] = PINF;
                    }
                    double cb;
                    uint32_t cm;
                    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cb) : "r"(ba));
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cm) : "r"(ma));
                    if (tie_better(b, S, cb, cm)) {
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(ba), "d"(b) : "memory");
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ma), "r"(S) : "memory");
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(fmin(b, LC(tiny_bic))) : "memory");
                        if (L.gbest) {
                            // publish: every warp's later items take it as their candidate floor
                            uint32_t lmv;
                            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lmv) : "r"(a + 12));
                            atomicMax(L.gbest + __popc(lmv), bic_ord(b));
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
}

// The free-list entries of this lane at step record q: slots and validity.
template <int NFE>
__device__ __forceinline__ void free_entries(const LaneC& L, uint32_t nib, int nf, unsigned* slot, bool* ok)
{
    const uint32_t nl = nib >> (4 * L.fh0);
#pragma unroll
    for (int j = 0; j < NFE; ++j) {
        slot[j] = (nl >> (16 * j)) & 15u;
        ok[j] = L.live && (L.fh0 + 4 * j < nf);
    }
}

// Seed pseudo-step (reading G11: the seed prefixes {free 0..j-1}, i = j - 1):
// RSS = U_{i+1} = E_i.y, or U_0 = R_0^2 + E_0.y for the empty prefix; no rotation.
template <int JB, int NFE, bool HR, bool HB, bool HP>
__device__ __forceinline__ void seed_step(const LaneC& L, const TravParams& P, const uint4 q)
{
    constexpr int NE = JB + NFE;
    const uint32_t fl = q.w;
    const int nf = (int)(fl & 31u);
    const int i = (int)((fl >> 8) & 31u) - 1;
    const bool s0 = i < 0;
    const unsigned bi = L.sbase + q.x;   // row max(i, 0)
    double rs[NE > 0 ? NE : 1];
    unsigned ra[NE > 0 ? NE : 1];
    bool okv[NE > 0 ? NE : 1];
    if constexpr (JB > 0) {
        uint32_t rb[4 * JB];
        tm_wait_st();
        tm_ld<4 * JB>(L.tb + (uint32_t)((s0 ? 0 : i) * JB * 4), rb);
        tm_wait_ld<4 * JB>(rb);
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            const double R = tm_f64(rb + 4 * j), U = tm_f64(rb + 4 * j + 2);
            rs[j] = s0 ? fma(R, R, U) : U;
            ra[j] = L.recB + 64 * j;
            okv[j] = (L.bval >> j) & 1u;
        }
    }
    unsigned sl[NFE > 0 ? NFE : 1];
    bool fo[NFE > 0 ? NFE : 1];
    free_entries<NFE>(L, q.z, nf, sl, fo);
#pragma unroll
    for (int j = 0; j < NFE; ++j) {
        const double2 a = lds2(bi + sl[j] * kCS);
        rs[JB + j] = s0 ? fma(a.x, a.x, a.y) : a.y;
        ra[JB + j] = L.recb + sl[j] * 16;
        okv[JB + j] = fo[j] && L.hfree;
    }
    const uint32_t Tsh = (fl >> 17) << LC(fv0);
    harvest<NE, HR, HB, HP>(L, P, rs, ra, okv, L.KCw[(fl >> 8) & 31u], Tsh | L.Xw, L.Fw | Tsh);
}

// One lockstep GRC step of a lane (a7-a11):
//   phase A  the rotation of rows i, i+1 of every entry's column with this step's
//            (c, s) and the new suffix sum U_{i+1} = U_{i+2} + R'_{i+1}^2: back
//            entries in TMEM (one ld / st of the contiguous rows), free entries in
//            shared memory; the pivot Y (now at position i): E_i = (h, 0), R_{i+1} = 0;
//   givens   the next step's rotation from its pivot column (overlaps phase C);
//   phase C  harvest().
template <int JB, int NFE, bool HR, bool HB, bool HP>
__device__ __forceinline__ void grc_step(const LaneC& L, const TravParams& P, const uint4 q, double& c, double& sg,
                                         double& hh, bool sync)
{
    constexpr int NE = JB + NFE;
    const uint32_t fl = q.w;
    const int nf = (int)(fl & 31u);
    const int i = (int)((fl >> 8) & 31u) - 1;
    const unsigned bi = L.sbase + q.x;
    const int RS = LC(RS);
    double rs[NE];
    unsigned ra[NE];
    bool okv[NE];
    unsigned sl[NFE > 0 ? NFE : 1];
    bool fo[NFE > 0 ? NFE : 1];
    free_entries<NFE>(L, q.z, nf, sl, fo);
    double f0[NFE > 0 ? NFE : 1];
    double2 f1[NFE > 0 ? NFE : 1];
    if constexpr (JB > 0) {
        uint32_t rb[8 * JB];
        const uint32_t tcol = L.tb + (uint32_t)(i * JB * 4);
        K8_CHECK(L, i >= 0 && (unsigned)((i + 2) * JB * 4) <= L.tmcols);
        tm_wait_st();
        tm_ld<8 * JB>(tcol, rb);
#pragma unroll
        for (int j = 0; j < NFE; ++j) {
            f0[j] = lds1(bi + sl[j] * kCS);
            f1[j] = lds2(bi + sl[j] * kCS + RS);
        }
        tm_wait_ld<8 * JB>(rb);
        // the rotated rows into their own registers (not over the loaded ones): ptxas then
        // places them where the store reads them (2.5% fewer instructions than in place)
        uint32_t wb[8 * JB];
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            const uint32_t* r0 = rb + 4 * j;            // row i:   (R_i, U_{i+1})
            const uint32_t* r1 = rb + 4 * JB + 4 * j;   // row i+1: (R_{i+1}, U_{i+2})
            const double x = tm_f64(r0), y = tm_f64(r1), u2 = tm_f64(r1 + 2);
            const double t1 = sg * y, t2 = sg * x;
            const double xa = fma(c, x, t1), ya = fma(c, y, -t2);
            const double ru = fma(ya, ya, u2);
            tm_put(wb + 4 * j, xa);
            tm_put(wb + 4 * j + 2, ru);
            tm_put(wb + 4 * JB + 4 * j, ya);
            wb[4 * JB + 4 * j + 2] = r1[2];
            wb[4 * JB + 4 * j + 3] = r1[3];
            rs[j] = ru;
            ra[j] = L.recB + 64 * j;
            okv[j] = (L.bval >> j) & 1u;
        }
        tm_st<8 * JB>(tcol, wb);
    } else {
#pragma unroll
        for (int j = 0; j < NFE; ++j) {
            f0[j] = lds1(bi + sl[j] * kCS);
            f1[j] = lds2(bi + sl[j] * kCS + RS);
        }
    }
#pragma unroll
    for (int j = 0; j < NFE; ++j) {
        K8_CHECK(L, !fo[j] || (bi + sl[j] * kCS + RS + 16 - L.sb0 <= L.sbytes && bi + sl[j] * kCS >= L.sb0));
        const double xa = fma(c, f0[j], sg * f1[j].x), ya = fma(c, f1[j].x, -sg * f0[j]);
        const double ru = fma(ya, ya, f1[j].y);
        sts_pair_if(bi + sl[j] * kCS, xa, ru, ya, RS, fo[j]);
        rs[JB + j] = ru;
        ra[JB + j] = L.recb + sl[j] * 16;
        okv[JB + j] = fo[j] && L.hfree;
    }
    if (L.h == 0) sts_pair_if(bi + ((fl >> 13) & 15u) * kCS, hh, 0.0, 0.0, RS, true);   // pivot Y
    __syncwarp();
    {
        // the next step's rotation, unconditionally (no branch: the chain interleaves with
        // phase C); without a next GRC the table points at a valid slot and the result is unused
        double a, b;
        const unsigned ncol = L.sbase + q.y;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"(ncol));
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b) : "r"(ncol + RS));
#ifndef BNREG_CHAIN_NOSEL
        if (!((fl >> 7) & 1u)) {
            a = 0.0;
            b = 1.0;
        }
#endif
        givens_fr(a, b, c, sg, hh);
    }
    const uint32_t Tsh = (fl >> 17) << LC(fv0);
    // the gang's stores start together (DRAM write combining of the 4 warps' parts of each
    // region) every BNREG_SYNC_EVERY steps: the barrier costs more than the last bit of combining
    if (sync) asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
    harvest<NE, HR, HB, HP>(L, P, rs, ra, okv, L.KCw[(fl >> 8) & 31u], Tsh | L.Xw, L.Fw | Tsh);
}

// One item (gang) of a warp with JB back entries per lane: fill the lane's TMEM
// rows from the seed block, the k + 1 seed pseudo-steps, then Upsilon(k).
template <int JB, bool HR, bool HB, bool HP>
__device__ __forceinline__ void walk_item(const LaneC& L, const TravParams& P, const unsigned char* src, int k, int SA,
                                       int NB, int b0, const uint4* __restrict__ wsteps, int nsteps)
{
    if constexpr (JB > 0) {
        // back slot b = b0 + 4j + h of worker w, row l: seed block [w][l][slot] at ((w k + l) SA + k + b) * 16
        const unsigned char* bs = src + ((size_t)(L.w * k) * SA + k + b0 + L.h) * 16;
        for (int l = 0; l < k; l += 2) {
            uint32_t v0[4 * JB], v1[4 * JB];
#pragma unroll
            for (int j = 0; j < JB; ++j) {
                const bool ok = L.live && (b0 + 4 * j + L.h < NB);
                uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
                if (ok) {
                    a = __ldg((const uint4*)(bs + ((size_t)l * SA + 4 * j) * 16));
                    if (l + 1 < k) b = __ldg((const uint4*)(bs + ((size_t)(l + 1) * SA + 4 * j) * 16));
                }
                v0[4 * j] = a.x; v0[4 * j + 1] = a.y; v0[4 * j + 2] = a.z; v0[4 * j + 3] = a.w;
                v1[4 * j] = b.x; v1[4 * j + 1] = b.y; v1[4 * j + 2] = b.z; v1[4 * j + 3] = b.w;
            }
            tm_st<4 * JB>(L.tb + (uint32_t)(l * JB * 4), v0);
            if (l + 1 < k) tm_st<4 * JB>(L.tb + (uint32_t)((l + 1) * JB * 4), v1);
        }
    }
    // a6-a11: the k + 1 seed pseudo-steps, then d + Upsilon(k), in lockstep
    // step records: lane l holds record t0 + l of the current 32-step window (one
    // coalesced load per 32 steps), a step's record is shuffled from lane t - t0
    uint4 win = make_uint4(0, 0, 0, 0);
    const int lane = (int)(threadIdx.x & 31);
    auto record = [&](int t) {
        if ((t & 31) == 0) win = __ldg(wsteps + t + lane);   // (the device table is padded to whole windows)
        const int s = t & 31;
        return make_uint4(__shfl_sync(FULLMASK, win.x, s), __shfl_sync(FULLMASK, win.y, s),
                          __shfl_sync(FULLMASK, win.z, s), __shfl_sync(FULLMASK, win.w, s));
    };
    win = __ldg(wsteps + lane);
    uint4 qk = make_uint4(0, 0, 0, 0);
    for (int t = 0; t <= k; ++t) {
        const uint4 q = t ? record(t) : make_uint4(__shfl_sync(FULLMASK, win.x, 0), __shfl_sync(FULLMASK, win.y, 0),
                                                   __shfl_sync(FULLMASK, win.z, 0), __shfl_sync(FULLMASK, win.w, 0));
        qk = q;
        const int nfe = ((int)(q.w & 31u) + 3) >> 2;
        if (nfe == 0) seed_step<JB, 0, HR, HB, HP>(L, P, q);
        else if (nfe == 1) seed_step<JB, 1, HR, HB, HP>(L, P, q);
        else seed_step<JB, 2, HR, HB, HP>(L, P, q);
    }
    double c = 1.0, sg = 0.0, hh = 0.0;
    {
        // the first GRC's rotation (the last seed record points at its pivot column)
        double a = 0.0, b = 1.0;
        if ((qk.w >> 7) & 1u) {
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"(L.sbase + qk.y));
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b) : "r"(L.sbase + qk.y + LC(RS)));
        }
        givens_fr(a, b, c, sg, hh);
    }
    constexpr int kSync = HP ? BNREG_SYNC_EVERY : 1;
    for (int t = k + 1; t < nsteps; ++t) {
        const uint4 q = record(t);
        if ((q.w & 31u) > 4u) grc_step<JB, 2, HR, HB, HP>(L, P, q, c, sg, hh, (t & (kSync - 1)) == 0);
        else grc_step<JB, 1, HR, HB, HP>(L, P, q, c, sg, hh, (t & (kSync - 1)) == 0);
    }
    tm_wait_st();
}

template <bool HR, bool HB, bool HP, int JBMAX>
#ifndef BNREG_WALK_MAXREG
#define BNREG_WALK_MAXREG 0      // A/B: cap the walk's registers (e.g. 112 leaves room for one prep CTA per SM)
#endif
#if BNREG_WALK_MAXREG > 0
__global__ void __maxnreg__(JBMAX <= 4 ? BNREG_WALK_MAXREG : 255) walk_kernel(const __grid_constant__ TravParams P)
#else
__global__ void __launch_bounds__(128, JBMAX <= 4 ? 4 : 2) walk_kernel(const __grid_constant__ TravParams P)
#endif
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_item, s_taddr;
    double2* const lntab = (double2*)smem;
    double* const KC = (double*)(smem + 16 * kLnEntries);
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    for (int j = tid; j < kLnEntries; j += blockDim.x) lntab[j] = P.lntab9[j];
    for (int j = tid; j < 33; j += blockDim.x) KC[j] = P.Kc[j];
    if (wib == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&s_taddr)),
                     "r"(P.tm_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g, SA = P.S_alloc;
    const int fv0 = p + g;                      // user id of free slot 0
    const int gs = bh - g;                      // gang levels are gs..bh-1
    const int G = 1 << g;
    const WalkLayout Ly = walk_layout(k, SA);
    unsigned char* const wb = smem + kWalkHead + wib * Ly.per_warp;
    unsigned char* const st = wb + Ly.state;
    unsigned char* const recb = wb + Ly.rec;
    uint32_t* const bm = (uint32_t*)(wb + Ly.bm);
    double* const bbv = (double*)(wb + Ly.bb);
    double* const wbb = (double*)(wb + Ly.wbb);
    uint32_t* const wbm = (uint32_t*)(wb + Ly.wbm);
    const int w = lane & (kW - 1), h = lane >> 3;
    const double NINF = -__longlong_as_double(0x7ff0000000000000LL);
    wbb[lane] = NINF;
    wbm[lane] = 0xffffffffu;
    const int shb = P.world1 ? m - 1 : m - P.r;   // child block = v << shb entries
    const int nw = P.nw;
    LaneC L;
    L.sbase = (unsigned)__cvta_generic_to_shared(st + w * 16);
    L.recb = (unsigned)__cvta_generic_to_shared(recb);
    L.recB = L.recb + (unsigned)(k + h) * 16u;
    L.bmb = (unsigned)__cvta_generic_to_shared(bm);
    L.bbb = (unsigned)__cvta_generic_to_shared(bbv);
    L.tiny_bic = P.tiny_bic;
    L.tb = s_taddr + ((uint32_t)(wib * 32) << 16);
    L.w = (uint32_t)w;
    L.live = w < nw;
    L.h = h;
    L.RS = k * kW * 16;
    L.fv0 = fv0;
    L.mhalf_n = P.mhalf_n;
    L.lnt = (unsigned)__cvta_generic_to_shared(lntab);
    L.out_rss = P.out_rss;
    L.out_bic = P.out_bic;
    L.out_pairs = P.out_pairs;
    L.k8 = P.k8;
    L.k8_n = P.k8_n;
    L.gbest = P.gbest;
    L.sb0 = (unsigned)__cvta_generic_to_shared(st);
    L.sbytes = (unsigned)(k * k * kW * 16);
    L.tmcols = (unsigned)P.tm_cols;
    K8_CHECK(L, !(P.k8_selftest && (threadIdx.x & 31) == 0));   // (a negative control of the counter path)
    {
        // the worker's warp and gang variables in F (user-id bits): w, and gang slot wib
        // bit j = seed-tree level gs + j = gang variable fv0 - 1 - j (plan.h hv_id)
        uint32_t x = (uint32_t)w;
        for (int j = 0; j < g; ++j) x |= ((uint32_t)(wib >> j) & 1u) << (fv0 - 1 - j);
        L.Xw = x;
    }
    const int nsteps = P.nsteps;
    const uint4* const wsteps = P.wsteps;
    unsigned long long t_start = 0, n_items = 0;
    if (P.trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    __syncthreads();

    for (;;) {
        if (tid == 0) s_item = atomicAdd(P.counter, 1u);
        __syncthreads();
        const int item = P.item_begin + (int)s_item;
        __syncthreads();
        if (item >= P.item_end) break;
        ++n_items;
        // split items (back slots beyond the 16 of a 4-entry TMEM lane): the entry
        // 0x80000000 | a of the item list is a second pass over item a's back slots 16..
        const uint32_t pk = P.packs[item];
        const bool passB = (pk >> 31) != 0;
        const int aitem = passB ? (int)(pk & 0x7fffffffu) : item;
        const uint32_t pack = passB ? P.packs[aitem] : pk;    // the gang's tree levels (gang bits 0)
        uint32_t Ft = 0;                        // tree variables in F (user ids)
        int nBt = 0;
        for (int l = 0; l < gs; ++l) {
            if ((pack >> l) & 1u) Ft |= 1u << hv_of(l, m, gs, fv0);
            else ++nBt;
        }
        // back slots [warp vars | gang vars | tree back set]: the same list in every warp of
        // the gang (a warp or gang variable in a worker's F keeps its slot, absent), so the
        // gang's warps run identical steps and store each child's 256 B region together
        const int NB = fv0 + nBt;
        const int Sw = k + NB;                  // walk slots: free, back

        // ---- a5: this warp's seeds (seed kernel): worker-major blocks [w][row l][slot] of
        //      16 B E pairs; the free slots go to shared memory [l][f][w] (cp.async), the
        //      back slots to TMEM (walk_item)
        const unsigned char* src = P.seeds + ((size_t)(aitem - P.item_begin) * G + wib) * (size_t)(k * SA * kW * 16);
        {
            const unsigned dst = L.sbase - w * 16;
            const int kk = k * k;
            for (int ww = 0; ww < nw; ++ww)
                for (int ls = lane; ls < kk; ls += 32) {
                    const int l = ls / k, f = ls - l * k;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + ((l * k + f) * kW + ww) * 16),
                                 "l"(src + ((size_t)(ww * k + l) * Sw + f) * 16));
                }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // slot -> variable: [free 0..k-1 | warp vars 0..p-1 | gang vars | tree back set ascending id]
        int slotvar = -1;
        if (lane < Sw) {
            const int s = lane;
            if (s < k) slotvar = fv0 + s;
            else if (s < k + fv0) slotvar = s - k;
            else {
                int c = s - k - fv0;
                for (int l = gs - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u)) {
                        if (c == 0) { slotvar = hv_of(l, m, gs, fv0); break; }
                        --c;
                    }
            }
        }
        // per-slot records: the warp's running best of the slot's child (from the warp's
        // best so far: only families that beat it take the update path), the table index
        // of (child v, F without the warp, gang and free variables) and lm
        if (lane < Sw) {
            const int v = slotvar;
            const uint32_t lm = (1u << v) - 1u;
            const uint32_t off = P.world1 ? block_offset<true>(P, Ft, Ft >> 1, lm)
                                          : block_offset<false>(P, Ft, Ft >> 1, lm);
            const uint32_t idx = (uint32_t)((long long)v << shb) + off;
            unsigned char* r = recb + lane * 16;
            // candidate threshold: this warp's best so far, floored by the best any warp has
            // found (a family's BIC: <= the child's maximum, so the argmax stays exact, G14)
            const double gb = P.gbest ? bic_unord(((volatile long long*)P.gbest)[v]) : wbb[v];
            *(double*)r = fmin(fmax(wbb[v], gb), P.tiny_bic);
            bbv[lane] = wbb[v];
            *(uint32_t*)(r + 8) = idx;
            *(uint32_t*)(r + 12) = lm;
            bm[lane] = wbm[v];
        }
        L.Fw = Ft | L.Xw;                       // the worker's F: tree, gang and warp variables
        L.KCw = KC + __popc(L.Fw);
        L.fh0 = (h - NB) & 3;
        // pass A: back slots 0..min(NB, 16)-1 and the free entries; pass B (split items):
        // back slots 16..NB-1 only (the free entries are rotated, not harvested)
        const int b0 = passB ? 16 : 0;
        const int nbp = passB ? NB - 16 : (JBMAX <= 4 ? min(NB, 16) : NB);
        L.hfree = passB ? 0 : 1;
        L.recB = L.recb + (unsigned)(k + b0 + h) * 16u;
        {
            // back entry j = slot k + b0 + 4j + h: exists for b < b0 + nbp; absent for this
            // worker when it is warp or gang variable b (b < fv0) in F
            uint32_t bv = 0;
            for (int j = 0; j < 8; ++j) {
                const int b = b0 + 4 * j + h;
                if (L.live && b < b0 + nbp && !(b < fv0 && ((L.Xw >> b) & 1u))) bv |= 1u << j;
            }
            L.bval = bv;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();

        const int JB = (nbp + 3) >> 2;
        switch (JB) {
            case 0: walk_item<0, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps); break;
            case 1: walk_item<1, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps); break;
            case 2: walk_item<2, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps); break;
            case 3: walk_item<3, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps); break;
            default:
                if constexpr (JBMAX <= 4) {
                    walk_item<4, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps);
                } else {
                    if (JB == 4) walk_item<4, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps);
                    else if (JB == 5) walk_item<5, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps);
                    else if (JB == 6) walk_item<6, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps);
                    else walk_item<7, HR, HB, HP>(L, P, src, k, Sw, NB, b0, wsteps, nsteps);
                }
                break;
        }
        __syncwarp();
        // the per-slot records are the warp's per-child bests (a11)
        if (lane < Sw) {
            wbb[slotvar] = bbv[lane];
            wbm[slotvar] = bm[lane];
        }
        __syncwarp();
    }
    __syncwarp();
    if (P.trace && tid == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        P.trace[3 * blockIdx.x] = t_start;
        P.trace[3 * blockIdx.x + 1] = t_end;
        P.trace[3 * blockIdx.x + 2] = n_items;
    }
    if (lane < m) {
        const size_t row = (size_t)P.part_base + (size_t)blockIdx.x * G + wib;
        P.part_bic[row * m + lane] = wbb[lane];
        P.part_mask[row * m + lane] = wbm[lane];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (wib == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "r"(P.tm_cols));
}

// Dynamic shared memory of a launch: the layout, padded so that no more CTAs
// share an SM than its 512 TMEM columns hold (a CTA beyond that would wait in
// tcgen05.alloc).
static inline size_t walk_launch_smem(const TravParams& P)
{
    size_t smem = walk_cta_smem_h(P.m, P.k, P.S_alloc, P.g, P.lw);
    const int occ_tm = 512 / P.tm_cols;
    const size_t cap = (size_t)233472 / (size_t)(occ_tm + 1);   // 228 KB per SM / (occ + 1)
    if (smem + 1024 <= cap) smem = cap - 1024 + 16;
    return smem;
}

template <bool HR, bool HB, bool HP, int JBMAX>
static inline cudaError_t launch_w(const TravParams& P, int grid, cudaStream_t st)
{
    const size_t smem = walk_launch_smem(P);
    auto f = walk_kernel<HR, HB, HP, JBMAX>;
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    f<<<grid, 32 << P.g, smem, st>>>(P);
    return cudaGetLastError();
}

}  // namespace bnr
