// walk7_kernel.cu -- the hot kernel of the bnreg path, with
// 32 lockstep workers per warp, one lane each.
//
// What it computes (as walk_kernel.cuh): Alg.2 workers each walk
// d + Upsilon(k) (Alg.1 with Eq.10's +1) from their seed
// R, one GRC per step (Eq.3-4 with reading G1); every step exposes
// one new prefix set, whose families (child = each column after the prefix) get
// RSS = the column's tail sum of squares (Eq.5, reading G3, kept
// as suffix sums by addition only), the BIC (a9, reading G5), one 16 B (RSS, BIC)
// record store (a10) and the per-child running best (a11, G14).
//
// B200 mapping:
//   * lane w = worker w: the 32 workers of a warp differ in the 5 lowest user ids
//     (the "warp variables"), so for every (child, step) the warp's 32 records are
//     adjacent in the table: ONE STG.128 instruction writes a whole 512 B region
//     (no gang of warps, no barriers: the 4 warps of an SM are independent);
//   * all workers of a warp follow the same step records: control flow and every
//     slot index are warp-uniform (records broadcast from shared memory);
//   * walk state E(l, slot) = (R_l, U_{l+1}) of the k free rows l of a column,
//     U_l = sum_{r >= l} R_r^2 (+ the rows below the free block).  Back slots
//     (statically placed) live in TENSOR MEMORY, the lane's own TMEM lane: 512
//     columns = TB back slots x k rows x 4 words, in chunks of 4 slots; a chunk row
//     l is 16 columns [R_l of the 4 slots | U_{l+1} of the 4 slots], so rows i, i+1
//     are one 32-column range [R_i | U_{i+1} | R_{i+1} | U_{i+2}]; the
//     free slots (their list position moves every step) and the rare overflow
//     back slots (items with more than TB back slots) live in shared memory,
//     worker-interleaved (a row of one slot = 32 x 16 B = 512 B).
//   * one CTA of 4 warps per SM (one warp per TMEM lane quarter and per SM
//     sub-partition): the latency of a step is hidden by the ~20 independent
//     entries every lane processes, not by more warps.
#include <cstdint>
#include <cmath>
#include <algorithm>
#include "kernels.h"
#include "device.cuh"
#include "tmem.cuh"

namespace bnr {

#ifndef BNREG_PAIRS
#define BNREG_PAIRS 1            // back chunks two per harvest (A/B: 0 = one)
#endif
constexpr int kW7 = 32;          // lockstep workers per warp
constexpr int kCS7 = kW7 * 16;   // bytes between slots of a shared-memory row

// ---------------------------------------------------------------- shared memory layout
// Per CTA: [log table 16 kLnEntries][K(s) 33 doubles][step table nsteps x 16 B], then per warp:
//   state   k * KA * 512 B   E(l, slot, w) at ((l * KA + slot) * 32 + w) * 16 (slots: k free, then
//                            the overflow back slots)
//   rec     NS * 16 B        per slot (shared by the warp's workers): the candidate threshold
//                            min(running best BIC of the slot's child, tiny_bic), the table
//                            index of (child, F without the warp and free variables), lm = 2^v - 1
//   bb      NS * 8 B         the running best BIC of the slot's child
//   bm      NS * 4 B         the mask of that running best
//   wbb/wbm 32 * 12 B        the warp's running best per child (kept across items)
struct W7Layout {
    int state, rec, bb, bm, wbb, wbm, per_warp;
};

__host__ __device__ inline int al16_7(int x) { return (x + 15) & ~15; }

__host__ __device__ inline W7Layout w7_layout(int k, int KA, int NS)
{
    W7Layout L;
    int o = 0;
    L.state = o;
    o += k * KA * kCS7;
    L.rec = o;
    L.bb = o + NS * 16;
    L.bm = o + NS * 24;
    o += al16_7(NS * 28);
    L.wbb = o;
    o += 32 * 8;
    L.wbm = o;
    o += 32 * 4;
    L.per_warp = al16_7(o);
    return L;
}

__host__ __device__ inline int w7_head(int nsteps) { return 16 * kLnEntries + 272 + al16_7((nsteps + 1) * 16); }

// Per-lane constants of the current item.
struct L7 {
    unsigned sbase;   // shared address of this worker's free state (row 0, slot 0)
    unsigned recb;    // shared address of rec[slot 0]
    unsigned bmb;     // shared address of bm[slot 0]
    unsigned bbb;     // shared address of bb[slot 0]
    double tiny_bic;  // a lower bound of the BIC of any RSS <= 1e-300 (G13)
    uint32_t tb;      // TMEM address of (this warp's lane quarter, column 0)
    uint32_t bval;    // bit b: back slot b holds a family of this worker
    uint32_t Xw;      // the worker's warp variables in F (user-id bits) = its lane bits
    uint32_t Fw;      // the worker's F (user ids)
    int live;         // lane < 2^p
    int RS;           // bytes between free rows l and l+1 (KA * 512)
    int k;            // free variables
    int fv0;          // user id of free slot 0 (= p)
    int NBT;          // this item's back slots in TMEM
    int NSO;          // this item's overflow back slots (shared memory slots k ..)
    double mhalf_n;
    const double* KCw;   // K(|S|) = KCw[i + 1] (K shifted by the worker's d)
    unsigned lnt;        // shared address of the log table
    double* out_rss;
    double* out_bic;
    double* out_pairs;
    unsigned* k8;        // BNREG_K8: write counters (+ the violation counter k8[k8_n])
    unsigned long long k8_n;
    unsigned sb0;        // BNREG_K8 bounds checks: the warp's shared state [sb0, sb0 + sbytes)
    unsigned sbytes;
    unsigned tmcols;     // and the TMEM columns it may address
};

// Harvest of NE entries (a9-a11): ln RSS, BIC, the record / table stores and the
// running-best candidates; new bests (rare) are resolved warp-serially (G14).
template <int NE, bool HT, bool HP>
__device__ __forceinline__ void harvest7(const L7& L, const double* rs, const unsigned* ra, const bool* okv, double Kw,
                                         uint32_t X, uint32_t S)
{
    const double PINF = __longlong_as_double(0x7ff0000000000000LL);
    const uint32_t X1 = X >> 1;
    uint32_t upd = 0;
    double bics[NE > 0 ? NE : 1];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const double rss = rs[e];
        const double lnr = fast_ln9s(rss, L.lnt);
        const double bic = fma(L.mhalf_n, lnr, Kw);
        bics[e] = bic;
        const double2 rr = lds2(ra[e]);                              // (threshold, (idx, lm)): one broadcast
        const uint32_t idx = (uint32_t)__double2loint(rr.y);        // table index of (child, F_w)
        const uint32_t lm = (uint32_t)__double2hiint(rr.y);         // (1 << child) - 1
        const uint32_t ix = idx + ((X & lm) | (X1 & ~lm));           // + compress(T | w-bits, child)
        if (HT) {
            stg_cs_if(L.out_rss + ix, rss, okv[e] && L.out_rss != nullptr);
            stg_cs_if(L.out_bic + ix, bic, okv[e] && L.out_bic != nullptr);
        }
        if (HP) stg2_cs_if(L.out_pairs + 2 * (size_t)ix, rss, bic, okv[e]);
        K8_COUNT(L, okv[e], ix);   // K8 debug builds: every entry written exactly once, in range
        upd |= (okv[e] && bic >= rr.x) ? (1u << e) : 0u;
    }
    unsigned bal = __ballot_sync(FULLMASK, upd != 0);
    while (bal) {
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
                        if (HT && L.out_bic) L.out_bic[idx + ((X & lm) | (X1 & ~lm))] = PINF;
                        if (HP) L.out_pairs[2 * (size_t)(idx + ((X & lm) | (X1 & ~lm))) + 1] = PINF;
                    }
                    double cb;
                    uint32_t cm;
                    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cb) : "r"(ba));
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cm) : "r"(ma));
                    if (tie_better(b, S, cb, cm)) {
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(ba), "d"(b) : "memory");
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ma), "r"(S) : "memory");
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(fmin(b, L.tiny_bic)) : "memory");
                    }
                }
            }
        }
        __syncwarp();
    }
}

// Seed pseudo-step j (reading G11: the seed prefixes {free 0..j-1}, i = j - 1):
// RSS = U_{i+1} = E_i.y, or U_0 = R_0^2 + E_0.y for the empty prefix; no rotation.
// Entries: the back slots (NBC TMEM chunks + the overflow slots), then the free
// list (positions j..k-1: NFC chunks of 4).
template <int NFC, bool HT, bool HP>
__device__ __forceinline__ void seed_step7(const L7& L, const uint4 q, int NBC)
{
    const uint32_t fl = q.w;
    const int nf = (int)(fl & 31u);
    const int i = (int)((fl >> 8) & 31u) - 1;
    const bool s0 = i < 0;
    const int r = s0 ? 0 : i;
    const unsigned bi = L.sbase + q.x;   // row max(i, 0)
    const uint32_t Tsh = (fl >> 17) << L.fv0;
    const double Kw = L.KCw[(fl >> 8) & 31u];
    const uint32_t X = Tsh | L.Xw, S = L.Fw | Tsh;
    tm_wait_st();
#pragma unroll 1
    for (int c = 0; c < NBC; ++c) {
        uint32_t rb[16];
        tm_ld<16>(L.tb + (uint32_t)((c * L.k + r) * 16), rb);
        tm_wait_ld<16>(rb);
        double rs[4];
        unsigned ra[4];
        bool okv[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int e = 4 * c + s;
            const double R = tm_f64(rb + 2 * s), U = tm_f64(rb + 8 + 2 * s);
            rs[s] = s0 ? fma(R, R, U) : U;
            ra[s] = L.recb + (unsigned)(L.k + e) * 16u;
            okv[s] = (L.bval >> e) & 1u;
        }
        harvest7<4, HT, HP>(L, rs, ra, okv, Kw, X, S);
    }
#pragma unroll
    for (int c = 0; c < NFC; ++c) {
        double rs[4];
        unsigned ra[4];
        bool okv[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int j = 4 * c + s;
            const unsigned sl = (q.z >> (4 * j)) & 15u;
            const double2 a = lds2(bi + sl * kCS7);
            rs[s] = s0 ? fma(a.x, a.x, a.y) : a.y;
            ra[s] = L.recb + sl * 16u;
            okv[s] = L.live && j < nf;
        }
        harvest7<4, HT, HP>(L, rs, ra, okv, Kw, X, S);
    }
    // the overflow back slots (items with more back slots than TMEM holds; rare)
    for (int o = 0; o < L.NSO; ++o) {
        const int b = L.NBT + o;
        const double2 a = lds2(bi + (unsigned)(L.k + o) * kCS7);
        double r1[1] = {s0 ? fma(a.x, a.x, a.y) : a.y};
        unsigned a1[1] = {L.recb + (unsigned)(L.k + b) * 16u};
        bool o1[1] = {((L.bval >> b) & 1u) != 0};
        harvest7<1, HT, HP>(L, r1, a1, o1, Kw, X, S);
    }
}

// rotation of one shared-memory entry at row i (E_i at a, E_{i+1} at a + RS)
__device__ __forceinline__ double rot_smem(unsigned a, int RS, double c, double sg, bool ok)
{
    const double x = lds1(a);
    const double2 y = lds2(a + RS);
    const double xa = fma(c, x, sg * y.x), ya = fma(c, y.x, -sg * x);
    const double ru = fma(ya, ya, y.y);
    sts_pair_if(a, xa, ru, ya, RS, ok);
    return ru;
}

// Rotation of NC back chunks (cc0, cc0 + 1, ..) at rows i, i+1 in TMEM: the chunk's
// 32 columns [R_i | U_{i+1} | R_{i+1} | U_{i+2}] (4 slots each) are loaded, R_i, U_{i+1}
// and R_{i+1} replaced (x16 + x8 stores); rs = the new U_{i+1} (computed a second time
// into the harvest's registers: one DFMA is cheaper than the register moves the two
// uses would otherwise cost).
template <int NC>
__device__ __forceinline__ void back_rot2(const L7& L, int i, int cc0, double c, double sg, double* rs, unsigned* ra,
                                          bool* okv)
{
    K8_CHECK(L, i >= 0 && (unsigned)(((cc0 + NC - 1) * L.k + i) * 16 + 32) <= L.tmcols);
    uint32_t ab[NC][16], cd[NC][16];
#pragma unroll
    for (int h = 0; h < NC; ++h) {
        const uint32_t ta = L.tb + (uint32_t)(((cc0 + h) * L.k + i) * 16);
        tm_ld<8>(ta, ab[h]);
        tm_ld<16>(ta + 16, cd[h]);
    }
    tm_wait_ld<8>(ab[0]);
#pragma unroll
    for (int h = 0; h < NC; ++h) {
        tm_pin<16>(cd[h]);
        if (h) tm_pin<8>(ab[h]);
    }
#pragma unroll
    for (int h = 0; h < NC; ++h) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const double x = tm_f64(ab[h] + 2 * s), y = tm_f64(cd[h] + 2 * s), u2 = tm_f64(cd[h] + 8 + 2 * s);
            const double xa = fma(c, x, sg * y), ya = fma(c, y, -sg * x);
            tm_put(ab[h] + 2 * s, xa);
            tm_put(ab[h] + 8 + 2 * s, fma(ya, ya, u2));
            tm_put(cd[h] + 2 * s, ya);
            const int e = 4 * h + s, b = 4 * (cc0 + h) + s;
            rs[e] = fma(ya, ya, u2);
            ra[e] = L.recb + (unsigned)(L.k + b) * 16u;
            okv[e] = (L.bval >> b) & 1u;
        }
        const uint32_t ta = L.tb + (uint32_t)(((cc0 + h) * L.k + i) * 16);
        tm_st<16>(ta, ab[h]);
        tm_st<8>(ta + 16, cd[h]);
    }
}

// One lockstep GRC step (a7-a11): rotation of rows i, i+1 of every entry's column
// with this step's (c, s) and the new suffix sum U_{i+1} = U_{i+2} + R'_{i+1}^2, then
// the entry's harvest.  Order: the free entries (shared memory) and the pivot Y (now
// at position i: E_i = (h, 0), R_{i+1} = 0) first, so that the next step's rotation
// (from its pivot column, a free slot) can start; then the back chunks (TMEM, the
// next chunk's load in flight while a chunk is harvested), the free entries' harvest
// and the overflow back slots.
template <int NFC, bool HT, bool HP>
__device__ __forceinline__ void grc_step7(const L7& L, const uint4 q, double& c, double& sg, double& hh, int NBC)
{
    const uint32_t fl = q.w;
    const int nf = (int)(fl & 31u);
    const int i = (int)((fl >> 8) & 31u) - 1;
    const unsigned bi = L.sbase + q.x;
    const int RS = L.RS;
    const uint32_t Tsh = (fl >> 17) << L.fv0;
    const uint32_t X = Tsh | L.Xw, S = L.Fw | Tsh;
    // free entries: rotate and store now, harvest later
    double rf[4 * NFC];
#pragma unroll
    for (int j = 0; j < 4 * NFC; ++j) {
        const unsigned fa = bi + ((q.z >> (4 * j)) & 15u) * kCS7;
        K8_CHECK(L, j >= nf || (fa + RS + 16 - L.sb0 <= L.sbytes && fa >= L.sb0));
        const double x = lds1(fa);
        const double2 y = lds2(fa + RS);
        const double xa = fma(c, x, sg * y.x), ya = fma(c, y.x, -sg * x);
        rf[j] = fma(ya, ya, y.y);
        sts_pair_if(fa, xa, rf[j], ya, RS, j < nf);
    }
    // the pivot Y
    sts_pair_if(bi + ((fl >> 13) & 15u) * kCS7, hh, 0.0, 0.0, RS, true);
    // the next step's rotation (without a next GRC the table points at a valid slot and the
    // result is unused)
    double cn, sn, hn;
    {
        const unsigned ncol = L.sbase + q.y;
        const double a = lds1(ncol), b = lds1(ncol + RS);
        givens_fr(a, b, cn, sn, hn);
    }
    const double Kw = L.KCw[(fl >> 8) & 31u];
    tm_wait_st();
    // back chunks, two per iteration (8 independent entries per harvest)
#pragma unroll 1
    for (int cc = 0; cc + 1 < NBC && BNREG_PAIRS; cc += 2) {
        double rs[8];
        unsigned ra[8];
        bool okv[8];
        back_rot2<2>(L, i, cc, c, sg, rs, ra, okv);
        harvest7<8, HT, HP>(L, rs, ra, okv, Kw, X, S);
    }
    for (int cc = BNREG_PAIRS ? (NBC & ~1) : 0; cc < NBC; ++cc) {
        double rs[4];
        unsigned ra[4];
        bool okv[4];
        back_rot2<1>(L, i, cc, c, sg, rs, ra, okv);
        harvest7<4, HT, HP>(L, rs, ra, okv, Kw, X, S);
    }
#pragma unroll
    for (int cc = 0; cc < NFC; ++cc) {
        double rs[4];
        unsigned ra[4];
        bool okv[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int j = 4 * cc + s;
            rs[s] = rf[j];
            ra[s] = L.recb + ((q.z >> (4 * j)) & 15u) * 16u;
            okv[s] = L.live && j < nf;
        }
        harvest7<4, HT, HP>(L, rs, ra, okv, Kw, X, S);
    }
    // the overflow back slots (rare: items with more back slots than TMEM holds)
    for (int o = 0; o < L.NSO; ++o) {
        const int b = L.NBT + o;
        double r1[1] = {rot_smem(bi + (unsigned)(L.k + o) * kCS7, RS, c, sg, true)};
        unsigned a1[1] = {L.recb + (unsigned)(L.k + b) * 16u};
        bool o1[1] = {((L.bval >> b) & 1u) != 0};
        harvest7<1, HT, HP>(L, r1, a1, o1, Kw, X, S);
    }
    c = cn;
    sg = sn;
    hh = hn;
}

// Seed block of an item (seed7 layout, doubles): R(s, l, w) at (s k + l) 32 + w for the
// walk slots s < k + NB (s < k free, s = k + b back slot b), the tail sum of squares of
// back slot b at (k + nbmax) k 32 + b 32 + w.  Fill this worker's walk state:
// E(l) = (R_l, U_{l+1}), U_k = tail (0 for free columns), U_l = U_{l+1} + R_l^2.
__device__ __forceinline__ void load_seed7(const L7& L, const double* __restrict__ blk, int nbmax, int lane, int NBC)
{
    const int k = L.k;
    const double* tails = blk + (size_t)(k + nbmax) * k * kW7;
    // free slots and overflow back slots -> shared memory, two slots at a time
    const int nsm = k + L.NSO;
    for (int s0 = 0; s0 < nsm; s0 += 2) {
        double R[2][kMaxFreeWalk7];
        double U[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int ss = s0 + s;
            const int ws = ss < k ? ss : k + L.NBT + (ss - k);     // walk slot
            U[s] = 0.0;
            if (ss < nsm) {
                if (ss >= k) U[s] = __ldg(tails + (size_t)(ws - k) * kW7 + lane);
#pragma unroll
                for (int l = 0; l < kMaxFreeWalk7; ++l)
                    if (l < k) R[s][l] = __ldg(blk + ((size_t)ws * k + l) * kW7 + lane);
            }
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int ss = s0 + s;
            if (ss < nsm) {
#pragma unroll
                for (int l = kMaxFreeWalk7 - 1; l >= 0; --l)
                    if (l < k) {
                        const unsigned a = L.sbase + (unsigned)(l * L.RS + ss * kCS7);
                        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(R[s][l]), "d"(U[s]) : "memory");
                        U[s] = fma(R[s][l], R[s][l], U[s]);
                    }
            }
        }
    }
    // TMEM back slots: chunk c holds back slots 4c..4c+3, row l at columns (c k + l) 16:
    // [R_l of the 4 slots | U_{l+1} of the 4 slots]; two slots at a time
#pragma unroll 1
    for (int pr = 0; pr < 2 * NBC; ++pr) {
        const int c = pr >> 1, h2 = pr & 1;
        double R[2][kMaxFreeWalk7];
        double U[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int b = 2 * pr + s;
            U[s] = 0.0;
#pragma unroll
            for (int l = 0; l < kMaxFreeWalk7; ++l) R[s][l] = 0.0;
            if (b < L.NBT) {
                U[s] = __ldg(tails + (size_t)b * kW7 + lane);
#pragma unroll
                for (int l = 0; l < kMaxFreeWalk7; ++l)
                    if (l < k) R[s][l] = __ldg(blk + ((size_t)(k + b) * k + l) * kW7 + lane);
            }
        }
        // rows from the bottom
#pragma unroll
        for (int l = kMaxFreeWalk7 - 1; l >= 0; --l)
            if (l < k) {
                uint32_t vr[4], vu[4];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    tm_put(vr + 2 * s, R[s][l]);
                    tm_put(vu + 2 * s, U[s]);
                    U[s] = fma(R[s][l], R[s][l], U[s]);
                }
                tm_st<4>(L.tb + (uint32_t)((c * k + l) * 16 + 4 * h2), vr);
                tm_st<4>(L.tb + (uint32_t)((c * k + l) * 16 + 8 + 4 * h2), vu);
            }
    }
}

// One item (a pack of 32 workers) with NBC TMEM back chunks.
template <bool HT, bool HP>
__device__ __forceinline__ void walk_item7(L7& L, const double* blk, int nbmax, const uint4* stab, int nsteps, int lane,
                                        int NBC)
{
    load_seed7(L, blk, nbmax, lane, NBC);
    // a6-a11: the k + 1 seed pseudo-steps, then d + Upsilon(k), in lockstep
    const int k = L.k;
    uint4 q = stab[0];
    for (int t = 0; t <= k; ++t) {
        const uint4 qn = stab[t + 1];              // prefetch (the table is padded by one record)
        const int nfe = ((int)(q.w & 31u) + 3) >> 2;
        if (nfe == 0) seed_step7<0, HT, HP>(L, q, NBC);
        else if (nfe == 1) seed_step7<1, HT, HP>(L, q, NBC);
        else seed_step7<2, HT, HP>(L, q, NBC);
        if (t == k) break;
        q = qn;
    }
    double c, sg, hh;
    {
        // the first GRC's rotation (the last seed record points at its pivot column)
        double a = 0.0, b = 1.0;
        if ((q.w >> 7) & 1u) {
            a = lds1(L.sbase + q.y);
            b = lds1(L.sbase + q.y + L.RS);
        }
        givens_fr(a, b, c, sg, hh);
    }
    q = stab[k + 1];
    for (int t = k + 1; t < nsteps; ++t) {
        const uint4 qn = stab[t + 1];
        if ((q.w & 31u) > 4u) grc_step7<2, HT, HP>(L, q, c, sg, hh, NBC);
        else grc_step7<1, HT, HP>(L, q, c, sg, hh, NBC);
        q = qn;
    }
    tm_wait_st();
}

template <bool HT, bool HP>
__global__ void __launch_bounds__(128, 1) walk7_kernel(const __grid_constant__ TravParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_taddr;
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5, nwarps = blockDim.x >> 5;
    const int nsteps = P.nsteps;
    double2* const lntab = (double2*)smem;
    double* const KC = (double*)(smem + 16 * kLnEntries);
    uint4* const stab = (uint4*)(smem + 16 * kLnEntries + 272);
    for (int j = tid; j < kLnEntries; j += blockDim.x) lntab[j] = P.lntab9[j];
    for (int j = tid; j < 33; j += blockDim.x) KC[j] = P.Kc[j];
    for (int j = tid; j <= nsteps; j += blockDim.x) stab[j] = j < nsteps ? P.wsteps[j] : make_uint4(0, 0, 0, 0);
    if (wib == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&s_taddr)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int m = P.m, k = P.k, p = P.p, gs = P.bh;   // no gang variables: every tree level is an item level
    const int fv0 = p;
    const int NS = k + P.nbmax;
    const W7Layout Ly = w7_layout(k, P.KA, NS);
    unsigned char* const wb = smem + w7_head(nsteps) + wib * Ly.per_warp;
    unsigned char* const recb = wb + Ly.rec;
    uint32_t* const bm = (uint32_t*)(wb + Ly.bm);
    double* const bbv = (double*)(wb + Ly.bb);
    double* const wbb = (double*)(wb + Ly.wbb);
    uint32_t* const wbm = (uint32_t*)(wb + Ly.wbm);
    const double NINF = -__longlong_as_double(0x7ff0000000000000LL);
    wbb[lane] = NINF;
    wbm[lane] = 0xffffffffu;
    const int shb = P.world1 ? m - 1 : m - P.r;   // child block = v << shb entries
    L7 L;
    L.sbase = (unsigned)__cvta_generic_to_shared(wb + Ly.state) + lane * 16;
    L.recb = (unsigned)__cvta_generic_to_shared(recb);
    L.bmb = (unsigned)__cvta_generic_to_shared(bm);
    L.bbb = (unsigned)__cvta_generic_to_shared(bbv);
    L.tiny_bic = P.tiny_bic;
    L.tb = s_taddr + ((uint32_t)((wib & 3) * 32) << 16);
    L.live = lane < P.nw;
    L.Xw = L.live ? (uint32_t)lane : 0u;
    L.RS = P.KA * kCS7;
    L.k = k;
    L.fv0 = fv0;
    L.mhalf_n = P.mhalf_n;
    L.lnt = (unsigned)__cvta_generic_to_shared(lntab);
    L.out_rss = P.out_rss;
    L.out_bic = P.out_bic;
    L.out_pairs = P.out_pairs;
    L.k8 = P.k8;
    L.k8_n = P.k8_n;
    L.sb0 = (unsigned)__cvta_generic_to_shared(wb + Ly.state);
    L.sbytes = (unsigned)(k * P.KA * kCS7);
    L.tmcols = 512u;
    K8_CHECK(L, !(P.k8_selftest && (threadIdx.x & 31) == 0));   // (a negative control of the counter path)
    const uint4* const st = stab;
    __syncwarp();

    for (;;) {
        uint32_t it = 0;
        if (lane == 0) it = atomicAdd(P.counter, 1u);
        it = __shfl_sync(FULLMASK, it, 0);
        const int item = P.item_begin + (int)it;
        if (item >= P.item_end) break;
        const uint32_t pack = P.packs[item];    // the item's tree levels
        uint32_t Ft = 0;                        // tree variables in F (user ids)
        int nBt = 0;
        for (int l = 0; l < gs; ++l) {
            if ((pack >> l) & 1u) Ft |= 1u << hv_of(l, m, gs, fv0);
            else ++nBt;
        }
        const int NB = p + nBt;                 // back slots [warp vars | tree back set ascending id]
        const int Sw = k + NB;                  // walk slots: free, back
        // slot -> variable
        int slotvar = -1;
        if (lane < Sw) {
            const int s = lane;
            if (s < k) slotvar = fv0 + s;
            else if (s < k + p) slotvar = s - k;
            else {
                int cq = s - k - p;
                for (int l = gs - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u)) {
                        if (cq == 0) { slotvar = hv_of(l, m, gs, fv0); break; }
                        --cq;
                    }
            }
        }
        // per-slot records (the warp's running best of the slot's child, the table index of
        // (child v, F without the warp and free variables), lm)
        if (lane < Sw) {
            const int v = slotvar;
            const uint32_t lm = (1u << v) - 1u;
            const uint32_t off = P.world1 ? block_offset<true>(P, Ft, Ft >> 1, lm)
                                          : block_offset<false>(P, Ft, Ft >> 1, lm);
            const uint32_t idx = (uint32_t)((long long)v << shb) + off;
            unsigned char* r = recb + lane * 16;
            *(double*)r = fmin(wbb[v], P.tiny_bic);
            bbv[lane] = wbb[v];
            *(uint32_t*)(r + 8) = idx;
            *(uint32_t*)(r + 12) = lm;
            bm[lane] = wbm[v];
        }
        L.Fw = Ft | L.Xw;
        L.KCw = KC + __popc(L.Fw);
        L.NBT = min(NB, P.TB);
        L.NSO = NB - L.NBT;
        {
            // back slot b holds a family of this worker unless it is a warp variable in F
            uint32_t bv = 0;
            for (int b = 0; b < NB; ++b)
                if (L.live && !(b < p && ((L.Xw >> b) & 1u))) bv |= 1u << b;
            L.bval = bv;
        }
        __syncwarp();
        const double* blk = (const double*)P.seeds + (size_t)(item - P.item_begin) * P.sblk;
        walk_item7<HT, HP>(L, blk, P.nbmax, st, nsteps, lane, (L.NBT + 3) >> 2);
        __syncwarp();
        // the per-slot records are the warp's per-child bests (a11)
        if (lane < Sw) {
            wbb[slotvar] = bbv[lane];
            wbm[slotvar] = bm[lane];
        }
        __syncwarp();
    }
    __syncwarp();
    if (lane < m) {
        const size_t row = (size_t)P.part_base + (size_t)blockIdx.x * nwarps + wib;
        P.part_bic[row * m + lane] = wbb[lane];
        P.part_mask[row * m + lane] = wbm[lane];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (wib == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "r"(512));
}

template <bool HT, bool HP>
static cudaError_t launch_w7(const TravParams& P, int grid, int warps, cudaStream_t st)
{
    const size_t smem = (size_t)w7_head(P.nsteps) + (size_t)warps * w7_layout(P.k, P.KA, P.k + P.nbmax).per_warp;
    auto f = walk7_kernel<HT, HP>;
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    f<<<grid, 32 * warps, smem, st>>>(P);
    return cudaGetLastError();
}

#ifdef BNREG_WALK7_TABLES
// the separate-table layouts (bnreg_run, bnreg_all_rss, bnreg_bic): each table written if non-null
cudaError_t launch_walk7_tables(const TravParams& P, int grid, int warps, cudaStream_t st)
{
    return launch_w7<true, false>(P, grid, warps, st);
}
#else
cudaError_t launch_walk7_tables(const TravParams& P, int grid, int warps, cudaStream_t st);   // walk7_tables.cu

size_t walk7_cta_smem(int k, int KA, int nslots, int warps)
{
    // (the step table is at most 2^8 - 8 - 1 + 9 = 256 records at k = 8, + one pad record)
    return (size_t)w7_head(1 << kMaxFreeWalk7) + (size_t)warps * (size_t)w7_layout(k, KA, nslots).per_warp;
}

cudaError_t launch_walk7(const TravParams& P, int grid, int warps, cudaStream_t st)
{
    if (P.k > kMaxFreeWalk7 || P.TB > 20 || P.KA - P.k > 4 || warps < 1 || warps > 4) return cudaErrorInvalidValue;
    if (P.out_pairs) return launch_w7<false, true>(P, grid, warps, st);
    return launch_walk7_tables(P, grid, warps, st);
}
#endif

}  // namespace bnr
