// walk_kernel.cu -- the hot kernel of the bnreg path:
// Alg.2 workers each walk d + Upsilon(k) (Alg.1 with Eq.10's
// +1) from their seed R, one GRC per step
// (Eq.3-4 with reading G1), harvesting every new family from
// suffix sums of squares (Eq.5, reading G3), computing its
// BIC (a9, reading G5), storing RSS and BIC into the (child, mask)-indexed
// table (a10) and keeping a per-child running best (a11, G14).
//
// B200 mapping:
//   * a warp runs W = 8 workers in lockstep; lane = (worker w = lane % W,
//     part h = lane / W).  All workers of a warp follow the same step records,
//     so control flow is uniform; part h takes list entries h, h+4, h+8, ...
//   * the W workers differ in the W lowest user ids (the "warp variables"), the
//     CTA's 4 warps in the next 2 ids (the "gang variables"): for every child
//     and step a CTA writes 32 adjacent entries = 256 B of each table at the same
//     time (DRAM write combining needs that: profiles/r01_storebench.txt)
//   * walk state in shared memory, E(l, slot, w) = (R_l, U_{l+1}) of free row l
//     of the slot's column, U_l = sum_{r >= l} R_r^2 (+ the rows below the free
//     block), worker-interleaved so that every LDS/STS.128 phase reads 128
//     contiguous bytes; suffix sums are updated by addition only
//   * seeds: the gang's node at tree depth L1 (global memory, tree_level_kernel)
//     -> the remaining tree levels in-warp -> the W workers' seeds along a Gray
//     path over the warp variables (each flip moves one variable across the free
//     block: k + j GRCs), each seed converted into its worker's walk state.
#include <cstdint>
#include <cmath>
#include <algorithm>
#include "kernels.h"
#include "device.cuh"

namespace bnr {

// ---------------------------------------------------------------- shared memory layout
// Per CTA: [log table 512 x 16 B][K(s) 33 doubles] then per warp:
//   state   k * SA * W * 16 B   E(l, slot, w) at ((l*SA + slot)*W + w)*16
//   rec     SA * 16 B           per slot (shared by the warp's workers): the warp's running
//                               best BIC of the slot's child, the table index of (child,
//                               F without the warp and free variables), lm = (1 << v) - 1
//   bm      SA * 4 B            the mask of that running best
//   wbb/wbm 32 * 12 B           the warp's running best per child (kept across items)
//   slotof  32 B                variable -> slot
struct WalkLayout {
    int state, scratch, bm, wbb, wbm, slotof, per_warp;
};

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline WalkLayout walk_layout(int m, int k, int SA, int W)
{
    WalkLayout L;
    int o = 0;
    L.state = o;
    o += al16(k * SA * W * 16);
    L.scratch = o;
    L.bm = o + SA * 16;
    o += al16(SA * 20);
    L.wbb = o;
    o += 32 * 8;
    L.wbm = o;
    o += 32 * 4;
    L.slotof = o;
    o += 32;
    L.per_warp = al16(o);
    return L;
}

constexpr int kWalkHead = 8192 + 272;   // log table + K(s) table

size_t walk_cta_smem(int m, int k, int SA, int g, int lw)
{
    return (size_t)kWalkHead + ((size_t)1 << g) * (size_t)walk_layout(m, k, SA, 1 << lw).per_warp;
}

// user id of seed-tree level l (plan.h hv_id): top ids first, the gang ids last
__device__ __forceinline__ int hv_of(int l, int m, int gs, int fv0) { return l < gs ? m - 1 - l : fv0 - 1 - (l - gs); }


// Predicated stores that stay predicated (no branch around them, so the
// entries of a step remain one basic block the scheduler can interleave).
__device__ __forceinline__ void stg_cs_if(double* p, double v, bool q)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cs.f64 [%0], %1;\n\t}" ::"l"(p), "d"(v),
                 "r"((unsigned)q));
}
__device__ __forceinline__ void sts_pair_if(unsigned a, double x, double u, double y, int rs, bool q)
{
    // E_i = (x, u) at a, E_{i+1}.x = y at a + rs
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.shared.v2.f64 [%0], {%1, %2};\n\t"
                 "@q st.shared.f64 [%3], %4;\n\t}" ::"r"(a), "d"(x), "d"(u), "r"(a + rs), "d"(y), "r"((unsigned)q)
                 : "memory");
}

// Givens coefficients without the rank-deficiency guard: in the walk, b is the
// diagonal entry r_{i+1,i+1} of the pivot column, nonzero for full-rank data
// (checked at create, G26), so h2 > 0.
__device__ __forceinline__ void givens_fr(double a, double b, double& c, double& s, double& h)
{
    const double h2 = fma(a, a, b * b);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(h2));
    double e = fma(-h2, y * y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-h2, y * y, 1.0);
    y = fma(0.5 * y, e, y);
    c = a * y;
    s = b * y;
    h = h2 * y;
}

// Per-step values of a lane (entries e = h + PP j of the step's list: the free
// slots after the prefix, in position order, then the back slots).
struct StepV {
    unsigned bi;          // shared address of (row i, slot 0, worker w) of the walk state
    unsigned bb0;         // shared address of the lane's first back entry: bi + (kb + h) * CSb
    unsigned rb0;         // record address of the lane's first back entry: rec + (kb + h) * 16
    unsigned rf;          // record array base (free entries: rf + f * 16)
    int RS;               // bytes between rows i and i+1
    int nvalid;           // entries j < nvalid exist for this lane
    int nfj;              // entries j < nfj are free slots (from the nibble list)
    uint32_t nl, nh;      // the free-list nibbles shifted to this lane's first entry
    uint32_t ab0;         // absent >> (kb + h): bit PP j = back entry j's variable is in F
    uint32_t X, X1;       // free part of the prefix set | this worker's warp-variable bits, and >> 1
    double c, sg;         // this step's rotation
    double Kw;            // BIC constant of |S|
    int seed0;            // seed pseudo-step with i = -1 (RSS = U_0)
};

// Record address of a free entry from its state address (same slot index; the
// state's slot stride is W*16 bytes, the records' 16 bytes).
__device__ __forceinline__ unsigned rec_of(const StepV& v, unsigned sa) { return v.rf + ((sa - v.bi) >> 3); }

constexpr int kMaxE = 16;   // list entries per lane and step (PP * kMaxE >= 32 > m - 1)

// state address of entry j (free entries from the nibble list, back entries at fixed strides)
template <int PP, int CSB>
__device__ __forceinline__ unsigned entry_addr(const StepV& v, int j)
{
    constexpr int JF = 8 / PP;                               // free entries only for e < nf <= k - 1 <= 8
    const unsigned back = v.bb0 + j * (PP * CSB);
    if (j < JF) {
        const int sh = 4 * PP * j;                           // nibble of entry e = h + PP j
        const unsigned f = ((sh < 32 ? v.nl >> (sh & 31) : v.nh >> ((sh - 32) & 31)) & 15u);
        return j < v.nfj ? v.bi + f * CSB : back;
    }
    return back;
}

// One lockstep step of a lane over its NE = ceil(L / PP) entries:
//   phase A  the GRC's rotation of rows i, i+1 of every entry's column and the
//            new suffix sum U_{i+1} = U_{i+2} + R'_{i+1}^2 (a7, a8), or the seed
//            pseudo-step's read of U_{i+1};
//   pivot    Y (now at position i): E_i = (h, 0), R_{i+1} = 0;
//   givens   the next step's rotation from its pivot column (overlaps phase C);
//   phase C  ln RSS, BIC (a9), the two table stores (a10), running-best
//            candidates; new bests (rare) resolved at the end (a11, G14).
template <bool SEED, int NE, int PP, int CSB, bool HR, bool HB>
__device__ __forceinline__ void walk_step(const StepV& v, const double2* lntab, double mhalf_n, double* out_rss,
                                          double* out_bic, bool pivot, unsigned pcol, double hh, bool has_next,
                                          unsigned ncol, double& cn, double& sn, double& hn, uint32_t S,
                                          unsigned rec_sh, unsigned bm_sh)
{
    constexpr int NA = NE > 0 ? NE : 1;                       // (NE = 0: an empty list, e.g. the last seed step)
    double rs[NA];
    unsigned ad[NA];
    {
        double2 a0[NA], a1[NA];
#pragma unroll
        for (int j = 0; j < NE; ++j) {
            ad[j] = entry_addr<PP, CSB>(v, j);
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a0[j].x), "=d"(a0[j].y) : "r"(ad[j]));
            if (!SEED)
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a1[j].x), "=d"(a1[j].y) : "r"(ad[j] + v.RS));
        }
#pragma unroll
        for (int j = 0; j < NE; ++j) {
            if (SEED) {
                rs[j] = v.seed0 ? fma(a0[j].x, a0[j].x, a0[j].y) : a0[j].y;   // U_0 or U_{i+1}
            } else {
                const double xa = fma(v.c, a0[j].x, v.sg * a1[j].x), ya = fma(v.c, a1[j].x, -v.sg * a0[j].x);
                const double ra = fma(ya, ya, a1[j].y);
                rs[j] = ra;
                sts_pair_if(ad[j], xa, ra, ya, v.RS, j < v.nvalid);
            }
        }
    }
    if (!SEED && pivot) sts_pair_if(pcol, hh, 0.0, 0.0, v.RS, true);
    __syncwarp();
    {
        // unconditional (no branch: the chain interleaves with phase C); without a next
        // GRC the table points at a valid slot and the result is unused
        double a, b;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a) : "r"(ncol));
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b) : "r"(ncol + v.RS));
        if (!has_next) {
            a = 0.0;
            b = 1.0;
        }
        givens_fr(a, b, cn, sn, hn);
    }
    const double PINF = __longlong_as_double(0x7ff0000000000000LL);
    constexpr int JF = 8 / PP;
    uint32_t upd = 0;
    double bics[NA];
#pragma unroll
    for (int j = 0; j < NE; ++j) {
        const double rss = rs[j];
        const double lnr = fast_ln9(rss, lntab);
        const double bic = fma(mhalf_n, lnr, v.Kw);
        const bool tiny = rss <= 1e-300;                             // G13: BIC = +inf, fixed on the rare path
        bics[j] = bic;
        const unsigned ra = (j < JF) ? rec_of(v, ad[j]) : v.rb0 + j * (PP * 16);
        double bb, rr;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(bb), "=d"(rr) : "r"(ra));
        const uint32_t idx = (uint32_t)__double2loint(rr);          // table index of (child, F_w)
        const uint32_t lm = (uint32_t)__double2hiint(rr);           // (1 << child) - 1
        const uint32_t ix = idx + ((v.X & lm) | (v.X1 & ~lm));       // + compress(T | w-bits, child)
        bool ok = j < v.nvalid;
        if (j < JF) ok = ok && (j < v.nfj || !((v.ab0 >> (PP * j)) & 1u));
        else ok = ok && !((v.ab0 >> (PP * j)) & 1u);
        if (HR) stg_cs_if(out_rss + ix, rss, ok);
        if (HB) stg_cs_if(out_bic + ix, bic, ok);
        upd |= (ok && (bic >= bb || tiny)) ? (1u << j) : 0u;
    }
    unsigned bal = __ballot_sync(FULLMASK, upd != 0);
    while (bal) {
        // rare: a family beats (or ties, G14) the warp's running best of its child; the
        // 8 workers share the record, so lanes with candidates take turns
        const int l = __ffs(bal) - 1;
        bal &= bal - 1;
        if ((int)(threadIdx.x & 31) == l) {
#pragma unroll
            for (int j = 0; j < NE; ++j) {
                if ((upd >> j) & 1u) {
                    const unsigned ra = (j < JF) ? rec_of(v, ad[j]) : v.rb0 + j * (PP * 16);
                    const unsigned ma = bm_sh + ((ra - rec_sh) >> 2);   // bm[slot] beside rec[slot]
                    if (rs[j] <= 1e-300) {
                        // a perfect fit (G13): BIC = +inf, stored over the finite value written above
                        bics[j] = PINF;
                        double rr;
                        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(rr) : "r"(ra + 8));
                        const uint32_t idx = (uint32_t)__double2loint(rr), lm = (uint32_t)__double2hiint(rr);
                        if (HB) out_bic[idx + ((v.X & lm) | (v.X1 & ~lm))] = PINF;
                    }
                    double cb;
                    uint32_t cm;
                    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cb) : "r"(ra));
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cm) : "r"(ma));
                    if (tie_better(bics[j], S, cb, cm)) {
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(ra), "d"(bics[j]) : "memory");
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ma), "r"(S) : "memory");
                    }
                }
            }
        }
        __syncwarp();
    }
}

// NE-dispatch of the step body (NE = entries per lane, at most 32 / PP).
template <bool SEED, int PP, int CSB, bool HR, bool HB, int NE>
__device__ __forceinline__ void step_ne(const StepV& v, const double2* lntab, double mhalf_n, double* out_rss,
                                        double* out_bic, bool pv, unsigned pcol, double hh, bool has_next,
                                        unsigned ncol, double& cn, double& sn, double& hn, uint32_t S,
                                        unsigned rec_sh, unsigned bm_sh)
{
    if constexpr (NE * PP <= 32)
        walk_step<SEED, NE, PP, CSB, HR, HB>(v, lntab, mhalf_n, out_rss, out_bic, pv, pcol, hh, has_next, ncol, cn, sn,
                                             hn, S, rec_sh, bm_sh);
}

template <int LW, bool WORLD1, bool HR, bool HB>
__global__ void __launch_bounds__(128, 1) walk_kernel(const __grid_constant__ TravParams P)
{
    constexpr int W = 1 << LW;
    constexpr int PP = 32 / W;                  // lanes (parts) per worker
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_item;
    double2* const lntab = (double2*)smem;
    double* const KC = (double*)(smem + 8192);
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    for (int j = tid; j < 512; j += blockDim.x) lntab[j] = P.lntab9[j];
    for (int j = tid; j < 33; j += blockDim.x) KC[j] = P.Kc[j];
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g, SA = P.S_alloc;
    const int fv0 = p + g;                      // user id of free slot 0
    const int gs = bh - g;                      // gang levels are gs..bh-1
    const int G = 1 << g;
    const WalkLayout Ly = walk_layout(m, k, SA, W);
    unsigned char* const wb = smem + kWalkHead + wib * Ly.per_warp;
    unsigned char* const st = wb + Ly.state;
    unsigned char* const recb = wb + Ly.scratch;            // rec[slot], 16 B
    uint32_t* const bm = (uint32_t*)(wb + Ly.bm);           // bm[slot]
    static_assert(W == 8, "rec_of assumes a state slot stride of 8 x 16 B");
    double* const wbb = (double*)(wb + Ly.wbb);
    uint32_t* const wbm = (uint32_t*)(wb + Ly.wbm);
    const int w = lane & (W - 1), h = lane >> LW;
    const double NINF = -__longlong_as_double(0x7ff0000000000000LL);
    wbb[lane] = NINF;
    wbm[lane] = 0xffffffffu;
    const int shb = WORLD1 ? m - 1 : m - P.r;   // child block = v << shb entries
    const int RS = SA * W * 16;                 // bytes between free rows l and l+1 of a slot
    constexpr int CSb = W * 16;                 // bytes between slots (state and rec)
    const int nw = P.nw;
    double* const out_rss = P.out_rss;
    double* const out_bic = P.out_bic;
    const double mhalf_n = P.mhalf_n;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(st + w * 16);     // state of (row 0, slot 0, w)
    const unsigned rbase = (unsigned)__cvta_generic_to_shared(recb);            // rec[slot 0]
    const unsigned recb_sh = (unsigned)__cvta_generic_to_shared(recb);
    const unsigned bm_sh = (unsigned)__cvta_generic_to_shared(bm);
    const int nsteps = P.nsteps;                // kernel parameters the step loop needs, in registers
    const uint4* const wsteps = P.wsteps;
    __syncthreads();

    for (;;) {
        if (tid == 0) s_item = atomicAdd(P.counter, 1u);
        __syncthreads();
        const int item = P.item_begin + (int)s_item;
        __syncthreads();
        if (item >= P.item_end) break;
        const uint32_t pack = P.packs[item] | ((uint32_t)wib << gs);
        uint32_t Fhi = 0;                       // tree/gang variables in F (user ids)
        int nB = 0;
        for (int l = 0; l < bh; ++l) {
            if ((pack >> l) & 1u) Fhi |= 1u << hv_of(l, m, gs, fv0);
            else ++nB;
        }
        const int Sw = k + p + nB;              // walk slots of this warp: free, warp vars, back set

        // ---- a5: this warp's seeds (seed kernel): worker-major blocks [w][row l][slot] of
        //      16 B E pairs, transposed into the interleaved state [l][slot][w] (cp.async)
        {
            const unsigned char* src =
                P.seeds + ((size_t)(item - P.item_begin) * G + wib) * (size_t)(k * RS);
            const unsigned dst = sbase - w * 16;
            for (int r = 0; r < nw * k; ++r) {          // (worker, row) pairs; lane = slot
                const int ww = r / k, l = r - ww * k;
                if (lane < Sw)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + ((l * SA + lane) * W + ww) * 16),
                                 "l"(src + ((size_t)(ww * k + l) * SA + lane) * 16));
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // slot -> variable: [free 0..k-1 | warp vars 0..p-1 | back set ascending id]
        int slotvar = -1;
        if (lane < Sw) {
            const int s = lane;
            if (s < k) slotvar = fv0 + s;
            else if (s < k + p) slotvar = s - k;
            else {
                int c = s - k - p;
                for (int l = bh - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u)) {
                        if (c == 0) { slotvar = hv_of(l, m, gs, fv0); break; }
                        --c;
                    }
            }
        }
        // per-slot records: the warp's running best of the slot's child (from the warp's
        // best so far: only families that beat it take the update path), the table index
        // of (child v, F without the warp and free variables) and lm
        if (lane < Sw) {
            const int v = slotvar;
            const uint32_t lm = (1u << v) - 1u;
            const uint32_t idx = (uint32_t)((long long)v << shb) + block_offset<WORLD1>(P, Fhi, Fhi >> 1, lm);
            unsigned char* r = recb + lane * 16;
            *(double*)r = wbb[v];
            *(uint32_t*)(r + 8) = idx;
            *(uint32_t*)(r + 12) = lm;
            bm[lane] = wbm[v];
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();

        // ---- a6-a11: the walk, k+1 seed pseudo-steps then d + Upsilon(k), in lockstep
        const uint32_t Fw = Fhi | (uint32_t)w;  // warp variable j (user id j) in F iff bit j of w
        const int dw = __popc(Fw);
        const uint32_t absent = (w < nw) ? ((uint32_t)w << k) : 0xffffffffu;
        const int NB = Sw - k;
        double c = 1.0, sg = 0.0, hh = 0.0;
        const unsigned sb_h = sbase + h * CSb;              // + kbCS: the lane's first back entry
        const unsigned rb_h = rbase + h * 16;
        const uint32_t ab_h = absent >> h;
        const double* const KCw = KC + dw;                  // K(|S|) = KC[dw + i + 1]
        const int nv_h = (w < nw) ? NB + (PP - 1) - h : -64; // entries: nvalid = (nf + nv_h) / PP (absent workers: none)
        const int nfj_h = (PP - 1) - h;                      // free entries: nfj = (nf + nfj_h) / PP
        uint4 r0 = __ldg(wsteps);
        for (int t = 0; t < nsteps; ++t) {
            const uint4 q = r0;
            if (t + 1 < nsteps) r0 = __ldg(wsteps + t + 1);
            const uint32_t fl = q.w;
            const int nf = (int)(fl & 31u);
            const int L = nf + NB;
            const uint32_t Tsh = (fl >> 17) << fv0;              // the free part of the prefix set
            const uint32_t S = Fw | Tsh;
            StepV v;
            v.bi = sbase + q.x;
            const unsigned kbcs = (unsigned)(k - nf) * CSb;
            v.bb0 = sb_h + q.x + kbcs;
            v.rf = rbase;
            v.rb0 = rb_h + (unsigned)(k - nf) * 16;
            v.RS = RS;
            v.nvalid = (nf + nv_h) >> (5 - LW);               // / PP (arithmetic: negative = none)
            v.nfj = (nf + nfj_h) >> (5 - LW);
            v.nl = q.z >> (4 * h);
            v.nh = 0;
            v.ab0 = ab_h >> (k - nf);
            v.X = Tsh | (uint32_t)w;
            v.X1 = v.X >> 1;
            v.c = c;
            v.sg = sg;
            v.Kw = KCw[(fl >> 8) & 31u];                          // read-only table: plain load
            v.seed0 = (fl >> 6) & 1u;
            const bool seed = (fl >> 5) & 1u;
            const bool has_next = (fl >> 7) & 1u;
            const unsigned ncol = sbase + q.y;
            const unsigned pcol = v.bi + ((fl >> 13) & 15u) * CSb;
            const bool pv = h == 0;
            const int ne = (L + PP - 1) >> (5 - LW);
            double cn = c, sn = sg, hn = hh;
#define BN_STEP(SEEDV, NEV)                                                                                   \
    step_ne<SEEDV, PP, CSb, HR, HB, NEV>(v, lntab, mhalf_n, out_rss, out_bic, pv, pcol, hh, has_next, ncol, cn, sn, \
                                         hn, S, recb_sh, bm_sh)
#define BN_SWITCH(SEEDV)                                                                                      \
    switch (ne) {                                                                                             \
        case 0: BN_STEP(SEEDV, 0); break;                                                                     \
        case 1: BN_STEP(SEEDV, 1); break;                                                                     \
        case 2: BN_STEP(SEEDV, 2); break;                                                                     \
        case 3: BN_STEP(SEEDV, 3); break;                                                                     \
        case 4: BN_STEP(SEEDV, 4); break;                                                                     \
        case 5: BN_STEP(SEEDV, 5); break;                                                                     \
        case 6: BN_STEP(SEEDV, 6); break;                                                                     \
        case 7: BN_STEP(SEEDV, 7); break;                                                                     \
        case 8: BN_STEP(SEEDV, 8); break;                                                                     \
        case 9: BN_STEP(SEEDV, 9); break;                                                                     \
        case 10: BN_STEP(SEEDV, 10); break;                                                                   \
        case 11: BN_STEP(SEEDV, 11); break;                                                                   \
        case 12: BN_STEP(SEEDV, 12); break;                                                                   \
        case 13: BN_STEP(SEEDV, 13); break;                                                                   \
        case 14: BN_STEP(SEEDV, 14); break;                                                                   \
        case 15: BN_STEP(SEEDV, 15); break;                                                                   \
        default: BN_STEP(SEEDV, 16); break;                                                                   \
    }
            if (seed) {
                BN_SWITCH(true)
            } else {
                BN_SWITCH(false)
            }
#undef BN_SWITCH
#undef BN_STEP
            c = cn;
            sg = sn;
            hh = hn;
            // the gang's warps write the two halves of each 256 B region: keep them in step
        }
        __syncwarp();
        // the per-slot records are the warp's per-child bests (a11)
        if (lane < Sw) {
            wbb[slotvar] = *(const double*)(recb + lane * 16);
            wbm[slotvar] = bm[lane];
        }
        __syncwarp();
    }
    __syncwarp();
    if (lane < m) {
        const size_t row = (size_t)P.part_base + (size_t)blockIdx.x * G + wib;
        P.part_bic[row * m + lane] = wbb[lane];
        P.part_mask[row * m + lane] = wbm[lane];
    }
}

// ---------------------------------------------------------------- a5: the seed kernel
// One warp per pack (item, warp of the gang): the pack's node at tree depth L1
// (tree_level_kernel), the remaining tree levels, then the W workers' seeds
// along a Gray path over the warp variables, each converted into walk state
// (E pairs of the free rows + suffix sums) and written to the pack's block of
// `seeds`.  Separate from the walk so that its serial GRC chains run at high
// occupancy.
//
// The node lives in a square array A[row position][physical column] and each
// lane owns one physical column (its variable never changes) and tracks the
// column's position: a GRC at positions J, J+1 rotates rows
// J, J+1 of every column at a position >= J and exchanges the two positions --
// no data moves for the swap itself.
__host__ __device__ size_t seed_block_bytes(int k, int S_alloc, int lw) { return (size_t)k * S_alloc * (16u << lw); }

// GRC at positions J, J+1 on the square node (lane = physical column, pos = its position).
__device__ __forceinline__ void grc_cols(double* A, int SA, int J, int lane, int& pos)
{
    const int Y = __ffs(__ballot_sync(FULLMASK, pos == J + 1)) - 1;   // the column at position J+1
    const double a = A[J * SA + Y], b = A[(J + 1) * SA + Y];
    double c, s, h;
    givens_fr(a, b, c, s, h);
    const bool live = pos < 32;                                        // lanes past the node's columns idle
    double* const p0 = A + J * SA + (live ? lane : 0);
    const double x = p0[0], y = p0[SA];
    __syncwarp();
    const bool isY = lane == Y;
    const double xn = isY ? h : fma(c, x, s * y);
    const double yn = isY ? 0.0 : fma(c, y, -s * x);
    const unsigned sa = (unsigned)__cvta_generic_to_shared(p0);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t@q st.shared.f64 [%0], %1;\n\t"
                 "@q st.shared.f64 [%2], %3;\n\t}" ::"r"(sa), "d"(xn), "r"(sa + SA * 8), "d"(yn),
                 "r"((unsigned)(live && pos >= J))
                 : "memory");
    __syncwarp();
    pos = pos == J ? J + 1 : (pos == J + 1 ? J : pos);
}

// Seed -> walk state of one worker, written to its part of a worker-major seed
// block ([row l][slot] of 16 B E pairs, row stride SA*16): the columns at
// positions >= og = [free block (k) | back columns].  Rows are processed
// bottom-up in lockstep (suffix sums of squares by addition; rows below the
// free block form the tail), so each row's stores are contiguous.
__device__ __forceinline__ void snapshot_sq(const double* A, int SAq, int sn, int og, int k, int SA, int lane, int pos,
                                            int slot, unsigned char* wblk)
{
    const bool mine = pos >= og && pos < sn;
    double acc = 0.0;
    const double* pa = A + (sn - 1) * SAq + lane;
    int r = sn - 1;
    // the tail: rows below the free block only add to the suffix sum
    for (; r >= og + k; --r, pa -= SAq) {
        const double x = (mine && r <= pos) ? *pa : 0.0;
        acc = fma(x, x, acc);
    }
    // the free rows og..og+k-1: E_l = (R_l, U_{l+1}), l = r - og
    double2* pw = (double2*)(wblk + (size_t)slot * 16) + (size_t)(r - og) * SA;
    for (; r >= og; --r, pa -= SAq, pw -= SA) {
        const double x = (mine && r <= pos) ? *pa : 0.0;
        if (mine) *pw = make_double2(x, acc);
        acc = fma(x, x, acc);
    }
}

// The seed tree's nodes at depth L1, all in one launch: one warp per node
// derives it from the root R directly (the same GRC sequence the level-by-level
// tree applies: a level's variable in F stays at the front and is dropped, one
// not in F is bubbled behind the remaining tree levels, the warp variables and
// the free block).  Output: m x m row-major, top-left sn x sn in position order.
__global__ void __launch_bounds__(128) tree_direct_kernel(const double* __restrict__ root, double* __restrict__ nodes,
                                                          int m, int L1, int bh, int p, int k)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int SAq = m | 1;
    double* const A = (double*)smem + (size_t)wib * m * SAq;
    const uint32_t nid = blockIdx.x * (blockDim.x >> 5) + wib;
    if (nid >= (1u << L1)) return;
    if (lane < m)
        for (int r = 0; r < m; ++r) A[r * SAq + lane] = root[r * m + lane];
    __syncwarp();
    int pos = lane < m ? lane : 1 << 20;
    int org = 0;
    for (int l = 0; l < L1; ++l) {
        if ((nid >> l) & 1u) {
            ++org;
            continue;
        }
        const int T = (bh - l - 1) + p + k;
        for (int j = 0; j < T; ++j) grc_cols(A, SAq, org + j, lane, pos);
    }
    // write the node in position order, without the dropped front
    const int sn = m - org;
    double* const dst = nodes + (size_t)nid * m * m;
    if (pos < 32 && pos >= org) {
        const int cq = pos - org;
        for (int r = org; r < m; ++r) dst[(r - org) * m + cq] = A[r * SAq + lane];
    }
    (void)sn;
}

cudaError_t launch_tree_direct(const double* root, double* nodes, int m, int L1, int bh, int p, int k,
                               cudaStream_t st)
{
    if (L1 <= 0) return cudaSuccess;
    const size_t smem = (size_t)4 * m * (m | 1) * sizeof(double);
    const unsigned n = 1u << L1;
    cudaError_t e = cudaFuncSetAttribute(tree_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tree_direct_kernel<<<(n + 3) / 4, 128, smem, st>>>(root, nodes, m, L1, bh, p, k);
    return cudaGetLastError();
}

template <int LW>
__global__ void __launch_bounds__(128) seed_kernel(const __grid_constant__ SeedParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g;
    const int fv0 = p + g, gs = bh - g, G = 1 << g;
    const int SAq = m | 1;
    double* const A = (double*)smem + (size_t)wib * m * SAq;
    const int npk = (P.item_end - P.item_begin) * G;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int q = blockIdx.x * (blockDim.x >> 5) + wib; q < npk; q += nwarps) {
        const int item = P.item_begin + q / G, gw = q % G;
        int c = 0;
        while (c + 1 < P.nclass && item >= P.cls_end[c]) ++c;
        const int SA = P.cls_SA[c];
        unsigned char* const blk =
            P.seeds + P.cls_off[c] + ((size_t)(item - P.cls_begin[c]) * G + gw) * seed_block_bytes(k, SA, LW);
        const uint32_t pack = P.packs[item] | ((uint32_t)gw << gs);
        // the node at depth L1: sn x sn, row-major (stride m) in global memory
        const uint32_t nid = pack & ((1u << P.L1) - 1u);
        const int sn = m - __popc(nid);
        {
            const double* src = P.nodes + (size_t)nid * m * m;
            if (lane < sn)
                for (int r = 0; r < sn; ++r) {
                    const unsigned sa = (unsigned)__cvta_generic_to_shared(A + r * SAq + lane);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + r * m + lane));
                }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
        }
        // the lane's physical column: its position (initially the column index) and variable,
        // node order [hv[L1..bh-1], warp vars p-1..0, free, back set (ascending id)]
        int pos = lane < sn ? lane : 1 << 20;
        int myvar = -1;
        {
            const int nlev = bh - P.L1;
            const int qq = lane;
            if (qq < nlev) myvar = hv_of(P.L1 + qq, m, gs, fv0);
            else if (qq < nlev + p) myvar = p - 1 - (qq - nlev);
            else if (qq < nlev + p + k) myvar = fv0 + (qq - nlev - p);
            else if (qq < sn) {
                int cc = qq - nlev - p - k;
                for (int l = P.L1 - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u)) {
                        if (cc == 0) { myvar = hv_of(l, m, gs, fv0); break; }
                        --cc;
                    }
            }
        }
        // the column's walk slot: [free 0..k-1 | warp vars 0..p-1 | back set ascending id]
        int slot = 0;
        if (myvar >= 0) {
            if (myvar >= fv0 && myvar < fv0 + k) slot = myvar - fv0;
            else if (myvar < p) slot = k + myvar;
            else {
                int cnt = 0;                           // back variables with a smaller id (not in F)
                for (int l = bh - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u) && hv_of(l, m, gs, fv0) < myvar) ++cnt;
                slot = k + p + cnt;
            }
        }
        // remaining tree levels: F -> the leading position joins the front (dropped),
        // B -> bubble it behind the remaining tree levels, the warp variables and the free block
        int org = 0;
        for (int l = P.L1; l < bh; ++l) {
            if ((pack >> l) & 1u) {
                ++org;
                continue;
            }
            const int T = (bh - l - 1) + p + k;
            for (int j = 0; j < T; ++j) grc_cols(A, SAq, org + j, lane, pos);
        }
        // Gray path over the warp variables: start with all of them in F (front
        // region [w_{p-1} .. w_0 | free]), flip bit ctz(i) at step i; a flip moves
        // variable j across the free block and the j lower warp variables
        const size_t wsz = (size_t)k * SA * 16;      // one worker's part of the block
        int wcur = P.nw - 1;
        snapshot_sq(A, SAq, sn, org + p, k, SA, lane, pos, slot, blk + wcur * wsz);
        for (int i = 1; i < P.nw; ++i) {
            const int j = __ffs(i) - 1;
            const int pj = __shfl_sync(FULLMASK, pos, __ffs(__ballot_sync(FULLMASK, myvar == j)) - 1);
            const int d = k + j;
            if ((wcur >> j) & 1) {
                for (int t = 0; t < d; ++t) grc_cols(A, SAq, pj + t, lane, pos);
            } else {
                for (int t = 1; t <= d; ++t) grc_cols(A, SAq, pj - t, lane, pos);
            }
            wcur ^= 1 << j;
            snapshot_sq(A, SAq, sn, org + __popc(wcur), k, SA, lane, pos, slot, blk + wcur * wsz);
        }
        __syncwarp();
    }
}

cudaError_t launch_seed(const SeedParams& P, cudaStream_t st)
{
    const int m = P.m;
    const size_t smem = (size_t)4 * m * (m | 1) * sizeof(double);
    const int npk = (P.item_end - P.item_begin) << P.g;
    if (npk <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min((npk + 3) / 4, sms * 16);
    if (P.lw != 3) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(seed_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    seed_kernel<3><<<grid, 128, smem, st>>>(P);
    return cudaGetLastError();
}

template <int LW, bool W1, bool HR, bool HB>
static cudaError_t launch_w(const TravParams& P, int grid, cudaStream_t st)
{
    const size_t smem = walk_cta_smem(P.m, P.k, P.S_alloc, P.g, LW);
    auto f = walk_kernel<LW, W1, HR, HB>;
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    f<<<grid, 32 << P.g, smem, st>>>(P);
    return cudaGetLastError();
}

template <int LW>
static cudaError_t launch_lw(const TravParams& P, int grid, cudaStream_t st)
{
    const int key = (P.world1 ? 4 : 0) | (P.out_rss ? 2 : 0) | (P.out_bic ? 1 : 0);
    switch (key) {
        case 7: return launch_w<LW, true, true, true>(P, grid, st);
        case 6: return launch_w<LW, true, true, false>(P, grid, st);
        case 5: return launch_w<LW, true, false, true>(P, grid, st);
        case 4: return launch_w<LW, true, false, false>(P, grid, st);
        case 3: return launch_w<LW, false, true, true>(P, grid, st);
        case 2: return launch_w<LW, false, true, false>(P, grid, st);
        case 1: return launch_w<LW, false, false, true>(P, grid, st);
        default: return launch_w<LW, false, false, false>(P, grid, st);
    }
}

cudaError_t launch_walk(const TravParams& P, int grid, cudaStream_t st)
{
    if (P.lw != 3) return cudaErrorInvalidValue;   // 8 workers per warp (plan.h kPackBits)
    return launch_lw<3>(P, grid, st);
}

int walk_max_ctas_per_sm(int m, int k, int S_alloc, int g, int world1, int lw)
{
    const size_t smem = walk_cta_smem(m, k, S_alloc, g, lw);
    int n = 0;
    if (lw != 3) return 0;
    auto f = world1 ? walk_kernel<3, true, true, true> : walk_kernel<3, false, true, true>;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, 32 << g, smem) != cudaSuccess) return 0;
    return n;
}

}  // namespace bnr
