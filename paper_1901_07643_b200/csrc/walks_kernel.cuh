// walks_kernel.cuh -- the walk kernel, slot-split design (DESIGN.md §4 "design S"; opt-in,
// BNREG_WALK_S=1: measured slower than walk_kernel.cuh): the same Alg.2 workers
// walking d + Upsilon(k) (Alg.1 with Eq.10's +1, PAPER.md:160-174,
// :207-212), one GRC per step (Eq.3-4, reading G1), harvesting every new
// family's RSS from suffix sums (Eq.5, G3), its BIC (G5), the
// (child, mask)-indexed store and the per-child running best (G14) -- with the gang
// transposed:
//
//   * a CTA's 4 warps run the same 32 workers: lane = worker (its 3 warp and 2 gang
//     variables = the 5 lowest user ids), so for every child and step ONE warp store
//     writes the whole 512 B region of the 32 workers' (RSS, BIC) records;
//   * the warps split the walk SLOTS instead of the workers: warp w owns the back slots
//     b = w (mod 4) (state in its TMEM lane quarter) and takes the step's free-list
//     entries f = w (mod 4) of the free-slot state the 4 warps share, so a warp executes
//     only entries that exist;
//   * steps are ordered by kSD mbarriers (every thread arrives after its rotations of a
//     step, waits before the next step's): the harvest between the arrive and the wait is
//     the slack; every warp computes the step's rotation itself from the pivot rows one
//     warp copies to a staging buffer (DESIGN.md §4 lists the measured variants).
#pragma once
#include "walk_kernel.cuh"

namespace bnr {

constexpr int kSD = 4;          // step mbarriers (reused every kSD GRCs)
constexpr int kSCS = 32 * 16;   // bytes between free slots of the shared state (32 workers x 16 B)

// per-CTA shared memory after the log/K head: the pivot-row staging (2 of kSD x 32 x 16 B), the kSD
// step mbarriers, the free-slot state E(l, s, lane) at ((l k + s) 32 + lane) 16 (shared by
// the gang's warps: the free list is dealt anew every step), then per warp its per-slot
// records rec / bb / bm and its per-child bests wbb / wbm as in walk_kernel.cuh
struct WalkSLayout {
    int ring, mbar, state, warps, rec, bb, bm, wbb, wbm, per_warp;
};

__host__ __device__ inline WalkSLayout walks_layout(int k, int SA)
{
    WalkSLayout L;
    L.ring = kWalkHead;
    L.mbar = L.ring + kSD * kSCS;
    L.state = L.mbar + kSD * 8 + 16;
    L.state = al16(L.state);
    L.warps = L.state + k * k * kSCS;
    int o = 0;
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

inline size_t walks_cta_smem_h(int k, int SA) { return (size_t)walks_layout(k, SA).warps + 4 * (size_t)walks_layout(k, SA).per_warp; }

__device__ __forceinline__ void mbar_init(unsigned a, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned a)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void sts2(unsigned a, double x, double y)
{
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}

// per-lane constants of design S: walk_kernel.cuh's LaneC (the harvest reads it) plus
struct LaneS : LaneC {
    unsigned wib;      // this warp: back slots b = wib (mod 4), free-list entries f = wib (mod 4)
    unsigned lane;
    unsigned ring;     // shared address of ring slot 0, this lane's (c, s)
    unsigned mbar;     // step barrier 0 (barrier r at + 8 r)
};

// Step barriers (GRC number g of this CTA: barrier g mod kSD, phase g / kSD): all 128
// threads arrive after their rotations of GRC g - 1 (after the seed steps for an item's
// first GRC) -- the stager of g's pivot rows after copying them -- and wait before the
// rotations of GRC g: the free-slot state, the pivot and the staged rows of g are then
// visible to every warp.  Between the arrive and the wait lies the warp's harvest of
// g - 1, the slack that keeps the warps from waiting on each other.  Staging buffer g mod 2
// is rewritten (for g + 2, after the rotations of g + 1) only after every warp has passed
// the wait of g + 1, i.e. read the rows of g.
__device__ __forceinline__ void step_arrive(const LaneS& L, uint32_t g) { mbar_arrive(L.mbar + 8 * (g & (kSD - 1))); }
__device__ __forceinline__ void step_wait(const LaneS& L, uint32_t g)
{
    mbar_wait(L.mbar + 8 * (g & (kSD - 1)), (g / kSD) & 1u);
}

// this warp's free-list entries f = wib + 4j of a step (nib: the list's slot nibbles)
template <int NFE>
__device__ __forceinline__ void free_s(const LaneS& L, uint32_t nib, unsigned* slot)
{
    const uint32_t nl = nib >> (4 * L.wib);
#pragma unroll
    for (int j = 0; j < NFE; ++j) slot[j] = (nl >> (16 * j)) & 15u;
}

// seed pseudo-step (reading G11): RSS = U_{i+1} = E_i.y, or U_0 = R_0^2 + E_0.y
template <int JB, int NFE, bool HR, bool HB, bool HP>
__device__ __forceinline__ void seed_step_s(const LaneS& L, const TravParams& P, const uint4 q)
{
    constexpr int NE = JB + NFE;
    const uint32_t fl = q.w;
    const int i = (int)((fl >> 8) & 31u) - 1;
    const bool s0 = i < 0;
    const unsigned bi = L.sbase + q.x;
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
    free_s<NFE>(L, q.z, sl);
#pragma unroll
    for (int j = 0; j < NFE; ++j) {
        const double2 a = lds2(bi + sl[j] * kSCS);
        rs[JB + j] = s0 ? fma(a.x, a.x, a.y) : a.y;
        ra[JB + j] = L.recb + sl[j] * 16;
        okv[JB + j] = L.hfree != 0;
    }
    const uint32_t Tsh = ((fl >> 17) & 255u) << LC(fv0);   // (bits 25.. hold prod)
    harvest<NE, HR, HB, HP>(L, P, rs, ra, okv, L.KCw[(fl >> 8) & 31u], Tsh | L.Xw, L.Fw | Tsh);
}

// the staging writer of GRC g: copies the pivot column's rows (ncol: byte offset of row in
// of the pivot in the free state) of the 32 workers to staging buffer g mod 2
__device__ __forceinline__ void stage_pivot(const LaneS& L, uint32_t ncol, uint32_t g, int RS)
{
    __syncwarp();
    const unsigned a0 = L.sbase + ncol;
    const double a = lds1(a0), b = lds1(a0 + RS);
    sts2(L.ring + (g & 1u) * kSCS, a, b);
}

// one GRC step of a warp: wait for the step, its rotation from the staged pivot rows, its
// back entries (TMEM) and free-list entries (shared state), the pivot (warp 3), the next
// step's pivot rows (its stager), arrive, harvest
template <int JB, int NFE, bool HR, bool HB, bool HP>
__device__ __forceinline__ void grc_step_s(const LaneS& L, const TravParams& P, const uint4 q, uint32_t& gi)
{
    constexpr int NE = JB + NFE;
    const uint32_t fl = q.w;
    const int i = (int)((fl >> 8) & 31u) - 1;
    const unsigned bi = L.sbase + q.x;
    const int RS = LC(RS);
    double rs[NE > 0 ? NE : 1];
    unsigned ra[NE > 0 ? NE : 1];
    bool okv[NE > 0 ? NE : 1];
    unsigned sl[NFE > 0 ? NFE : 1];
    free_s<NFE>(L, q.z, sl);
    double c, sg, hh;
    step_wait(L, gi);
    {
        // this step's rotation from its pivot rows (every warp: no warp waits for another's chain)
        const double2 ab = lds2(L.ring + (gi & 1u) * kSCS);
        givens_fr(ab.x, ab.y, c, sg, hh);
    }
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
            f0[j] = lds1(bi + sl[j] * kSCS);
            f1[j] = lds2(bi + sl[j] * kSCS + RS);
        }
        tm_wait_ld<8 * JB>(rb);
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            uint32_t* r0 = rb + 4 * j;            // row i:   (R_i, U_{i+1})
            uint32_t* r1 = rb + 4 * JB + 4 * j;   // row i+1: (R_{i+1}, U_{i+2})
            const double x = tm_f64(r0), y = tm_f64(r1), u2 = tm_f64(r1 + 2);
            const double xa = fma(c, x, sg * y), ya = fma(c, y, -sg * x);
            const double ru = fma(ya, ya, u2);
            tm_put(r0, xa);
            tm_put(r0 + 2, ru);
            tm_put(r1, ya);
            rs[j] = ru;
            ra[j] = L.recB + 64 * j;
            okv[j] = (L.bval >> j) & 1u;
        }
        tm_st<8 * JB>(tcol, rb);
    } else {
#pragma unroll
        for (int j = 0; j < NFE; ++j) {
            f0[j] = lds1(bi + sl[j] * kSCS);
            f1[j] = lds2(bi + sl[j] * kSCS + RS);
        }
    }
#pragma unroll
    for (int j = 0; j < NFE; ++j) {
        K8_CHECK(L, bi + sl[j] * kSCS + RS + 16 - L.sb0 <= L.sbytes && bi + sl[j] * kSCS >= L.sb0);
        const double xa = fma(c, f0[j], sg * f1[j].x), ya = fma(c, f1[j].x, -sg * f0[j]);
        const double ru = fma(ya, ya, f1[j].y);
        sts_pair_if(bi + sl[j] * kSCS, xa, ru, ya, RS, true);
        rs[JB + j] = ru;
        ra[JB + j] = L.recb + sl[j] * 16;
        okv[JB + j] = L.hfree != 0;
    }
    // the pivot Y (now at position i): E_i = (h, 0), R_{i+1} = 0 -- by warp 3 (the fewest
    // free-list entries); no other warp touches Y's state in this step (the others read
    // its rows from the staging buffer)
    if (L.wib == 3) sts_pair_if(bi + ((fl >> 13) & 15u) * kSCS, hh, 0.0, 0.0, RS, true);
    ++gi;
    if ((fl >> 7) & 1u) {
        if (((q.y >> 16) & 3u) == L.wib) stage_pivot(L, q.y & 0xffffu, gi, RS);
        step_arrive(L, gi);
    }
    const uint32_t Tsh = ((fl >> 17) & 255u) << LC(fv0);   // (bits 25.. hold prod)
    harvest<NE, HR, HB, HP>(L, P, rs, ra, okv, L.KCw[(fl >> 8) & 31u], Tsh | L.Xw, L.Fw | Tsh);
}

template <int JB, bool HR, bool HB, bool HP>
__device__ __forceinline__ void walk_item_s(const LaneS& L, const TravParams& P, const unsigned char* src, int k, int Sw,
                                         int b0, const uint4* __restrict__ wsteps, int nsteps, uint32_t& gi)
{
    if constexpr (JB > 0) {
        // back slot b = b0 + 4j + wib of this lane's worker, row l: ((l Sw) + k + b) * 16 from src
        const unsigned char* bs = src + ((size_t)k + b0 + L.wib) * 16;
        for (int l = 0; l < k; l += 2) {
            uint32_t v0[4 * JB], v1[4 * JB];
#pragma unroll
            for (int j = 0; j < JB; ++j) {
                const bool ok = (L.bval >> (8 + j)) & 1u;   // the slot exists
                uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
                if (ok) {
                    a = __ldg((const uint4*)(bs + ((size_t)l * Sw + 4 * j) * 16));
                    if (l + 1 < k) b = __ldg((const uint4*)(bs + ((size_t)(l + 1) * Sw + 4 * j) * 16));
                }
                v0[4 * j] = a.x; v0[4 * j + 1] = a.y; v0[4 * j + 2] = a.z; v0[4 * j + 3] = a.w;
                v1[4 * j] = b.x; v1[4 * j + 1] = b.y; v1[4 * j + 2] = b.z; v1[4 * j + 3] = b.w;
            }
            tm_st<4 * JB>(L.tb + (uint32_t)(l * JB * 4), v0);
            if (l + 1 < k) tm_st<4 * JB>(L.tb + (uint32_t)((l + 1) * JB * 4), v1);
        }
    }
    uint4 win = make_uint4(0, 0, 0, 0);
    const int lane = (int)L.lane;
    auto record = [&](int t) {
        if ((t & 31) == 0) win = __ldg(wsteps + t + lane);
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
        const int nf = (int)(q.w & 31u);
        const int nfe = (nf - (int)L.wib + 3) >> 2;   // entries f = wib + 4j < nf
        if (nfe <= 0) seed_step_s<JB, 0, HR, HB, HP>(L, P, q);
        else if (nfe == 1) seed_step_s<JB, 1, HR, HB, HP>(L, P, q);
        else seed_step_s<JB, 2, HR, HB, HP>(L, P, q);
    }
    if ((qk.w >> 7) & 1u) {
        // the first GRC's pivot rows (the last seed record points at its pivot column)
        if (((qk.y >> 16) & 3u) == L.wib) stage_pivot(L, qk.y & 0xffffu, gi, LC(RS));
        step_arrive(L, gi);
    }
    for (int t = k + 1; t < nsteps; ++t) {
        const uint4 q = record(t);
        const int nf = (int)(q.w & 31u);
        const int nfe = (nf - (int)L.wib + 3) >> 2;
        if (nfe <= 0) grc_step_s<JB, 0, HR, HB, HP>(L, P, q, gi);
        else if (nfe == 1) grc_step_s<JB, 1, HR, HB, HP>(L, P, q, gi);
        else grc_step_s<JB, 2, HR, HB, HP>(L, P, q, gi);
    }
    tm_wait_st();
}

template <bool HR, bool HB, bool HP>
__global__ void __launch_bounds__(128, 4) walks_kernel(const __grid_constant__ TravParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_item, s_taddr;
    double2* const lntab = (double2*)smem;
    double* const KC = (double*)(smem + 16 * kLnEntries);
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g, SA = P.S_alloc;
    const WalkSLayout Ly = walks_layout(k, SA);
    for (int j = tid; j < kLnEntries; j += blockDim.x) lntab[j] = P.lntab9[j];
    for (int j = tid; j < 33; j += blockDim.x) KC[j] = P.Kc[j];
    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(smem + Ly.mbar);
    if (tid == 0) {
        for (int r = 0; r < kSD; ++r) mbar_init(mb0 + 8 * r, 128);   // step barriers: every thread arrives
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (wib == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&s_taddr)),
                     "r"(P.tm_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int fv0 = p + g;                      // user id of free slot 0
    const int gs = bh - g;                      // gang levels are gs..bh-1
    const int G = 1 << g;                       // = 4 (design S requires p = 3, g = 2)
    unsigned char* const wb = smem + Ly.warps + wib * Ly.per_warp;
    unsigned char* const st = smem + Ly.state;
    unsigned char* const recb = wb + Ly.rec;
    uint32_t* const bm = (uint32_t*)(wb + Ly.bm);
    double* const bbv = (double*)(wb + Ly.bb);
    double* const wbb = (double*)(wb + Ly.wbb);
    uint32_t* const wbm = (uint32_t*)(wb + Ly.wbm);
    const double NINF = -__longlong_as_double(0x7ff0000000000000LL);
    wbb[lane] = NINF;
    wbm[lane] = 0xffffffffu;
    const int shb = P.world1 ? m - 1 : m - P.r;   // child block = v << shb entries
    const int gw = lane >> 3, w = lane & 7;       // the lane's worker: gang slot, warp-variable bits
    LaneS L;
    L.sbase = (unsigned)__cvta_generic_to_shared(st + lane * 16);
    L.recb = (unsigned)__cvta_generic_to_shared(recb);
    L.bmb = (unsigned)__cvta_generic_to_shared(bm);
    L.bbb = (unsigned)__cvta_generic_to_shared(bbv);
    L.tiny_bic = P.tiny_bic;
    L.tb = s_taddr + ((uint32_t)(wib * 32) << 16);
    L.w = (uint32_t)w;
    L.live = 1;
    L.h = wib;
    L.wib = (unsigned)wib;
    L.lane = (unsigned)lane;
    L.ring = (unsigned)__cvta_generic_to_shared(smem + Ly.ring) + lane * 16;
    L.mbar = mb0;
    L.RS = k * kSCS;
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
    L.sbytes = (unsigned)(k * k * kSCS);
    L.tmcols = (unsigned)P.tm_cols;
    K8_CHECK(L, !(P.k8_selftest && lane == 0));   // (a negative control of the counter path)
    {
        // the worker's warp and gang variables in F (user-id bits): w, and gang slot gw
        // bit j = seed-tree level gs + j = gang variable fv0 - 1 - j (plan.h hv_id)
        uint32_t x = (uint32_t)w;
        for (int j = 0; j < g; ++j) x |= ((uint32_t)(gw >> j) & 1u) << (fv0 - 1 - j);
        L.Xw = x;
    }
    const int nsteps = P.nsteps;
    const uint4* const wsteps = P.wsteps;
    uint32_t gi = 0;                             // GRC steps of this CTA so far (the step barriers' clock)
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
        const uint32_t pk = P.packs[item];
        const bool passB = (pk >> 31) != 0;
        const int aitem = passB ? (int)(pk & 0x7fffffffu) : item;
        const uint32_t pack = passB ? P.packs[aitem] : pk;
        uint32_t Ft = 0;
        int nBt = 0;
        for (int l = 0; l < gs; ++l) {
            if ((pack >> l) & 1u) Ft |= 1u << hv_of(l, m, gs, fv0);
            else ++nBt;
        }
        const int NB = fv0 + nBt;
        const int Sw = k + NB;
        // this lane's worker's seed block (block of gang slot gw, worker w): [l][slot] rows of Sw
        const unsigned char* src = P.seeds + ((size_t)(aitem - P.item_begin) * G + gw) * (size_t)(k * SA * kW * 16) +
                                   (size_t)(w * k) * Sw * 16;
        {
            // the free slots' state of the 32 workers (warp wib copies slots wib, wib + 4)
            const unsigned dst = L.sbase;
            for (int s = wib; s < k; s += 4)
                for (int l = 0; l < k; ++l)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (l * k + s) * kSCS),
                                 "l"(src + ((size_t)l * Sw + s) * 16));
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
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
        if (lane < Sw) {
            const int v = slotvar;
            const uint32_t lm = (1u << v) - 1u;
            const uint32_t off = P.world1 ? block_offset<true>(P, Ft, Ft >> 1, lm)
                                          : block_offset<false>(P, Ft, Ft >> 1, lm);
            const uint32_t idx = (uint32_t)((long long)v << shb) + off;
            unsigned char* r = recb + lane * 16;
            const double gb = P.gbest ? bic_unord(((volatile long long*)P.gbest)[v]) : wbb[v];
            *(double*)r = fmin(fmax(wbb[v], gb), P.tiny_bic);
            bbv[lane] = wbb[v];
            *(uint32_t*)(r + 8) = idx;
            *(uint32_t*)(r + 12) = lm;
            bm[lane] = wbm[v];
        }
        L.Fw = Ft | L.Xw;
        L.KCw = KC + __popc(L.Fw);
        const int b0 = passB ? 16 : 0;
        const int nbp = passB ? NB - 16 : min(NB, 16);
        L.hfree = passB ? 0 : 1;
        L.recB = L.recb + (unsigned)(k + b0 + wib) * 16u;
        // the same JB in the gang's 4 warps (one code path per CTA: instruction-cache footprint)
        const int JB = (nbp + 3) >> 2;
        {
            // back entry j = slot k + b0 + 4j + wib: exists for b < b0 + nbp; absent for this
            // worker when it is warp or gang variable b (b < fv0) in F
            uint32_t bv = 0;
            for (int j = 0; j < JB; ++j) {
                const int b = b0 + 4 * j + wib;
                if (b < b0 + nbp) bv |= 1u << (8 + j);                        // the slot exists
                if (b < b0 + nbp && !(b < fv0 && ((L.Xw >> b) & 1u))) bv |= 1u << j;
            }
            L.bval = bv;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();                         // the free state is shared by the gang's warps
        switch (JB) {
            case 0: walk_item_s<0, HR, HB, HP>(L, P, src, k, Sw, b0, wsteps, nsteps, gi); break;
            case 1: walk_item_s<1, HR, HB, HP>(L, P, src, k, Sw, b0, wsteps, nsteps, gi); break;
            case 2: walk_item_s<2, HR, HB, HP>(L, P, src, k, Sw, b0, wsteps, nsteps, gi); break;
            case 3: walk_item_s<3, HR, HB, HP>(L, P, src, k, Sw, b0, wsteps, nsteps, gi); break;
            default: walk_item_s<4, HR, HB, HP>(L, P, src, k, Sw, b0, wsteps, nsteps, gi); break;
        }
        __syncwarp();
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

static inline size_t walks_launch_smem(const TravParams& P)
{
    size_t smem = walks_cta_smem_h(P.k, P.S_alloc);
    const int occ_tm = 512 / P.tm_cols;
    const size_t cap = (size_t)233472 / (size_t)(occ_tm + 1);   // no more CTAs per SM than TMEM holds
    if (smem + 1024 <= cap) smem = cap - 1024 + 16;
    return smem;
}

template <bool HR, bool HB, bool HP>
static inline cudaError_t launch_ws(const TravParams& P, int grid, cudaStream_t st)
{
    const size_t smem = walks_launch_smem(P);
    auto f = walks_kernel<HR, HB, HP>;
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    f<<<grid, 128, smem, st>>>(P);
    return cudaGetLastError();
}

}  // namespace bnr
