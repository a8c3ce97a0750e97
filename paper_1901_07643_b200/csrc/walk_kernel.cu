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
#include "kernels.h"
#include "device.cuh"

namespace bnr {

// ---------------------------------------------------------------- shared memory layout
// Per CTA: [lntab 128 x 16 B][K(s) 33 doubles] then per warp:
//   state   k * SA * W * 16 B   E(l, slot, w) at ((l*SA + slot)*W + w)*16
//   scratch max(tri, SA*W*12)   derivation triangle (packed, side <= m) | per-(slot, worker) best
//   desc    SA * 16 B           (RSS row ptr, BIC row ptr) of each slot's child
//   lm      SA * 4 B            (1 << v) - 1 of each slot's child v
//   wbb/wbm 32 * 12 B           the warp's running best per child (kept across items)
//   slotof  32 B                variable -> slot
struct WalkLayout {
    int state, scratch, bm, desc, lm, wbb, wbm, slotof, per_warp;
};

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline WalkLayout walk_layout(int m, int k, int SA, int W)
{
    WalkLayout L;
    int o = 0;
    L.state = o;
    o += al16(k * SA * W * 16);
    L.scratch = o;
    L.bm = o + SA * W * 8;
    const int tri = (m * (m + 1) / 2) * 8, bst = SA * W * 12;
    o += al16(tri > bst ? tri : bst);
    L.desc = o;
    o += al16(SA * 16);
    L.lm = o;
    o += al16(SA * 4);
    L.wbb = o;
    o += 32 * 8;
    L.wbm = o;
    o += 32 * 4;
    L.slotof = o;
    o += 32;
    L.per_warp = al16(o);
    return L;
}

constexpr int kWalkHead = 2048 + 272;   // lntab + K(s) table

size_t walk_cta_smem(int m, int k, int SA, int g)
{
    return (size_t)kWalkHead + ((size_t)1 << g) * (size_t)walk_layout(m, k, SA, 1 << kWalkLW).per_warp;
}

// user id of seed-tree level l (plan.h hv_id): top ids first, the gang ids last
__device__ __forceinline__ int hv_of(int l, int m, int gs, int fv0) { return l < gs ? m - 1 - l : fv0 - 1 - (l - gs); }

// GRC on the derivation triangle; myvar (lane = position) follows the swap.
__device__ __forceinline__ void grc_pv(double* A, int s, int J, int lane, int& myvar)
{
    grc_packed(A, s, J, s, lane);
    const int src = lane == J ? J + 1 : (lane == J + 1 ? J : lane);
    myvar = __shfl_sync(FULLMASK, myvar, src);
}

// Seed -> walk state of worker wc: the sub-triangle from position og (side
// sn - og) = [free block (k) | back columns]; lane = position q.  For every
// column: its free rows og..og+k-1 and the suffix sums of squares down to the
// diagonal (rows below the free block form the tail), by addition from the
// bottom.
template <int W>
__device__ __forceinline__ void snapshot(const double* A, int sn, int og, int k, int SA, int wc, int lane, int myvar,
                                         const uint8_t* slotof, unsigned char* st)
{
    const int q = lane;
    if (q >= og && q < sn) {
        const int slot = slotof[myvar];
        unsigned char* col = st + (slot * W + wc) * 16;
        const int RS = SA * W * 16;
        double acc = 0.0;
        for (int l = q - og + 1; l < k; ++l)                 // rows below the diagonal (free columns)
            *(double2*)(col + l * RS) = make_double2(0.0, 0.0);
        for (int r = q; r >= og; --r) {
            const double x = A[poff(r, sn) + q - r];
            const int l = r - og;
            if (l < k) *(double2*)(col + l * RS) = make_double2(x, acc);
            acc = fma(x, x, acc);
        }
    }
}

// One family (child of list entry `slot`, prefix set S of this worker):
// BIC, the two table stores, the running best of (slot, worker).
template <bool WORLD1, bool HR, bool HB>
__device__ __forceinline__ void harvest(const TravParams& P, const double2* lntab, const ulonglong2* desc,
                                        const uint32_t* lmt, double* bb, uint32_t* bm, int W, int w, int slot,
                                        bool present, double rss, uint32_t S, uint32_t S1, double Kw)
{
    const double bic = bic_of(rss, fast_ln(rss, lntab), P.mhalf_n, Kw);   // rss <= 1e-300 -> +inf
    const ulonglong2 d = desc[slot];
    const uint32_t off = block_offset<WORLD1>(P, S, S1, lmt[slot]);
    if (present) {
        if (HR) __stcs((double*)d.x + off, rss);
        if (HB) __stcs((double*)d.y + off, bic);
        double* bp = bb + slot * W + w;
        if (bic >= *bp) {                      // rare: a new best (or a tie) for this (child, worker)
            uint32_t* mp = bm + slot * W + w;
            if (tie_better(bic, S, *bp, *mp)) {
                *bp = bic;
                *mp = S;
            }
        }
    }
}

__device__ __forceinline__ int entry_slot(int e, int nf, int k, uint64_t nib)
{
    return e < nf ? (int)((nib >> (4 * e)) & 15u) : k + e - nf;
}

template <bool WORLD1, bool HR, bool HB>
__global__ void __launch_bounds__(128, 1) walk_kernel(const __grid_constant__ TravParams P)
{
    constexpr int LW = kWalkLW;
    constexpr int W = 1 << LW;
    constexpr int PP = 32 / W;                  // lanes (parts) per worker
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_item;
    double2* const lntab = (double2*)smem;
    double* const KC = (double*)(smem + 2048);
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    for (int j = tid; j < 128; j += blockDim.x) lntab[j] = P.lntab[j];
    for (int j = tid; j < 33; j += blockDim.x) KC[j] = P.Kc[j];
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g, SA = P.S_alloc;
    const int fv0 = p + g;                      // user id of free slot 0
    const int gs = bh - g;                      // gang levels are gs..bh-1
    const int G = 1 << g;
    const WalkLayout Ly = walk_layout(m, k, SA, W);
    unsigned char* const wb = smem + kWalkHead + wib * Ly.per_warp;
    unsigned char* const st = wb + Ly.state;
    double* const tri = (double*)(wb + Ly.scratch);
    double* const bb = (double*)(wb + Ly.scratch);
    uint32_t* const bm = (uint32_t*)(wb + Ly.bm);
    ulonglong2* const desc = (ulonglong2*)(wb + Ly.desc);
    uint32_t* const lmt = (uint32_t*)(wb + Ly.lm);
    double* const wbb = (double*)(wb + Ly.wbb);
    uint32_t* const wbm = (uint32_t*)(wb + Ly.wbm);
    uint8_t* const slotof = wb + Ly.slotof;
    const int w = lane & (W - 1), h = lane >> LW;
    const double NINF = -__longlong_as_double(0x7ff0000000000000LL);
    wbb[lane] = NINF;
    wbm[lane] = 0xffffffffu;
    const int shb = WORLD1 ? m - 1 : m - P.r;   // child block = v << shb entries
    const int RS = SA * W * 16;                 // bytes between free rows l and l+1 of a slot
    const int CSb = W * 16;                     // bytes between slots
    const int nw = P.nw;
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

        // ---- a5: node at depth L1 (all loads in flight at once)
        const uint32_t nid = pack & ((1u << P.L1) - 1u);
        const int sn = m - __popc(nid);
        {
            const double* src = P.nodes + (size_t)nid * m * m;
            const int tot = sn * (sn + 1) / 2;
            for (int e = lane; e < tot; e += 32) {
                int r = (int)((2.0f * sn + 1.0f - sqrtf((2.0f * sn + 1.0f) * (2.0f * sn + 1.0f) - 8.0f * e)) * 0.5f);
                if (r < 0) r = 0;
                while (r > 0 && poff(r, sn) > e) --r;
                while (r + 1 < sn && poff(r + 1, sn) <= e) ++r;
                const int c = r + (e - poff(r, sn));
                const unsigned sa = (unsigned)__cvta_generic_to_shared(tri + e);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + r * m + c));
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        // variable at each node position (lane = position):
        // [hv[L1..bh-1], warp vars p-1..0, free, back set (ascending id)]
        int myvar = -1;                          // -1: no column at this position
        {
            const int nlev = bh - P.L1;
            const int q = lane;
            if (q < nlev) myvar = hv_of(P.L1 + q, m, gs, fv0);
            else if (q < nlev + p) myvar = p - 1 - (q - nlev);
            else if (q < nlev + p + k) myvar = fv0 + (q - nlev - p);
            else if (q < sn) {
                int c = q - nlev - p - k;
                for (int l = P.L1 - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u)) {
                        if (c == 0) { myvar = hv_of(l, m, gs, fv0); break; }
                        --c;
                    }
            }
        }
        // slot tables: slots [free 0..k-1 | warp vars 0..p-1 | back set ascending id]
        if (lane < SA) {
            int v = -1;
            const int s = lane;
            if (s < k) v = fv0 + s;
            else if (s < k + p) v = s - k;
            else if (s < Sw) {
                int c = s - k - p;
                for (int l = bh - 1; l >= 0; --l)
                    if (!((pack >> l) & 1u)) {
                        if (c == 0) { v = hv_of(l, m, gs, fv0); break; }
                        --c;
                    }
            }
            if (v >= 0) {
                slotof[v] = (uint8_t)s;
                desc[s] = make_ulonglong2(HR ? (unsigned long long)(P.out_rss + ((long long)v << shb)) : 0ull,
                                          HB ? (unsigned long long)(P.out_bic + ((long long)v << shb)) : 0ull);
                lmt[s] = (1u << v) - 1u;
            } else {
                desc[s] = make_ulonglong2(0ull, 0ull);
                lmt[s] = 0u;
            }
        }
        __syncwarp();
        // remaining tree levels in-warp: F -> drop the leading row/column, B -> bubble it behind the free block
        int org = 0;
        for (int l = P.L1; l < bh; ++l) {
            if ((pack >> l) & 1u) {
                ++org;
                continue;
            }
            const int T = (bh - l - 1) + p + k;
            for (int j = 0; j < T; ++j) grc_pv(tri, sn, org + j, lane, myvar);
        }
        // Gray path over the warp variables: start with all of them in F (front
        // region [w_{p-1} .. w_0 | free]), flip bit ctz(i) at step i; a flip moves
        // variable j across the free block and the j lower warp variables
        int wcur = nw - 1;
        snapshot<W>(tri, sn, org + p, k, SA, wcur, lane, myvar, slotof, st);
        for (int i = 1; i < nw; ++i) {
            const int j = __ffs(i) - 1;
            const int pj = __ffs(__ballot_sync(FULLMASK, myvar == j)) - 1;
            const int d = k + j;
            __syncwarp();
            if ((wcur >> j) & 1) {
                for (int t = 0; t < d; ++t) grc_pv(tri, sn, pj + t, lane, myvar);
            } else {
                for (int t = 1; t <= d; ++t) grc_pv(tri, sn, pj - t, lane, myvar);
            }
            wcur ^= 1 << j;
            snapshot<W>(tri, sn, org + __popc(wcur), k, SA, wcur, lane, myvar, slotof, st);
        }
        __syncwarp();
        for (int e = lane; e < SA * W; e += 32) {      // the best arrays overlay the triangle
            bb[e] = NINF;
            bm[e] = 0xffffffffu;
        }
        __syncwarp();

        // ---- a6-a11: the walk, k+1 seed pseudo-steps then d + Upsilon(k), in lockstep
        const uint32_t Fw = Fhi | (uint32_t)w;  // warp variable j (user id j) in F iff bit j of w
        const int dw = __popc(Fw);
        const uint32_t absent = (w < nw) ? ((uint32_t)w << k) : 0xffffffffu;
        const int NB = Sw - k;
        unsigned char* const sw = st + w * 16;
        double c = 1.0, sg = 0.0, hh = 0.0;
        uint4 rec = __ldg(P.steps);
        for (int t = 0; t < P.nsteps; ++t) {
            const uint4 nrec = (t + 1 < P.nsteps) ? __ldg(P.steps + t + 1) : make_uint4(1u << 18, 0, 0, 0);
            const int i = (int)(rec.x & 31u) - 1;
            const int nf = (int)((rec.x >> 13) & 31u);
            const int L = nf + NB;
            const uint32_t S = Fw | (rec.y << fv0);
            const uint32_t S1 = S >> 1;
            const double Kw = KC[dw + i + 1];
            const uint64_t nib = ((uint64_t)rec.w << 32) | rec.z;
            if ((rec.x >> 18) & 1u) {
                // seed pseudo-step: prefix = free positions 0..i, RSS = U_{i+1} = E_i.y (U_0 = E_0.x^2 + E_0.y)
                const unsigned char* bi = sw + (i < 0 ? 0 : i) * RS;
                for (int e = h; e < L; e += PP) {
                    const int slot = entry_slot(e, nf, k, nib);
                    const double2 e0 = *(const double2*)(bi + slot * CSb);
                    const double rss = i < 0 ? fma(e0.x, e0.x, e0.y) : e0.y;
                    harvest<WORLD1, HR, HB>(P, lntab, desc, lmt, bb, bm, W, w, slot, !((absent >> slot) & 1u), rss,
                                            S, S1, Kw);
                }
            } else {
                // GRC at free position i: rotate rows i, i+1 of every column after the prefix
                unsigned char* const bi = sw + i * RS;
                int e = h;
                for (; e + PP < L; e += 2 * PP) {
                    const int sa = entry_slot(e, nf, k, nib), sb = entry_slot(e + PP, nf, k, nib);
                    unsigned char* const pa = bi + sa * CSb;
                    unsigned char* const pb = bi + sb * CSb;
                    const double2 a0 = *(const double2*)pa, a1 = *(const double2*)(pa + RS);
                    const double2 b0 = *(const double2*)pb, b1 = *(const double2*)(pb + RS);
                    const double xa = fma(c, a0.x, sg * a1.x), ya = fma(c, a1.x, -sg * a0.x);
                    const double xb = fma(c, b0.x, sg * b1.x), yb = fma(c, b1.x, -sg * b0.x);
                    const double ra = fma(ya, ya, a1.y), rb = fma(yb, yb, b1.y);
                    *(double2*)pa = make_double2(xa, ra);
                    *(double*)(pa + RS) = ya;
                    *(double2*)pb = make_double2(xb, rb);
                    *(double*)(pb + RS) = yb;
                    harvest<WORLD1, HR, HB>(P, lntab, desc, lmt, bb, bm, W, w, sa, !((absent >> sa) & 1u), ra, S, S1,
                                            Kw);
                    harvest<WORLD1, HR, HB>(P, lntab, desc, lmt, bb, bm, W, w, sb, !((absent >> sb) & 1u), rb, S, S1,
                                            Kw);
                }
                if (e < L) {
                    const int sa = entry_slot(e, nf, k, nib);
                    unsigned char* const pa = bi + sa * CSb;
                    const double2 a0 = *(const double2*)pa, a1 = *(const double2*)(pa + RS);
                    const double xa = fma(c, a0.x, sg * a1.x), ya = fma(c, a1.x, -sg * a0.x);
                    const double ra = fma(ya, ya, a1.y);
                    *(double2*)pa = make_double2(xa, ra);
                    *(double*)(pa + RS) = ya;
                    harvest<WORLD1, HR, HB>(P, lntab, desc, lmt, bb, bm, W, w, sa, !((absent >> sa) & 1u), ra, S, S1,
                                            Kw);
                }
                if (h == 0) {
                    // the pivot Y (now at position i): R_i = h, U_{i+1} = 0, R_{i+1} = 0
                    unsigned char* const py = bi + (int)((rec.x >> 9) & 15u) * CSb;
                    *(double2*)py = make_double2(hh, 0.0);
                    *(double*)(py + RS) = 0.0;
                }
            }
            __syncwarp();
            if (!((nrec.x >> 18) & 1u)) {
                // the next step's rotation: entries (in, in+1) of its pivot column
                const int in = (int)(nrec.x & 31u) - 1, Yn = (int)((nrec.x >> 9) & 15u);
                const unsigned char* col = sw + in * RS + Yn * CSb;
                givens(*(const double*)col, *(const double*)(col + RS), c, sg, hh);
            }
            rec = nrec;
            // the gang's warps write the two halves of each 256 B region: keep them in step
            if (G > 1 && (t % P.bar_every) == P.bar_every - 1) __syncthreads();
        }
        __syncwarp();
        // fold the per-(slot, worker) bests into the warp's per-child best (a11)
        for (int s = 0; s < Sw; ++s) {
            double b = NINF;
            uint32_t mk = 0xffffffffu;
            if (lane < W) {
                b = bb[s * W + lane];
                mk = bm[s * W + lane];
            }
#pragma unroll
            for (int o = 1; o < W; o <<= 1) {
                const double ob = __shfl_xor_sync(FULLMASK, b, o);
                const uint32_t om = __shfl_xor_sync(FULLMASK, mk, o);
                if (better(ob, om, b, mk)) {
                    b = ob;
                    mk = om;
                }
            }
            if (lane == 0) {
                const int v = __popc(lmt[s]);
                if (better(b, mk, wbb[v], wbm[v])) {
                    wbb[v] = b;
                    wbm[v] = mk;
                }
            }
            __syncwarp();
        }
    }
    __syncwarp();
    if (lane < m) {
        const size_t row = (size_t)P.part_base + (size_t)blockIdx.x * G + wib;
        P.part_bic[row * m + lane] = wbb[lane];
        P.part_mask[row * m + lane] = wbm[lane];
    }
}

template <bool W1, bool HR, bool HB>
static cudaError_t launch_w(const TravParams& P, int grid, cudaStream_t st)
{
    const size_t smem = walk_cta_smem(P.m, P.k, P.S_alloc, P.g);
    cudaError_t e = cudaFuncSetAttribute(walk_kernel<W1, HR, HB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    walk_kernel<W1, HR, HB><<<grid, 32 << P.g, smem, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_walk(const TravParams& P, int grid, cudaStream_t st)
{
    const int key = (P.world1 ? 4 : 0) | (P.out_rss ? 2 : 0) | (P.out_bic ? 1 : 0);
    switch (key) {
        case 7: return launch_w<true, true, true>(P, grid, st);
        case 6: return launch_w<true, true, false>(P, grid, st);
        case 5: return launch_w<true, false, true>(P, grid, st);
        case 4: return launch_w<true, false, false>(P, grid, st);
        case 3: return launch_w<false, true, true>(P, grid, st);
        case 2: return launch_w<false, true, false>(P, grid, st);
        case 1: return launch_w<false, false, true>(P, grid, st);
        default: return launch_w<false, false, false>(P, grid, st);
    }
}

int walk_max_ctas_per_sm(int m, int k, int S_alloc, int g, int world1)
{
    const size_t smem = walk_cta_smem(m, k, S_alloc, g);
    int n = 0;
    auto f = world1 ? walk_kernel<true, true, true> : walk_kernel<false, true, true>;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, 32 << g, smem) != cudaSuccess) return 0;
    return n;
}

}  // namespace bnr
