// bnreg_kernels.cu -- sm_100a kernels of the bnreg hot path.
//
//   centre_kernel      a1  centre the columns (fixed-order sums), NaN/Inf flag
//   tsqr_kernel        a2  TSQR: Householder QR of 256-row leaves in shared
//                          memory, then a binary tree of [R_a; R_b] merges
//                          (last-arriving CTA merges), diag > 0, rank check
//   tree_level_kernel  a5  one level of the Alg.2 seed tree: a node's R for
//                          the residual of the not-yet-decided variables
//                          after projecting out the front set F; a pinned
//                          variable either joins F (drop the leading row and
//                          column) or the back set B (bubble it behind the
//                          free block with GRCs)
//   traverse_kernel    a5-a11 (the hot kernel): one warp runs a PACK of 4
//                          Alg.2 workers in lockstep (their pinned sets differ
//                          only in variables 0 and 1), walking d + Upsilon(k)
//                          with one GRC per step per worker, harvesting every
//                          new family from suffix sums of squares, computing
//                          its BIC, storing RSS and BIC (the 4 workers' entries
//                          of a family are adjacent -> full 32 B sectors), and
//                          keeping a per-child running best
//   best_reduce_kernel a11 deterministic argmax over per-warp bests
//
// Notation follows the paper: R the triangular factor, GRC_i the swap of
// positions i,i+1 plus one Givens rotation (Eq.3-4 with the
// fix G1: c = r_{i,i+1}/h, s = r_{i+1,i+1}/h), Upsilon(k) the greedy schedule.
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include "kernels.h"
#include "device.cuh"

namespace bnr {

// ---------------------------------------------------------------- a1 centre
// grid = m CTAs (root position j), 256 threads.  Xr is column-major n x m in
// ROOT order: Xr[:, j] = X[:, root_order[j]] - mean.
__global__ void __launch_bounds__(256) centre_kernel(const double* __restrict__ X, int64_t n, int m,
                                                     const int* __restrict__ root_order,
                                                     double* __restrict__ Xr, int* status)
{
    __shared__ double red[8];
    int j = blockIdx.x;
    int u = root_order[j];
    const double* x = X + (int64_t)u * n;
    double s = 0.0;
    bool bad = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double v = x[i];
        bad |= !isfinite(v);
        s += v;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, 2);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];   // fixed order
    double mu = tot / (double)n;
    double* y = Xr + (int64_t)j * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) y[i] = x[i] - mu;
}

// ---------------------------------------------------------------- a2 TSQR
// Householder QR in shared memory of a column-major nr x m tile (ld = nr),
// 256 threads.  On return the upper triangle holds R (diag may be negative).
__device__ void householder_tile(double* T, int nr, int m, double* sh)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int j = 0; j < m && j < nr; ++j) {
        double* cj = T + (int64_t)j * nr;
        if (warp == 0) {
            double s = 0.0;
            for (int i = j + lane; i < nr; i += 32) s = fma(cj[i], cj[i], s);
            s = warp_sum(s);
            if (lane == 0) {
                double x0 = cj[j];
                double nrm = sqrt(s);
                double alpha = (x0 > 0.0) ? -nrm : nrm;
                double v0 = x0 - alpha;
                double vtv = s - x0 * x0 + v0 * v0;
                cj[j] = v0;
                sh[0] = alpha;
                sh[1] = vtv;
            }
        }
        __syncthreads();
        double vtv = sh[1];
        if (vtv > 0.0) {
            for (int c = j + 1 + warp; c < m; c += nwarp) {
                double* cc = T + (int64_t)c * nr;
                double d = 0.0;
                for (int i = j + lane; i < nr; i += 32) d = fma(cj[i], cc[i], d);
                d = warp_sum(d);
                double f = 2.0 * d / vtv;
                for (int i = j + lane; i < nr; i += 32) cc[i] = fma(-f, cj[i], cc[i]);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) cj[j] = (vtv > 0.0) ? sh[0] : cj[j];
        for (int i = j + 1 + (int)threadIdx.x; i < nr; i += blockDim.x) cj[i] = 0.0;
        __syncthreads();
    }
}

// rbuf: heap-ordered binary tree of R's (slot 1 = root, leaves at nleaf2 + b),
// each m*m row-major.  counters: nleaf2 zeroed arrival counters (self-resetting).
__global__ void __launch_bounds__(256) tsqr_kernel(const double* __restrict__ Xr, int64_t n, int m, int rb,
                                                   double* rbuf, unsigned* counters, int nleaf2,
                                                   double* Rroot, int* status)
{
    extern __shared__ double smem[];
    __shared__ double sh[4];
    __shared__ int s_old;
    const int b = blockIdx.x;
    const int64_t r0 = (int64_t)b * rb;
    int nr = 0;
    if (r0 < n) nr = (int)((n - r0) < rb ? (n - r0) : rb);
    int nrp = nr < m ? m : nr;                    // pad to at least m rows
    double* T = smem;                             // nrp x m, column-major
    for (int c = 0; c < m; ++c)
        for (int i = threadIdx.x; i < nrp; i += blockDim.x)
            T[(int64_t)c * nrp + i] = (i < nr) ? Xr[(int64_t)c * n + r0 + i] : 0.0;
    __syncthreads();
    householder_tile(T, nrp, m, sh);
    int node = nleaf2 + b;
    double* dst = rbuf + (int64_t)node * m * m;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        int i = e / m, c = e % m;
        dst[e] = (c >= i) ? T[(int64_t)c * nrp + i] : 0.0;
    }
    while (node > 1) {
        __threadfence();
        __syncthreads();
        int parent = node >> 1;
        if (threadIdx.x == 0) s_old = (int)atomicAdd(&counters[parent], 1u);
        __syncthreads();
        if (s_old == 0) return;                   // first arriver: sibling will merge
        if (threadIdx.x == 0) counters[parent] = 0u;   // reset for the next launch
        // second arriver: stack [R_left; R_right] (2m x m) and re-factor
        const double* Lr = rbuf + (int64_t)(2 * parent) * m * m;
        const double* Rr = rbuf + (int64_t)(2 * parent + 1) * m * m;
        int nr2 = 2 * m;
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
            int i = e / m, c = e % m;
            T[(int64_t)c * nr2 + i] = __ldcg(Lr + e);
            T[(int64_t)c * nr2 + m + i] = __ldcg(Rr + e);
        }
        __syncthreads();
        householder_tile(T, nr2, m, sh);
        node = parent;
        dst = rbuf + (int64_t)node * m * m;
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
            int i = e / m, c = e % m;
            dst[e] = (c >= i) ? T[(int64_t)c * nr2 + i] : 0.0;
        }
        nrp = nr2;
    }
    // root: sign-normalise rows (diag > 0), rank check (G26)
    __syncthreads();
    const double* R = rbuf + (int64_t)1 * m * m;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        int i = e / m, c = e % m;
        double d = __ldcg(R + i * m + i);
        double v = __ldcg(R + e);
        Rroot[e] = (c < i) ? 0.0 : (d < 0.0 ? -v : v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int c = 0; c < m; ++c) {
            double s = 0.0;
            for (int i = 0; i <= c; ++i) s = fma(Rroot[i * m + c], Rroot[i * m + c], s);
            mx = fmax(mx, sqrt(s));
        }
        bool deficient = !(mx > 0.0);
        for (int j = 0; j < m; ++j)
            if (!(fabs(Rroot[j * m + j]) > 1e-12 * mx)) deficient = true;
        if (deficient) atomicOr(status, 4);
    }
}

// ---------------------------------------------------------------- GRC on a square R in smem
// A: row-major with stride SA.  Swap (physical) columns J, J+1 and restore the
// triangle with one rotation of rows J, J+1.  Columns
// J+2..end-1 are rotated; rows above J only swap their two entries.
// Warp-collective (lane = row index for the swap, column index for the rotation).
__device__ __forceinline__ void grc_square(double* A, int SA, int J, int end, int lane)
{
    double a = A[J * SA + J + 1];
    double b = A[(J + 1) * SA + J + 1];
    double rjj = A[J * SA + J];
    double c, s, h;
    givens(a, b, c, s, h);
    __syncwarp();
    int q = lane;
    if (q < J) {
        double t0 = A[q * SA + J], t1 = A[q * SA + J + 1];
        A[q * SA + J] = t1;
        A[q * SA + J + 1] = t0;
    } else if (q == J) {
        A[J * SA + J] = h;
        A[(J + 1) * SA + J] = 0.0;
        A[J * SA + J + 1] = c * rjj;
        A[(J + 1) * SA + J + 1] = -s * rjj;
    } else if (q >= J + 2 && q < end) {
        double x = A[J * SA + q], y = A[(J + 1) * SA + q];
        A[J * SA + q] = fma(c, x, s * y);
        A[(J + 1) * SA + q] = fma(c, y, -s * x);
    }
    __syncwarp();
}

// ---------------------------------------------------------------- a5 seed tree level
// One warp per child node at depth L+1.  Node layout: m*m doubles row-major,
// top-left s x s used, s = m - |F|.  Node order: [hv[L..bh-1], pack, free, B].
__global__ void __launch_bounds__(128) tree_level_kernel(const double* __restrict__ parent, double* __restrict__ child,
                                                         int m, int L, int bh, int p, int k)
{
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int SA = m | 1;
    double* A = smem + (size_t)wib * m * SA;
    const uint32_t q = (uint32_t)(blockIdx.x * (blockDim.x >> 5) + wib);
    if (q >= (1u << (L + 1))) return;
    const uint32_t par = q & ((1u << L) - 1u);
    const int bit = (q >> L) & 1;
    const int sp = m - __popc(par);
    const double* src = parent + (size_t)par * m * m;
    for (int e = lane; e < sp * sp; e += 32) {
        int r = e / sp, c = e % sp;
        A[r * SA + c] = src[r * m + c];
    }
    __syncwarp();
    int org = 0;
    if (bit) {
        org = 1;
    } else {
        int T = (bh - L - 1) + p + k;
        for (int j = 0; j < T; ++j) grc_square(A, SA, j, sp, lane);
    }
    const int sc = sp - bit;
    double* dst = child + (size_t)q * m * m;
    for (int e = lane; e < sc * sc; e += 32) {
        int r = e / sc, c = e % sc;
        dst[r * m + c] = A[(org + r) * SA + org + c];
    }
}

// ---------------------------------------------------------------- walk state layout
// Per warp (one pack = 4 workers w):
//   W[w]  column-contiguous walk state, for every slot s (a column of the
//         worker's R restricted to its k free rows) the k pairs
//           E_l = (R_l, U_{l+1}),  l = 0..k-1,
//         U_l = sum_{r >= l} R_r^2 (+ the tail below the free rows for back
//         columns): a GRC at free position i reads E_i, E_{i+1} and writes
//         E_i = (R'_i, U'_{i+1}), E_{i+1}.x = R'_{i+1}  (a8: suffix sums by
//         addition only).  Column stride CS = 16 (k|1) bytes (odd number of
//         16 B units), worker stride WS = 16 ws16 with ws16 = 2 (mod 8): the 8
//         lanes of an LDS.128 phase hit distinct bank groups.
//   A     the packed seed triangle of the derivation; it overlaps the region
//         of the worker snapshotted last (placed last in memory).
//   rec   per slot: row pointers (this child's block of the RSS / BIC table)
//   bb,bm per child: the warp's running best (a11)
struct WarpSmem {
    unsigned char* Wb;      // worker regions
    double* A;              // packed derivation triangle
    ulonglong2* rec;        // [32] (rss row ptr, bic row ptr)
    double* bb;             // [32]
    uint32_t* bm;           // [32]
    uint8_t* slotvar;       // [32] slot -> user id
};

__host__ __device__ inline void walk_geometry(int m, int k, int& CS, int& WS)
{
    const int cs16 = k | 1;
    int ws16 = m * cs16;
    ws16 += (2 - (ws16 & 7) + 8) & 7;
    CS = cs16 * 16;
    WS = ws16 * 16;
}

__host__ __device__ inline size_t warp_smem_bytes(int m, int k)
{
    int CS, WS;
    walk_geometry(m, k, CS, WS);
    size_t asz = (size_t)(m * (m + 1) / 2) * 8;
    size_t w = (size_t)4 * WS;
    if ((size_t)3 * WS + asz > w) w = (size_t)3 * WS + asz;
    size_t tot = w + 32 * 16 + 32 * 8 + 32 * 4 + 32;
    return (tot + 15) & ~(size_t)15;
}

size_t traverse_smem_per_warp(int m, int k) { return warp_smem_bytes(m, k); }

// region index of worker w: the worker snapshotted last owns the last region
__device__ __forceinline__ int region_of(int w, int p)
{
    const int last = (p == 2) ? 2 : 0;
    return w == last ? 3 : (w < last ? w : w - 1);
}

// Logical position (relative to the snapshot origin) of a walk slot for worker
// w, or -1 when the slot's variable is in that worker's front set.
__device__ __forceinline__ int slot_pos(int slot, int w, int k, int p, int nw)
{
    if (slot < k) return slot;
    if (slot < k + p) {
        int j = slot - k;
        if ((w >> j) & 1) return -1;
        uint32_t absent_below = (~(uint32_t)w) & ((1u << j) - 1u) & (uint32_t)(nw - 1);
        return k + __popc(absent_below);
    }
    int present = p - __popc((uint32_t)w & (uint32_t)(nw - 1));
    return k + present + (slot - k - p);
}

// Snapshot: convert the sub-triangle of A starting at physical origin `org`
// (side s) into worker w's walk state (E pairs of its slots).  The seed
// prefixes are harvested afterwards by the walk's seed pseudo-steps.  Lanes =
// walk slots.  STAGE: A overlaps this worker's region, so each lane first
// reads its whole column into registers.
template <bool STAGE>
__device__ void snapshot(const TravParams& P, const WarpSmem& ws, int s, int org, int w, int lane, int CS, int WS,
                         int ncsp)
{
    const int k = P.k;
    if (w >= P.nw) return;
    const int slot = lane;
    const int pos = (slot < ncsp) ? slot_pos(slot, w, k, P.p, P.nw) : -1;
    double col[STAGE ? 32 : 1];
    if (STAGE) {
#pragma unroll
        for (int r = 0; r < 32; ++r)
            col[r] = (r <= pos) ? ws.A[poff(org + r, s) + pos - r] : 0.0;
        __syncwarp();
    }
    double* E = (double*)(ws.Wb + region_of(w, P.p) * WS + slot * CS);
    if (slot < P.m) {
        for (int l = 0; l < k; ++l) { E[2 * l] = 0.0; E[2 * l + 1] = 0.0; }
        double acc = 0.0;
        if (STAGE) {
#pragma unroll
            for (int r = 31; r >= 0; --r) {
                if (r <= pos) {
                    const double x = col[r];
                    acc = fma(x, x, acc);
                    if (r < k) E[2 * r] = x;
                    if (r >= 1 && r <= k) E[2 * (r - 1) + 1] = acc;       // U_r
                }
            }
        } else {
            for (int r = pos; r >= 0; --r) {
                const double x = ws.A[poff(org + r, s) + pos - r];
                acc = fma(x, x, acc);
                if (r < k) E[2 * r] = x;
                if (r >= 1 && r <= k) E[2 * (r - 1) + 1] = acc;           // U_r
            }
        }
    }
    __syncwarp();
}

struct StepCtx {
    unsigned char* wl;     // this lane's worker region
    int CS;
    double c, sn, h;       // the GRC's rotation and the new diagonal
    uint32_t S, S1;        // new prefix set of this worker (user ids), S >> 1
    double Kw;             // BIC constant for |S|
    int X, Y, i, nf, L, cl, k;
    uint32_t lo, hi;       // free slots at positions i+1.. (nibbles)
    uint32_t absent;       // slots whose variable is in this worker's front set
    int in, Yn;            // next step's position / pivot (in < 0: no Givens needed)
};

// One lockstep step over NCH chunks of 8 list entries per worker (list = the
// free slots at positions i+1.., then the back slots).
//   SEED: a seed pseudo-step harvests prefix j = i+1 of the seed order:
//         RSS = U_j = E_i.y (U_0 = E_0.x^2 + E_0.y).
//   else: (A) the GRC at i: rotate rows i, i+1, new suffix sums, store state;
//   (B) the NEXT step's Givens coefficients (only needs values (A) stored);
//   (C) this step's harvest: index, log, BIC, table stores, running best.
//   (B) and (C) are independent chains; so are the NCH families of a lane.
template <bool WORLD1, bool HR, bool HB, bool SEED, int NCH>
__device__ __forceinline__ void walk_step(const TravParams& P, const double2* lntab, const WarpSmem& ws,
                                          const StepCtx& s, double& cn, double& snn, double& hn)
{
    int slot[NCH];
    bool act[NCH];
    double rss[NCH];
    const int sh = 4 * s.cl;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        const int e = s.cl + 8 * q;
        act[q] = e < s.L;
        int sl;
        if (q == 0) sl = (e < s.nf) ? (int)((s.lo >> sh) & 15u) : s.k + e - s.nf;
        else if (q == 1) sl = (e < s.nf) ? (int)((s.hi >> sh) & 15u) : s.k + e - s.nf;
        else sl = s.k + e - s.nf;
        slot[q] = act[q] ? sl : 0;
    }
    if (SEED) {
        const int i0 = s.i < 0 ? 0 : s.i;
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
            const double2 e0 = *(const double2*)(s.wl + slot[q] * s.CS + 16 * i0);
            rss[q] = (s.i < 0) ? fma(e0.x, e0.x, e0.y) : e0.y;
        }
    } else {
        unsigned char* const base = s.wl + 16 * s.i;
        double2 e0[NCH], e1[NCH];
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
            const unsigned char* col = base + slot[q] * s.CS;
            e0[q] = *(const double2*)col;
            e1[q] = *(const double2*)(col + 16);
        }
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
            const double xn = fma(s.c, e0[q].x, s.sn * e1[q].x);
            const double yn = fma(s.c, e1[q].x, -s.sn * e0[q].x);
            rss[q] = fma(yn, yn, e1[q].y);
            if (act[q]) {
                unsigned char* col = base + slot[q] * s.CS;
                *(double2*)col = make_double2(xn, rss[q]);
                *(double*)(col + 16) = yn;
            }
        }
        if (s.cl == 0) {
            unsigned char* col = base + s.Y * s.CS;
            *(double2*)col = make_double2(s.h, 0.0);   // Y now at position i: (h, U_{i+1} = 0)
            *(double*)(col + 16) = 0.0;                // R_{i+1} = 0
        }
    }
    __syncwarp();
#ifdef BNREG_STEP_CLOCKS
    if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0 && P.dbg[0] < 4000) P.dbg[2 + 3 * P.dbg[0]] = clock64();
#endif
    // ---- (B) next step's rotation
    if (s.in >= 0) {
        const unsigned char* col = s.wl + 16 * s.in + s.Yn * s.CS;
        givens(*(const double*)col, *(const double*)(col + 16), cn, snn, hn);
    }
    // ---- (C)
    bool hv[NCH];
    double bic[NCH];
    ulonglong2 rp[NCH];
    uint32_t off[NCH];
    int vv[NCH];
    bool up = false;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        hv[q] = act[q] && !((s.absent >> slot[q]) & 1u);
        const int v = ws.slotvar[slot[q]];
        vv[q] = v;
        off[q] = block_offset<WORLD1>(P, s.S, s.S1, (1u << v) - 1u);
        rp[q] = ws.rec[slot[q]];
        bic[q] = bic_of(rss[q], fast_ln(rss[q], lntab), P.mhalf_n, s.Kw);   // rss <= 1e-300 -> +inf
        up |= hv[q] && bic[q] >= ws.bb[v];
    }
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        if (hv[q]) {
            if (HR) __stcs((double*)rp[q].x + off[q], rss[q]);
            if (HB) __stcs((double*)rp[q].y + off[q], bic[q]);
        }
    }
    // running best (a11): the 4 lanes of a column group share a child; record
    // improvements are rare, so they are resolved lane by lane (ascending id)
    unsigned bal = __ballot_sync(FULLMASK, up);
    while (bal) {
        const int l = __ffs(bal) - 1;
        bal &= bal - 1;
        if ((int)(threadIdx.x & 31) == l) {
#pragma unroll
            for (int q = 0; q < NCH; ++q) {
                const int v = vv[q];
                if (hv[q] && tie_better(bic[q], s.S, ws.bb[v], ws.bm[v])) {
                    ws.bb[v] = bic[q];
                    ws.bm[v] = s.S;
                }
            }
        }
        __syncwarp();
    }
}

template <bool WORLD1, bool HR, bool HB>
__global__ void __launch_bounds__(128) traverse_kernel(const __grid_constant__ TravParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double2 s_lntab[128];
    __shared__ uint32_t s_item;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g;
    const int fv0 = p + g;                      // user id of free slot 0
    for (int j = threadIdx.x; j < 128; j += blockDim.x) s_lntab[j] = P.lntab[j];
    __syncthreads();
    int CS, WS;
    walk_geometry(m, k, CS, WS);
    const double K0 = P.Kc[0];
    const double mhlnn = P.Kc[1] - P.Kc[0];     // -(1/2) ln n
    const size_t per = warp_smem_bytes(m, k);
    unsigned char* base = smem_raw + (size_t)wib * per;
    size_t wbytes = (size_t)4 * WS;
    {
        size_t asz = (size_t)(m * (m + 1) / 2) * 8;
        if ((size_t)3 * WS + asz > wbytes) wbytes = (size_t)3 * WS + asz;
    }
    WarpSmem ws;
    ws.Wb = base;
    ws.A = (double*)(base + 3 * WS);
    ws.rec = (ulonglong2*)(base + wbytes);
    ws.bb = (double*)(ws.rec + 32);
    ws.bm = (uint32_t*)(ws.bb + 32);
    ws.slotvar = (uint8_t*)(ws.bm + 32);

    ws.bb[lane] = -__longlong_as_double(0x7ff0000000000000LL);
    ws.bm[lane] = 0xffffffffu;
    __syncwarp();
    const int gwarp = blockIdx.x * (blockDim.x >> 5) + wib;
    const int w = lane & 3;           // worker of this lane within the pack
    const int cl = lane >> 2;         // lane's column group (0..7)
    // slots of pack variables in a worker's front set are never harvested
    uint32_t absent = 0;
    if (w >= P.nw) absent = 0xffffffffu;
    else
        for (int j = 0; j < p; ++j)
            if ((w >> j) & 1) absent |= 1u << (k + j);
    unsigned char* const Wlane = ws.Wb + region_of(w, p) * WS;
    const int shb = WORLD1 ? m - 1 : m - P.r;   // child block = v << shb entries

    for (;;) {
        // one work item = one gang: the CTA's 2^g warps take the 2^g packs that
        // differ in the gang variables and walk them in lockstep
        if (threadIdx.x == 0) s_item = atomicAdd(P.counter, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        __syncthreads();
        if ((int)item >= P.npacks) break;
        const uint32_t pack = P.packs[item] | ((uint32_t)wib << (bh - g));

        // ---- seed: load the depth-L1 node, derive the remaining tree levels (a5)
        const uint32_t nid = pack & ((1u << P.L1) - 1u);
        const int sn = m - __popc(nid);
        const double* src = P.nodes + (size_t)nid * m * m;
        {
            // all loads in flight at once (the node comes from HBM/L2): cp.async 8 B per entry
            const int tot = sn * (sn + 1) / 2;
            for (int e = lane; e < tot; e += 32) {
                // packed index e -> (r, c): row r starts at poff(r, sn)
                int r = (int)((2.0f * sn + 1.0f - sqrtf((2.0f * sn + 1.0f) * (2.0f * sn + 1.0f) - 8.0f * e)) * 0.5f);
                if (r < 0) r = 0;
                while (r > 0 && poff(r, sn) > e) --r;
                while (r + 1 < sn && poff(r + 1, sn) <= e) ++r;
                const int c = r + (e - poff(r, sn));
                const unsigned sa = (unsigned)__cvta_generic_to_shared(ws.A + e);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa), "l"(src + r * m + c));
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
        }
        int org = 0;
        for (int l = P.L1; l < bh; ++l) {
            if ((pack >> l) & 1u) {
                ++org;
            } else {
                const int T = (bh - l - 1) + p + k;
                for (int j = 0; j < T; ++j) grc_packed(ws.A, sn, org + j, sn, lane);
            }
        }
        uint32_t Fhi = 0;                                   // tree-level vars in F (user ids)
        for (int l = 0; l < bh; ++l)
            if ((pack >> l) & 1u) Fhi |= 1u << (l < bh - g ? m - 1 - l : fv0 - 1 - (l - (bh - g)));
        const int dh = __popc(pack);
        const int NCSp = k + p + (bh - dh);                 // slots in use for this pack
        {
            int v = 0;
            if (lane < k) v = fv0 + lane;
            else if (lane < k + p) v = lane - k;
            else if (lane < NCSp) {
                // back set: tree-level vars not in F, ascending id (= latest deferred first)
                int q = lane - k - p, cnt = 0;
                for (int id = p; id < m; ++id) {
                    if (id >= fv0 && id < fv0 + k) continue;
                    if (!((Fhi >> id) & 1u)) { if (cnt == q) { v = id; break; } ++cnt; }
                }
            }
            ws.slotvar[lane] = (uint8_t)v;
            ws.rec[lane] = make_ulonglong2(
                HR ? (unsigned long long)(P.out_rss + ((long long)v << shb)) : 0ull,
                HB ? (unsigned long long)(P.out_bic + ((long long)v << shb)) : 0ull);
        }
        __syncwarp();

        // ---- pack derivation: the 2^p workers' seeds along one GRC path (a5)
        const int o = org, sz = sn, end = sn;
        if (p == 2) {
            snapshot<false>(P, ws, sz, o + 2, 3, lane, CS, WS, NCSp);
            for (int j = 1; j <= k; ++j) grc_packed(ws.A, sz, o + j, end, lane);
            snapshot<false>(P, ws, sz, o + 1, 1, lane, CS, WS, NCSp);
            for (int j = 0; j < k; ++j) grc_packed(ws.A, sz, o + j, end, lane);
            snapshot<false>(P, ws, sz, o, 0, lane, CS, WS, NCSp);
            for (int j = k; j >= 0; --j) grc_packed(ws.A, sz, o + j, end, lane);
            snapshot<true>(P, ws, sz, o + 1, 2, lane, CS, WS, NCSp);
        } else if (p == 1) {
            snapshot<false>(P, ws, sz, o + 1, 1, lane, CS, WS, NCSp);
            for (int j = 0; j < k; ++j) grc_packed(ws.A, sz, o + j, end, lane);
            snapshot<true>(P, ws, sz, o, 0, lane, CS, WS, NCSp);
        } else {
            snapshot<true>(P, ws, sz, o, 0, lane, CS, WS, NCSp);
        }

        // ---- the walk: k+1 seed pseudo-steps, then d + Upsilon(k), in lockstep (a6-a11)
        const uint32_t Fw = Fhi | (uint32_t)w;          // pack var j = user id j
        const int dw = dh + __popc((uint32_t)w);
        const int NBp = NCSp - k;
        double c = 1.0, sg = 0.0, h = 0.0;
        uint4 rec = __ldg(P.steps);
        for (int t = 0; t < P.nsteps; ++t) {
            const uint4 nrec = (t + 1 < P.nsteps) ? __ldg(P.steps + t + 1) : make_uint4(1u << 18, 0, 0, 0);
            const int i = (int)(rec.x & 31u) - 1;
            const bool seed = (rec.x >> 18) & 1u;
            const int nf = (int)((rec.x >> 13) & 31u);
            const int L = nf + NBp;
            const uint32_t S = Fw | (rec.y << fv0);
            const bool nreal = !((nrec.x >> 18) & 1u);
            StepCtx sc{Wlane, CS, c, sg, h, S, S >> 1, fma((double)(dw + i + 1), mhlnn, K0),
                       (int)((rec.x >> 5) & 15u), (int)((rec.x >> 9) & 15u), i, nf, L, cl, k, rec.z, rec.w, absent,
                       nreal ? (int)(nrec.x & 31u) - 1 : -1, (int)((nrec.x >> 9) & 15u)};
            double cn = 1.0, snn = 0.0, hn = 0.0;
            const int nch = (L + 7) >> 3;
#ifdef BNREG_STEP_CLOCKS
            if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0 && P.dbg[0] < 4000) P.dbg[1 + 3 * P.dbg[0]] = clock64();
#endif
            if (seed) {
                switch (nch) {
                    case 1: walk_step<WORLD1, HR, HB, true, 1>(P, s_lntab, ws, sc, cn, snn, hn); break;
                    case 2: walk_step<WORLD1, HR, HB, true, 2>(P, s_lntab, ws, sc, cn, snn, hn); break;
                    case 3: walk_step<WORLD1, HR, HB, true, 3>(P, s_lntab, ws, sc, cn, snn, hn); break;
                    default: walk_step<WORLD1, HR, HB, true, 4>(P, s_lntab, ws, sc, cn, snn, hn); break;
                }
            } else {
                switch (nch) {
                    case 1: walk_step<WORLD1, HR, HB, false, 1>(P, s_lntab, ws, sc, cn, snn, hn); break;
                    case 2: walk_step<WORLD1, HR, HB, false, 2>(P, s_lntab, ws, sc, cn, snn, hn); break;
                    case 3: walk_step<WORLD1, HR, HB, false, 3>(P, s_lntab, ws, sc, cn, snn, hn); break;
                    default: walk_step<WORLD1, HR, HB, false, 4>(P, s_lntab, ws, sc, cn, snn, hn); break;
                }
            }
#ifdef BNREG_STEP_CLOCKS
            if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0 && P.dbg[0] < 4000) {
                P.dbg[3 + 3 * P.dbg[0]] = clock64();
                P.dbg[0] += 1;
            }
#endif
            c = cn; sg = snn; h = hn;
            rec = nrec;
            // the gang's warps write one 128 B line per (child, T): keep them
            // within a few steps of each other (lines complete in L2 long
            // before eviction) without paying a barrier every step
            if (g && ((t & 3) == 3 || t + 1 == P.nsteps)) __syncthreads();
            else __syncwarp();
        }
    }
    // ---- per-warp best -> global partials (a11)
    __syncwarp();
    if (lane < m) {
        P.part_bic[(size_t)gwarp * m + lane] = ws.bb[lane];
        P.part_mask[(size_t)gwarp * m + lane] = ws.bm[lane];
    }
}

// ---------------------------------------------------------------- warp-specialised traversal
// The harvest (a8-a11: index, log, BIC, table stores, best) needs none of the
// per-pack walk state except the suffix sums the GRC just stored, so each pack
// gets a PRODUCER warp (seed derivation + the GRCs, state in shared memory) and
// a CONSUMER warp (the harvest of step t, read from the state while the
// producer already runs step t+1).  A CTA = a gang of 2^g packs = 2^(g+1)
// warps; one named barrier per pack per step.  Safety of the overlap: the GRC
// at step t+1 (position i +- 1) and its pivot update never write E_i.y, the
// value the consumer reads for step t, and the producer cannot get two steps
// ahead of the pack barrier.
__host__ __device__ inline size_t pack_smem_bytes(int m, int k)
{
    int CS, WS;
    walk_geometry(m, k, CS, WS);
    size_t asz = (size_t)(m * (m + 1) / 2) * 8;
    size_t w = (size_t)4 * WS;
    if ((size_t)3 * WS + asz > w) w = (size_t)3 * WS + asz;
    size_t tot = w + 32 * 16 + 32;          // state (+ derivation triangle), rec, slotvar
    return (tot + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t ws_cta_smem(int m, int k, int G)
{
    return (pack_smem_bytes(m, k) + 32 * 8 + 32 * 4) * (size_t)G;   // + consumer best arrays
}

__device__ __forceinline__ void named_bar(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <bool WORLD1, bool HR, bool HB, int NCH>
__device__ __forceinline__ void consume_step(const TravParams& P, const double2* lntab, const WarpSmem& ws,
                                             const unsigned char* wl, int CS, int i, int nf, int L, int cl, int k,
                                             uint32_t lo, uint32_t hi, uint32_t absent, uint32_t S, double Kw)
{
    const int sh = 4 * cl;
    const uint32_t S1 = S >> 1;
    int slot[NCH];
    bool hv[NCH];
    double rss[NCH], bic[NCH];
    ulonglong2 rp[NCH];
    uint32_t off[NCH];
    int vv[NCH];
    bool up = false;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        const int e = cl + 8 * q;
        const bool act = e < L;
        int sl;
        if (q == 0) sl = (e < nf) ? (int)((lo >> sh) & 15u) : k + e - nf;
        else if (q == 1) sl = (e < nf) ? (int)((hi >> sh) & 15u) : k + e - nf;
        else sl = k + e - nf;
        slot[q] = act ? sl : 0;
        hv[q] = act && !((absent >> slot[q]) & 1u);
        const double2 e0 = *(const double2*)(wl + slot[q] * CS + 16 * (i < 0 ? 0 : i));
        rss[q] = (i < 0) ? fma(e0.x, e0.x, e0.y) : e0.y;      // U_0, or U_{i+1} = E_i.y
    }
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        const int v = ws.slotvar[slot[q]];
        vv[q] = v;
        off[q] = block_offset<WORLD1>(P, S, S1, (1u << v) - 1u);
        rp[q] = ws.rec[slot[q]];
        bic[q] = bic_of(rss[q], fast_ln(rss[q], lntab), P.mhalf_n, Kw);   // rss <= 1e-300 -> +inf
        up |= hv[q] && bic[q] >= ws.bb[v];
    }
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        if (hv[q]) {
            if (HR) __stcs((double*)rp[q].x + off[q], rss[q]);
            if (HB) __stcs((double*)rp[q].y + off[q], bic[q]);
        }
    }
    unsigned bal = __ballot_sync(FULLMASK, up);
    while (bal) {
        const int l = __ffs(bal) - 1;
        bal &= bal - 1;
        if ((int)(threadIdx.x & 31) == l) {
#pragma unroll
            for (int q = 0; q < NCH; ++q) {
                const int v = vv[q];
                if (hv[q] && tie_better(bic[q], S, ws.bb[v], ws.bm[v])) {
                    ws.bb[v] = bic[q];
                    ws.bm[v] = S;
                }
            }
        }
        __syncwarp();
    }
}

template <int NCH>
__device__ __forceinline__ void produce_step(unsigned char* wl, int CS, int i, int X, int Y, int nf, int L, int cl,
                                             int k, uint32_t lo, uint32_t hi, double c, double sn, double h)
{
    const int sh = 4 * cl;
    unsigned char* const base = wl + 16 * i;
    int slot[NCH];
    bool act[NCH];
    double2 e0[NCH], e1[NCH];
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        const int e = cl + 8 * q;
        act[q] = e < L;
        int sl;
        if (q == 0) sl = (e < nf) ? (int)((lo >> sh) & 15u) : k + e - nf;
        else if (q == 1) sl = (e < nf) ? (int)((hi >> sh) & 15u) : k + e - nf;
        else sl = k + e - nf;
        slot[q] = act[q] ? sl : 0;
        const unsigned char* col = base + slot[q] * CS;
        e0[q] = *(const double2*)col;
        e1[q] = *(const double2*)(col + 16);
    }
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        const double xn = fma(c, e0[q].x, sn * e1[q].x);
        const double yn = fma(c, e1[q].x, -sn * e0[q].x);
        const double r = fma(yn, yn, e1[q].y);
        if (act[q]) {
            unsigned char* col = base + slot[q] * CS;
            *(double2*)col = make_double2(xn, r);
            *(double*)(col + 16) = yn;
        }
    }
    if (cl == 0) {
        unsigned char* col = base + Y * CS;
        *(double2*)col = make_double2(h, 0.0);   // Y now at position i: (h, U_{i+1} = 0)
        *(double*)(col + 16) = 0.0;              // R_{i+1} = 0
    }
    (void)X;
}

template <bool WORLD1, bool HR, bool HB>
__global__ void __launch_bounds__(256, 3) traverse_ws_kernel(const __grid_constant__ TravParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double2 s_lntab[128];
    __shared__ uint32_t s_item;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int m = P.m, k = P.k, p = P.p, bh = P.bh, g = P.g;
    const int G = 1 << g;
    const int pk = wib & (G - 1);            // pack of this warp within the gang
    const bool producer = wib < G;
    const int fv0 = p + g;
    for (int j = threadIdx.x; j < 128; j += blockDim.x) s_lntab[j] = P.lntab[j];
    int CS, WS;
    walk_geometry(m, k, CS, WS);
    const double K0 = P.Kc[0];
    const double mhlnn = P.Kc[1] - P.Kc[0];     // -(1/2) ln n
    const size_t per = pack_smem_bytes(m, k);
    unsigned char* base = smem_raw + (size_t)pk * per;
    size_t wbytes = (size_t)4 * WS;
    {
        size_t asz = (size_t)(m * (m + 1) / 2) * 8;
        if ((size_t)3 * WS + asz > wbytes) wbytes = (size_t)3 * WS + asz;
    }
    WarpSmem ws;
    ws.Wb = base;
    ws.A = (double*)(base + 3 * WS);
    ws.rec = (ulonglong2*)(base + wbytes);
    ws.slotvar = (uint8_t*)(ws.rec + 32);
    ws.bb = (double*)(smem_raw + (size_t)G * per + (size_t)pk * (32 * 8 + 32 * 4));
    ws.bm = (uint32_t*)(ws.bb + 32);
    if (!producer) {
        ws.bb[lane] = -__longlong_as_double(0x7ff0000000000000LL);
        ws.bm[lane] = 0xffffffffu;
    }
    __syncthreads();
    const int gwarp = blockIdx.x * (blockDim.x >> 5) + wib;
    const int w = lane & 3;           // worker of this lane within the pack
    const int cl = lane >> 2;         // lane's column group (0..7)
    uint32_t absent = 0;
    if (w >= P.nw) absent = 0xffffffffu;
    else
        for (int j = 0; j < p; ++j)
            if ((w >> j) & 1) absent |= 1u << (k + j);
    unsigned char* const Wlane = ws.Wb + region_of(w, p) * WS;
    const int shb = WORLD1 ? m - 1 : m - P.r;   // child block = v << shb entries
    const int pbar = 1 + pk;                     // named barrier of this pack (producer + consumer)

    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(P.counter, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        __syncthreads();
        if ((int)item >= P.npacks) break;
        const uint32_t pack = P.packs[item] | ((uint32_t)pk << (bh - g));
        uint32_t Fhi = 0;                                   // tree-level vars in F (user ids)
        for (int l = 0; l < bh; ++l)
            if ((pack >> l) & 1u) Fhi |= 1u << (l < bh - g ? m - 1 - l : fv0 - 1 - (l - (bh - g)));
        const int dh = __popc(pack);
        const int NCSp = k + p + (bh - dh);
        const int NBp = NCSp - k;
        const uint32_t Fw = Fhi | (uint32_t)w;
        const int dw = dh + __popc((uint32_t)w);

        if (producer) {
            // ---- seed: node load, remaining tree levels, slot tables, pack derivation (a5)
            const uint32_t nid = pack & ((1u << P.L1) - 1u);
            const int sn = m - __popc(nid);
            const double* src = P.nodes + (size_t)nid * m * m;
            {
                const int tot = sn * (sn + 1) / 2;
                for (int e = lane; e < tot; e += 32) {
                    int r = (int)((2.0f * sn + 1.0f - sqrtf((2.0f * sn + 1.0f) * (2.0f * sn + 1.0f) - 8.0f * e)) * 0.5f);
                    if (r < 0) r = 0;
                    while (r > 0 && poff(r, sn) > e) --r;
                    while (r + 1 < sn && poff(r + 1, sn) <= e) ++r;
                    const int c = r + (e - poff(r, sn));
                    const unsigned sa = (unsigned)__cvta_generic_to_shared(ws.A + e);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + r * m + c));
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
            }
            int org = 0;
            for (int l = P.L1; l < bh; ++l) {
                if ((pack >> l) & 1u) {
                    ++org;
                } else {
                    const int T = (bh - l - 1) + p + k;
                    for (int j = 0; j < T; ++j) grc_packed(ws.A, sn, org + j, sn, lane);
                }
            }
            {
                int v = 0;
                if (lane < k) v = fv0 + lane;
                else if (lane < k + p) v = lane - k;
                else if (lane < NCSp) {
                    int q = lane - k - p, cnt = 0;
                    for (int id = p; id < m; ++id) {
                        if (id >= fv0 && id < fv0 + k) continue;
                        if (!((Fhi >> id) & 1u)) { if (cnt == q) { v = id; break; } ++cnt; }
                    }
                }
                ws.slotvar[lane] = (uint8_t)v;
                ws.rec[lane] = make_ulonglong2(
                    HR ? (unsigned long long)(P.out_rss + ((long long)v << shb)) : 0ull,
                    HB ? (unsigned long long)(P.out_bic + ((long long)v << shb)) : 0ull);
            }
            __syncwarp();
            const int o = org, sz = sn, end = sn;
            if (p == 2) {
                snapshot<false>(P, ws, sz, o + 2, 3, lane, CS, WS, NCSp);
                for (int j = 1; j <= k; ++j) grc_packed(ws.A, sz, o + j, end, lane);
                snapshot<false>(P, ws, sz, o + 1, 1, lane, CS, WS, NCSp);
                for (int j = 0; j < k; ++j) grc_packed(ws.A, sz, o + j, end, lane);
                snapshot<false>(P, ws, sz, o, 0, lane, CS, WS, NCSp);
                for (int j = k; j >= 0; --j) grc_packed(ws.A, sz, o + j, end, lane);
                snapshot<true>(P, ws, sz, o + 1, 2, lane, CS, WS, NCSp);
            } else if (p == 1) {
                snapshot<false>(P, ws, sz, o + 1, 1, lane, CS, WS, NCSp);
                for (int j = 0; j < k; ++j) grc_packed(ws.A, sz, o + j, end, lane);
                snapshot<true>(P, ws, sz, o, 0, lane, CS, WS, NCSp);
            } else {
                snapshot<true>(P, ws, sz, o, 0, lane, CS, WS, NCSp);
            }
            // ---- the GRCs (a6, a7, a8's suffix sums); step t's state is released to the consumer
            double c = 1.0, sg = 0.0, h = 0.0;
            uint4 rec = __ldg(P.steps);
            for (int t = 0; t < P.nsteps; ++t) {
                const uint4 nrec = (t + 1 < P.nsteps) ? __ldg(P.steps + t + 1) : make_uint4(1u << 18, 0, 0, 0);
                if (!((rec.x >> 18) & 1u)) {
                    const int i = (int)(rec.x & 31u) - 1;
                    const int nf = (int)((rec.x >> 13) & 31u);
                    const int L = nf + NBp;
                    const int X = (int)((rec.x >> 5) & 15u), Y = (int)((rec.x >> 9) & 15u);
                    switch ((L + 7) >> 3) {
                        case 1: produce_step<1>(Wlane, CS, i, X, Y, nf, L, cl, k, rec.z, rec.w, c, sg, h); break;
                        case 2: produce_step<2>(Wlane, CS, i, X, Y, nf, L, cl, k, rec.z, rec.w, c, sg, h); break;
                        case 3: produce_step<3>(Wlane, CS, i, X, Y, nf, L, cl, k, rec.z, rec.w, c, sg, h); break;
                        default: produce_step<4>(Wlane, CS, i, X, Y, nf, L, cl, k, rec.z, rec.w, c, sg, h); break;
                    }
                }
                __syncwarp();
                named_bar(pbar, 64);                 // step t's state is complete
                if (!((nrec.x >> 18) & 1u)) {        // next step's Givens (reads only)
                    const int in = (int)(nrec.x & 31u) - 1, Yn = (int)((nrec.x >> 9) & 15u);
                    const unsigned char* col = Wlane + 16 * in + Yn * CS;
                    givens(*(const double*)col, *(const double*)(col + 16), c, sg, h);
                }
                rec = nrec;
                if (g && (t & 7) == 7) __syncthreads();
            }
        } else {
            // ---- the harvest of every step (a8-a11)
            for (int t = 0; t < P.nsteps; ++t) {
                named_bar(pbar, 64);
                const uint4 rec = __ldg(P.steps + t);
                const int i = (int)(rec.x & 31u) - 1;
                const int nf = (int)((rec.x >> 13) & 31u);
                const int L = nf + NBp;
                const uint32_t S = Fw | (rec.y << fv0);
                const double Kw = fma((double)(dw + i + 1), mhlnn, K0);
                switch ((L + 7) >> 3) {
                    case 1: consume_step<WORLD1, HR, HB, 1>(P, s_lntab, ws, Wlane, CS, i, nf, L, cl, k, rec.z, rec.w, absent, S, Kw); break;
                    case 2: consume_step<WORLD1, HR, HB, 2>(P, s_lntab, ws, Wlane, CS, i, nf, L, cl, k, rec.z, rec.w, absent, S, Kw); break;
                    case 3: consume_step<WORLD1, HR, HB, 3>(P, s_lntab, ws, Wlane, CS, i, nf, L, cl, k, rec.z, rec.w, absent, S, Kw); break;
                    default: consume_step<WORLD1, HR, HB, 4>(P, s_lntab, ws, Wlane, CS, i, nf, L, cl, k, rec.z, rec.w, absent, S, Kw); break;
                }
                if (g && (t & 7) == 7) __syncthreads();
            }
        }
    }
    __syncwarp();
    if (!producer && lane < m) {
        P.part_bic[(size_t)gwarp * m + lane] = ws.bb[lane];
        P.part_mask[(size_t)gwarp * m + lane] = ws.bm[lane];
    } else if (producer && lane < m) {
        P.part_bic[(size_t)gwarp * m + lane] = -__longlong_as_double(0x7ff0000000000000LL);
        P.part_mask[(size_t)gwarp * m + lane] = 0xffffffffu;
    }
}

__global__ void debug_ln_kernel(const double* x, double* y, int64_t n, const double2* tab)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = fast_ln9(x[i], tab);   // the walk kernel's log (512-entry table)
}

cudaError_t launch_debug_ln(const double* x, double* y, int64_t n, const double2* tab, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    debug_ln_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, y, n, tab);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a11 best reduce
// One CTA per child: strided scan over the per-warp partials, then a fixed
// tree reduction -> deterministic.
__global__ void __launch_bounds__(256) best_reduce_kernel(const double* __restrict__ part_bic,
                                                          const uint32_t* __restrict__ part_mask, int nparts, int m,
                                                          double* best_bic, uint32_t* best_mask)
{
    __shared__ double sb[256];
    __shared__ uint32_t sm[256];
    const int v = blockIdx.x;
    double bb = -__longlong_as_double(0x7ff0000000000000LL);
    uint32_t bm = 0xffffffffu;
    for (int q = threadIdx.x; q < nparts; q += blockDim.x) {
        double b = part_bic[(size_t)q * m + v];
        uint32_t mk = part_mask[(size_t)q * m + v];
        if (better(b, mk, bb, bm)) { bb = b; bm = mk; }
    }
    sb[threadIdx.x] = bb;
    sm[threadIdx.x] = bm;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o && better(sb[threadIdx.x + o], sm[threadIdx.x + o], sb[threadIdx.x], sm[threadIdx.x])) {
            sb[threadIdx.x] = sb[threadIdx.x + o];
            sm[threadIdx.x] = sm[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        best_bic[v] = sb[0];
        best_mask[v] = sm[0];
    }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_centre(const double* X, int64_t n, int m, const int* root_order_dev, double* Xr, int* status,
                          cudaStream_t st)
{
    centre_kernel<<<m, 256, 0, st>>>(X, n, m, root_order_dev, Xr, status);
    return cudaGetLastError();
}

cudaError_t launch_tsqr(const double* Xr, int64_t n, int m, double* rbuf, unsigned* counters, int nleaf2, int rb,
                        double* Rroot, int* status, cudaStream_t st)
{
    int rows = rb > 2 * m ? rb : 2 * m;
    if (rows < m) rows = m;
    size_t smem = (size_t)rows * m * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(tsqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tsqr_kernel<<<nleaf2, 256, smem, st>>>(Xr, n, m, rb, rbuf, counters, nleaf2, Rroot, status);
    return cudaGetLastError();
}

cudaError_t launch_tree_level(const double* parent, double* child, int m, int L, int bh, int p, int k,
                              cudaStream_t st)
{
    const int wpc = 4;
    int nchild = 1 << (L + 1);
    int grid = (nchild + wpc - 1) / wpc;
    size_t smem = (size_t)wpc * m * (m | 1) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(tree_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tree_level_kernel<<<grid, wpc * 32, smem, st>>>(parent, child, m, L, bh, p, k);
    return cudaGetLastError();
}

static size_t traverse_smem(int m, int k, int wpc) { return warp_smem_bytes(m, k) * wpc; }

static bool use_legacy() { return getenv("BNREG_LEGACY_TRAVERSE") != nullptr; }

template <bool W1, bool HR, bool HB>
static cudaError_t launch_tv(const TravParams& P, int grid, int wpc, cudaStream_t st)
{
    if (use_legacy()) {
        size_t smem = traverse_smem(P.m, P.k, wpc);
        cudaError_t e = cudaFuncSetAttribute(traverse_kernel<W1, HR, HB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        traverse_kernel<W1, HR, HB><<<grid, wpc * 32, smem, st>>>(P);
    } else {
        size_t smem = ws_cta_smem(P.m, P.k, wpc);
        cudaError_t e = cudaFuncSetAttribute(traverse_ws_kernel<W1, HR, HB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        traverse_ws_kernel<W1, HR, HB><<<grid, wpc * 64, smem, st>>>(P);
    }
    return cudaGetLastError();
}

int traverse_max_ctas_per_sm(int m, int k, int warps_per_cta)
{
    int n = 0;
    if (use_legacy()) {
        size_t smem = traverse_smem(m, k, warps_per_cta);
        cudaFuncSetAttribute(traverse_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, traverse_kernel<true, true, true>, warps_per_cta * 32,
                                                          smem) != cudaSuccess)
            return 1;
    } else {
        size_t smem = ws_cta_smem(m, k, warps_per_cta);
        cudaFuncSetAttribute(traverse_ws_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, traverse_ws_kernel<true, true, true>,
                                                          warps_per_cta * 64, smem) != cudaSuccess)
            return 1;
    }
    return n > 0 ? n : 1;
}

int traverse_warps_per_cta_factor() { return use_legacy() ? 1 : 2; }

cudaError_t launch_traverse(const TravParams& P, int grid, int wpc, cudaStream_t st)
{
    const int key = (P.world1 ? 4 : 0) | (P.out_rss ? 2 : 0) | (P.out_bic ? 1 : 0);
    switch (key) {
        case 7: return launch_tv<true, true, true>(P, grid, wpc, st);
        case 6: return launch_tv<true, true, false>(P, grid, wpc, st);
        case 5: return launch_tv<true, false, true>(P, grid, wpc, st);
        case 4: return launch_tv<true, false, false>(P, grid, wpc, st);
        case 3: return launch_tv<false, true, true>(P, grid, wpc, st);
        case 2: return launch_tv<false, true, false>(P, grid, wpc, st);
        case 1: return launch_tv<false, false, true>(P, grid, wpc, st);
        default: return launch_tv<false, false, false>(P, grid, wpc, st);
    }
}

cudaError_t launch_best_reduce(const double* part_bic, const uint32_t* part_mask, int nparts, int m,
                               double* best_bic, uint32_t* best_mask, cudaStream_t st)
{
    best_reduce_kernel<<<m, 256, 0, st>>>(part_bic, part_mask, nparts, m, best_bic, best_mask);
    return cudaGetLastError();
}

}  // namespace bnr
