// bnreg_kernels.cu -- sm_100a kernels of the bnreg hot path.
//
//   centre_kernel      a1  centre the columns (fixed-order sums), NaN/Inf flag
//   tsqr_kernel        a2  TSQR: Householder QR of 256-row leaves in shared
//                          memory, then an 8-ary tree of stacked-R merges
//                          (last-arriving CTA merges), diag > 0, rank check
//   tree_level_kernel  a5  one level of the Alg.2 seed tree: a node's R for
//                          the residual of the not-yet-decided variables
//                          after projecting out the front set F; a pinned
//                          variable either joins F (drop the leading row and
//                          column) or the back set B (bubble it behind the
//                          free block with GRCs)
//   best_reduce_kernel a11 deterministic argmax over per-warp bests
// (the seed and walk kernels of a5-a11 are in walk_kernel.cu)
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
// Householder QR in shared memory of a column-major nr x m tile (ld = nr), a CTA of
// kTsqrThreads.  On return the upper triangle holds R (diag may be negative); below
// it are the Householder vectors (callers read the upper triangle only).  Reflection
// j: x = column j (rows j..), alpha = -sign(x0) ||x||, v = x - alpha e_j; the other
// columns c > j get c -= 2 (v.c / v.v) v.  One barrier per column: every thread
// derives alpha and v.v from ||x||^2, which the warp that updated column j (in step
// j - 1) summed on the fly (double-buffered in sh[0..1]); v's head v0 replaces x0 in
// registers, so the tile is not written between the barriers except by the updates.
#ifndef TSQR_THREADS
#define TSQR_THREADS 1024
#endif
constexpr int kTsqrThreads = TSQR_THREADS;
__device__ __forceinline__ void householder_tile(double* T, int nr, int m, double* sh /* 2 + m */)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    double* const diag = sh + 2;
    if (warp == 0) {
        double s = 0.0;
        for (int i = lane; i < nr; i += 32) s = fma(T[i], T[i], s);
        s = warp_sum(s);
        if (lane == 0) sh[0] = s;
    }
    __syncthreads();
    const int nj = m < nr ? m : nr;
    for (int j = 0; j < nj; ++j) {
        const double* cj = T + (int64_t)j * nr;
        if (warp == 0 || j + 1 + warp < m) {           // (warps without a column skip the scalars)
        const double s = sh[j & 1];
        const double x0 = cj[j];
        const double nrm = sqrt(s);
        const double alpha = (x0 > 0.0) ? -nrm : nrm;
        const double v0 = x0 - alpha;
        const double vtv = s - x0 * x0 + v0 * v0;      // 0 only for a zero column (alpha = 0)
        if (threadIdx.x == 0) diag[j] = alpha;
        const double tv = vtv > 0.0 ? 2.0 / vtv : 0.0;   // (off the dot product's chain)
        for (int c = j + 1 + warp; c < m; c += nwarp) {
            double* cc = T + (int64_t)c * nr;
            // row j (v's head v0) by lane 0, rows j+1.. (v = x) by all lanes: no per-row selects
            // two accumulators (rows 64 apart): half the dependent-FMA chain of the column's warp,
            // which every other warp waits for at the column's barrier
            double d = lane == 0 ? v0 * cc[j] : 0.0, d1 = 0.0;
            int i = j + 1 + lane;
#pragma unroll 2
            for (; i + 32 < nr; i += 64) {
                d = fma(cj[i], cc[i], d);
                d1 = fma(cj[i + 32], cc[i + 32], d1);
            }
            if (i < nr) d = fma(cj[i], cc[i], d);
            const double f = warp_sum(d + d1) * tv;
            if (lane == 0) cc[j] = fma(-f, v0, cc[j]);
            double s2 = 0.0, s3 = 0.0;                  // ||column, rows j+1..||^2 after the update
            i = j + 1 + lane;
#pragma unroll 2
            for (; i + 32 < nr; i += 64) {
                const double y = fma(-f, cj[i], cc[i]), y1 = fma(-f, cj[i + 32], cc[i + 32]);
                cc[i] = y;
                cc[i + 32] = y1;
                s2 = fma(y, y, s2);
                s3 = fma(y1, y1, s3);
            }
            if (i < nr) {
                const double y = fma(-f, cj[i], cc[i]);
                cc[i] = y;
                s2 = fma(y, y, s2);
            }
            s2 += s3;
            if (c == j + 1) {
                s2 = warp_sum(s2);
                if (lane == 0) sh[(j + 1) & 1] = s2;
            }
        }
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < nj; j += blockDim.x) T[(int64_t)j * nr + j] = diag[j];
    __syncthreads();
}

// rbuf: the merge tree's R's level by level (leaves first, then ceil(c / F) nodes per
// level up to the root), each m*m row-major.  counters: one zeroed arrival counter per
// internal node (self-resetting).  A merge of F children is one Householder QR of
// their stacked R's (F m x m): fewer sequential levels than a binary tree.
constexpr int kTsqrFanIn = 16;   // (kernels.h kTsqrFanInH: the host picks the leaf rows)
__global__ void __launch_bounds__(kTsqrThreads) tsqr_kernel(const double* __restrict__ Xr, int64_t n, int m, int rb,
                                                   double* rbuf, unsigned* counters, int nleaf2,
                                                   double* Rroot, int* status)
{
    extern __shared__ double smem[];
    __shared__ double sh[2 + 32];
    __shared__ int s_old;
    const int b = blockIdx.x;
    const int64_t r0 = (int64_t)b * rb;
    int nr = 0;
    if (r0 < n) nr = (int)((n - r0) < rb ? (n - r0) : rb);
    int nrp = nr < m ? m : nr;                    // pad to at least m rows
    double* T = smem;                             // nrp x m, column-major
    // flat element loop, unrolled: the loads of several elements are in flight at once
#pragma unroll 4
    for (int e = threadIdx.x; e < nrp * m; e += blockDim.x) {
        const int c = e / nrp, i = e - c * nrp;
        T[e] = (i < nr) ? __ldg(Xr + (int64_t)c * n + r0 + i) : 0.0;
    }
    __syncthreads();
    householder_tile(T, nrp, m, sh);
    // the merge tree: level 0 = the nl leaves, level l+1 has ceil(c_l / F) nodes; the
    // last of a node's (up to F) children to arrive stacks their R's and re-factors
    constexpr int F = kTsqrFanIn;
    const int nl = (int)((n + rb - 1) / rb);
    int c_l = nl, off = 0, idx = b;              // this level's size, its first node, our node
    double* dst = rbuf + (int64_t)(off + idx) * m * m;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        int i = e / m, c = e % m;
        dst[e] = (c >= i) ? T[(int64_t)c * nrp + i] : 0.0;
    }
    while (c_l > 1) {
        __threadfence();
        __syncthreads();
        const int parent = idx / F;
        const int nch = min(F, c_l - F * parent);
        const int c_next = (c_l + F - 1) / F;
        const int poff = off + c_l;              // the next level's first node
        if (threadIdx.x == 0) s_old = (int)atomicAdd(&counters[poff - nl + parent], 1u);
        __syncthreads();
        if (s_old < nch - 1) return;             // not the last child: the last one merges
        if (threadIdx.x == 0) counters[poff - nl + parent] = 0u;   // reset for the next launch
        // last arriver: stack the children's R's (nch * m x m) and re-factor
        const int nr2 = nch * m;
        const double* R0 = rbuf + (int64_t)(off + F * parent) * m * m;   // the children are consecutive
#pragma unroll 4
        for (int e = threadIdx.x; e < nch * m * m; e += blockDim.x) {
            const int q = e / (m * m), r = e - q * m * m;
            const int i = r / m, c = r - i * m;
            T[(int64_t)c * nr2 + q * m + i] = __ldcg(R0 + e);
        }
        __syncthreads();
        householder_tile(T, nr2, m, sh);
        off = poff;
        idx = parent;
        c_l = c_next;
        dst = rbuf + (int64_t)(off + idx) * m * m;
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
            int i = e / m, c = e % m;
            dst[e] = (c >= i) ? T[(int64_t)c * nr2 + i] : 0.0;
        }
        nrp = nr2;
    }
    // root: sign-normalise rows (diag > 0), rank check (G26), from the tile
    // (T holds the root R in its upper triangle, ld = nrp)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int i = e / m, c = e - i * m;
        const double d = T[(int64_t)i * nrp + i];
        const double v = T[(int64_t)c * nrp + i];
        Rroot[e] = (c < i) ? 0.0 : (d < 0.0 ? -v : v);
    }
    if (threadIdx.x < 32) {
        const int c = threadIdx.x;
        double s = 0.0;
        if (c < m)
            for (int i = 0; i <= c; ++i) s = fma(T[(int64_t)c * nrp + i], T[(int64_t)c * nrp + i], s);
        double mx = sqrt(s);
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const bool bad = c < m && !(fabs(T[(int64_t)c * nrp + c]) > 1e-12 * mx);
        if (__any_sync(0xffffffffu, bad || !(mx > 0.0)) && c == 0) atomicOr(status, 4);
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

__global__ void debug_ln_kernel(const double* x, double* y, int64_t n, const double2* tab)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = fast_ln9(x[i], tab);   // the walk kernel's log (kLnEntries-entry table)
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
                                                          size_t sb_bytes, size_t sm_bytes, double* best_bic,
                                                          uint32_t* best_mask, uint32_t* mask_copy)
{
    __shared__ double sb[256];
    __shared__ uint32_t sm[256];
    const int v = blockIdx.x;
    double bb = -__longlong_as_double(0x7ff0000000000000LL);
    uint32_t bm = 0xffffffffu;
    for (int q = threadIdx.x; q < nparts; q += blockDim.x) {
        double b = ((const double*)((const char*)part_bic + (size_t)q * sb_bytes))[v];
        uint32_t mk = ((const uint32_t*)((const char*)part_mask + (size_t)q * sm_bytes))[v];
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
        if (mask_copy) mask_copy[v] = sm[0];   // the handle's copy (bnreg_coefficients after an async run)
    }
}

// ---------------------------------------------------------------- a11 candidate floor
// The shared floor of the walk's running-best thresholds starts at the score of families
// the run visits, found greedily: a base set (the empty set, a12: RSS(v|{}) = ||x_v||^2, the
// squared norm of R's column), then up to kFloorDepth forward steps, each adding the parent
// with the best score (RSS by Householder reflections of R's columns applied to column v:
// the stable route of the oracle's O2; X = Q0 R0).  The floor must not exceed the child's
// maximum over this rank's shard (else its argmax would be missed), so
//   * with world > 1 every visited set is one the rank owns: the base set is the rank's
//     selector pattern (root positions 0..r-1 are the selector variables; for a selector
//     child the pattern with its bit clear, plan.h) and only non-selector parents are
//     added -- the rank's reported best is its shard's maximum, and the merge is exact;
//   * every RSS is raised by a generous bound of its rounding error (64 m (s+1) eps
//     ||x_v||^2 for a set of s parents) before the score and 1e-6 is subtracted:
//     near-collinear sets only weaken the floor (G14 stays exact).
// One warp per child (root position), lane = row of R.
constexpr int kFloorRefl = kFloorDepth + kFloorSel;   // reflections of the base set + the steps

__global__ void __launch_bounds__(32) gbest_init_kernel(const double* __restrict__ R, const int* __restrict__ order,
                                                        int m, double mhalf_n, const FloorK K, long long* gbest,
                                                        int r, uint32_t t0, uint32_t t1)
{
    const int pv = blockIdx.x, lane = threadIdx.x;
    const double NINF = -__longlong_as_double(0x7ff0000000000000LL);
    if (pv >= 32) return;
    if (pv >= m) {
        if (lane == 0) gbest[pv] = bic_ord(NINF);
        return;
    }
    double yr = (lane <= pv && lane < m) ? R[lane * m + pv] : 0.0;   // column v, reflected as S grows
    const double yy = warp_sum(yr * yr);
    const double eps = 64.0 * m * 1.1102230246251565e-16 * yy;
    double W[kFloorRefl], WW[kFloorRefl];                            // the reflections of S (lane's row)
    uint32_t S = 0;
    int t = 0;                                                       // |S|
    // S += {pu}: its reflection in the current coordinates, applied to column v
    auto add = [&](int pu) {
        double a = (lane <= pu && lane < m) ? R[lane * m + pu] : 0.0;
#pragma unroll
        for (int q = 0; q < kFloorRefl; ++q)
            if (q < t) a = fma(-2.0 * warp_sum(W[q] * a) / WW[q], W[q], a);
        const double at = lane >= t ? a : 0.0;
        const double nrm = sqrt(warp_sum(at * at));
        const double a0 = __shfl_sync(FULLMASK, a, t);
        const double alpha = a0 >= 0.0 ? nrm : -nrm;
#pragma unroll
        for (int q = 0; q < kFloorRefl; ++q)
            if (q == t) {
                W[q] = lane == t ? at + alpha : at;
                WW[q] = 2.0 * nrm * (nrm + fabs(a0));
                yr = fma(-2.0 * warp_sum(W[q] * yr) / WW[q], W[q], yr);
            }
        S |= 1u << pu;
        ++t;
    };
    if (r > 0) {
        // the base set: this rank's selector pattern (selector variables = root positions < r)
        const uint32_t pat = (pv < r && ((t0 >> pv) & 1u)) ? t1 : t0;
        const uint32_t S0 = pat & ((1u << r) - 1u) & ~(1u << pv);
        for (int pu = 0; pu < r; ++pu)
            if ((S0 >> pu) & 1u) add(pu);
    }
    const double rss0 = warp_sum(lane >= t ? yr * yr : 0.0);
    double best = fma(mhalf_n, log(rss0 + (t + 1) * eps), K.k[t]);
    const uint32_t excl = (r > 0) ? (1u << r) - 1u : 0u;             // never add a selector variable
    for (int step = 0; step < kFloorDepth && t < m - 1; ++step) {
        double bs = NINF;
        int bu = -1;
        for (int pu = 0; pu < m; ++pu) {
            if (pu == pv || ((S >> pu) & 1u) || ((excl >> pu) & 1u)) continue;
            double a = (lane <= pu && lane < m) ? R[lane * m + pu] : 0.0;
#pragma unroll
            for (int q = 0; q < kFloorRefl; ++q)
                if (q < t) a = fma(-2.0 * warp_sum(W[q] * a) / WW[q], W[q], a);
            const double at = lane >= t ? a : 0.0;                  // the part orthogonal to S
            const double aa = warp_sum(at * at);
            if (!(aa > 0.0)) continue;
            const double nrm = sqrt(aa);
            const double a0 = __shfl_sync(FULLMASK, a, t);
            const double alpha = a0 >= 0.0 ? nrm : -nrm;
            const double w = lane == t ? at + alpha : at;
            const double ww = 2.0 * nrm * (nrm + fabs(a0));
            const double y2 = fma(-2.0 * warp_sum(w * yr) / ww, w, yr);
            const double rss = warp_sum(lane > t ? y2 * y2 : 0.0);
            const double sc = fma(mhalf_n, log(rss + (t + 2) * eps), K.k[t + 1]);
            if (sc > bs) { bs = sc; bu = pu; }
        }
        if (bu < 0) break;
        best = fmax(best, bs);
        add(bu);
    }
    const double fl = best - (1e-9 * fabs(best) + 1e-6);
    if (lane == 0)
        gbest[order[pv]] = bic_ord(isfinite(fl) ? fl : (fl > 0 ? __longlong_as_double(0x7ff0000000000000LL) : NINF));
}

cudaError_t launch_gbest_init(const double* R, const int* order, int m, double mhalf_n, const FloorK& K, long long* gbest,
                              int r, uint32_t t0, uint32_t t1, cudaStream_t st)
{
    gbest_init_kernel<<<32, 32, 0, st>>>(R, order, m, mhalf_n, K, gbest, r, t0, t1);
    return cudaGetLastError();
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
    int rows = rb > kTsqrFanIn * m ? rb : kTsqrFanIn * m;
    if (rows < m) rows = m;
    size_t smem = (size_t)rows * m * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(tsqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nl = (int)((n + rb - 1) / rb);
    (void)nleaf2;
    tsqr_kernel<<<nl, kTsqrThreads, smem, st>>>(Xr, n, m, rb, rbuf, counters, nleaf2, Rroot, status);
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

cudaError_t launch_best_reduce(const double* part_bic, const uint32_t* part_mask, int nparts, int m,
                               double* best_bic, uint32_t* best_mask, uint32_t* mask_copy, cudaStream_t st,
                               size_t row_bytes)
{
    const size_t sb = row_bytes ? row_bytes : (size_t)m * sizeof(double);
    const size_t sm = row_bytes ? row_bytes : (size_t)m * sizeof(uint32_t);
    best_reduce_kernel<<<m, 256, 0, st>>>(part_bic, part_mask, nparts, m, sb, sm, best_bic, best_mask, mask_copy);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- coefficients
// The least-squares coefficients of child v on parent set S ("solve the
// regression equations"), from the root R: X~ = Q0 R0 with Q0 orthonormal, so the
// regression of x~_v on X~_S is that of R0[:, v] on R0[:, S].  One warp per child,
// lane = row of the m x (|S| + 1) matrix [R0[:, S] | R0[:, v]] (columns by ascending
// user id): Householder QR, then back-substitution on the |S| x |S| triangle.  A batch
// of families (children[f], masks[f]) runs one CTA per family (children NULL: family f
// is child f); a child outside [0, m) gets a row of NaN.
__global__ void __launch_bounds__(32) coef_kernel(const double* __restrict__ R, const int* __restrict__ order, int m,
                                                  const int32_t* __restrict__ children,
                                                  const uint32_t* __restrict__ masks, int64_t count,
                                                  double* __restrict__ beta)
{
    __shared__ double M[32 * 33];          // column-major, ld 32
    __shared__ int cols[32];
    const int lane = threadIdx.x;
    for (int64_t f = blockIdx.x; f < count; f += gridDim.x) {
        const int v = children ? children[f] : (int)f;
        if (v < 0 || v >= m) {
            if (lane < m) beta[f * m + lane] = __longlong_as_double(0x7ff8000000000000LL);
            continue;
        }
        const uint32_t S = masks[f] & ~(1u << v) & (m == 32 ? 0xffffffffu : ((1u << m) - 1u));
        // position of user id u in the root order
        int k = 0;
        if (lane == 0) {
            for (int u = 0; u < m; ++u)
                if ((S >> u) & 1u) cols[k++] = u;
            cols[k] = v;
        }
        __syncwarp();
        k = __popc(S);
        for (int j = 0; j <= k; ++j) {
            const int u = cols[j];
            int pu = 0;
            for (int c = 0; c < m; ++c)
                if (order[c] == u) pu = c;
            M[j * 32 + lane] = lane < m ? R[(size_t)lane * m + pu] : 0.0;
        }
        __syncwarp();
        for (int j = 0; j < k; ++j) {
            const double xj = M[j * 32 + lane];
            const double x = lane >= j ? xj : 0.0;
            const double nrm2 = warp_sum(x * x);
            const double x0 = __shfl_sync(FULLMASK, xj, j);
            const double alpha = x0 > 0.0 ? -sqrt(nrm2) : sqrt(nrm2);
            const double vr = lane == j ? x0 - alpha : x;          // Householder vector (rows >= j)
            const double vn2 = nrm2 - x0 * x0 + (x0 - alpha) * (x0 - alpha);
            for (int c = j + 1; c <= k; ++c) {
                const double mc = M[c * 32 + lane];
                const double d = warp_sum(vr * mc);
                if (lane >= j && vn2 > 0.0) M[c * 32 + lane] = mc - 2.0 * vr * d / vn2;
            }
            __syncwarp();
            if (lane == j) M[j * 32 + j] = alpha;
            __syncwarp();
        }
        if (lane == 0) {
            double b[32];
            for (int i = k - 1; i >= 0; --i) {
                double t = M[k * 32 + i];
                for (int c = i + 1; c < k; ++c) t -= M[c * 32 + i] * b[c];
                b[i] = t / M[i * 32 + i];
            }
            for (int u = 0; u < m; ++u) beta[f * m + u] = 0.0;
            for (int i = 0; i < k; ++i) beta[f * m + cols[i]] = b[i];
        }
        __syncwarp();
    }
}

cudaError_t launch_coefficients(const double* R, const int* order, int m, const int32_t* children,
                                const uint32_t* masks, int64_t count, double* beta, cudaStream_t st)
{
    if (count <= 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>(count, (int64_t)148 * 32 * 8);
    coef_kernel<<<grid, 32, 0, st>>>(R, order, m, children, masks, count, beta);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a2 alternative: Gram + Cholesky
// SURVEY §8(f) NEXT 2, the paper's covariance alternative (it "comes at
// cost of numerical accuracy"): R = chol(X~^T X~) instead of the TSQR.  Same R up to
// rounding in exact arithmetic, but the Gram matrix squares the condition number.
// gram_kernel: one CTA per (i <= j) column pair, G[i][j] = sum_r X~[r][i] X~[r][j].
__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ Xr, int64_t n, int m,
                                                   double* __restrict__ G)
{
    __shared__ double red[8];
    int p = blockIdx.x, i = 0;
    while (p >= m - i) { p -= m - i; ++i; }
    const int j = i + p;
    const double* a = Xr + (int64_t)i * n;
    const double* b = Xr + (int64_t)j * n;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) s = fma(a[r], b[r], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];   // fixed order
        G[(size_t)i * m + j] = t;
        G[(size_t)j * m + i] = t;
    }
}

// chol_kernel: one warp, upper Cholesky factor R (row-major, diag > 0) of G in place
// into Rroot; rank check as the TSQR's (G26), a non-positive pivot is rank deficient.
__global__ void __launch_bounds__(32) chol_kernel(const double* __restrict__ G, int m, double* __restrict__ R,
                                                  int* status)
{
    __shared__ double A[32 * 33];
    const int lane = threadIdx.x;
    for (int r = 0; r < m; ++r)
        if (lane < m) A[r * 33 + lane] = G[(size_t)r * m + lane];
    __syncwarp();
    bool bad = false;
    double mx = 0.0;
    for (int c = 0; c < m; ++c) mx = fmax(mx, sqrt(fabs(A[c * 33 + c])));
    for (int k = 0; k < m; ++k) {
        const double d = A[k * 33 + k];
        bad |= !(d > 0.0);
        const double rkk = d > 0.0 ? sqrt(d) : 0.0;
        __syncwarp();
        // row k of R: R[k][j] = A[k][j] / rkk for j > k; trailing update A[i][j] -= R[k][i] R[k][j]
        if (lane > k && lane < m) A[k * 33 + lane] = rkk > 0.0 ? A[k * 33 + lane] / rkk : 0.0;
        if (lane == k) A[k * 33 + k] = rkk;
        __syncwarp();
        if (lane > k && lane < m)
            for (int i = k + 1; i <= lane; ++i) A[i * 33 + lane] = fma(-A[k * 33 + i], A[k * 33 + lane], A[i * 33 + lane]);
        __syncwarp();
        if (!(rkk > 1e-12 * mx)) bad = true;
    }
    if (lane < m)
        for (int r = 0; r < m; ++r) R[(size_t)r * m + lane] = lane >= r ? A[r * 33 + lane] : 0.0;
    if (lane == 0 && bad) atomicOr(status, 4);
}

cudaError_t launch_gram_chol(const double* Xr, int64_t n, int m, double* G, double* Rroot, int* status,
                             cudaStream_t st)
{
    gram_kernel<<<m * (m + 1) / 2, 256, 0, st>>>(Xr, n, m, G);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    chol_kernel<<<1, 32, 0, st>>>(G, m, Rroot, status);
    return cudaGetLastError();
}

}  // namespace bnr
