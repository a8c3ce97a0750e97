// seed_kernel.cu -- a5 of the bnreg path: the seed tree's
// nodes at depth L1 (tree_direct_kernel) and every pack's worker seeds
// (seed_kernel), written in the layout the walk kernel (walk_kernel.cu) loads.
// Alg.2's seeds (readings G7-G11) are derived by GRCs
// (Eq.3-4 with reading G1) from the root R.
#include <cstdint>
#include <cmath>
#include <algorithm>
#include "kernels.h"
#include "device.cuh"

namespace bnr {

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

// A bubble: d consecutive GRCs that move one column across d others (each
// GRC swaps two adjacent columns and restores the triangle with one rotation of their two
// rows), with every column (lane) carrying its current row in a register: per GRC one
// shared load and one store per column instead of two each, no per-GRC position updates.
// Entries below a column's diagonal are exact zeros (the pivot of every GRC gets (h, 0)),
// so columns a rotation does not touch just rotate zeros: the sweeps need no predicates.
// The arithmetic is a single GRC's (givens_fr on the pivot's rows J, J+1; x' = c x + s y,
// y' = c y - s x), so the result is that of the d GRCs one after the other.

// forward: the column at position pj moves to pj + d (GRCs at pj, pj+1, .., pj+d-1); the
// pivot of GRC t is the column at position pj + t + 1 (it moves to pj + t): its current row
// J (the carried register) and row J + 1 come from its lane by shuffles
__device__ __forceinline__ void bubble_fwd(double* A, int SA, int pj, int d, int lane, int& pos, double* cs)
{
    int* const lanemap = (int*)cs;           // position -> lane
    const bool live = pos < 32;
    if (live) lanemap[pos] = lane;
    __syncwarp();
    double* p = A + pj * SA + (live ? lane : 0);
    double x = live ? p[0] : 0.0;            // the carried row J
    for (int t = 0; t < d; ++t, p += SA) {
        const double y = live ? p[SA] : 0.0;
        const int Y = lanemap[pj + t + 1];
        double c, s, h;
        givens_fr(__shfl_sync(FULLMASK, x, Y), __shfl_sync(FULLMASK, y, Y), c, s, h);
        const bool isY = lane == Y;
        const double xn = isY ? h : fma(c, x, s * y);
        const double yn = isY ? 0.0 : fma(c, y, -s * x);
        if (live) p[0] = xn;
        x = yn;
    }
    if (live) p[0] = x;
    __syncwarp();
    pos = pos == pj ? pj + d : (pos > pj && pos <= pj + d ? pos - 1 : pos);
}

// backward: the column Z at position pj moves to pj - d (GRCs at pj-1, pj-2, .., pj-d);
// Z is every GRC's pivot: its rows are (h, 0) after each, so the chain needs only its
// original entries above the diagonal
__device__ __forceinline__ void bubble_bwd(double* A, int SA, int pj, int d, int lane, int& pos, double* cs)
{
    const int Z = __ffs(__ballot_sync(FULLMASK, pos == pj)) - 1;
    const double* cz = A + Z;
    double h = cz[pj * SA];
    for (int t = 1; t <= d; ++t) {
        const int J = pj - t;
        double c, s;
        givens_fr(cz[J * SA], h, c, s, h);
        if (lane == 0) {
            cs[3 * t - 3] = c;
            cs[3 * t - 2] = s;
            cs[3 * t - 1] = h;
        }
    }
    __syncwarp();
    const bool live = pos < 32 && lane != Z;
    double* p = A + pj * SA + (live ? lane : 0);
    double y = live ? p[0] : 0.0;            // the carried row J + 1
    for (int t = 1; t <= d; ++t) {
        p -= SA;                             // row J = pj - t
        const double ct = cs[3 * t - 3], st = cs[3 * t - 2];
        const double x = live ? p[0] : 0.0;
        const double xn = fma(ct, x, st * y), yn = fma(ct, y, -st * x);
        if (live) p[SA] = yn;
        y = xn;
    }
    if (live) p[0] = y;
    if (lane == Z) {                         // Z: (h_d, 0, .., 0) in rows pj-d .. pj
        double* q = A + (pj - d) * SA + Z;
        q[0] = h;
        for (int r = 1; r <= d; ++r) q[r * SA] = 0.0;
    }
    __syncwarp();
    pos = pos == pj ? pj - d : (pos >= pj - d && pos < pj ? pos + 1 : pos);
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
// With a rank selector (rsel > 0, multi-GPU), only the nodes whose low rsel
// levels match one of the rank's two patterns t0, t1 are derived (the rank's
// work items lie below them): warp q takes node ((q >> 1) << rsel) | t_{q & 1}.
__global__ void __launch_bounds__(128) tree_direct_kernel(const double* __restrict__ root, double* __restrict__ nodes,
                                                          int m, int L1, int bh, int p, int k, int rsel, uint32_t t0,
                                                          uint32_t t1)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int SAq = m | 1;
    double* const A = (double*)smem + (size_t)wib * m * SAq;
    double* const cs = (double*)smem + (size_t)(blockDim.x >> 5) * m * SAq + 48 * wib;   // bubble scratch: 3 d <= 36 doubles, or 32 ints
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + wib;
    const uint32_t nid = rsel > 0 ? (((q >> 1) << rsel) | ((q & 1u) ? t1 : t0)) : q;
    if ((rsel > 0 ? (q >> 1) << rsel : q) >= (1u << L1)) return;
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
        bubble_fwd(A, SAq, org, T, lane, pos, cs);
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

cudaError_t launch_tree_direct(const double* root, double* nodes, int m, int L1, int bh, int p, int k, int rsel,
                               uint32_t t0, uint32_t t1, cudaStream_t st)
{
    if (L1 <= 0) return cudaSuccess;
    const size_t smem = (size_t)4 * (m * (m | 1) + 48) * sizeof(double);
    if (rsel > L1) rsel = 0;                       // the selector is below the global tree: all nodes
    const unsigned n = rsel > 0 ? 2u << (L1 - rsel) : 1u << L1;
    cudaError_t e = cudaFuncSetAttribute(tree_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tree_direct_kernel<<<(n + 3) / 4, 128, smem, st>>>(root, nodes, m, L1, bh, p, k, rsel, t0, t1);
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
    double* const cs = (double*)smem + (size_t)(blockDim.x >> 5) * m * SAq + 48 * wib;   // bubble scratch: 3 d <= 36 doubles, or 32 ints
    const int npk = (P.item_end - P.item_begin) * G;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int q = blockIdx.x * (blockDim.x >> 5) + wib; q < npk; q += nwarps) {
        const int item = P.item_begin + q / G, gw = q % G;
        int c = 0;
        while (c + 1 < P.nclass && item >= P.cls_end[c]) ++c;
        const int SA = P.cls_SA[c];
        unsigned char* const blk =
            P.seeds + P.cls_off[c] + ((size_t)(item - P.cls_begin[c]) * G + gw) * seed_block_bytes(k, SA, LW);
        if (P.packs[item] >> 31) continue;       // a split item's second pass: the first pass's seeds
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
        // the column's walk slot: [free 0..k-1 | warp vars 0..p-1 | gang vars 0..g-1 |
        // tree back set ascending id]; a warp or gang variable in F keeps its (unused) slot
        int slot = 0;
        if (myvar >= 0) {
            if (myvar >= fv0 && myvar < fv0 + k) slot = myvar - fv0;
            else if (myvar < fv0) slot = k + myvar;
            else {
                // tree back variables with a smaller id: tree level l < gs is user id m - 1 - l
                // (plan.h hv_id), so the back set's id mask is the bit-reversed free levels
                const uint32_t lv = ~pack & ((1u << gs) - 1u);
                const uint32_t bmask = (uint32_t)(__brev(lv) >> (32 - m));
                slot = k + fv0 + __popc(bmask & ((1u << myvar) - 1u));
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
            bubble_fwd(A, SAq, org, T, lane, pos, cs);
        }
        // Gray path over the warp variables: start with all of them in F (front
        // region [w_{p-1} .. w_0 | free]), flip bit ctz(i) at step i; a flip moves
        // variable j across the free block and the j lower warp variables
        // the block is packed with this item's own slot count Sw (<= SA) as the row stride
        const int SW = k + fv0 + (gs - __popc(P.packs[item] & ((1u << gs) - 1u)));
        const size_t wsz = (size_t)k * SW * 16;      // one worker's part of the block
        int wcur = P.nw - 1;
        snapshot_sq(A, SAq, sn, org + p, k, SW, lane, pos, slot, blk + wcur * wsz);
        for (int i = 1; i < P.nw; ++i) {
            const int j = __ffs(i) - 1;
            const int pj = __shfl_sync(FULLMASK, pos, __ffs(__ballot_sync(FULLMASK, myvar == j)) - 1);
            const int d = k + j;
            if ((wcur >> j) & 1) bubble_fwd(A, SAq, pj, d, lane, pos, cs);
            else bubble_bwd(A, SAq, pj, d, lane, pos, cs);
            wcur ^= 1 << j;
            snapshot_sq(A, SAq, sn, org + __popc(wcur), k, SW, lane, pos, slot, blk + wcur * wsz);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- a5 for the 32-worker walk (walk7)
// Seed -> compact seed7 block of worker w: R(slot, l, w) of the k free rows l for
// every walk slot (slot-major, worker fastest: the walk reads 256 B per (slot, row)),
// and the tail sum of squares (rows below the free block) of every back slot; the
// walk rebuilds the suffix sums.  A warp variable in the worker's F (absent back
// slot) gets zeros.
__device__ __forceinline__ void snapshot7(const double* A, int SAq, int sn, int og, int k, int lane, int pos, int slot,
                                          bool haveslot, double* blk, double* tails, int w)
{
    const bool mine = haveslot && pos >= og && pos < sn;
    const bool zero = haveslot && pos < og && slot >= k;
    double acc = 0.0;
    const double* pa = A + (sn - 1) * SAq + lane;
    for (int r = sn - 1; r >= og + k; --r, pa -= SAq) {
        const double x = (mine && r <= pos) ? *pa : 0.0;
        acc = fma(x, x, acc);
    }
    if ((mine || zero) && slot >= k) tails[(size_t)(slot - k) * 32 + w] = mine ? acc : 0.0;
    for (int l = 0; l < k; ++l) {
        const int r = og + l;
        const double x = (mine && r <= pos) ? A[r * SAq + lane] : 0.0;
        if (mine || zero) blk[((size_t)slot * k + l) * 32 + w] = x;
    }
}

// One warp per item (= pack of 2^p workers, p <= 5): the node at tree depth L1, the
// remaining tree levels, the workers' seeds along a Gray path over the warp variables.
__global__ void __launch_bounds__(128) seed7_kernel(const __grid_constant__ SeedParams P)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int m = P.m, k = P.k, p = P.p, bh = P.bh;
    const int fv0 = p, gs = bh;
    const int SAq = m | 1;
    double* const A = (double*)smem + (size_t)wib * m * SAq;
    double* const cs = (double*)smem + (size_t)(blockDim.x >> 5) * m * SAq + 48 * wib;   // bubble scratch: 3 d <= 36 doubles, or 32 ints
    const int npk = P.item_end - P.item_begin;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int q = blockIdx.x * (blockDim.x >> 5) + wib; q < npk; q += nwarps) {
        const int item = P.item_begin + q;
        double* const blk = (double*)P.seeds + (size_t)q * P.sblk;
        double* const tails = blk + (size_t)(k + P.nbmax) * k * 32;
        const uint32_t pack = P.packs[item];
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
        // walk slot: [free 0..k-1 | warp vars 0..p-1 | tree back set ascending id]
        int slot = 0;
        const bool haveslot = myvar >= 0 && !(myvar >= fv0 + k && ((pack >> (m - 1 - myvar)) & 1u));
        if (myvar >= 0) {
            if (myvar >= fv0 && myvar < fv0 + k) slot = myvar - fv0;
            else if (myvar < fv0) slot = k + myvar;
            else {
                const uint32_t lv = ~pack & ((1u << gs) - 1u);
                const uint32_t bmask = (uint32_t)(__brev(lv) >> (32 - m));
                slot = k + fv0 + __popc(bmask & ((1u << myvar) - 1u));
            }
        }
        int org = 0;
        for (int l = P.L1; l < bh; ++l) {
            if ((pack >> l) & 1u) {
                ++org;
                continue;
            }
            const int T = (bh - l - 1) + p + k;
            bubble_fwd(A, SAq, org, T, lane, pos, cs);
        }
        int wcur = P.nw - 1;
        snapshot7(A, SAq, sn, org + p, k, lane, pos, slot, haveslot, blk, tails, wcur);
        for (int i = 1; i < P.nw; ++i) {
            const int j = __ffs(i) - 1;
            const int pj = __shfl_sync(FULLMASK, pos, __ffs(__ballot_sync(FULLMASK, myvar == j)) - 1);
            const int d = k + j;
            if ((wcur >> j) & 1) bubble_fwd(A, SAq, pj, d, lane, pos, cs);
            else bubble_bwd(A, SAq, pj, d, lane, pos, cs);
            wcur ^= 1 << j;
            snapshot7(A, SAq, sn, org + __popc(wcur), k, lane, pos, slot, haveslot, blk, tails, wcur);
        }
        __syncwarp();
    }
}

cudaError_t launch_seed7(const SeedParams& P, cudaStream_t st)
{
    const int m = P.m;
    const size_t smem = (size_t)4 * (m * (m | 1) + 48) * sizeof(double);
    const int npk = P.item_end - P.item_begin;
    if (npk <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min((npk + 3) / 4, sms * 16);
    cudaError_t e = cudaFuncSetAttribute(seed7_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    seed7_kernel<<<grid, 128, smem, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_seed(const SeedParams& P, cudaStream_t st)
{
    const int m = P.m;
    const size_t smem = (size_t)4 * (m * (m | 1) + 48) * sizeof(double);
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

}  // namespace bnr
