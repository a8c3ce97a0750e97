// kernels.h -- launch interface between the C-ABI (bnreg_api.cu) and the
// sm_100a kernels (bnreg_kernels.cu).  Plain structs, no torch types.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace bnr {

// fast log of the BIC epilogue (device.cuh fast_ln9): polynomial degree and table size
#ifndef BNREG_LN_DEG
#define BNREG_LN_DEG 4
#endif
constexpr int kMaxFreeWalk7 = 8;   // walk7: free variables per worker (a step's free list = one u32 of nibbles)
constexpr int kLnBits = BNREG_LN_DEG == 3 ? 10 : 9;
constexpr int kLnEntries = 1 << kLnBits;

// Parameters of the fused traversal kernel (K4 seed derivation + K5 walk +
// a8 harvest + a9 BIC + a10 store + a11 per-child running best).
struct TravParams {
    int m, k, p, bh, L1, nw;
    int g;                      // gang bits: 2^g lockstep warps per CTA
    int lw;                     // log2 workers per warp
    int world1;                 // 1: single rank, identity table layout
    int nsteps;                 // k + 1 seed pseudo-steps + Upsilon(k)
    const uint32_t* packs;      // this rank's work items = gang base pack ids (costliest first)
    unsigned int* counter;      // this launch's work-queue counter (zeroed before the launches)
    double* out_rss;            // rank-local RSS table (device) or nullptr
    double* out_bic;            // rank-local BIC table (device) or nullptr
    double* out_pairs;          // rank-local (RSS, BIC) record table (device, 16 B per family) or nullptr
    double* part_bic;           // [warps of all launches][m] per-warp best BIC
    uint32_t* part_mask;        // [warps of all launches][m] per-warp best mask
    double mhalf_n;             // -n/2
    double tiny_bic;            // lower bound of the BIC (fast log) of any RSS <= 1e-300 (G13 candidates)
    const double2* lntab9;      // fast-log table (kLnEntries x (r_j, -ln r_j))
    double Kc[33];              // BIC constant per parent-set size
    int r;                      // rank-selector bits (world > 1)
    unsigned patlo;             // smaller selector pattern of this rank (non-selector children)
    int S_alloc;                // walk slots allocated per warp (>= every item's slot count)
    int item_begin, item_end;   // this launch's work items [begin, end) of `packs`
    int part_base;              // first row of this launch's warps in part_bic / part_mask
    const uint4* wsteps;        // this launch's walk step table (plan.h WalkStep, one uint4 per step)
    const unsigned char* seeds; // this launch's seed blocks (seed kernel), one per (item, warp)
    int jbmax;                  // most back entries per lane of this launch's warps (ceil(back slots / 4))
    int tm_cols;                // TMEM columns per CTA (walk_tmem_cols(k, jbmax))
    // walk7 (32 lockstep workers per warp, one lane each):
    int KA;                     // shared-memory slots per free row: k free + overflow back slots
    int TB;                     // back slots held in TMEM (512 columns / (4 k))
    int nbmax;                  // most back slots of any item (p + tree levels)
    unsigned long long sblk;    // doubles per item of the seed blocks (seed7 layout)
    unsigned* k8;               // BNREG_K8 debug builds: per-entry write counters (rank-local index), or null;
                                // k8[k8_n] counts out-of-range accesses (table index, shared state, TMEM)
    unsigned long long k8_n;    // this rank's table entries
    int k8_selftest;            // BNREG_K8: lane 0 of every warp reports one deliberate violation
    unsigned long long* trace;  // diagnostic (BNREG_TRACE): per CTA [start ns, end ns, items] or null
    long long* gbest;           // per child: the best BIC any warp has found so far (order-preserving int64
                                // of the double), a shared floor for the warps' candidate thresholds; or null
};
// order-preserving map of doubles to int64 (atomicMax on the running bests)
__host__ __device__ inline long long bic_ord(double x)
{
    long long b;
    memcpy(&b, &x, 8);
    return b < 0 ? b ^ 0x7fffffffffffffffLL : b;
}
__host__ __device__ inline double bic_unord(long long o)
{
    const long long b = o < 0 ? o ^ 0x7fffffffffffffffLL : o;
    double x;
    memcpy(&x, &b, 8);
    return x;
}

// seed kernel: one warp per pack derives its 2^p workers' seeds (the remaining
// tree levels + the Gray path over the warp variables) and writes them in the
// walk kernel's state layout to `seeds` (one block per (item, warp) of each class)
constexpr int kMaxClasses = 8;
struct SeedParams {
    int m, k, p, bh, g, L1, nw, lw;
    int nclass;
    int cls_begin[kMaxClasses], cls_end[kMaxClasses], cls_SA[kMaxClasses];
    unsigned long long cls_off[kMaxClasses];   // byte offset of the class's first block
    int item_begin, item_end;                  // items (gangs) of this launch
    const double* nodes;                       // seed-tree nodes at depth L1
    const uint32_t* packs;
    unsigned char* seeds;
    int TB, nbmax;                             // seed7: back slots in TMEM, most back slots of an item
    unsigned long long sblk;                   // seed7: doubles per item
};
// seed7: the compact seed blocks of the 32-worker walk (R of the free rows, slot-major,
// worker fastest, + the tail sum of squares of every back slot); one warp per item
cudaError_t launch_seed7(const SeedParams& P, cudaStream_t st);
// walk7: 32 lockstep workers per warp, one CTA of `warps` independent warps per SM
size_t walk7_cta_smem(int k, int KA, int nslots, int warps);
cudaError_t launch_walk7(const TravParams& P, int grid, int warps, cudaStream_t st);
__host__ __device__ size_t seed_block_bytes(int k, int S_alloc, int lw);
cudaError_t launch_seed(const SeedParams& P, cudaStream_t st);
// the seed tree's nodes at depth L1 in one launch (one warp per node, derived from the root)
// rsel > 0: only the nodes under this rank's selector patterns t0, t1 (low rsel levels)
cudaError_t launch_tree_direct(const double* root, double* nodes, int m, int L1, int bh, int p, int k, int rsel,
                               uint32_t t0, uint32_t t1, cudaStream_t st);

// walk kernel: 2^lw = 8 lockstep workers per warp, gang of 2^g warps per CTA; the back
// slots' walk state in TMEM (walk_tmem_cols per CTA), the free slots' in shared memory
size_t walk_cta_smem(int m, int k, int S_alloc, int g, int lw);
int walk_tmem_cols(int k, int jbmax);
int walk_max_ctas_per_sm(int m, int k, int S_alloc, int g, int jbmax);
cudaError_t launch_walk(const TravParams& P, int grid_ctas, cudaStream_t st);
// slot-split walk (design S, measured slower: DESIGN.md §4): the gang's 4 warps run the same 32
// workers (one lane each) and split the walk slots; the same seed blocks and items, the step
// table of walk_step_table_s, step mbarriers instead of the gang barrier
size_t walks_cta_smem(int k, int S_alloc);
cudaError_t launch_walks(const TravParams& P, int grid_ctas, cudaStream_t st);


// TSQR: leaves of rb rows, merged 16 at a time (one merge level whenever n <= 16 rb): the
// host picks rb >= 256 so that n fits one level if the leaf tile (rb x m doubles) fits
constexpr int kTsqrFanInH = 16;
inline int tsqr_leaf_rows(int64_t n, int m)
{
    int rb = (int)(((n + kTsqrFanInH - 1) / kTsqrFanInH + 31) / 32 * 32);
    const int cap = (227 * 1024 / (8 * m)) / 32 * 32;
    if (rb < 256) rb = 256;
    if (rb > cap) rb = cap;
    return rb;
}
cudaError_t launch_centre(const double* X, int64_t n, int m, const int* root_order_dev,
                          double* Xr, int* status, cudaStream_t st);
cudaError_t launch_tsqr(const double* Xr, int64_t n, int m, double* rbuf, unsigned* counters,
                        int nleaf2, int rb, double* Rroot, int* status, cudaStream_t st);
// a2 alternative: root R by Cholesky of the Gram matrix (G: m*m scratch)
cudaError_t launch_gram_chol(const double* Xr, int64_t n, int m, double* G, double* Rroot, int* status,
                             cudaStream_t st);
cudaError_t launch_tree_level(const double* parent, double* child, int m, int L, int bh, int p, int k,
                              cudaStream_t st);
// the walk's shared candidate floor: each child's empty-set score less a margin
constexpr int kFloorDepth = 3;                 // greedy forward steps of the candidate floor
constexpr int kFloorSel = 6;                   // selector variables of a rank's base set (world <= 32)
struct FloorK {
    double k[kFloorDepth + kFloorSel + 1];     // the score constants K(0..kFloorDepth + kFloorSel)
};
// r, t0, t1: this rank's selector bits and patterns (plan.h; r = 0 for a single rank)
cudaError_t launch_gbest_init(const double* R, const int* order, int m, double mhalf_n, const FloorK& K, long long* gbest,
                              int r, uint32_t t0, uint32_t t1, cudaStream_t st);
cudaError_t launch_best_reduce(const double* part_bic, const uint32_t* part_mask, int nparts, int m,
                               double* best_bic, uint32_t* best_mask, uint32_t* mask_copy, cudaStream_t st,
                               size_t row_bytes = 0);   // bytes between rows (0: dense m-entry rows)

// best parent set within every candidate set (subset-max transform of a score column)
cudaError_t launch_bps(const double* scores, int64_t stride, int m, double* out_s, uint32_t* out_m, cudaStream_t st);
// least-squares coefficients of every child on masks[child] from the root R (one warp per child)
cudaError_t launch_coefficients(const double* R, const int* order, int m, const int32_t* children,
                                const uint32_t* masks, int64_t count, double* beta, cudaStream_t st);
cudaError_t launch_debug_ln(const double* x, double* y, int64_t n, const double2* tab, cudaStream_t st);

}  // namespace bnr
