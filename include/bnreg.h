/*
 * bnreg.h -- C ABI of the B200-native all-family regression library.
 *
 * The method (arXiv 1901.07643): for m continuous variables compute, for every
 * child v and every parent set S not containing v (m 2^(m-1) "families",
 * PAPER.md:15, §1), the least-squares residual sum of squares RSS(v|S) of the
 * regression of the centred x_v on the centred x_S, and the Gaussian BIC local
 * score.  It starts from ONE QR decomposition of the data ("The algorithm
 * starts with calculating the QRD of the data matrix", §2) and
 * walks the paper's shortest sequence of adjacent-column swaps re-triangularised
 * by Givens rotations (GRC, Eq.3-4; schedule Alg.1
 * and Eq.10 :207-212), split over workers as in Alg.2.
 *
 * Conventions (all functions):
 *   - fp64 throughout; all calls are synchronous with respect to the host unless
 *     named *_async; status codes are returned, never thrown; the message of the
 *     last failing call is in bnreg_last_error() (thread-local).
 *   - Table layout (reading D6): entry of family (child v, parent
 *     mask S, bit u of S = user variable u, 0-based) is at
 *         index = v * 2^(m-1) + compress(S, v)
 *     where compress deletes bit v.  Sorting by index = sorting by (v, S).
 *     With world > 1 a rank writes only its shard: the concatenation, in index
 *     order, of the ranges bnreg_shard_ranges reports (bnreg_local_index maps).
 *   - BIC (reading G5): -(n/2) ln(RSS/n) - (n/2)(1 + ln 2pi) - (|S|/2) ln n,
 *     higher is better; +INF when RSS <= 1e-300 (perfect fit, G13).
 *   - Best (reading G14): per child the parent set of largest BIC; on exact ties
 *     the smaller |S|, then the smaller mask.
 *   - A handle is not thread-safe; distinct handles are independent.  Output is
 *     bit-identical across runs at a fixed world size and build.
 *   - Limits: 2 <= m <= 30, n >= m + 1.  One rank writes at most 2^32 table
 *     entries (32-bit entry offsets in the walk kernel): m <= 28 on one rank,
 *     m = 29 needs world >= 2 and m = 30 world >= 4 (bnreg_create_ex returns
 *     BNREG_E_INVAL otherwise).  Device memory limits m further: the RSS+BIC
 *     tables take 16 m 2^(m-1) bytes per job (60 GB at m = 28).
 */
#ifndef BNREG_H
#define BNREG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bnreg bnreg_t;   /* opaque; owns all device state it allocates */

typedef enum {
    BNREG_OK = 0,
    BNREG_E_INVAL = 1,      /* bad argument (sizes, NULL handle, world/rank, k)              */
    BNREG_E_NONFINITE = 2,  /* X holds a NaN or Inf (SPEC.md:54 NonFinite)                    */
    BNREG_E_RANK = 3,       /* |r_jj| <= 1e-12 max_j ||x_j - mean||  (reading G26) */
    BNREG_E_NOMEM = 4,      /* device allocation failed                                       */
    BNREG_E_CUDA = 5,       /* any other CUDA error (message in bnreg_last_error)             */
    BNREG_E_STATE = 6,      /* call out of order (e.g. run before data/root is loaded)        */
    BNREG_E_NCCL = 7        /* NCCL missing or failing (bnreg_create_dist, bnreg_run_pairs_dist) */
} bnreg_status;

typedef struct {
    int32_t free_vars;        /* k, the free block each worker permutes with Upsilon(k);
                                 0 = auto (min(m, 8)); 2 <= k <= min(m, 8) (the walk
                                 kernel keeps a step's free list in one u32 of nibbles) */
    int32_t levels_in_warp;   /* seed-tree levels each warp derives itself; -1 = auto (4) */
    int32_t world;            /* ranks sharing the walk (power of two); 0 or 1 = single */
    int32_t rank;             /* this rank, 0 <= rank < world                             */
    int32_t pack_bits;        /* log2 of the lockstep workers a walk warp runs: 0 = auto
                                 (3: 8 workers x 4 lanes, gangs of 4 warps); 5 = 32
                                 workers, one lane each (walk7: a warp's record store
                                 writes one whole 512 B region; slower)     */
    int32_t ctas_per_sm;      /* traversal CTAs per SM; 0 = occupancy maximum             */
} bnreg_options;

/* Create a handle for n x m data and load X (centre + QR, steps a1-a2).
 * X: HOST pointer, column-major n x m (ld = n), read-only, copied; the caller
 * keeps ownership.  On error *out = NULL.  Equivalent to
 * bnreg_create_ex(NULL options) + bnreg_load(h, X, 0). */
bnreg_status bnreg_create(const double* X, int64_t n, int32_t m, bnreg_t** out);

/* Create without loading data.  opt may be NULL (defaults).  Allocates the
 * device state on the current CUDA device. */
bnreg_status bnreg_create_ex(int64_t n, int32_t m, const bnreg_options* opt, bnreg_t** out);

/* (Re)load data of the handle's n, m: centre each column (a1; reading G4) and
 * factor it (a2: TSQR of 256-row Householder leaves).  X: column-major n x m,
 * a HOST pointer when x_on_device == 0 (copied host->device here), else a
 * DEVICE pointer (read in place).  Errors: BNREG_E_NONFINITE, BNREG_E_RANK. */
bnreg_status bnreg_load(bnreg_t* h, const double* X, int32_t x_on_device);

/* As bnreg_load, enqueued on the handle's stream without waiting for it (no host
 * synchronisation inside a pipelined step).  A host X must stay valid (and, for
 * an asynchronous copy, be pinned) until the stream has passed the load.  The
 * NaN/Inf and rank checks are deferred: the next synchronous call on the handle
 * (bnreg_sync, bnreg_run, bnreg_run_pairs) reports BNREG_E_NONFINITE /
 * BNREG_E_RANK; work enqueued in between computes on the rejected data. */
bnreg_status bnreg_load_async(bnreg_t* h, const double* X, int32_t x_on_device);

/* Wait for the handle's stream(s); report a CUDA error or a deferred load error. */
bnreg_status bnreg_sync(bnreg_t* h);

/* Pipelined datasets: run later loads (bnreg_load / bnreg_load_async / bnreg_set_root_device:
 * the H2D copy, centring, the root QR) and the seed tree of the following run on this
 * second CUDA stream, so that dataset s+1 is prepared while dataset s is walked.  The load
 * waits (on the device) until the previous run's seed kernel has consumed the root and the
 * tree; the next run waits until the load is done.  NULL = loads on the handle's stream
 * (the default, no overlap).  Synchronises with the previous load stream. */
bnreg_status bnreg_set_load_stream(bnreg_t* h, void* stream);

/* Number of table entries this handle writes: m 2^(m-1), or this rank's share. */
int64_t bnreg_num_families(const bnreg_t* h);

/* Global index of (child, mask); -1 if bit `child` is set or child is out of range. */
int64_t bnreg_index(int32_t m, int32_t child, uint32_t mask);

/* Rank-local offset of a global index, -1 if another rank owns it. */
int64_t bnreg_local_index(const bnreg_t* h, int64_t global_index);

/* The fused hot path (a5-a11): seed tree, seed kernel, walk with harvest, BIC,
 * stores, per-child best.  out_rss / out_bic: caller-owned DEVICE buffers of
 * bnreg_num_families(h) doubles; either may be NULL (not written).  The work is
 * ordered on the handle's stream (its own non-blocking stream unless
 * bnreg_set_stream): device buffers the caller fills or reads on another stream
 * must be ordered against it by the caller (e.g. a device synchronise).
 * best_mask / best_bic: HOST arrays of m entries (either may be NULL); with
 * world > 1 they hold this rank's best only (merge with bnreg_best_merge). */
bnreg_status bnreg_run(bnreg_t* h, double* out_rss, double* out_bic, uint32_t* best_mask, double* best_bic);

/* As bnreg_run but asynchronous on the handle's stream; best_mask / best_bic
 * are DEVICE arrays of m entries (either may be NULL).  Errors surface on the
 * next synchronous call. */
bnreg_status bnreg_run_async(bnreg_t* h, double* out_rss, double* out_bic, uint32_t* best_mask_dev,
                             double* best_bic_dev);

/* The fused hot path writing one 16 B record per family (the north star's
 * 128-bit stores): out_pairs is a caller-owned DEVICE buffer of
 * 2 * bnreg_num_families(h) doubles, 16-byte aligned; family i's RSS is
 * out_pairs[2i] and its BIC out_pairs[2i + 1] (same index as the separate
 * tables).  best_mask / best_bic as in bnreg_run (HOST). */
bnreg_status bnreg_run_pairs(bnreg_t* h, double* out_pairs, uint32_t* best_mask, double* best_bic);

/* As bnreg_run_pairs, asynchronous on the handle's stream; DEVICE best arrays. */
bnreg_status bnreg_run_pairs_async(bnreg_t* h, double* out_pairs, uint32_t* best_mask_dev, double* best_bic_dev);

/* The score the BIC table / record column and the per-child best hold (SURVEY.md §8(f)
 * NEXT 4): BNREG_SCORE_BIC (default; reading G5), BNREG_SCORE_AIC
 * (loglik - |S|, higher is better), BNREG_SCORE_LOGLIK (loglik = -(n/2) ln(RSS/n)
 * - (n/2)(1 + ln 2pi)).  +inf for RSS <= 1e-300 in every score (G13).  Applies to
 * later runs; BNREG_E_INVAL for another value. */
enum { BNREG_SCORE_BIC = 0, BNREG_SCORE_AIC = 1, BNREG_SCORE_LOGLIK = 2 };
bnreg_status bnreg_set_score(bnreg_t* h, int32_t score);

/* How bnreg_load factors the centred data:
 * BNREG_ROOT_TSQR (default): Householder QR of 256-row tiles and a merge tree.
 * BNREG_ROOT_CHOLESKY: R = chol(X~^T X~), the paper's covariance alternative
 * (PAPER.md:31): faster, but the Gram matrix squares the condition number, so
 * ill-conditioned data (cfg3's near-collinear pair) loses accuracy -- a
 * comparison path.  Applies to later loads; BNREG_E_INVAL for another value. */
enum { BNREG_ROOT_TSQR = 0, BNREG_ROOT_CHOLESKY = 1 };
bnreg_status bnreg_set_root_method(bnreg_t* h, int32_t method);

/* Best parent set within every candidate set (the step after
 * the score table in exact structure search): for every child v and
 * candidate set C (entry i = bnreg_index(m, v, C)), best_score[i] = the maximum over
 * S subset of C of the score of (v, S) and best_mask[i] = that S (user ids; G14
 * tie-break: larger score, then smaller |S|, then smaller mask).  scores: DEVICE, the
 * score column of a run on this handle: the BIC table (stride 1) or the record
 * table's column (out_pairs + 1, stride 2).  best_score / best_mask: DEVICE,
 * bnreg_num_families entries each.  best_score may alias scores only exactly and
 * with stride == 1; any other overlap of [scores, scores + stride * entries) with
 * best_score or best_mask is rejected (BNREG_E_INVAL).
 * Single rank only (world 1: a child's candidate lattice is not split).
 * Asynchronous on the handle's stream. */
bnreg_status bnreg_best_subsets(bnreg_t* h, const double* scores, int64_t stride, double* best_score,
                                uint32_t* best_mask);

/* Least-squares coefficients ("solve the regression equations"; SURVEY.md
 * §8(f) NEXT 1) of each child's regression on one parent set per child, from the
 * root R (X~ = Q0 R0: the regression of R0[:,v] on R0[:,S]).  masks: HOST, m
 * entries (bit v of masks[v] is ignored), or NULL for the per-child best sets of
 * the last run.  beta: HOST, m*m doubles, row-major: beta[v*m + u] is the
 * coefficient of parent u in child v's regression on the centred data, 0 for u
 * outside the set.  Synchronous.  BNREG_E_STATE before data is loaded (or, with
 * masks NULL, before a run on the currently loaded data or root). */
bnreg_status bnreg_coefficients(bnreg_t* h, const uint32_t* masks, double* beta);

/* The same for a batch of families (coefficients per family,
 * e.g. every family of a small m, or the families a search selected): family f is
 * child children[f] regressed on masks[f] (bit children[f] ignored, bits >= m
 * ignored).  children, masks: DEVICE, count entries; beta: DEVICE, count*m doubles,
 * row f as in bnreg_coefficients; a child outside [0, m) gets a row of NaN.
 * Asynchronous on the handle's stream; count == 0 is a no-op.  BNREG_E_INVAL for
 * count < 0 or NULL pointers with count > 0, BNREG_E_STATE before data is loaded. */
bnreg_status bnreg_coefficients_batch(bnreg_t* h, const int32_t* children, const uint32_t* masks, int64_t count,
                                      double* beta);

/* The north-star calls: the RSS table alone (the residual sum of squares of every
 * family, §1 "regressions for all child and parent-set combinations",
 * Eq.5 PAPER.md:109-113 read with G3) / the BIC table alone (reading G5).
 * out: caller-owned DEVICE buffer of bnreg_num_families(h) doubles, table layout as
 * above.  = bnreg_run(h, out, NULL, NULL, NULL) / bnreg_run(h, NULL, out, NULL, NULL):
 * synchronous; BNREG_E_STATE before data (or a root) is loaded. */
bnreg_status bnreg_all_rss(bnreg_t* h, double* out);
bnreg_status bnreg_bic(bnreg_t* h, double* out);

/* Use this CUDA stream (a cudaStream_t) for all further work; NULL = the
 * handle's own stream. */
bnreg_status bnreg_set_stream(bnreg_t* h, void* stream);

/* Root factor R (m x m row-major, diag > 0) in the walk's root variable order,
 * and that order (order[pos] = user id).  Either pointer may be NULL. HOST. */
bnreg_status bnreg_root_r(const bnreg_t* h, double* R_host, int32_t* order_host);

/* Multi-GPU step a3 (§6: every processor walks from the root QRD;
 * the north star broadcasts it from rank 0 instead of refactoring X per rank):
 * copy the root R (m*m doubles, row-major, root order) into / out of a
 * caller-owned DEVICE buffer, so the harness can broadcast it with NCCL over
 * NVLink.  Ranks that receive it call bnreg_set_root_device instead of
 * bnreg_load.  Both are enqueued on the handle's stream WITHOUT host
 * synchronisation: order the collective on the same stream (or synchronise).
 * get: BNREG_E_STATE before a load. */
bnreg_status bnreg_get_root_device(bnreg_t* h, double* R_dev);
bnreg_status bnreg_set_root_device(bnreg_t* h, const double* R_dev);

/* Index ranges of this rank's shard (global index space).  *count receives the
 * number of ranges (<= 2m); starts/lens (capacity 2m) receive them in order. */
bnreg_status bnreg_shard_ranges(const bnreg_t* h, int64_t* count, int64_t* starts, int64_t* lens);

/* Host-only equivalents for a plan (no GPU, no handle): the shard ranges and
 * the rank-local offset of a global index (-1 if another rank owns it). */
bnreg_status bnreg_plan_shard_ranges(int32_t m, int64_t n, const bnreg_options* opt, int64_t* count, int64_t* starts,
                                     int64_t* lens);
int64_t bnreg_plan_local_index(int32_t m, int64_t n, const bnreg_options* opt, int64_t global_index);

/* Deterministic merge of per-rank bests (step a11 after the all-gather; reading
 * G14): masks/bics are nparts x m row-major HOST arrays; a mask 0xffffffff marks
 * "no candidate". */
bnreg_status bnreg_best_merge(int32_t m, int32_t nparts, const uint32_t* masks, const double* bics,
                              uint32_t* out_mask, double* out_bic);

/* The same merge on the device, enqueued on the handle's stream (no host round
 * trip inside a multi-GPU step): row q (q < nparts) of masks_dev / bics_dev holds
 * m DEVICE entries at byte offset q * row_bytes (row_bytes = 0: dense rows, 4m /
 * 8m bytes; else a multiple of 8, >= 8m -- e.g. one all-gathered record per rank
 * [m BICs | m masks | pad] with row_bytes = 16m); out_* DEVICE arrays of m.
 * Bit-identical to bnreg_best_merge. */
bnreg_status bnreg_best_merge_async(bnreg_t* h, int32_t nparts, const uint32_t* masks_dev, const double* bics_dev,
                                    int64_t row_bytes, uint32_t* out_mask_dev, double* out_bic_dev);

/* Per-phase device time of the runs since the last reset, from CUDA events on
 * the launching stream.  enable: 1 = start recording (and reset), 0 = stop,
 * -1 = just read.  out_ms (6 entries): [0] = whole run, [1] = seed tree + seed
 * kernel, [2] = walk kernel, [3] = best reduce, [4] = loads (centre + root QR) of
 * timed loads, [5] = number of those loads; *runs = number of runs accumulated.
 * Collecting the events synchronises once per run. */
bnreg_status bnreg_timing(bnreg_t* h, int32_t enable, double* out_ms, int64_t* runs);

/* Kernel launches of one bnreg_run / bnreg_run_async on this handle (the seed
 * tree levels, the seed kernel, one walk launch per shared-memory class, the
 * best reduction); bnreg_load adds 2 (centre, TSQR).  -1 for a NULL handle. */
int64_t bnreg_launches_per_run(const bnreg_t* h);

/* Plan introspection (host only, no GPU): info must hold 13 entries:
 * info[0..12] = k, b, p, bh, L1, LW, npacks (this rank), schedule length, local
 * families, total families, traversal smem bytes per warp, r (rank selector
 * bits), g (gang bits: 2^g lockstep warps per walk CTA). */
bnreg_status bnreg_plan_query(int32_t m, int64_t n, const bnreg_options* opt, int64_t* info);

/* Upsilon(k) (1-based swap positions) as the kernels use it; returns its length
 * (2^k - k - 1) or -1; writes min(length, cap) entries. Host only. */
int64_t bnreg_schedule(int32_t k, int8_t* out, int64_t cap);

/* Pack ids of a plan in launch order (host only); returns the count. */
int64_t bnreg_plan_packs(int32_t m, int64_t n, const bnreg_options* opt, uint32_t* out, int64_t cap);

/* Test hook: the fp64 natural log the BIC epilogue uses (a9), applied to
 * count DEVICE doubles x_dev (> 1e-300, finite) -> out_dev.  Synchronous. */
bnreg_status bnreg_debug_ln(bnreg_t* h, const double* x_dev, double* out_dev, int64_t count);

/* Test hook (reading G11 "every family exactly once"): in the debug
 * build libbnreg_k8.so (-DBNREG_K8) every table store of later runs also increments
 * counts_dev[local index] (a caller-owned, zeroed DEVICE array of bnreg_num_families + 1
 * uint32; NULL = stop counting), so a test can assert each entry is written exactly once;
 * counts_dev[bnreg_num_families] counts violated bounds checks of the walk kernels (a table
 * index out of range, a shared-memory state or TMEM address outside the warp's region).
 * The release library returns BNREG_E_INVAL. */
bnreg_status bnreg_debug_write_counts(bnreg_t* h, uint32_t* counts_dev);

const char* bnreg_last_error(void);

void bnreg_destroy(bnreg_t* h);   /* NULL-safe; frees device state (and a dist handle's communicator) */

/* ---- Multi-GPU with the library's own NCCL communicator (SURVEY §8(b) bnreg_create_dist;
 * PAPER.md:299-324 §6 Alg.2: the lattice split over p processors; north_star: R
 * NCCL-broadcast from rank 0, per-child maxima gathered with NCCL).  One process per GPU;
 * NCCL is opened at run time (libnccl.so.2: the copy the process already has, e.g.
 * torch's, else the system one), so the library has no link-time NCCL dependency.
 *
 * bnreg_nccl_unique_id: rank 0 creates the communicator id (128 bytes, caller-owned
 * HOST buffer) and hands it to the other ranks out of band (e.g. torch.distributed).
 * bnreg_create_dist: a rank-r handle of a world-rank job on the current device (world a
 * power of two); X is rank 0's HOST column-major n x m data (NULL on the other ranks).
 * Collective: every rank calls it.  Rank 0 centres and factors X (a1-a2); R is broadcast
 * (a3, ncclBroadcast of 8 m^2 bytes) and every rank prepares its shard (a4-a5).
 * bnreg_load_dist: the same for new data of the same n, m (collective).
 * bnreg_run_pairs_dist: every rank writes its shard (out_pairs: DEVICE buffer of
 * bnreg_num_families(h) 16 B records, the rank-local layout of bnreg_shard_ranges), then
 * the ranks all-gather their 16 m-byte best records (ncclAllGather) and merge them on the
 * device (G14): best_mask / best_bic (HOST, m entries, may be NULL) receive the GLOBAL
 * per-child best on every rank.  Collective, synchronous.
 * Errors: BNREG_E_NCCL (NCCL not loadable, or an NCCL call failing: message in
 * bnreg_last_error), the errors of bnreg_create_ex / bnreg_load / bnreg_run_pairs.
 * bnreg_run_pairs_dist on a handle not made by bnreg_create_dist: BNREG_E_STATE. */
bnreg_status bnreg_nccl_unique_id(void* id128);
bnreg_status bnreg_create_dist(const double* X, int64_t n, int32_t m, const void* nccl_id, int32_t rank,
                               int32_t world, bnreg_t** out);
bnreg_status bnreg_load_dist(bnreg_t* h, const double* X);
bnreg_status bnreg_run_pairs_dist(bnreg_t* h, double* out_pairs, uint32_t* best_mask, double* best_bic);

#ifdef __cplusplus
}
#endif

#endif /* BNREG_H */
