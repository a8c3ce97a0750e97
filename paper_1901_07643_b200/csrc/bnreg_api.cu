// bnreg_api.cu -- the C ABI (include/bnreg.h): argument checks, device state,
// host plan (plan.h) and the launch sequence of the sm_100a kernels.
#include <cuda_runtime.h>
#include <nccl.h>          // types only: NCCL is opened at run time (dlopen), never linked
#include <dlfcn.h>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <stdexcept>
#include <cmath>

#include "../../include/bnreg.h"
#include "kernels.h"
#include "plan.h"

using namespace bnr;

static thread_local std::string g_err;

// Wait for the stream by polling: cudaStreamSynchronize under the default
// "auto" schedule may yield the host thread, and its wake-up costs ~1 ms per
// synchronous call (measured: tools/e2e_probe.py); the calls that wait are
// short and the caller asked to block anyway.
static cudaError_t stream_wait(cudaStream_t st)
{
    for (;;) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaErrorNotReady) return e;
    }
}
static cudaError_t event_wait(cudaEvent_t ev)
{
    for (;;) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e != cudaErrorNotReady) return e;
    }
}


static bnreg_status fail(bnreg_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? BNREG_E_NOMEM : BNREG_E_CUDA,             \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                        \
        }                                                                                           \
    } while (0)

struct bnreg {
    Plan plan;
    bnreg_options opt{};
    int device = 0;
    int num_sms = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    // device buffers
    double* dX = nullptr;          // host-loaded copy of X (n*m)
    double* dXr = nullptr;         // centred, root-ordered X
    int* d_order = nullptr;        // root order
    double* d_rbuf = nullptr;      // TSQR tree slots
    unsigned* d_tcnt = nullptr;    // TSQR arrival counters
    int nleaf2 = 1;
    int rb = 256;                  // TSQR leaf rows (tsqr_leaf_rows)
    double* d_root = nullptr;      // root R (m*m)
    double* d_nodes[2] = {nullptr, nullptr};
    uint32_t* d_packs = nullptr;
    double* d_part_bic = nullptr;
    uint32_t* d_part_mask = nullptr;
    double* d_best_bic = nullptr;
    uint32_t* d_best_mask = nullptr;
    int* d_status = nullptr;
    double2* d_lntab9 = nullptr;   // fast-log table (a9), 512 entries (walk kernel, debug_ln)
    int wpc = 4;                   // warps per walk CTA (one gang)
    bool loaded = false;
    bool pending = false;          // an asynchronous load's status flags are not checked yet
    int* h_status = nullptr;       // pinned host copy of d_status (deferred checks)
    // timing
    bool timing = false;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    double acc_ms[6] = {0, 0, 0, 0, 0, 0};   // run, seeds, walk, reduce, load (centre + root QR), loads
    cudaEvent_t evl[2] = {nullptr, nullptr};
    // pipelined loads (bnreg_set_load_stream): load + seed tree of the next dataset on a
    // second stream, overlapping the current walk
    cudaStream_t load_stream = nullptr;
    cudaEvent_t ev_seeds = nullptr;   // run stream: the seed kernel has consumed d_root / d_nodes
    cudaEvent_t ev_prep = nullptr;    // load stream: root R and seed tree of the next run are ready
    // the candidate floor (gbest_init: a latency-bound warp per child) runs on its own stream
    // beside the seed tree and seeds: forked when the root R is ready, joined before the walk
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_root = nullptr, ev_floor = nullptr;
    bool prepared = false;
    bool load_timed = false;       // a timed load is waiting to be collected
    int64_t runs = 0;
    // walk kernel: one launch per shared-memory class of work items
    struct WalkClass {
        int begin, end, S_alloc, grid, part_base, jbmax;
    };
    std::vector<WalkClass> classes;
    int nparts = 0;                // rows of d_part_bic / d_part_mask
    unsigned* d_counters = nullptr;
    int score = 0;                     // BNREG_SCORE_*
    int root_method = 0;               // BNREG_ROOT_*
    double* d_gram = nullptr;          // Gram scratch (BNREG_ROOT_CHOLESKY)
    bool ran = false;                  // a run wrote d_best_mask
    double* d_coef = nullptr;          // bnreg_coefficients output (m*m)
    uint32_t* d_cmask = nullptr;       // bnreg_coefficients input masks
    uint4* d_wsteps = nullptr;     // per-class walk step tables (plan.h WalkStep)
    unsigned char* d_seeds = nullptr;   // seed kernel output: per class, one walk-state block per (item, warp)
    unsigned char* d_seeds2 = nullptr;  // pipelined mode: the second buffer (dataset s+1's seeds while s walks)
    size_t seed_bytes = 0;
    int cur_buf = 0;                    // the buffer the next / last walk reads
    cudaEvent_t ev_walk[2] = {nullptr, nullptr};   // a walk reading buffer b has finished
    unsigned long long* d_trace = nullptr;          // BNREG_TRACE diagnostic
    long long* d_gbest = nullptr;                   // per child: the best BIC any warp has found (bic_ord)
    std::vector<size_t> seed_off;       // byte offset of each class's blocks
    size_t wsteps_len = 0;         // steps per class table
    // walk7 (32 lockstep workers per warp; P.lw == 5)
    bool w7 = false;
    bool ws = false;                    // slot-split walk (design S, walks_kernel.cuh; BNREG_WALK_S=1)
    int w7_warps = 4, w7_TB = 16, w7_KA = 8, w7_nbmax = 0;
    unsigned long long w7_sblk = 0;     // doubles per item of the seed blocks
    unsigned* k8 = nullptr;             // BNREG_K8 debug builds: caller's per-entry write counters
    // bnreg_create_dist: the library's NCCL communicator and its device buffers
    ncclComm_t comm = nullptr;
    double* d_Rt = nullptr;             // the broadcast root R (m*m)
    double* d_rec = nullptr;            // world rows of [m BICs | m masks]: the all-gathered bests
    uint32_t* d_gm = nullptr;           // the merged best
    double* d_gb = nullptr;
};

// NCCL, opened at run time: the process's copy if one is loaded (torch's), else the system's
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};
static NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            api.why = std::string("cannot open libnccl.so.2: ") + dlerror();
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(lib, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(lib, "ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))dlsym(lib, "ncclCommDestroy");
        api.broadcast = (decltype(api.broadcast))dlsym(lib, "ncclBroadcast");
        api.allGather = (decltype(api.allGather))dlsym(lib, "ncclAllGather");
        api.errorString = (decltype(api.errorString))dlsym(lib, "ncclGetErrorString");
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.broadcast && api.allGather && api.errorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks an NCCL entry point";
    });
    return api;
}

static bnreg_options defaults(const bnreg_options* o)
{
    bnreg_options d{};
    d.free_vars = 0; d.levels_in_warp = -1; d.world = 1; d.rank = 0; d.pack_bits = 0; d.ctas_per_sm = 0;
    if (o) {
        d = *o;
        if (d.world <= 0) d.world = 1;
    }
    return d;
}

static void free_all(bnreg* h)
{
    if (!h) return;
    if (h->comm && nccl().ok) nccl().commDestroy(h->comm);
    h->comm = nullptr;
    void* ptrs[] = {h->d_Rt, h->d_rec, h->d_gm, h->d_gb, h->dX, h->dXr, h->d_order, h->d_rbuf, h->d_tcnt, h->d_root, h->d_nodes[0], h->d_nodes[1],
                    h->d_packs, h->d_part_bic, h->d_part_mask, h->d_best_bic,
                    h->d_best_mask, h->d_status, h->d_lntab9, h->d_counters, h->d_wsteps, h->d_seeds, h->d_coef, h->d_cmask, h->d_gram, h->d_seeds2, h->d_trace, h->d_gbest};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : h->evl)
        if (e) cudaEventDestroy(e);
    if (h->ev_seeds) cudaEventDestroy(h->ev_seeds);
    for (auto& e : h->ev_walk)
        if (e) cudaEventDestroy(e);
    if (h->ev_prep) cudaEventDestroy(h->ev_prep);
    if (h->ev_root) cudaEventDestroy(h->ev_root);
    if (h->ev_floor) cudaEventDestroy(h->ev_floor);
    if (h->aux_stream) cudaStreamDestroy(h->aux_stream);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    if (h->h_status) cudaFreeHost(h->h_status);
}

extern "C" {

const char* bnreg_last_error(void) { return g_err.c_str(); }

int64_t bnreg_index(int32_t m, int32_t child, uint32_t mask)
{
    if (m < 2 || m > kMaxM) return -1;
    return family_index(m, child, mask);
}

int64_t bnreg_schedule(int32_t k, int8_t* out, int64_t cap)
{
    if (k < 2 || k > kMaxFree) return -1;
    auto s = greedy_swaps(k);
    if (out)
        for (int64_t t = 0; t < (int64_t)s.size() && t < cap; ++t) out[t] = s[t];
    return (int64_t)s.size();
}

bnreg_status bnreg_plan_query(int32_t m, int64_t n, const bnreg_options* o, int64_t* info)
{
    if (!info) return fail(BNREG_E_INVAL, "info is NULL");
    bnreg_options d = defaults(o);
    try {
        Plan P = make_plan(m, n, d.free_vars, d.levels_in_warp, d.world, d.rank, d.pack_bits);
        info[0] = P.k; info[1] = P.b; info[2] = P.p; info[3] = P.bh; info[4] = P.L1; info[5] = P.LW;
        info[6] = (int64_t)P.packs.size(); info[7] = (int64_t)P.sched.size(); info[8] = P.local_families;
        info[9] = P.total_families; info[10] = (int64_t)walk_cta_smem(P.m, P.k, P.m, P.g, P.lw) >> P.g; info[11] = P.r;
        info[12] = P.g;
    } catch (std::exception& e) {
        return fail(BNREG_E_INVAL, e.what());
    }
    return BNREG_OK;
}

int64_t bnreg_plan_packs(int32_t m, int64_t n, const bnreg_options* o, uint32_t* out, int64_t cap)
{
    bnreg_options d = defaults(o);
    try {
        Plan P = make_plan(m, n, d.free_vars, d.levels_in_warp, d.world, d.rank, d.pack_bits);
        if (out)
            for (int64_t i = 0; i < (int64_t)P.packs.size() && i < cap; ++i) out[i] = P.packs[i];
        return (int64_t)P.packs.size();
    } catch (std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

bnreg_status bnreg_create_ex(int64_t n, int32_t m, const bnreg_options* o, bnreg_t** out)
{
    if (!out) return fail(BNREG_E_INVAL, "out is NULL");
    *out = nullptr;
    bnreg_options d = defaults(o);
    Plan P;
    try {
        P = make_plan(m, n, d.free_vars, d.levels_in_warp, d.world, d.rank, d.pack_bits);
    } catch (std::exception& e) {
        return fail(BNREG_E_INVAL, e.what());
    }
    bnreg* h = new bnreg();
    h->plan = P;
    h->opt = d;
    auto bail = [&](bnreg_status s) {
        free_all(h);
        delete h;
        return s;
    };
#define CKH(call)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return bail(fail(e_ == cudaErrorMemoryAllocation ? BNREG_E_NOMEM : BNREG_E_CUDA,      \
                             std::string(#call) + ": " + cudaGetErrorString(e_)));               \
    } while (0)
    CKH(cudaGetDevice(&h->device));
    CKH(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
    CKH(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    const size_t nm = (size_t)n * m;
    CKH(cudaMalloc(&h->dX, nm * sizeof(double)));
    CKH(cudaMalloc(&h->dXr, nm * sizeof(double)));
    CKH(cudaMalloc(&h->d_order, m * sizeof(int)));
    CKH(cudaMemcpy(h->d_order, P.root_order.data(), m * sizeof(int), cudaMemcpyHostToDevice));
    h->rb = tsqr_leaf_rows(n, m);
    int nleaf = (int)((n + h->rb - 1) / h->rb);
    h->nleaf2 = 1;
    while (h->nleaf2 < nleaf) h->nleaf2 <<= 1;
    CKH(cudaMalloc(&h->d_rbuf, (size_t)2 * h->nleaf2 * m * m * sizeof(double)));
    CKH(cudaMalloc(&h->d_tcnt, (size_t)h->nleaf2 * sizeof(unsigned)));
    CKH(cudaMemset(h->d_tcnt, 0, (size_t)h->nleaf2 * sizeof(unsigned)));
    CKH(cudaMalloc(&h->d_root, (size_t)m * m * sizeof(double)));
    if (P.L1 > 0) {
        size_t nodes = (size_t)1 << P.L1;
        CKH(cudaMalloc(&h->d_nodes[0], nodes * m * m * sizeof(double)));
        CKH(cudaMalloc(&h->d_nodes[1], nodes * m * m * sizeof(double)));
    }
    CKH(cudaMalloc(&h->d_packs, std::max<size_t>(1, P.packs.size()) * sizeof(uint32_t)));
    if (!P.packs.empty())
        CKH(cudaMemcpy(h->d_packs, P.packs.data(), P.packs.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    h->wpc = 1 << P.g;                                    // one CTA = one gang of lockstep warps
    if (P.local_families > (int64_t)0xffffffffLL)
        return bail(fail(BNREG_E_INVAL, "this rank's table exceeds 2^32 entries (use more ranks)"));
    if (P.lw == 5) {
        // walk7: one launch over every item; one CTA of up to 4 independent warps per SM (one per
        // TMEM lane quarter); back slots beyond the TMEM capacity TB go to shared memory
        h->w7 = true;
        const int k = P.k;
        h->w7_TB = std::min(20, 4 * (32 / k));
        h->w7_nbmax = P.b;
        const int so = std::max(0, h->w7_nbmax - h->w7_TB);
        if (so > 4) return bail(fail(BNREG_E_INVAL, "too many back slots for the walk's state (lower m or raise k)"));
        h->w7_KA = k + so;
        int warps = 4;
        while (warps > 0 && walk7_cta_smem(k, h->w7_KA, k + h->w7_nbmax, warps) > (size_t)227 * 1024) --warps;
        if (warps < 1) return bail(fail(BNREG_E_NOMEM, "walk7 state does not fit in shared memory"));
        h->w7_warps = warps;
        h->w7_sblk = (unsigned long long)(k + h->w7_nbmax) * k * 32 + (unsigned long long)h->w7_nbmax * 32;
        const int64_t ni = (int64_t)P.packs.size();
        bnreg::WalkClass c;
        c.begin = 0; c.end = (int)ni; c.S_alloc = 0; c.jbmax = 0;
        c.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->num_sms, (ni + warps - 1) / warps));
        c.part_base = 0;
        h->nparts = c.grid * warps;
        h->classes.push_back(c);
        h->seed_off.push_back(0);
        h->seed_bytes = std::max<size_t>((size_t)ni * h->w7_sblk * sizeof(double), 16);
        CKH(cudaMalloc(&h->d_seeds, h->seed_bytes));
        CKH(cudaMalloc(&h->d_counters, sizeof(unsigned)));
        const auto recs = step_records(P.k, P.sched);
        h->wsteps_len = recs.size();
        auto tb = walk_step_table(recs, P.k, h->w7_KA, 32);
        tb.push_back(WalkStep{});
        CKH(cudaMalloc(&h->d_wsteps, tb.size() * sizeof(WalkStep)));
        CKH(cudaMemcpy(h->d_wsteps, tb.data(), tb.size() * sizeof(WalkStep), cudaMemcpyHostToDevice));
        if (getenv("BNREG_VERBOSE"))
            fprintf(stderr, "walk7: items %lld grid %d warps %d TB %d KA %d nbmax %d smem %zu seed blocks %.2f GB\n",
                    (long long)ni, c.grid, warps, h->w7_TB, h->w7_KA, h->w7_nbmax,
                    walk7_cta_smem(k, h->w7_KA, k + h->w7_nbmax, warps), ni * h->w7_sblk * 8.0 / 1e9);
    } else if (!getenv("BNREG_NO_SPLIT")) {
        // walk kernel, one launch: every item at 4 CTAs per SM (4 back entries per lane in TMEM,
        // 16 back slots per warp); an item with more back slots gets a second pass over back
        // slots 16.. (entry 0x80000000 | item appended to the item list; it rotates the free
        // entries without harvesting them).  Items stay sorted costliest first.
        const int gs = P.bh - P.g;
        std::vector<uint32_t> items(P.packs.begin(), P.packs.end());
        const int64_t na = (int64_t)items.size();
        int nbmax = 0;
        for (int64_t i = 0; i < na; ++i) {
            const int nb = P.p + P.g + (gs - popc(P.packs[i] & ((1u << gs) - 1u)));
            nbmax = std::max(nbmax, nb);
            if (nb > 16) items.push_back(0x80000000u | (uint32_t)i);
        }
        if (nbmax > 32) return bail(fail(BNREG_E_INVAL, "too many back slots per item (raise k)"));
        const int S0 = P.k + nbmax;
        int occ = d.ctas_per_sm > 0 ? d.ctas_per_sm : walk_max_ctas_per_sm(m, P.k, S0, P.g, 4);
        if (occ <= 0) return bail(fail(BNREG_E_NOMEM, "walk kernel does not fit in shared memory / TMEM"));
        bnreg::WalkClass c;
        c.begin = 0; c.end = (int)items.size(); c.S_alloc = S0; c.jbmax = 4;
        c.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->num_sms * occ, (int64_t)items.size()));
        c.part_base = 0;
        h->nparts = c.grid * h->wpc;
        h->classes.push_back(c);
        if (!items.empty()) {
            cudaFree(h->d_packs);
            h->d_packs = nullptr;
            CKH(cudaMalloc(&h->d_packs, items.size() * sizeof(uint32_t)));
            CKH(cudaMemcpy(h->d_packs, items.data(), items.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        }
        h->seed_off.push_back(0);
        h->seed_bytes = std::max<size_t>((size_t)na * (size_t)h->wpc * seed_block_bytes(P.k, S0, P.lw), 16);
        CKH(cudaMalloc(&h->d_seeds, h->seed_bytes));
        CKH(cudaMalloc(&h->d_counters, sizeof(unsigned)));
        const auto recs = step_records(P.k, P.sched);
        h->wsteps_len = recs.size();
        h->ws = P.p == 3 && P.g == 2 && getenv("BNREG_WALK_S") != nullptr;
        auto tb = h->ws ? walk_step_table_s(recs, P.k)                 // design S: shared free-slot state
                        : walk_step_table(recs, P.k, P.k, 1 << P.lw);   // free-slot state: k slots
        for (int j = 0; j < 32; ++j) tb.push_back(WalkStep{});   // pad: the walk kernel loads 32-record windows
        CKH(cudaMalloc(&h->d_wsteps, tb.size() * sizeof(WalkStep)));
        CKH(cudaMemcpy(h->d_wsteps, tb.data(), tb.size() * sizeof(WalkStep), cudaMemcpyHostToDevice));
        if (getenv("BNREG_VERBOSE"))
            fprintf(stderr, "walk: items %zu (%lld split) S_alloc %d grid %d occ %d\n", items.size(),
                    (long long)(items.size() - na), S0, c.grid, occ);
    } else {
        // walk kernel: items are sorted costliest first = most walk slots first
        // (a gang's slots: m - |F among its tree levels|).  A launch ("class") takes
        // the items whose warps need the same TMEM allocation (back entries per lane
        // JB = ceil(back slots / 4): JB <= 4 or more), sized for its first item
        const int gs = P.bh - P.g;
        int64_t i0 = 0;
        const int64_t ni = (int64_t)P.packs.size();
        auto slots_of = [&](int64_t i) { return m - popc(P.packs[i] & ((1u << gs) - 1u)); };
        auto jb_of = [&](int S) { return (S - P.k + 3) / 4; };
        while (i0 < ni) {
            const int S0 = slots_of(i0);
            const int jb0 = jb_of(S0);
            const bool big = jb0 > 4;
            int occ = d.ctas_per_sm > 0 ? d.ctas_per_sm : walk_max_ctas_per_sm(m, P.k, S0, P.g, big ? jb0 : 4);
            if (occ <= 0) return bail(fail(BNREG_E_NOMEM, "walk kernel does not fit in shared memory / TMEM"));
            int64_t i1 = i0 + 1;
            while (i1 < ni && (jb_of(slots_of(i1)) > 4) == big) ++i1;   // (slots are non-increasing)
            bnreg::WalkClass c;
            c.begin = (int)i0; c.end = (int)i1; c.S_alloc = S0;
            c.jbmax = big ? jb0 : std::min(jb0, 4);
            c.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->num_sms * occ, i1 - i0));
            c.part_base = h->nparts;
            h->nparts += c.grid * h->wpc;
            h->classes.push_back(c);
            i0 = i1;
        }
        {
            size_t off = 0;
            for (auto& c : h->classes) {
                h->seed_off.push_back(off);
                off += (size_t)(c.end - c.begin) * (size_t)h->wpc * seed_block_bytes(P.k, c.S_alloc, P.lw);
            }
            h->seed_bytes = std::max<size_t>(off, 16);
            CKH(cudaMalloc(&h->d_seeds, h->seed_bytes));
        }
        if (getenv("BNREG_VERBOSE"))
            for (auto& c : h->classes)
                fprintf(stderr, "walk class: items [%d, %d) S_alloc %d jbmax %d tmem %d grid %d smem %zu\n", c.begin,
                        c.end, c.S_alloc, c.jbmax, walk_tmem_cols(P.k, c.jbmax), c.grid,
                        walk_cta_smem(m, P.k, c.S_alloc, P.g, P.lw));
        if (h->classes.empty()) {            // no work items (cannot happen for m >= 2): keep the reduce well-defined
            h->nparts = 1;
        }
        CKH(cudaMalloc(&h->d_counters, std::max<size_t>(1, h->classes.size()) * sizeof(unsigned)));
        {
            const auto recs = step_records(P.k, P.sched);
            h->wsteps_len = recs.size();
            std::vector<WalkStep> all;
            for (auto& c : h->classes) {
                auto tb = walk_step_table(recs, P.k, P.k, 1 << P.lw);   // free-slot state: k slots
                all.insert(all.end(), tb.begin(), tb.end());
            }
            if (!all.empty()) {
                for (int j = 0; j < 32; ++j) all.push_back(WalkStep{});   // pad: the walk kernel loads 32-record windows
                CKH(cudaMalloc(&h->d_wsteps, all.size() * sizeof(WalkStep)));
                CKH(cudaMemcpy(h->d_wsteps, all.data(), all.size() * sizeof(WalkStep), cudaMemcpyHostToDevice));
            }
        }
    }
    size_t gw = (size_t)h->nparts;
    CKH(cudaMalloc(&h->d_part_bic, gw * m * sizeof(double)));
    CKH(cudaMalloc(&h->d_part_mask, gw * m * sizeof(uint32_t)));
    if (h->classes.empty()) {
        std::vector<double> nb(m, -INFINITY);
        std::vector<uint32_t> nm(m, 0xffffffffu);
        CKH(cudaMemcpy(h->d_part_bic, nb.data(), m * sizeof(double), cudaMemcpyHostToDevice));
        CKH(cudaMemcpy(h->d_part_mask, nm.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    CKH(cudaMalloc(&h->d_best_bic, m * sizeof(double)));
    CKH(cudaMalloc(&h->d_gbest, 2 * 32 * sizeof(long long)));   // one floor per seed buffer (pipelining)
    CKH(cudaMalloc(&h->d_best_mask, m * sizeof(uint32_t)));
    CKH(cudaMalloc(&h->d_status, sizeof(int)));
    CKH(cudaMallocHost(&h->h_status, sizeof(int)));
    {
        // (r_j, -ln r_j), r_j = fl(1 / (1 + (j + 1/2)/2^kLnBits)); -ln r_j in long double
        std::vector<double2> tab9(kLnEntries);
        for (int j = 0; j < kLnEntries; ++j) {
            long double t = 1.0L + ((long double)j + 0.5L) / (long double)kLnEntries;
            double r = (double)(1.0L / t);
            tab9[j].x = r;
            tab9[j].y = (double)(-logl((long double)r));
        }
        CKH(cudaMalloc(&h->d_lntab9, kLnEntries * sizeof(double2)));
        CKH(cudaMemcpy(h->d_lntab9, tab9.data(), kLnEntries * sizeof(double2), cudaMemcpyHostToDevice));
    }
    for (auto& e : h->ev) CKH(cudaEventCreate(&e));
    for (auto& e : h->evl) CKH(cudaEventCreate(&e));
    CKH(cudaEventCreateWithFlags(&h->ev_seeds, cudaEventDisableTiming));
    for (auto& e : h->ev_walk) CKH(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CKH(cudaEventCreateWithFlags(&h->ev_prep, cudaEventDisableTiming));
    CKH(cudaEventCreateWithFlags(&h->ev_root, cudaEventDisableTiming));
    CKH(cudaEventCreateWithFlags(&h->ev_floor, cudaEventDisableTiming));
    CKH(cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking));
#undef CKH
    *out = h;
    return BNREG_OK;
}

bnreg_status bnreg_create(const double* X, int64_t n, int32_t m, bnreg_t** out)
{
    if (!X) return fail(BNREG_E_INVAL, "X is NULL");
    bnreg_status s = bnreg_create_ex(n, m, nullptr, out);
    if (s != BNREG_OK) return s;
    s = bnreg_load(*out, X, 0);
    if (s != BNREG_OK) {
        std::string keep = g_err;
        bnreg_destroy(*out);
        *out = nullptr;
        g_err = keep;
    }
    return s;
}

bnreg_status bnreg_set_stream(bnreg_t* h, void* stream)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    h->stream = stream ? (cudaStream_t)stream : h->own_stream;
    return BNREG_OK;
}

// a5: the seed tree's nodes at depth L1 (one launch; BNREG_TREE_LEVELS=1: level by level)
static const double* seed_tree_nodes(const bnreg_t* h)
{
    const Plan& P = h->plan;
    if (P.L1 <= 0) return h->d_root;
    if (getenv("BNREG_TREE_LEVELS")) return h->d_nodes[(P.L1 - 1) & 1];
    return h->d_nodes[0];
}

static bnreg_status launch_seed_tree(bnreg_t* h, cudaStream_t st)
{
    const Plan& P = h->plan;
    if (P.L1 <= 0) return BNREG_OK;
    if (getenv("BNREG_TREE_LEVELS")) {
        for (int L = 0; L < P.L1; ++L) {
            const double* par = (L == 0) ? h->d_root : h->d_nodes[(L - 1) & 1];
            double* ch = h->d_nodes[L & 1];
            CK(launch_tree_level(par, ch, P.m, L, P.bh, P.p, P.k, st));
        }
    } else {
        // multi-GPU: only the nodes above this rank's work items (its two selector patterns)
        const uint32_t t0 = (uint32_t)P.rank, t1 = ((1u << P.r) - 1u) ^ (uint32_t)P.rank;
        CK(launch_tree_direct(h->d_root, h->d_nodes[0], P.m, P.L1, P.bh, P.p, P.k, P.world > 1 ? P.r : 0, t0, t1, st));
    }
    return BNREG_OK;
}

// a5: every pack's seeds into seed buffer `buf`, in the walk kernel's layout
static bnreg_status launch_seeds(bnreg_t* h, cudaStream_t st, int buf)
{
    const Plan& P = h->plan;
    const double* nodes = seed_tree_nodes(h);
    SeedParams SP{};
    SP.m = P.m; SP.k = P.k; SP.p = P.p; SP.bh = P.bh; SP.g = P.g; SP.L1 = P.L1; SP.nw = 1 << P.p; SP.lw = P.lw;
    SP.nclass = (int)h->classes.size();
    for (size_t c = 0; c < h->classes.size(); ++c) {
        SP.cls_begin[c] = h->classes[c].begin;
        SP.cls_end[c] = h->classes[c].end;
        SP.cls_SA[c] = h->classes[c].S_alloc;
        SP.cls_off[c] = h->seed_off[c];
    }
    SP.item_begin = 0;
    SP.item_end = (int)P.packs.size();
    SP.nodes = nodes; SP.packs = h->d_packs; SP.seeds = buf ? h->d_seeds2 : h->d_seeds;
    if (h->w7) {
        SP.TB = h->w7_TB; SP.nbmax = h->w7_nbmax; SP.sblk = h->w7_sblk;
        CK(launch_seed7(SP, st));
    } else {
        CK(launch_seed(SP, st));
    }
    return BNREG_OK;
}

// the walk's shared candidate floor for the dataset whose root is in d_root (seed buffer `buf`)
static bnreg_status gbest_init(bnreg_t* h, cudaStream_t st, int buf)
{
    const Plan& P = h->plan;
    long long* g = h->d_gbest + 32 * buf;
    if (getenv("BNREG_GBEST_NEGINF") || (P.world > 1 && P.r > kFloorSel)) {   // (no floor)
        CK(cudaMemsetAsync(g, 0x80, 32 * sizeof(long long), st));
    } else {
        double K[33];
        score_constants(P.n, h->score, K);
        FloorK fk;
        for (int q = 0; q <= kFloorDepth + kFloorSel; ++q) fk.k[q] = K[q];
        const uint32_t t0 = (uint32_t)P.rank, t1 = ((1u << P.r) - 1u) ^ (uint32_t)P.rank;
        CK(launch_gbest_init(h->d_root, h->d_order, P.m, P.mhalf_n, fk, g, P.world > 1 ? P.r : 0, t0, t1, st));
    }
    return BNREG_OK;
}

// the candidate floor of seed buffer `buf` on the auxiliary stream, forked from `st` (the root
// R is ready there); gbest_join makes `st` wait for it
static bnreg_status gbest_fork(bnreg_t* h, cudaStream_t st, int buf)
{
    CK(cudaEventRecord(h->ev_root, st));
    CK(cudaStreamWaitEvent(h->aux_stream, h->ev_root, 0));
    const bnreg_status s = gbest_init(h, h->aux_stream, buf);
    if (s != BNREG_OK) return s;
    CK(cudaEventRecord(h->ev_floor, h->aux_stream));
    return BNREG_OK;
}
static bnreg_status gbest_join(bnreg_t* h, cudaStream_t st)
{
    CK(cudaStreamWaitEvent(st, h->ev_floor, 0));
    return BNREG_OK;
}

// pipelined mode: after the root R is in place on the load stream, build the seed tree there too
static bnreg_status prepare_on_load_stream(bnreg_t* h)
{
    // the seeds of this dataset go to the buffer the current walk does not read; the walk
    // that read it last (two runs ago) must be done
    const int b = 1 - h->cur_buf;
    bnreg_status s = BNREG_OK;
    if (!h->w7) {
        CK(cudaStreamWaitEvent(h->load_stream, h->ev_walk[b], 0));   // (the floor of buffer b too)
        s = gbest_fork(h, h->load_stream, b);
        if (s != BNREG_OK) return s;
    }
    s = launch_seed_tree(h, h->load_stream);
    if (s != BNREG_OK) return s;
    CK(cudaStreamWaitEvent(h->load_stream, h->ev_walk[b], 0));
    s = launch_seeds(h, h->load_stream, b);
    if (s != BNREG_OK) return s;
    if (!h->w7) {
        s = gbest_join(h, h->load_stream);
        if (s != BNREG_OK) return s;
    }
    CK(cudaEventRecord(h->ev_prep, h->load_stream));
    h->prepared = true;
    return BNREG_OK;
}

// a1-a2 enqueued on the handle's stream; the status flags land in d_status
static bnreg_status load_enqueue(bnreg_t* h, const double* X, int32_t x_on_device)
{
    const Plan& P = h->plan;
    const size_t nm = (size_t)P.n * P.m;
    const double* src = X;
    // pipelined mode: the load (and the seed tree) run on the load stream once the previous
    // run's seed kernel has consumed the root and the tree
    cudaStream_t ls = h->load_stream ? h->load_stream : h->stream;
    if (h->load_stream) CK(cudaStreamWaitEvent(ls, h->ev_seeds, 0));
    if (!x_on_device) {
        CK(cudaMemcpyAsync(h->dX, X, nm * sizeof(double), cudaMemcpyHostToDevice, ls));
        src = h->dX;
    }
    if (h->timing) CK(cudaEventRecord(h->evl[0], ls));
    CK(cudaMemsetAsync(h->d_status, 0, sizeof(int), ls));
    CK(launch_centre(src, P.n, P.m, h->d_order, h->dXr, h->d_status, ls));
    if (h->root_method == 1) {
        if (!h->d_gram) CK(cudaMalloc(&h->d_gram, (size_t)P.m * P.m * sizeof(double)));
        CK(launch_gram_chol(h->dXr, P.n, P.m, h->d_gram, h->d_root, h->d_status, ls));
    } else {
        CK(launch_tsqr(h->dXr, P.n, P.m, h->d_rbuf, h->d_tcnt, h->nleaf2, h->rb, h->d_root, h->d_status, ls));
    }
    if (h->timing) {
        CK(cudaEventRecord(h->evl[1], ls));
        h->load_timed = true;
    }
    CK(cudaMemcpyAsync(h->h_status, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, ls));
    h->ran = false;
    if (h->load_stream) return prepare_on_load_stream(h);
    return BNREG_OK;
}

// the status flags of the last load, once the stream has passed it
static bnreg_status load_status(bnreg_t* h)
{
    const int status = *h->h_status;
    h->pending = false;
    if (status & 6) {
        h->loaded = false;
        if (status & 2) return fail(BNREG_E_NONFINITE, "X contains NaN or Inf");
        return fail(BNREG_E_RANK, "data is rank deficient (|r_jj| <= 1e-12 max column norm)");
    }
    return BNREG_OK;
}

bnreg_status bnreg_load(bnreg_t* h, const double* X, int32_t x_on_device)
{
    if (!h || !X) return fail(BNREG_E_INVAL, "NULL handle or X");
    h->loaded = false;
    bnreg_status s = load_enqueue(h, X, x_on_device);
    if (s != BNREG_OK) return s;
    CK(stream_wait(h->load_stream ? h->load_stream : h->stream));
    h->loaded = true;
    return load_status(h);
}

bnreg_status bnreg_load_async(bnreg_t* h, const double* X, int32_t x_on_device)
{
    if (!h || !X) return fail(BNREG_E_INVAL, "NULL handle or X");
    bnreg_status s = load_enqueue(h, X, x_on_device);
    if (s != BNREG_OK) {
        h->loaded = false;
        return s;
    }
    h->loaded = true;      // provisionally: the flags are checked by the next synchronous call
    h->pending = true;
    return BNREG_OK;
}

bnreg_status bnreg_sync(bnreg_t* h)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (h->load_stream) CK(stream_wait(h->load_stream));
    CK(stream_wait(h->stream));
    if (h->d_trace && !h->classes.empty()) {
        // BNREG_TRACE: the last walk launch's per-CTA [start, end, items] relative to the first start
        const int g = h->classes[0].grid;
        std::vector<unsigned long long> t(3 * (size_t)g);
        CK(cudaMemcpy(t.data(), h->d_trace, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull, t1 = 0;
        for (int c = 0; c < g; ++c) { t0 = std::min(t0, t[3 * c]); t1 = std::max(t1, t[3 * c + 1]); }
        std::vector<double> ends, starts;
        for (int c = 0; c < g; ++c) { ends.push_back((t[3 * c + 1] - t0) * 1e-6); starts.push_back((t[3 * c] - t0) * 1e-6); }
        std::sort(ends.begin(), ends.end());
        std::sort(starts.begin(), starts.end());
        unsigned long long cand = 0;
        CK(cudaMemcpy(&cand, h->d_trace + 3 * 4096, sizeof(cand), cudaMemcpyDeviceToHost));
        (void)cand;
        fprintf(stderr, "walk trace: span %.3f ms; CTA starts max %.3f ms; CTA ends min %.3f p10 %.3f p50 %.3f p90 %.3f max %.3f ms\n",
                (t1 - t0) * 1e-6, starts.back(), ends.front(), ends[g / 10], ends[g / 2], ends[9 * g / 10], ends.back());
    }
    CK(cudaGetLastError());
    if (h->pending) return load_status(h);
    return BNREG_OK;
}

bnreg_status bnreg_get_root_device(bnreg_t* h, double* R_dev)
{
    if (!h || !R_dev) return fail(BNREG_E_INVAL, "NULL argument");
    if (!h->loaded) return fail(BNREG_E_STATE, "no data loaded");
    const int m = h->plan.m;
    CK(cudaMemcpyAsync(R_dev, h->d_root, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice,
                       h->load_stream ? h->load_stream : h->stream));
    return BNREG_OK;
}

bnreg_status bnreg_set_root_device(bnreg_t* h, const double* R_dev)
{
    if (!h || !R_dev) return fail(BNREG_E_INVAL, "NULL argument");
    const int m = h->plan.m;
    cudaStream_t ls = h->load_stream ? h->load_stream : h->stream;
    if (h->load_stream) CK(cudaStreamWaitEvent(ls, h->ev_seeds, 0));
    CK(cudaMemcpyAsync(h->d_root, R_dev, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, ls));
    h->loaded = true;
    h->pending = false;    // the sender checked its data
    h->ran = false;
    if (h->load_stream) return prepare_on_load_stream(h);
    return BNREG_OK;
}

bnreg_status bnreg_set_load_stream(bnreg_t* h, void* stream)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (h->load_stream) CK(stream_wait(h->load_stream));
    if (h->prepared) CK(cudaStreamWaitEvent(h->stream, h->ev_prep, 0));
    CK(stream_wait(h->stream));
    if (stream && !h->d_seeds2) CK(cudaMalloc(&h->d_seeds2, h->seed_bytes));
    h->load_stream = (cudaStream_t)stream;
    h->prepared = false;
    h->cur_buf = 0;
    return BNREG_OK;
}

bnreg_status bnreg_root_r(const bnreg_t* h, double* R_host, int32_t* order_host)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (!h->loaded) return fail(BNREG_E_STATE, "no data loaded");
    const int m = h->plan.m;
    if (R_host) {
        if (h->load_stream) CK(stream_wait(h->load_stream));
        CK(stream_wait(h->stream));
        CK(cudaMemcpy(R_host, h->d_root, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (order_host)
        for (int j = 0; j < m; ++j) order_host[j] = h->plan.root_order[j];
    return BNREG_OK;
}

int64_t bnreg_num_families(const bnreg_t* h) { return h ? h->plan.local_families : -1; }

int64_t bnreg_launches_per_run(const bnreg_t* h)
{
    if (!h) return -1;
    return (int64_t)(h->plan.L1 > 0 ? 1 : 0) + 1 + (int64_t)h->classes.size() + 1;
}

int64_t bnreg_local_index(const bnreg_t* h, int64_t g)
{
    if (!h || g < 0 || g >= h->plan.total_families) return -1;
    return local_index(h->plan, g);
}

static void shard_ranges_of(const Plan& P, int64_t* count, int64_t* starts, int64_t* lens);

bnreg_status bnreg_shard_ranges(const bnreg_t* h, int64_t* count, int64_t* starts, int64_t* lens)
{
    if (!h || !count) return fail(BNREG_E_INVAL, "NULL argument");
    shard_ranges_of(h->plan, count, starts, lens);
    return BNREG_OK;
}

bnreg_status bnreg_plan_shard_ranges(int32_t m, int64_t n, const bnreg_options* o, int64_t* count, int64_t* starts,
                                     int64_t* lens)
{
    if (!count) return fail(BNREG_E_INVAL, "NULL argument");
    bnreg_options d = defaults(o);
    try {
        Plan P = make_plan(m, n, d.free_vars, d.levels_in_warp, d.world, d.rank, d.pack_bits);
        shard_ranges_of(P, count, starts, lens);
    } catch (std::exception& e) {
        return fail(BNREG_E_INVAL, e.what());
    }
    return BNREG_OK;
}

int64_t bnreg_plan_local_index(int32_t m, int64_t n, const bnreg_options* o, int64_t g)
{
    bnreg_options d = defaults(o);
    try {
        Plan P = make_plan(m, n, d.free_vars, d.levels_in_warp, d.world, d.rank, d.pack_bits);
        if (g < 0 || g >= P.total_families) return -1;
        return local_index(P, g);
    } catch (std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

static void shard_ranges_of(const Plan& P, int64_t* count, int64_t* starts, int64_t* lens)
{
    std::vector<std::pair<int64_t, int64_t>> r;
    for (int v = 0; v < P.m; ++v) {
        int64_t cb = (int64_t)v << (P.m - 1);
        if (P.world == 1) {
            r.push_back({cb, (int64_t)1 << (P.m - 1)});
            continue;
        }
        bool sel = v >= P.m - P.r;
        int sh = sel ? (P.m - P.r) : P.shard_shift;
        r.push_back({cb + ((int64_t)P.pat_lo[v] << sh), (int64_t)1 << sh});
        if (!sel) r.push_back({cb + ((int64_t)P.pat_hi[v] << sh), (int64_t)1 << sh});
    }
    *count = (int64_t)r.size();
    for (size_t i = 0; i < r.size(); ++i) {
        if (starts) starts[i] = r[i].first;
        if (lens) lens[i] = r[i].second;
    }
}

static bnreg_status run_impl(bnreg_t* h, double* out_rss, double* out_bic, uint32_t* bm_dev, double* bb_dev,
                             double* out_pairs = nullptr)
{
    if (out_pairs && (reinterpret_cast<uintptr_t>(out_pairs) & 15u))
        return fail(BNREG_E_INVAL, "out_pairs must be 16-byte aligned");
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (!h->loaded) return fail(BNREG_E_STATE, "no data loaded (bnreg_load / bnreg_root_received first)");
    const Plan& P = h->plan;
    cudaStream_t st = h->stream;
    if (h->timing) CK(cudaEventRecord(h->ev[0], st));
    // a5: the seed tree's nodes at depth L1 (already built on the load stream after a pipelined load)
    const bool prepared = h->prepared;
    if (prepared) {
        CK(cudaStreamWaitEvent(st, h->ev_prep, 0));
        h->prepared = false;
        h->cur_buf = 1 - h->cur_buf;           // the buffer the load stream filled
    } else {
        const bnreg_status ts = launch_seed_tree(h, st);
        if (ts != BNREG_OK) return ts;
    }
    TravParams T{};
    T.m = P.m; T.k = P.k; T.p = P.p; T.bh = P.bh; T.L1 = P.L1; T.nw = 1 << P.p; T.g = P.g; T.lw = P.lw;
    int sched_len = (int)P.sched.size();
    if (const char* dbg = getenv("BNREG_DEBUG_SCHED_LEN")) sched_len = std::min(sched_len, atoi(dbg));  // profiling aid
    T.nsteps = P.k + 1 + sched_len;
    T.packs = h->d_packs;
    T.out_rss = out_rss; T.out_bic = out_bic; T.out_pairs = out_pairs;
    T.part_bic = h->d_part_bic; T.part_mask = h->d_part_mask;
    T.mhalf_n = P.mhalf_n;
    double K[33];
    score_constants(P.n, h->score, K);
    // RSS <= 1e-300 (or 0, or subnormal: the fast log then returns ~-709) has ln RSS <= -690.77,
    // so its score >= (n/2) 690.77 + K(32) (K is non-increasing in |S|); 1 below that for rounding
    T.tiny_bic = (double)P.n / 2.0 * 690.7755278982137 + K[32] - 1.0;
    T.lntab9 = h->d_lntab9;
    T.world1 = P.world == 1 ? 1 : 0;
    for (int s = 0; s <= 32; ++s) T.Kc[s] = K[s];
    T.r = P.r;
    T.k8 = h->k8;
    T.k8_n = (unsigned long long)P.local_families;
    T.k8_selftest = getenv("BNREG_K8_SELFTEST") ? 1 : 0;
    if (getenv("BNREG_TRACE")) {
        // diagnostic: per-CTA start / end times of the walk launch, printed at the next sync
        if (!h->d_trace) CK(cudaMalloc(&h->d_trace, (3 * 4096 + 1) * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(h->d_trace + 3 * 4096, 0, sizeof(unsigned long long), st));
        T.trace = h->d_trace;
    }
    T.patlo = (P.world > 1) ? P.pat_lo[0] : 0u;   // child 0 is never a selector variable
    CK(cudaMemsetAsync(h->d_counters, 0, std::max<size_t>(1, h->classes.size()) * sizeof(unsigned), st));
    // the shared candidate floor starts below every BIC (bytes 0x80: bic_ord of about -7e305)
    if (!h->w7 && !getenv("BNREG_NO_GBEST")) {
        // (after a pipelined load the load stream has set this dataset's floor)
        if (!prepared) {
            const bnreg_status gs = gbest_fork(h, st, h->cur_buf);   // beside the seeds, joined before the walk
            if (gs != BNREG_OK) return gs;
        }
        T.gbest = h->d_gbest + 32 * h->cur_buf;
    }
    // a5: every pack's seeds, in the walk kernel's layout (already derived on the load stream
    //     after a pipelined load)
    if (!prepared) {
        const bnreg_status ss = launch_seeds(h, st, h->cur_buf);
        if (ss != BNREG_OK) return ss;
        if (T.gbest) {
            const bnreg_status js = gbest_join(h, st);
            if (js != BNREG_OK) return js;
        }
    }
    if (h->load_stream && !prepared) CK(cudaEventRecord(h->ev_seeds, st));   // the next load may overwrite root and tree
    if (h->timing) CK(cudaEventRecord(h->ev[1], st));
    // a6-a11: the walk, one launch per shared-memory class
    for (size_t c = 0; c < h->classes.size(); ++c) {
        const auto& C = h->classes[c];
        T.counter = h->d_counters + c;
        T.S_alloc = C.S_alloc;
        T.jbmax = C.jbmax;
        T.tm_cols = walk_tmem_cols(P.k, C.jbmax);
        T.item_begin = C.begin;
        T.item_end = C.end;
        T.part_base = C.part_base;
        T.wsteps = h->d_wsteps + c * h->wsteps_len;
        T.seeds = (h->cur_buf ? h->d_seeds2 : h->d_seeds) + h->seed_off[c];
        if (h->w7) {
            T.KA = h->w7_KA; T.TB = h->w7_TB; T.nbmax = h->w7_nbmax; T.sblk = h->w7_sblk;
            CK(launch_walk7(T, C.grid, h->w7_warps, st));
        } else if (h->ws) {
            CK(launch_walks(T, C.grid, st));
        } else {
            CK(launch_walk(T, C.grid, st));
        }
    }
    CK(cudaEventRecord(h->ev_walk[h->cur_buf], st));   // buffer cur_buf may be refilled after this
    if (h->timing) CK(cudaEventRecord(h->ev[2], st));
    // the handle keeps its own copy of the best masks whatever the caller's target
    // (bnreg_coefficients with masks NULL reads it)
    CK(launch_best_reduce(h->d_part_bic, h->d_part_mask, h->nparts, P.m,
                          bb_dev ? bb_dev : h->d_best_bic, bm_dev ? bm_dev : h->d_best_mask,
                          bm_dev ? h->d_best_mask : nullptr, st));
    if (h->timing) CK(cudaEventRecord(h->ev[3], st));
    h->ran = true;
    return BNREG_OK;
}

static bnreg_status collect_timing(bnreg_t* h)
{
    if (!h->timing) return BNREG_OK;
    CK(event_wait(h->ev[3]));
    float a = 0, b = 0, c = 0, d = 0;
    CK(cudaEventElapsedTime(&a, h->ev[0], h->ev[3]));
    CK(cudaEventElapsedTime(&b, h->ev[0], h->ev[1]));
    CK(cudaEventElapsedTime(&c, h->ev[1], h->ev[2]));
    CK(cudaEventElapsedTime(&d, h->ev[2], h->ev[3]));
    h->acc_ms[0] += a; h->acc_ms[1] += b; h->acc_ms[2] += c; h->acc_ms[3] += d;
    if (h->load_timed) {
        float l = 0;
        CK(cudaEventElapsedTime(&l, h->evl[0], h->evl[1]));
        h->acc_ms[4] += l;
        h->acc_ms[5] += 1;
        h->load_timed = false;
    }
    h->runs += 1;
    return BNREG_OK;
}

static bnreg_status run_sync(bnreg_t* h, double* out_rss, double* out_bic, double* out_pairs, uint32_t* best_mask,
                             double* best_bic)
{
    bnreg_status s = run_impl(h, out_rss, out_bic, nullptr, nullptr, out_pairs);
    if (s != BNREG_OK) return s;
    const int m = h->plan.m;
    if (best_mask)
        CK(cudaMemcpyAsync(best_mask, h->d_best_mask, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
    if (best_bic)
        CK(cudaMemcpyAsync(best_bic, h->d_best_bic, m * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h->stream));
    CK(cudaGetLastError());
    if (h->pending) {
        const bnreg_status ls = load_status(h);
        if (ls != BNREG_OK) return ls;
    }
    return collect_timing(h);
}

bnreg_status bnreg_run(bnreg_t* h, double* out_rss, double* out_bic, uint32_t* best_mask, double* best_bic)
{
    return run_sync(h, out_rss, out_bic, nullptr, best_mask, best_bic);
}

bnreg_status bnreg_run_pairs(bnreg_t* h, double* out_pairs, uint32_t* best_mask, double* best_bic)
{
    if (!out_pairs) return fail(BNREG_E_INVAL, "out_pairs is NULL");
    return run_sync(h, nullptr, nullptr, out_pairs, best_mask, best_bic);
}

bnreg_status bnreg_run_pairs_async(bnreg_t* h, double* out_pairs, uint32_t* bm_dev, double* bb_dev)
{
    if (!out_pairs) return fail(BNREG_E_INVAL, "out_pairs is NULL");
    bnreg_status s = run_impl(h, nullptr, nullptr, bm_dev, bb_dev, out_pairs);
    if (s != BNREG_OK) return s;
    if (h->timing) return collect_timing(h);
    return BNREG_OK;
}

bnreg_status bnreg_run_async(bnreg_t* h, double* out_rss, double* out_bic, uint32_t* bm_dev, double* bb_dev)
{
    bnreg_status s = run_impl(h, out_rss, out_bic, bm_dev, bb_dev);
    if (s != BNREG_OK) return s;
    if (h->timing) return collect_timing(h);   // timing needs the events: synchronises
    return BNREG_OK;
}

bnreg_status bnreg_set_root_method(bnreg_t* h, int32_t method)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (method != 0 && method != 1) return fail(BNREG_E_INVAL, "method must be BNREG_ROOT_TSQR or BNREG_ROOT_CHOLESKY");
    h->root_method = method;
    return BNREG_OK;
}

bnreg_status bnreg_best_subsets(bnreg_t* h, const double* scores, int64_t stride, double* best_score,
                                uint32_t* best_mask)
{
    if (!h || !scores || !best_score || !best_mask) return fail(BNREG_E_INVAL, "NULL argument");
    if (stride < 1) return fail(BNREG_E_INVAL, "stride must be >= 1");
    if (h->plan.world != 1) return fail(BNREG_E_INVAL, "bnreg_best_subsets needs the whole table (world 1)");
    {
        // the passes read and write in place across CTAs: an output may alias the scores
        // only exactly (best_score == scores, stride 1); any other overlap races
        const uintptr_t F = (uintptr_t)h->plan.local_families;
        const uintptr_t s0 = (uintptr_t)scores, s1 = s0 + ((uintptr_t)stride * (F - 1) + 1) * sizeof(double);
        const uintptr_t b0 = (uintptr_t)best_score, b1 = b0 + F * sizeof(double);
        const uintptr_t m0 = (uintptr_t)best_mask, m1 = m0 + F * sizeof(uint32_t);
        const bool exact = stride == 1 && (const void*)scores == (const void*)best_score;
        if (!exact && b0 < s1 && s0 < b1)
            return fail(BNREG_E_INVAL, "best_score overlaps scores (allowed only as best_score == scores with stride 1)");
        if (m0 < s1 && s0 < m1) return fail(BNREG_E_INVAL, "best_mask overlaps scores");
        if (m0 < b1 && b0 < m1) return fail(BNREG_E_INVAL, "best_mask overlaps best_score");
    }
    CK(launch_bps(scores, stride, h->plan.m, best_score, best_mask, h->stream));
    return BNREG_OK;
}

bnreg_status bnreg_coefficients(bnreg_t* h, const uint32_t* masks, double* beta)
{
    if (!h || !beta) return fail(BNREG_E_INVAL, "NULL handle or beta");
    if (!h->loaded) return fail(BNREG_E_STATE, "no data loaded");
    if (!masks && !h->ran) return fail(BNREG_E_STATE, "no run yet: pass the parent sets");
    const int m = h->plan.m;
    if (!h->d_coef) {
        CK(cudaMalloc(&h->d_coef, (size_t)m * m * sizeof(double)));
        CK(cudaMalloc(&h->d_cmask, (size_t)m * sizeof(uint32_t)));
    }
    const uint32_t* dm = h->d_best_mask;
    if (masks) {
        CK(cudaMemcpyAsync(h->d_cmask, masks, (size_t)m * sizeof(uint32_t), cudaMemcpyHostToDevice, h->stream));
        dm = h->d_cmask;
    }
    if (h->load_stream) CK(cudaStreamWaitEvent(h->stream, h->ev_prep, 0));   // a pipelined load's root
    CK(launch_coefficients(h->d_root, h->d_order, m, nullptr, dm, m, h->d_coef, h->stream));
    CK(cudaMemcpyAsync(beta, h->d_coef, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h->stream));
    return BNREG_OK;
}

bnreg_status bnreg_coefficients_batch(bnreg_t* h, const int32_t* children, const uint32_t* masks, int64_t count,
                                      double* beta)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (count < 0) return fail(BNREG_E_INVAL, "negative count");
    if (count > 0 && (!children || !masks || !beta)) return fail(BNREG_E_INVAL, "NULL children, masks or beta");
    if (!h->loaded) return fail(BNREG_E_STATE, "no data loaded");
    if (h->load_stream) CK(cudaStreamWaitEvent(h->stream, h->ev_prep, 0));
    CK(launch_coefficients(h->d_root, h->d_order, h->plan.m, children, masks, count, beta, h->stream));
    return BNREG_OK;
}

bnreg_status bnreg_set_score(bnreg_t* h, int32_t score)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (score < 0 || score > 2) return fail(BNREG_E_INVAL, "score must be BNREG_SCORE_BIC, _AIC or _LOGLIK");
    h->score = score;
    return BNREG_OK;
}

bnreg_status bnreg_all_rss(bnreg_t* h, double* out) { return bnreg_run(h, out, nullptr, nullptr, nullptr); }
bnreg_status bnreg_bic(bnreg_t* h, double* out) { return bnreg_run(h, nullptr, out, nullptr, nullptr); }

bnreg_status bnreg_best_merge(int32_t m, int32_t nparts, const uint32_t* masks, const double* bics,
                              uint32_t* out_mask, double* out_bic)
{
    if (m < 2 || m > kMaxM || nparts < 1 || !masks || !bics) return fail(BNREG_E_INVAL, "bad arguments");
    for (int v = 0; v < m; ++v) {
        double bb = -INFINITY;
        uint32_t bm = 0xffffffffu;
        int bs = 1 << 30;
        for (int q = 0; q < nparts; ++q) {
            uint32_t mk = masks[(size_t)q * m + v];
            if (mk == 0xffffffffu) continue;
            double b = bics[(size_t)q * m + v];
            int s = popc(mk);
            if (b > bb || (b == bb && (s < bs || (s == bs && mk < bm)))) { bb = b; bm = mk; bs = s; }
        }
        if (out_mask) out_mask[v] = bm;
        if (out_bic) out_bic[v] = bb;
    }
    return BNREG_OK;
}

bnreg_status bnreg_best_merge_async(bnreg_t* h, int32_t nparts, const uint32_t* masks_dev, const double* bics_dev,
                                    int64_t row_bytes, uint32_t* out_mask_dev, double* out_bic_dev)
{
    if (!h || nparts < 1 || !masks_dev || !bics_dev || !out_mask_dev || !out_bic_dev || row_bytes < 0 ||
        (row_bytes & 7) || (row_bytes > 0 && row_bytes < 8 * (int64_t)h->plan.m))
        return fail(BNREG_E_INVAL, "bad arguments");
    // the same deterministic G14 reduction as the per-warp partials (one CTA per child)
    CK(launch_best_reduce(bics_dev, masks_dev, nparts, h->plan.m, out_bic_dev, out_mask_dev, nullptr, h->stream,
                          (size_t)row_bytes));
    return BNREG_OK;
}

bnreg_status bnreg_debug_write_counts(bnreg_t* h, uint32_t* counts_dev)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
#ifdef BNREG_K8
    h->k8 = counts_dev;
    return BNREG_OK;
#else
    (void)counts_dev;
    return fail(BNREG_E_INVAL, "this library was built without BNREG_K8 (libbnreg_k8.so has the write counters)");
#endif
}

bnreg_status bnreg_timing(bnreg_t* h, int32_t enable, double* out_ms, int64_t* runs)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (out_ms)
        for (int i = 0; i < 6; ++i) out_ms[i] = h->acc_ms[i];
    if (runs) *runs = h->runs;
    if (enable == 1) {
        h->timing = true;
        for (double& a : h->acc_ms) a = 0;
        h->runs = 0;
    } else if (enable == 0) {
        h->timing = false;
    }
    return BNREG_OK;
}

bnreg_status bnreg_debug_ln(bnreg_t* h, const double* x_dev, double* out_dev, int64_t count)
{
    if (!h || (!x_dev && count > 0) || (!out_dev && count > 0)) return fail(BNREG_E_INVAL, "NULL argument");
    CK(launch_debug_ln(x_dev, out_dev, count, h->d_lntab9, h->stream));
    CK(stream_wait(h->stream));
    return BNREG_OK;
}

void bnreg_destroy(bnreg_t* h)
{
    if (!h) return;
    if (h->stream) cudaStreamSynchronize(h->stream);
    free_all(h);
    delete h;
}

// ---- multi-GPU with the library's own NCCL communicator (include/bnreg.h)
#define NCK(call)                                                                                  \
    do {                                                                                           \
        const ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess) return fail(BNREG_E_NCCL, std::string(#call) + ": " + nccl().errorString(r_)); \
    } while (0)

bnreg_status bnreg_nccl_unique_id(void* id128)
{
    if (!id128) return fail(BNREG_E_INVAL, "id is NULL");
    if (!nccl().ok) return fail(BNREG_E_NCCL, nccl().why);
    ncclUniqueId id;
    NCK(nccl().getUniqueId(&id));
    memcpy(id128, &id, sizeof(id));
    return BNREG_OK;
}

bnreg_status bnreg_load_dist(bnreg_t* h, const double* X)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (!h->comm) return fail(BNREG_E_STATE, "not a bnreg_create_dist handle");
    const Plan& P = h->plan;
    const size_t mm = (size_t)P.m * P.m;
    bnreg_status s = BNREG_OK;
    std::string why;
    if (P.rank == 0) {
        // rank 0 factors X; on failure it still takes part in the broadcast (a NaN R tells
        // the other ranks), then returns its error
        s = X ? bnreg_load(h, X, 0) : fail(BNREG_E_INVAL, "rank 0 needs X");
        why = g_err;
        if (s == BNREG_OK) s = bnreg_get_root_device(h, h->d_Rt);
        if (s == BNREG_OK) CK(stream_wait(h->load_stream ? h->load_stream : h->stream));
        else CK(cudaMemsetAsync(h->d_Rt, 0xff, mm * sizeof(double), h->stream));
    }
    NCK(nccl().broadcast(h->d_Rt, h->d_Rt, mm, ncclFloat64, 0, h->comm, h->stream));
    CK(stream_wait(h->stream));
    if (P.rank == 0) {
        if (s != BNREG_OK) g_err = why;
        return s;
    }
    double r00 = 0.0;
    CK(cudaMemcpy(&r00, h->d_Rt, sizeof(double), cudaMemcpyDeviceToHost));
    if (!(r00 == r00)) return fail(BNREG_E_STATE, "rank 0 could not load its data");
    s = bnreg_set_root_device(h, h->d_Rt);
    if (s != BNREG_OK) return s;
    CK(stream_wait(h->load_stream ? h->load_stream : h->stream));
    return BNREG_OK;
}

bnreg_status bnreg_create_dist(const double* X, int64_t n, int32_t m, const void* nccl_id, int32_t rank,
                               int32_t world, bnreg_t** out)
{
    if (!out || !nccl_id) return fail(BNREG_E_INVAL, "NULL argument");
    *out = nullptr;
    if (!nccl().ok) return fail(BNREG_E_NCCL, nccl().why);
    bnreg_options o = defaults(nullptr);
    o.world = world;
    o.rank = rank;
    bnreg_t* h = nullptr;
    bnreg_status s = bnreg_create_ex(n, m, &o, &h);
    if (s != BNREG_OK) return s;
    auto bail = [&](bnreg_status st) {
        const std::string keep = g_err;
        bnreg_destroy(h);
        g_err = keep;
        return st;
    };
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    const ncclResult_t r = nccl().commInitRank(&h->comm, world, id, rank);
    if (r != ncclSuccess) {
        h->comm = nullptr;
        return bail(fail(BNREG_E_NCCL, std::string("ncclCommInitRank: ") + nccl().errorString(r)));
    }
    if (cudaMalloc(&h->d_Rt, (size_t)m * m * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&h->d_rec, (size_t)world * 2 * m * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&h->d_gm, (size_t)m * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&h->d_gb, (size_t)m * sizeof(double)) != cudaSuccess)
        return bail(fail(BNREG_E_NOMEM, "cudaMalloc of the dist buffers"));
    s = bnreg_load_dist(h, X);
    if (s != BNREG_OK) return bail(s);
    *out = h;
    return BNREG_OK;
}

bnreg_status bnreg_run_pairs_dist(bnreg_t* h, double* out_pairs, uint32_t* best_mask, double* best_bic)
{
    if (!h) return fail(BNREG_E_INVAL, "NULL handle");
    if (!h->comm) return fail(BNREG_E_STATE, "not a bnreg_create_dist handle");
    const Plan& P = h->plan;
    const int m = P.m;
    // this rank's best into its row of the gather buffer: [m BICs | m masks]
    double* row = h->d_rec + (size_t)P.rank * 2 * m;
    bnreg_status s = bnreg_run_pairs_async(h, out_pairs, (uint32_t*)(row + m), row);
    if (s != BNREG_OK) return s;
    NCK(nccl().allGather(row, h->d_rec, (size_t)2 * m, ncclFloat64, h->comm, h->stream));
    s = bnreg_best_merge_async(h, P.world, (const uint32_t*)(h->d_rec + m), h->d_rec, (int64_t)16 * m, h->d_gm,
                               h->d_gb);
    if (s != BNREG_OK) return s;
    if (best_mask) CK(cudaMemcpyAsync(best_mask, h->d_gm, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
    if (best_bic) CK(cudaMemcpyAsync(best_bic, h->d_gb, m * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h->stream));
    if (h->pending) return load_status(h);
    return BNREG_OK;
}
#undef NCK

}  // extern "C"
