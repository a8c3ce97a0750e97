// plan.h -- host-side plan for the bnreg traversal (pure C++, no CUDA).
//
// Everything here is integer bookkeeping that tells the kernels WHAT to walk:
//   * Upsilon(k), the paper's greedy swap schedule (Alg.1 GreedySwaps with the
//     +1 of Eq.10; reading G2),
//   * the Alg.2 partition (readings G7-G11) re-labelled for
//     the B200 layout: which variables are pinned / free, the pack of 2^p
//     lockstep workers a warp runs, the order packs are scheduled in, and
//     which packs a rank owns (complementary top-bit patterns),
//   * the rank-local table layout (index ranges a rank writes),
//   * the BIC constants per parent-set size (reading G5).
//
// Variable roles (reading G27: any relabelling is valid; the table stays keyed
// by user ids):
//   pack vars  ids 0..p-1            (p = min(2, b)); lowest ids so the 2^p
//                                     workers of a pack (one warp) write
//                                     adjacent entries (a 32 B sector)
//   gang vars  ids p..p+g-1           (g <= 2) the 2^g warps of a CTA differ in
//                                     these and step in lockstep, so one step
//                                     writes 2^(p+g) adjacent entries (128 B)
//   free vars  ids p+g..p+g+k-1       the k variables Upsilon(k) permutes
//   hi vars    ids p+g+k..m-1         with the gang vars, the "pinned" levels of
//                                     the seed tree: hv[l] = m-1-l for the top
//                                     ids, then the gang ids p+g-1..p last;
//                                     bit l of the pack id P is hv[l] in F
// A worker = (pack P, w) with w bit j = 1 iff pack var j is in F.  A work item
// = a gang: the 2^g packs whose ids differ only in the top g bits.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>
#include <algorithm>

namespace bnr {

constexpr int kMaxM = 30;        // u32 masks, 64-bit indices; memory caps m far below
constexpr int kMaxFree = 16;     // free vars per worker: 4-bit permutation nibbles in a u64
constexpr int kMaxFreeWalk = 8;  // walk kernel: a step's free list (<= 8 slots) fits one u32 of nibbles, <= 2 per lane
constexpr int kPackBits = 3;     // default: 8 lockstep workers per warp in gangs of 4 warps (walk kernel);
                                 // 5 = 32 workers per warp, one lane each (walk7 kernel: measured slower,
                                 // DESIGN.md §4 "walk7")

// Alg.1 GreedySwaps(m) with Eq.10's +1.
// Returns 1-based swap positions, length 2^m - m - 1 (Eq.9).
inline std::vector<int8_t> greedy_swaps(int m)
{
    std::vector<int8_t> s;
    if (m < 2) return s;
    s.push_back(1);
    for (int q = 3; q <= m; ++q) {              // Upsilon(q) from Upsilon(q-1)
        size_t prev = s.size();
        for (int i = q - 1; i >= 1; --i) s.push_back((int8_t)i);
        for (size_t t = 0; t < prev; ++t) s.push_back((int8_t)(s[t] + 1));
    }
    return s;
}

// One record per lockstep step of a worker's walk (host-built, identical for
// every worker since all of them run Upsilon(k) on their free block):
//   seed pseudo-steps j = 0..k: harvest the seed prefix {free 0..j-1}
//     (reading G11: prefixes of sizes d..d+k), no rotation;
//   real steps t: the GRC at free position i = Upsilon(k)[t] - 1, which swaps
//     free slots X (position i) and Y (position i+1).
// meta: bits 0-4 = i + 1 (seed j: i = j - 1), 5-8 = X, 9-12 = Y, 13-17 = nf
// (free children after the prefix), bit 18 = seed.  T = free-slot mask of the
// new prefix set.  (lo, hi) = nibbles of the free slots at positions i+1.. .
struct StepRec {
    uint32_t meta, T, lo, hi;
};

inline std::vector<StepRec> step_records(int k, const std::vector<int8_t>& sched)
{
    std::vector<StepRec> out;
    std::vector<int> perm(k);
    for (int f = 0; f < k; ++f) perm[f] = f;
    auto list_of = [&](int from, StepRec& r) {
        uint64_t nib = 0;
        for (int pos = from, e = 0; pos < k; ++pos, ++e) nib |= (uint64_t)perm[pos] << (4 * e);
        r.lo = (uint32_t)nib;
        r.hi = (uint32_t)(nib >> 32);
    };
    for (int j = 0; j <= k; ++j) {
        StepRec r{};
        const int i = j - 1, nf = k - j;
        r.meta = (uint32_t)(i + 1) | ((uint32_t)nf << 13) | (1u << 18);
        r.T = (uint32_t)((1u << j) - 1u);
        list_of(j, r);
        out.push_back(r);
    }
    for (int8_t s1 : sched) {
        const int i = s1 - 1;
        const int X = perm[i], Y = perm[i + 1];
        std::swap(perm[i], perm[i + 1]);
        StepRec r{};
        const int nf = k - 1 - i;
        r.meta = (uint32_t)(i + 1) | ((uint32_t)X << 5) | ((uint32_t)Y << 9) | ((uint32_t)nf << 13);
        uint32_t T = 0;
        for (int q = 0; q <= i; ++q) T |= 1u << perm[q];
        r.T = T;
        list_of(i + 1, r);
        out.push_back(r);
    }
    return out;
}

// The walk kernel's per-step table for one shared-memory class: the step
// records above turned into byte offsets of its walk-state layout (slot stride
// CS = W*16 bytes, row stride RS = SA*W*16 bytes), one uint4 per step:
//   x: i*RS (0 for i < 0)
//   y: in*RS + Yn*CS, the next step's pivot column if the next step is a GRC (else 0)
//   z: the free-list nibbles (k <= 9: the list after a prefix has <= 8 slots)
//   w: nf | seed << 5 | (i < 0) << 6 | next-is-GRC << 7 | (i + 1) << 8 | Y << 13 | T << 17
struct WalkStep {
    uint32_t offA, offN, nib, flags;
};

inline std::vector<WalkStep> walk_step_table(const std::vector<StepRec>& recs, int k, int SA, int W)
{
    const uint32_t CS = (uint32_t)W * 16u, RS = (uint32_t)SA * W * 16u;
    std::vector<WalkStep> out(recs.size());
    for (size_t t = 0; t < recs.size(); ++t) {
        const StepRec& r = recs[t];
        const int i = (int)(r.meta & 31u) - 1;
        const int Y = (int)((r.meta >> 9) & 15u);
        const int nf = (int)((r.meta >> 13) & 31u);
        const bool seed = (r.meta >> 18) & 1u;
        WalkStep w{};
        w.offA = i < 0 ? 0u : (uint32_t)i * RS;
        bool next = false;
        if (t + 1 < recs.size() && !((recs[t + 1].meta >> 18) & 1u)) {
            next = true;
            const int in = (int)(recs[t + 1].meta & 31u) - 1;
            const int Yn = (int)((recs[t + 1].meta >> 9) & 15u);
            w.offN = (uint32_t)in * RS + (uint32_t)Yn * CS;
        }
        w.nib = r.lo;
        w.flags = (uint32_t)nf | ((seed ? 1u : 0u) << 5) | ((i < 0 ? 1u : 0u) << 6) | ((next ? 1u : 0u) << 7) |
                  ((uint32_t)(i + 1) << 8) | ((uint32_t)(seed ? 0 : Y) << 13) | (r.T << 17);
        out[t] = w;
    }
    return out;
}

// The same records for the slot-split walk (walks_kernel.cuh, "design S"): the gang's 4
// warps share the free-slot state E(l, s, worker) (slot stride CS = 32*16 B, row stride
// RS = k*CS) and deal each step's free list by position (entry f -> warp f mod 4).  Every
// warp computes a GRC's rotation itself from the pivot column's rows, which one warp,
// stg(t), copies to a staging buffer in step t - 1: the warp that rotated the pivot's
// column in step t - 1 (the owner of its list entry), else warp 3 (it writes every pivot,
// and rows written before the last step barrier are visible to it).
//   x: i*RS (0 for i < 0)
//   y: in*RS + Yn*CS | stg(t + 1) << 16, if the next step is a GRC (else 0)
//   z: the free-list nibbles (as walk_step_table)
//   w: the flags of walk_step_table
inline std::vector<WalkStep> walk_step_table_s(const std::vector<StepRec>& recs, int k)
{
    const uint32_t CS = 512u, RS = (uint32_t)k * 512u;
    std::vector<WalkStep> out = walk_step_table(recs, k, k, 8);
    for (size_t t = 0; t < recs.size(); ++t) {
        const StepRec& r = recs[t];
        const int i = (int)(r.meta & 31u) - 1;
        const int nf = (int)((r.meta >> 13) & 31u);
        const bool seed = (r.meta >> 18) & 1u;
        WalkStep& w = out[t];
        w.offA = i < 0 ? 0u : (uint32_t)i * RS;
        w.offN = 0;
        if ((w.flags >> 7) & 1u) {
            const int in = (int)(recs[t + 1].meta & 31u) - 1;
            const int Yn = (int)((recs[t + 1].meta >> 9) & 15u);
            uint32_t sw = 3;
            if (!seed) {
                const uint64_t nib = (uint64_t)r.lo | ((uint64_t)r.hi << 32);
                for (int e = 0; e < nf; ++e)
                    if ((int)((nib >> (4 * e)) & 15u) == Yn) sw = (uint32_t)(e % 4);
            }
            w.offN = ((uint32_t)in * RS + (uint32_t)Yn * CS) | (sw << 16);
        }
    }
    return out;
}

struct Plan {
    int m = 0, k = 0, b = 0, p = 0, bh = 0;   // b = m - k pinned, p pack bits, bh tree bits (incl. gang)
    int lw = kPackBits;                       // walk kernel: log2 lockstep workers per warp
    int g = 0;                                // gang bits (the top g of the bh tree bits)
    int L1 = 0, LW = 0;                       // tree depth in global memory / levels derived in-warp
    int world = 1, rank = 0, r = 0;           // rank selector bits r (0 when world == 1)
    int64_t n = 0;
    int64_t total_families = 0;               // m 2^(m-1)
    int64_t local_families = 0;               // this rank's share
    std::vector<int8_t> sched;                // Upsilon(k), 1-based
    std::vector<uint32_t> packs;              // this rank's work items (gang base pack ids), costliest first
    std::vector<int> root_order;              // position -> user id of the root R
    // rank-local layout: per child, up to 2 ranges of the child's 2^(m-1) block
    int64_t child_base[32] = {0};             // local offset of child v's first range
    int32_t shard_shift = 0;                  // m-1-r : low bits kept inside a range
    uint32_t pat_lo[32] = {0}, pat_hi[32] = {0}; // per child: selector patterns of range 0 / 1
    int32_t nrange[32] = {0};
    double bic_const[33] = {0};               // K(s) = (n/2)ln n - (n/2)(1+ln 2pi) - (s/2) ln n
    double mhalf_n = 0;                       // -n/2
};

inline int popc(uint32_t x) { return __builtin_popcount(x); }

// user id of tree level l (bit l of a pack id)
inline int hv_id(const Plan& P, int l)
{
    return l < P.bh - P.g ? P.m - 1 - l : P.p + P.g - 1 - (l - (P.bh - P.g));
}

// Cost of a pack in families (sum over its 2^p workers of 2^(k-1)(2(m-d)-k)).
inline int64_t pack_cost(const Plan& P, uint32_t pack)
{
    int64_t c = 0;
    int dh = popc(pack);
    for (int w = 0; w < (1 << P.p); ++w) {
        int d = dh + popc((uint32_t)w);
        c += (int64_t(1) << (P.k - 1)) * (2 * (P.m - d) - P.k);
    }
    return c;
}

// k: requested free count (0 = auto).  lw: tree levels derived in-warp (-1 = auto).
// pack_bits: log2 lockstep workers per warp (0 = auto = kPackBits; 3 or 5).
inline Plan make_plan(int m, int64_t n, int k, int lw, int world, int rank, int pack_bits = 0)
{
    Plan P;
    if (m < 2 || m > kMaxM) throw std::invalid_argument("m must be in [2, 30]");
    if (n < m + 1) throw std::invalid_argument("need n >= m + 1");
    if (world < 1 || rank < 0 || rank >= world || (world & (world - 1)))
        throw std::invalid_argument("world must be a power of two and 0 <= rank < world");
    // default k: the walk kernel's shared memory grows with k (k rows of state per slot);
    // k = 8 balances it against the seed derivation (~2k GRCs per worker, 2^k - k - 1 walk steps)
    if (k <= 0) k = std::min(m, 8);
    if (k < 2 || k > m || k > kMaxFree) throw std::invalid_argument("free count k must be in [2, min(m,16)]");
    if (k > kMaxFreeWalk)
        throw std::invalid_argument("the walk kernel takes at most 8 free variables (k <= 8)");
    P.m = m; P.n = n; P.k = k; P.b = m - k;
    if (pack_bits == 0) pack_bits = kPackBits;
    if (pack_bits != 3 && pack_bits != 5) throw std::invalid_argument("pack_bits must be 3 or 5 (8 or 32 workers per warp)");
    P.lw = pack_bits;
    P.p = std::min(P.lw, P.b);
    P.bh = P.b - P.p;
    // walk kernel: a CTA's 2^g warps x 2^lw workers = 32 workers = 256 B per (child, step)
    P.g = std::min(5 - P.lw, P.bh);
    if (lw < 0) lw = 4;
    P.LW = std::min(std::max(lw, P.g), P.bh);
    P.L1 = P.bh - P.LW;
    P.world = world; P.rank = rank;
    P.total_families = (int64_t)m << (m - 1);
    P.sched = greedy_swaps(k);
    // root order: [hv[0..bh-1], pack vars, free p+g..p+g+k-1]
    for (int l = 0; l < P.bh; ++l) P.root_order.push_back(hv_id(P, l));
    // the seed kernel's Gray path wants the warp variables in descending id
    // next to the free block ([w_{p-1} .. w_0 | free])
    for (int j = 0; j < P.p; ++j) P.root_order.push_back(P.p - 1 - j);
    for (int f = 0; f < k; ++f) P.root_order.push_back(P.p + P.g + f);

    // rank selector: top r hi bits (hv[0..r-1] = ids m-1..m-r), complementary patterns
    if (world > 1) {
        int r = 0;
        while ((1 << r) < 2 * world) ++r;
        if (r > P.bh - P.g) throw std::invalid_argument("too few pinned variables for this world size (lower k)");
        P.r = r;
    }
    uint32_t tmask = (1u << P.r) - 1u;
    uint32_t t0 = (uint32_t)rank, t1 = tmask ^ (uint32_t)rank;
    std::vector<uint32_t> all;
    const int gs = P.bh - P.g;                    // gang bits are the top g tree bits
    auto item_cost = [&](uint32_t q) {
        int64_t c = 0;
        for (uint32_t j = 0; j < (1u << P.g); ++j) c += pack_cost(P, q | (j << gs));
        return c;
    };
    for (uint32_t q = 0; q < (1u << gs); ++q)
        if (world == 1 || (q & tmask) == t0 || (q & tmask) == t1) all.push_back(q);
    std::stable_sort(all.begin(), all.end(), [&](uint32_t a, uint32_t b) {
        int64_t ca = item_cost(a), cb = item_cost(b);
        return ca != cb ? ca > cb : a < b;
    });
    P.packs = all;

    // rank-local layout.  Bits of the compressed mask of child v: the top r
    // positions (m-1-r .. m-2) hold hv[0..r-1] when v is not one of them.
    if (world == 1) {
        P.shard_shift = m - 1;
        for (int v = 0; v < m; ++v) {
            P.child_base[v] = (int64_t)v << (m - 1);
            P.nrange[v] = 1; P.pat_lo[v] = 0; P.pat_hi[v] = 0;
        }
        P.local_families = P.total_families;
    } else {
        int64_t off = 0;
        for (int v = 0; v < m; ++v) {
            P.child_base[v] = off;
            int lv = m - 1 - v;                          // hi level of v, if v is a selector var
            bool sel = v >= m - P.r;
            if (!sel) {
                // selector bits sit at compressed positions m-1-r..m-2, bit order:
                // compressed bit (m-1-r)+j  <->  user id m-r+j  <->  hi level r-1-j
                auto to_comp = [&](uint32_t t) {
                    uint32_t c = 0;
                    for (int l = 0; l < P.r; ++l)
                        if ((t >> l) & 1u) c |= 1u << (P.r - 1 - l);
                    return c;
                };
                uint32_t a = to_comp(t0), b = to_comp(t1);
                P.pat_lo[v] = std::min(a, b); P.pat_hi[v] = std::max(a, b);
                P.nrange[v] = 2;
                off += (int64_t)2 << (m - 1 - P.r);
            } else {
                // v is hv[lv]; it must be in B, so only the pattern with bit lv = 0 owns it
                uint32_t t = ((t0 >> lv) & 1u) ? t1 : t0;
                // remaining r-1 selector bits, compressed: positions m-r..m-2 after deleting v
                uint32_t c = 0;
                int pos = 0;
                for (int id = m - P.r; id < m; ++id) {
                    if (id == v) continue;
                    int l = m - 1 - id;
                    if ((t >> l) & 1u) c |= 1u << pos;
                    ++pos;
                }
                P.pat_lo[v] = c; P.pat_hi[v] = c;
                P.nrange[v] = 1;
                off += (int64_t)1 << (m - P.r);
            }
        }
        P.local_families = off;
    }
    P.shard_shift = (world == 1) ? (m - 1) : (m - 1 - P.r);

    long double nn = (long double)n;
    long double l2pi = logl(2.0L * 3.14159265358979323846264338327950288L);
    for (int s = 0; s <= 32; ++s)
        P.bic_const[s] = (double)((nn / 2) * logl(nn) - (nn / 2) * (1.0L + l2pi) - ((long double)s / 2) * logl(nn));
    P.mhalf_n = -(double)n / 2.0;
    return P;
}

// The score epilogue is score = -(n/2) ln RSS + K(|S|) for every decomposable Gaussian
// score: loglik = -(n/2) ln(RSS/n) - (n/2)(1 + ln 2pi),
// BIC (score 0, reading G5) = loglik - (s/2) ln n, AIC (1) = loglik - s, log-likelihood (2).
inline void score_constants(int64_t n, int score, double* K33)
{
    const long double nn = (long double)n;
    const long double l2pi = logl(2.0L * 3.14159265358979323846264338327950288L);
    for (int s = 0; s <= 32; ++s) {
        const long double ll = (nn / 2) * logl(nn) - (nn / 2) * (1.0L + l2pi);
        const long double pen = score == 1 ? (long double)s : score == 2 ? 0.0L : ((long double)s / 2) * logl(nn);
        K33[s] = (double)(ll - pen);
    }
}

// Global flat index (SPEC.md:179 / D6): child 2^(m-1) + compress(mask, child).
inline int64_t family_index(int m, int child, uint32_t mask)
{
    if (child < 0 || child >= m || ((mask >> child) & 1u)) return -1;
    uint64_t lo = mask & ((1u << child) - 1u);
    uint64_t hi = (uint64_t)mask >> (child + 1);
    return ((int64_t)child << (m - 1)) + (int64_t)(lo | (hi << child));
}

// Rank-local offset of a global index, or -1 if another rank owns it.
inline int64_t local_index(const Plan& P, int64_t gidx)
{
    int v = (int)(gidx >> (P.m - 1));
    uint64_t c = (uint64_t)gidx & ((1ull << (P.m - 1)) - 1ull);
    if (P.world == 1) return gidx;
    bool sel = v >= P.m - P.r;
    int sh = sel ? (P.m - P.r) : P.shard_shift;
    uint64_t pat = c >> sh, low = c & ((1ull << sh) - 1ull);
    if (pat == P.pat_lo[v]) return P.child_base[v] + (int64_t)low;
    if (!sel && pat == P.pat_hi[v]) return P.child_base[v] + ((int64_t)1 << sh) + (int64_t)low;
    return -1;
}

}  // namespace bnr
