/*
 * oracle.c -- the plain, slow, obviously-correct CPU fp64 oracle for bnreg.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this file.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1901_07643_b200/csrc/), and it never calls it.
 *
 * What it computes is the plain definition of the method's output: the paper
 * computes, "for an efficient and exact calculation of regressions for all
 * child and parent-set combinations" (Abstract/§1), the
 * least-squares regression of every child over every parent set; the naive
 * strategy it improves on is to "solve the regression equations for each
 * family independent of the other families" (§1.1).  That naive
 * strategy IS this oracle: one independent Householder QR
 * per family, nothing shared between families, no Givens, no schedule.
 *
 * Readings of the paper used here (all listed in DESIGN.md "Readings"):
 *   G4  intercept: columns are centred first; RSS(v|{}) = ||x_v - mean||^2.
 *   G5  score: Gaussian BIC, higher is better,
 *         BIC = -(n/2) ln(RSS/n) - (n/2)(1 + ln 2pi) - (|S|/2) ln n
 *       (parameter count = number of parents).
 *   G13 RSS <= 1e-300 (perfect fit) gives BIC = +inf.
 *   G14 argmax tie-break: larger BIC; on exact equality smaller |S|, then
 *       smaller mask.
 *   D6  table index = child * 2^(m-1) + compress(S, child), where compress
 *       deletes bit `child` from the user-id mask S.
 *   V17 RSS is the squared norm of the untouched tail of Q^T y (equivalently
 *       r_{k+1,k+1}^2); the "head subtraction" ||y||^2 - ||Q_S^T y||^2 of
 *       SPEC.md:354 is NOT used (it cancels on collinear data).
 *
 * Functions and the passage each follows:
 *   oracle_centre        a1 / G4: mean with a long double accumulator in index
 *                        order, then x - mean.
 *   oracle_householder_rss   PAPER.md:22 (naive per-family QR, O(2nk^2)):
 *                        k Householder reflections on [X_S | y], RSS = tail^2.
 *   oracle_rss           O1 for one family (gathers the columns, calls above).
 *   oracle_rss_residual  SPEC.md:354/:380 self-check: beta by back substitution
 *                        on the same factorization, then the explicit residual
 *                        ||y - X_S beta||^2 (a second, differently-rounded route).
 *   oracle_qr_r          Householder R of the whole centred X (PAPER.md:134
 *                        "starts with calculating the QRD of the data matrix");
 *                        rows sign-normalised so diag(R) > 0.
 *   oracle_rss_reduced   O2: the same per-family Householder
 *                        on the m x (k+1) slice [R0[:,S] | R0[:,v]] (valid since
 *                        X = Q0 R0 with Q0 orthonormal).
 *   oracle_bic           G5/G13.
 *   oracle_table         O1 over every family (OpenMP over families).
 *   oracle_best          G14 argmax per child over a full BIC table.
 *   oracle_reduced_table O2 + oracle_bic over every family (full-size parity).
 *   oracle_best_reduced  oracle_best over O2 + oracle_bic, streamed (no table):
 *                        per child the G14 best and runner-up (cfg4/cfg5 argmax
 *                        goldens, tests/golden/make_best_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_API __attribute__((visibility("default")))

/* ---- indexing (D6) ---------------------------------------------------- */
ORACLE_API int64_t oracle_index(int m, int child, uint32_t mask)
{
    if (child < 0 || child >= m || (mask >> child) & 1u) return -1;
    uint32_t lo = mask & ((1u << child) - 1u);
    uint32_t hi = (uint32_t)((uint64_t)mask >> (child + 1));
    uint64_t c = (uint64_t)lo | ((uint64_t)hi << child);
    return ((int64_t)child << (m - 1)) + (int64_t)c;
}

ORACLE_API uint32_t oracle_mask_of(int m, int64_t idx, int *child)
{
    int v = (int)(idx >> (m - 1));
    uint64_t c = (uint64_t)idx & ((1ull << (m - 1)) - 1ull);
    uint64_t lo = c & ((1ull << v) - 1ull);
    uint64_t hi = c >> v;
    if (child) *child = v;
    return (uint32_t)(lo | (hi << (v + 1)));
}

/* ---- a1: centring ------------------------------------------------------ */
/* X, Xc: column-major n x m.  Returns 0, or 2 if any entry is not finite. */
ORACLE_API int oracle_centre(const double *X, int64_t n, int m, double *Xc)
{
    for (int v = 0; v < m; ++v) {
        long double s = 0.0L;
        for (int64_t i = 0; i < n; ++i) {
            double x = X[(int64_t)v * n + i];
            if (!isfinite(x)) return 2;
            s += (long double)x;
        }
        double mu = (double)(s / (long double)n);
        for (int64_t i = 0; i < n; ++i) Xc[(int64_t)v * n + i] = X[(int64_t)v * n + i] - mu;
    }
    return 0;
}

/* ---- one Householder QR of an nr x (k+1) column-major block ------------ */
/* A is overwritten.  Applies k reflections (columns 0..k-1) to all k+1
 * columns; returns sum_{i>=k} A[i][k]^2, the squared norm of the part of the
 * last column (the response) orthogonal to the first k columns. */
ORACLE_API double oracle_householder_rss(double *A, int64_t nr, int k)
{
    for (int j = 0; j < k; ++j) {
        double *aj = A + (int64_t)j * nr;
        double norm2 = 0.0;
        for (int64_t i = j; i < nr; ++i) norm2 += aj[i] * aj[i];
        double norm = sqrt(norm2);
        if (norm == 0.0) continue;                 /* zero column: no reflection */
        double alpha = aj[j] > 0 ? -norm : norm;   /* avoid cancellation */
        /* v = x - alpha e1, stored in place of column j; v^T v = 2 norm (norm + |x0|) */
        aj[j] -= alpha;
        double vtv = 0.0;
        for (int64_t i = j; i < nr; ++i) vtv += aj[i] * aj[i];
        for (int c = j + 1; c <= k; ++c) {
            double *ac = A + (int64_t)c * nr;
            double d = 0.0;
            for (int64_t i = j; i < nr; ++i) d += aj[i] * ac[i];
            double f = 2.0 * d / vtv;
            for (int64_t i = j; i < nr; ++i) ac[i] -= f * aj[i];
        }
        aj[j] = alpha;                              /* R[j][j] */
        for (int64_t i = j + 1; i < nr; ++i) aj[i] = 0.0;
    }
    const double *y = A + (int64_t)k * nr;
    double rss = 0.0;
    for (int64_t i = k; i < nr; ++i) rss += y[i] * y[i];
    return rss;
}

static int gather(const double *Xc, int64_t n, int m, int child, uint32_t mask, double *A)
{
    int k = 0;
    for (int u = 0; u < m; ++u)
        if ((mask >> u) & 1u) {
            memcpy(A + (int64_t)k * n, Xc + (int64_t)u * n, sizeof(double) * (size_t)n);
            ++k;
        }
    memcpy(A + (int64_t)k * n, Xc + (int64_t)child * n, sizeof(double) * (size_t)n);
    return k;
}

/* O1 for one family.  work: n*(m+1) doubles (NULL: allocated here). */
ORACLE_API double oracle_rss(const double *Xc, int64_t n, int m, int child, uint32_t mask, double *work)
{
    double *A = work ? work : (double *)malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
    int k = gather(Xc, n, m, child, mask, A);
    double r = oracle_householder_rss(A, n, k);
    if (!work) free(A);
    return r;
}

/* SPEC.md:354/:380 self-check: beta from the Householder factorization by
 * back substitution (R beta = (Q^T y)_head), then the explicit residual
 * ||y - X_S beta||^2 computed from the ORIGINAL columns. */
ORACLE_API double oracle_rss_residual(const double *Xc, int64_t n, int m, int child, uint32_t mask)
{
    double *A = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
    int k = gather(Xc, n, m, child, mask, A);
    (void)oracle_householder_rss(A, n, k);
    double beta[64];
    for (int j = k - 1; j >= 0; --j) {
        double s = A[(int64_t)k * n + j];
        for (int c = j + 1; c < k; ++c) s -= A[(int64_t)c * n + j] * beta[c];
        beta[j] = s / A[(int64_t)j * n + j];
    }
    double rss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double r = Xc[(int64_t)child * n + i];
        int c = 0;
        for (int u = 0; u < m; ++u)
            if ((mask >> u) & 1u) { r -= Xc[(int64_t)u * n + i] * beta[c]; ++c; }
        rss += r * r;
    }
    free(A);
    return rss;
}

/* Householder R (m x m, row-major R[i*m+j]) of the centred X, diag > 0. */
ORACLE_API void oracle_qr_r(const double *Xc, int64_t n, int m, double *R)
{
    double *A = (double *)malloc(sizeof(double) * (size_t)n * (size_t)m);
    memcpy(A, Xc, sizeof(double) * (size_t)n * (size_t)m);
    for (int j = 0; j < m; ++j) {
        double *aj = A + (int64_t)j * n;
        double norm2 = 0.0;
        for (int64_t i = j; i < n; ++i) norm2 += aj[i] * aj[i];
        double norm = sqrt(norm2);
        if (norm == 0.0) continue;
        double alpha = aj[j] > 0 ? -norm : norm;
        aj[j] -= alpha;
        double vtv = 0.0;
        for (int64_t i = j; i < n; ++i) vtv += aj[i] * aj[i];
        for (int c = j + 1; c < m; ++c) {
            double *ac = A + (int64_t)c * n;
            double d = 0.0;
            for (int64_t i = j; i < n; ++i) d += aj[i] * ac[i];
            double f = 2.0 * d / vtv;
            for (int64_t i = j; i < n; ++i) ac[i] -= f * aj[i];
        }
        aj[j] = alpha;
    }
    for (int i = 0; i < m; ++i) {
        double sg = A[(int64_t)i * n + i] < 0 ? -1.0 : 1.0;
        for (int j = 0; j < m; ++j) R[i * m + j] = (j < i) ? 0.0 : sg * A[(int64_t)j * n + i];
    }
    free(A);
}

/* O2: per-family Householder on the m x (k+1) slice of R0 (row-major m x m). */
ORACLE_API double oracle_rss_reduced(const double *R0, int m, int child, uint32_t mask)
{
    double A[33 * 33];
    int k = 0;
    for (int u = 0; u < m; ++u)
        if ((mask >> u) & 1u) {
            for (int i = 0; i < m; ++i) A[k * m + i] = R0[i * m + u];
            ++k;
        }
    for (int i = 0; i < m; ++i) A[k * m + i] = R0[i * m + child];
    return oracle_householder_rss(A, m, k);
}

/* ---- a9: BIC (G5, G13) ------------------------------------------------- */
ORACLE_API double oracle_bic(double rss, int64_t n, int k)
{
    if (rss <= 1e-300) return INFINITY;
    double dn = (double)n;
    return -(dn / 2.0) * log(rss / dn) - (dn / 2.0) * (1.0 + log(2.0 * M_PI)) - ((double)k / 2.0) * log(dn);
}

/* ---- other decomposable Gaussian scores -----
 * score 0 = BIC (as oracle_bic), 1 = AIC in the same "higher is better" scale
 * (loglik - k), 2 = the maximised log-likelihood
 * loglik = -(n/2) ln(RSS/n) - (n/2)(1 + ln 2pi); +inf for RSS <= 1e-300 (G13). */
ORACLE_API double oracle_score(double rss, int64_t n, int k, int score)
{
    if (rss <= 1e-300) return INFINITY;
    double dn = (double)n;
    double ll = -(dn / 2.0) * log(rss / dn) - (dn / 2.0) * (1.0 + log(2.0 * M_PI));
    if (score == 1) return ll - (double)k;
    if (score == 2) return ll;
    return ll - ((double)k / 2.0) * log(dn);
}

static int popc32(uint32_t x) { return __builtin_popcount(x); }

/* ---- O1 over the whole table ------------------------------------------- */
/* rss, bic: m * 2^(m-1) entries each (either may be NULL).  threads <= 0: all. */
ORACLE_API void oracle_table(const double *Xc, int64_t n, int m, double *rss, double *bic, int threads)
{
    int64_t total = (int64_t)m << (m - 1);
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        double *work = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
        for (int64_t idx = 0; idx < total; ++idx) {
            int v;
            uint32_t S = oracle_mask_of(m, idx, &v);
            double r = oracle_rss(Xc, n, m, v, S, work);
            if (rss) rss[idx] = r;
            if (bic) bic[idx] = oracle_bic(r, n, popc32(S));
        }
        free(work);
    }
}

/* O1 on a list of flat indices. */
ORACLE_API void oracle_rss_indices(const double *Xc, int64_t n, int m, const int64_t *idx, int64_t count,
                                   double *out, int threads)
{
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        double *work = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
        for (int64_t q = 0; q < count; ++q) {
            int v;
            uint32_t S = oracle_mask_of(m, idx[q], &v);
            out[q] = oracle_rss(Xc, n, m, v, S, work);
        }
        free(work);
    }
}

/* O2 on a list of flat indices (or all of them when idx == NULL). */
ORACLE_API void oracle_rss_reduced_indices(const double *R0, int m, const int64_t *idx, int64_t count,
                                           double *out, int threads)
{
    int64_t total = idx ? count : ((int64_t)m << (m - 1));
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads)
#endif
    for (int64_t q = 0; q < total; ++q) {
        int v;
        uint32_t S = oracle_mask_of(m, idx ? idx[q] : q, &v);
        out[q] = oracle_rss_reduced(R0, m, v, S);
    }
}

/* O2 over the whole table with its BIC (either output may be NULL). */
ORACLE_API void oracle_reduced_table(const double *R0, int m, int64_t n, double *rss, double *bic, int threads)
{
    int64_t total = (int64_t)m << (m - 1);
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4096) num_threads(threads)
#endif
    for (int64_t q = 0; q < total; ++q) {
        int v;
        uint32_t S = oracle_mask_of(m, q, &v);
        double r = oracle_rss_reduced(R0, m, v, S);
        if (rss) rss[q] = r;
        if (bic) bic[q] = oracle_bic(r, n, popc32(S));
    }
}

/* ---- a11: argmax per child (G14) --------------------------------------- */
ORACLE_API void oracle_best(const double *bic, int m, uint32_t *best_mask, double *best_bic)
{
    int64_t per = (int64_t)1 << (m - 1);
    for (int v = 0; v < m; ++v) {
        double bb = -INFINITY;
        uint32_t bm = 0;
        int bp = 1 << 30;
        for (int64_t c = 0; c < per; ++c) {
            int64_t idx = (int64_t)v * per + c;
            int vv;
            uint32_t S = oracle_mask_of(m, idx, &vv);
            double b = bic[idx];
            int p = popc32(S);
            if (b > bb || (b == bb && (p < bp || (p == bp && S < bm)))) { bb = b; bm = S; bp = p; }
        }
        best_mask[v] = bm;
        best_bic[v] = bb;
    }
}

/* ---- a11 over O2 without storing the table (cfg4/cfg5 full size) -------- */
/* For every child v: over all 2^(m-1) parent sets, the G14 best (mask, BIC,
 * RSS) and the runner-up (the G14 best of the other sets) by O2 RSS
 * (oracle_rss_reduced) and oracle_bic -- the composition of oracle_rss_reduced,
 * oracle_bic and oracle_best, streamed so the table never exists.  out arrays
 * have m entries each (any may be NULL except best_mask / best_bic).
 * R0: row-major m x m (oracle_qr_r). */
static int g14_better(double b1, uint32_t s1, double b2, uint32_t s2)
{
    if (b1 != b2) return b1 > b2;
    int p1 = popc32(s1), p2 = popc32(s2);
    return p1 != p2 ? p1 < p2 : s1 < s2;
}

typedef struct { double b1, b2, r1; uint32_t m1, m2; int have1, have2; } top2_t;

static void top2_add(top2_t *t, double b, uint32_t S, double rss)
{
    if (!t->have1 || g14_better(b, S, t->b1, t->m1)) {
        if (t->have1) { t->b2 = t->b1; t->m2 = t->m1; t->have2 = 1; }
        t->b1 = b; t->m1 = S; t->r1 = rss; t->have1 = 1;
    } else if (!t->have2 || g14_better(b, S, t->b2, t->m2)) {
        t->b2 = b; t->m2 = S; t->have2 = 1;
    }
}

ORACLE_API void oracle_best_reduced(const double *R0, int m, int64_t n, uint32_t *best_mask, double *best_bic,
                                    double *best_rss, uint32_t *second_mask, double *second_bic, int threads)
{
    int64_t per = (int64_t)1 << (m - 1);
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#endif
    for (int v = 0; v < m; ++v) {
        top2_t all = {0};
#ifdef _OPENMP
#pragma omp parallel num_threads(threads)
#endif
        {
            top2_t t = {0};
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4096)
#endif
            for (int64_t c = 0; c < per; ++c) {
                int vv;
                uint32_t S = oracle_mask_of(m, (int64_t)v * per + c, &vv);
                double r = oracle_rss_reduced(R0, m, v, S);
                top2_add(&t, oracle_bic(r, n, popc32(S)), S, r);
            }
#ifdef _OPENMP
#pragma omp critical
#endif
            {
                if (t.have1) top2_add(&all, t.b1, t.m1, t.r1);
                if (t.have2) top2_add(&all, t.b2, t.m2, 0.0);
            }
        }
        best_mask[v] = all.m1;
        best_bic[v] = all.b1;
        if (best_rss) best_rss[v] = all.r1;
        if (second_mask) second_mask[v] = all.have2 ? all.m2 : 0xffffffffu;
        if (second_bic) second_bic[v] = all.have2 ? all.b2 : -INFINITY;
    }
}

ORACLE_API int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
