/*
 * wt_fit_core.h -- TEST INFRASTRUCTURE ONLY (oracle/).  Never linked into the
 * product; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may reach it.
 *
 * Plain-C restatement of the small dense linear algebra that the reference's
 * fit_bucket (proj/src/model.cpp:20-77) obtains from Eigen 3.4:
 *   - Eigen::ColPivHouseholderQR<MatrixXd>  (compute, setThreshold, rank,
 *     solve, colsPermutation)                       model.cpp:43-50
 *   - Eigen::HouseholderQR (via householderQr())   model.cpp:55
 *   - MatrixXd * Vector4d, squaredNorm, mean       model.cpp:64-68
 * Eigen is a third-party dependency that is NOT vendored under
 * /root/reference (proj/CMakeLists.txt:11 `find_package(Eigen3 REQUIRED)`,
 * no version pin).  Its published algorithm (Businger-Golub column pivoting
 * with the LAPACK xGEQPF norm-downdate rule, Householder reflectors
 * `makeHouseholderInPlace` / `applyHouseholderOnTheLeft`, unit-stride upper
 * back-substitution) is restated here.
 *
 * Reduction order.  Eigen's vectorised reductions have a build-dependent
 * association order, so bitwise parity with a real Eigen build is UNPINNED
 * (pinned only to 1e-9 by the reference's golden fits, test_model.cpp:23-61,
 * acceptance.cpp:313-323).  This restatement fixes ONE order per problem
 * size that the GPU fit kernels reproduce exactly (products rounded first,
 * sums from +0.0): problems of <= WTF_QROWS (24) rows -- every (macro, wave)
 * bucket of the synthetic plans --
 * reduce rows in plain ascending order (one GPU lane per design column);
 * larger problems (extrapolation windows, per-macro baselines) reduce the
 * QR's dot products as eight interleaved ascending partials in a fixed tree
 * (wtf_qsum; 8 GPU lanes per design column).  Diagnostics (R^2, MAPE) stay
 * ascending.  CPU and GPU agree bit for bit.
 * All arithmetic is IEEE binary64 with no contraction (-ffp-contract=off).
 */
#ifndef WT_FIT_CORE_H
#define WT_FIT_CORE_H

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Sum of v[r] for r in [r0, n), ascending. */
static inline double wtf_sum(const double* v, int r0, int n) {
    double p = 0.0;
    for (int r = r0; r < n; ++r) p = p + v[r];
    return p;
}

/* Problems of up to WTF_QROWS rows reduce in ascending order (the GPU's
 * quad kernel k_qfit: one lane per design column, the problem in a
 * WTF_QROWS-row shared slab); larger ones in the octet order (k_ofit). */
#define WTF_QROWS 24

/* Row sum of the QR's reductions over [r0, n) of an n-row problem.
 * n <= WTF_QROWS: ascending (one GPU lane per design column).  Otherwise eight
 * interleaved ascending partials p_j over the rows r = j (mod 8), combined
 * as ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7)) -- the GPU gives such problems a
 * warp, 8 lanes per column (k_ofit). */
static inline double wtf_qsum(const double* v, int r0, int n) {
    if (n <= WTF_QROWS) return wtf_sum(v, r0, n);
    double p[8];
    for (int j = 0; j < 8; ++j) {
        p[j] = 0.0;
        for (int r = r0 + ((j - r0 % 8) % 8 + 8) % 8; r < n; r += 8) p[j] = p[j] + v[r];
    }
    return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

/* dot(a[r0..n), b[r0..n)) with products rounded first (n = problem rows). */
static inline double wtf_dot(const double* a, const double* b, int r0, int n, double* scratch) {
    for (int r = r0; r < n; ++r) scratch[r] = a[r] * b[r];
    return wtf_qsum(scratch, r0, n);
}

/* Householder reflector for x = col[k..n): Eigen makeHouseholderInPlace.
 * Leaves the essential part in col[k+1..n), returns tau, writes beta. */
static inline double wtf_house(double* col, int k, int n, double* beta, double* scratch) {
    double c0 = col[k];
    double tailsq = (n - k == 1) ? 0.0 : wtf_dot(col, col, k + 1, n, scratch);
    if (tailsq <= DBL_MIN) {
        *beta = c0;
        for (int r = k + 1; r < n; ++r) col[r] = 0.0;
        return 0.0;
    }
    double b = sqrt(c0 * c0 + tailsq);
    if (c0 >= 0.0) b = -b;
    double d = c0 - b;
    for (int r = k + 1; r < n; ++r) col[r] = col[r] / d;
    *beta = b;
    return (b - c0) / b;
}

/* H = I - tau v v^T (v = [1; ess]) applied from the left to rows [k, n) of
 * one column y (Eigen applyHouseholderOnTheLeft, one column at a time). */
static inline void wtf_apply(const double* ess_col, double tau, double* y, int k, int n,
                             double* scratch) {
    if (n - k == 1) {
        y[k] = y[k] * (1.0 - tau);
        return;
    }
    if (tau == 0.0) return;
    double tmp = wtf_dot(ess_col, y, k + 1, n, scratch);
    tmp = tmp + y[k];
    y[k] = y[k] - tau * tmp;
    for (int r = k + 1; r < n; ++r) y[r] = y[r] - (tau * ess_col[r]) * tmp;
}

/* Column-pivoting QR of an n x nc column-major matrix (nc <= 4). */
typedef struct {
    int n, nc, size;
    double* a; /* n*nc, overwritten by R (upper) and reflectors (below) */
    double tau[4];
    int trans[4];
    int perm[4];
    int nonzero_pivots;
    double maxpivot;
} wtf_cpqr;

static inline void wtf_cpqr_compute(wtf_cpqr* q, double* scratch) {
    const int n = q->n, nc = q->nc;
    const int size = n < nc ? n : nc;
    q->size = size;
    double upd[4], direct[4];
    for (int c = 0; c < nc; ++c) {
        direct[c] = sqrt(wtf_dot(q->a + (size_t)c * n, q->a + (size_t)c * n, 0, n, scratch));
        upd[c] = direct[c];
    }
    double mx = upd[0];
    for (int c = 1; c < nc; ++c)
        if (upd[c] > mx) mx = upd[c];
    double th_help = (mx * DBL_EPSILON) * (mx * DBL_EPSILON) / (double)n;
    const double downdate_th = sqrt(DBL_EPSILON);
    q->nonzero_pivots = size;
    q->maxpivot = 0.0;
    for (int k = 0; k < size; ++k) {
        int big = k;
        double bigv = upd[k];
        for (int c = k + 1; c < nc; ++c)
            if (upd[c] > bigv) {
                bigv = upd[c];
                big = c;
            }
        double big_sq = bigv * bigv;
        if (q->nonzero_pivots == size && big_sq < th_help * (double)(n - k)) q->nonzero_pivots = k;
        q->trans[k] = big;
        if (big != k) {
            double* ck = q->a + (size_t)k * n;
            double* cb = q->a + (size_t)big * n;
            for (int r = 0; r < n; ++r) {
                double t = ck[r];
                ck[r] = cb[r];
                cb[r] = t;
            }
            double t = upd[k]; upd[k] = upd[big]; upd[big] = t;
            t = direct[k]; direct[k] = direct[big]; direct[big] = t;
        }
        double* colk = q->a + (size_t)k * n;
        double beta;
        q->tau[k] = wtf_house(colk, k, n, &beta, scratch);
        colk[k] = beta;
        if (fabs(beta) > q->maxpivot) q->maxpivot = fabs(beta);
        for (int j = k + 1; j < nc; ++j) wtf_apply(colk, q->tau[k], q->a + (size_t)j * n, k, n, scratch);
        for (int j = k + 1; j < nc; ++j) {
            if (upd[j] != 0.0) {
                double t = fabs(q->a[(size_t)j * n + k]) / upd[j];
                t = (1.0 + t) * (1.0 - t);
                if (t < 0.0) t = 0.0;
                double ratio = upd[j] / direct[j];
                double t2 = t * (ratio * ratio);
                if (t2 <= downdate_th) {
                    direct[j] = sqrt(wtf_dot(q->a + (size_t)j * n, q->a + (size_t)j * n, k + 1, n, scratch));
                    upd[j] = direct[j];
                } else {
                    upd[j] = upd[j] * sqrt(t);
                }
            }
        }
    }
    for (int c = 0; c < nc; ++c) q->perm[c] = c;
    for (int k = 0; k < size; ++k) {
        int t = q->perm[k];
        q->perm[k] = q->perm[q->trans[k]];
        q->perm[q->trans[k]] = t;
    }
}

static inline int wtf_cpqr_rank(const wtf_cpqr* q, double threshold) {
    double pre = fabs(q->maxpivot) * threshold;
    int rank = 0;
    for (int i = 0; i < q->nonzero_pivots; ++i)
        rank += fabs(q->a[(size_t)i * q->n + i]) > pre;
    return rank;
}

/* Upper back-substitution on c[0..m) with R = a (ld n); Eigen
 * triangular_solve_vector<Upper, ColMajor>, single panel (m <= 8). */
static inline void wtf_backsolve(const double* a, int n, int m, double* c) {
    for (int i = m - 1; i >= 0; --i) {
        if (c[i] != 0.0) {
            c[i] = c[i] / a[(size_t)i * n + i];
            for (int j = 0; j < i; ++j) c[j] = c[j] - c[i] * a[(size_t)i * n + j];
        }
    }
}

/* x (length nc) = least-squares solve with the nonzero pivots. */
static inline void wtf_cpqr_solve(const wtf_cpqr* q, const double* b, double* x, double* work,
                                  double* scratch) {
    const int n = q->n, nz = q->nonzero_pivots;
    if (nz == 0) {
        for (int c = 0; c < q->nc; ++c) x[c] = 0.0;
        return;
    }
    memcpy(work, b, sizeof(double) * (size_t)n);
    for (int k = 0; k < nz; ++k) wtf_apply(q->a + (size_t)k * n, q->tau[k], work, k, n, scratch);
    wtf_backsolve(q->a, n, nz, work);
    for (int i = 0; i < nz; ++i) x[q->perm[i]] = work[i];
    for (int i = nz; i < q->nc; ++i) x[q->perm[i]] = 0.0;
}

/* Unpivoted Householder QR solve of an n x m column-major matrix (m <= 4);
 * a is overwritten.  Eigen HouseholderQR::compute + solve. */
static inline void wtf_hhqr_solve(double* a, int n, int m, const double* b, double* x,
                                  double* work, double* scratch) {
    const int size = n < m ? n : m;
    double tau[4];
    for (int k = 0; k < size; ++k) {
        double* colk = a + (size_t)k * n;
        double beta;
        tau[k] = wtf_house(colk, k, n, &beta, scratch);
        colk[k] = beta;
        for (int j = k + 1; j < m; ++j) wtf_apply(colk, tau[k], a + (size_t)j * n, k, n, scratch);
    }
    memcpy(work, b, sizeof(double) * (size_t)n);
    for (int k = 0; k < size; ++k) wtf_apply(a + (size_t)k * n, tau[k], work, k, n, scratch);
    wtf_backsolve(a, n, size, work);
    for (int i = 0; i < size; ++i) x[i] = work[i];
    for (int i = size; i < m; ++i) x[i] = 0.0;
}

#endif /* WT_FIT_CORE_H */
