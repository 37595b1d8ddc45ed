/*
 * wt_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's WaveTune decision path.  See wt_oracle.h for the contract and
 * the rule on who may load this library.  Every function cites the reference
 * lines it restates (paths relative to /root/reference/proj).
 */
#include "wt_oracle.h"

#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "wt_fit_core.h"

/* ---- L1: mapping ------------------------------------------------------- */

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; } /* kernel_map.hpp:17 */

int wto_map_dense(int64_t m, int64_t n, int64_t k, int64_t t_m, int64_t t_n, int64_t t_k,
                  int64_t* g, int64_t* l) {
    /* kernel_map.cpp:236-243: dims < 1 -> invalid_argument */
    if (m < 1 || n < 1 || k < 1) return WTO_INVALID_ARGUMENT;
    *g = cdiv(m, t_m) * cdiv(n, t_n);
    *l = cdiv(k, t_k);
    return WTO_OK;
}

int wto_wave_count(int64_t g, int32_t n_sm, int32_t bps, int32_t* w) {
    /* kernel_map.cpp:266-271 */
    if (g < 1) return WTO_INVALID_ARGUMENT;
    if (n_sm < 1 || bps < 1) return WTO_INVALID_ARGUMENT;
    *w = (int32_t)cdiv(g, (int64_t)(n_sm * bps));
    return WTO_OK;
}

/* model.hpp:20-23: alpha*g*l + beta*g + gamma*l + delta, left to right. */
static double bilinear(const double* th, int64_t g, int64_t l) {
    double gd = (double)g, ld = (double)l;
    return th[0] * gd * ld + th[1] * gd + th[2] * ld + th[3];
}

/* ---- L4: predict_latency (tuner.cpp:11-42) ----------------------------- */

int wto_predict(const wto_tables* T, int32_t t, int64_t g, int64_t l, int32_t n_sm, int32_t bps,
                double* lat, int32_t* extrap, int32_t* w, int32_t* used_w) {
    if (g < 1 || l < 1) return WTO_INVALID_ARGUMENT;                 /* :14-15 */
    int32_t wc;
    int st = wto_wave_count(g, n_sm, bps, &wc);
    if (st) return st;
    *w = wc;
    *used_w = -1;
    if (wc > T->W[t]) {                                               /* :17-18 */
        *extrap = 1;
        *lat = bilinear(T->theta_ext + 4 * (size_t)t, g, l);
        return WTO_OK;
    }
    *extrap = 0;
    int32_t lo = T->coeff_off[t], hi = T->coeff_off[t + 1];
    for (int32_t i = lo; i < hi; ++i)
        if (T->coeff_w[i] == wc) {                                    /* :20 find */
            *lat = bilinear(T->coeff_theta + 4 * (size_t)i, g, l);
            return WTO_OK;
        }
    if (lo == hi) return WTO_RUNTIME_ERROR;                           /* :23-26 */
    int32_t best_w = 0, best_i = -1;                                  /* :27-35 */
    int best_dist = INT_MAX;
    for (int32_t i = lo; i < hi; ++i) {
        int cand = T->coeff_w[i];
        int dist = abs(cand - wc);
        if (dist < best_dist || (dist == best_dist && cand < best_w)) {
            best_w = cand;
            best_dist = dist;
            best_i = i;
        }
    }
    *used_w = best_w;                                                 /* :36-38 */
    *lat = bilinear(T->coeff_theta + 4 * (size_t)best_i, g, l);
    return WTO_OK;
}

/* ---- nearest_anchor (tuner.cpp:44-70) ---------------------------------- */

int wto_nearest_anchor(const int64_t* a, int32_t n, int64_t l, int64_t* out, int32_t* comps) {
    if (n <= 0) return WTO_INVALID_ARGUMENT;
    int32_t c = 0;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        ++c;
        if (a[mid] < l)
            lo = mid + 1;
        else
            hi = mid;
    }
    if (lo == 0) {
        *out = a[0];
    } else if (lo == n) {
        *out = a[n - 1];
    } else {
        int64_t below = a[lo - 1], above = a[lo];
        ++c;
        *out = (l - below <= above - l) ? below : above;
    }
    *comps = c;
    return WTO_OK;
}

/* ---- Stage I + II (tuner.cpp:76-166) ----------------------------------- */

static const wto_tables* g_sort_T;
static int by_macro(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    int32_t ma = g_sort_T->macro_id[a], mb = g_sort_T->macro_id[b];
    if (ma != mb) return ma < mb ? -1 : 1;
    return a < b ? -1 : (a > b);
}

static int32_t* sorted_order(const wto_tables* T) {
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)(T->n_tables > 0 ? T->n_tables : 1));
    for (int32_t i = 0; i < T->n_tables; ++i) ord[i] = i;
    g_sort_T = T;
    qsort(ord, (size_t)T->n_tables, sizeof(int32_t), by_macro);
    return ord;
}

/* retrieve_micro (tuner.cpp:76-113). */
static int retrieve_micro(const wto_tables* T, int32_t t, int32_t extrap, int32_t w, int64_t l,
                          int32_t* micro, int32_t* comps, int32_t* fb_wave) {
    const int64_t* keys = NULL;
    const int32_t* vals = NULL;
    int32_t cnt = 0;
    *fb_wave = -1;
    if (extrap) {
        int32_t a = T->ext_aoff[t], b = T->ext_aoff[t + 1];
        if (b > a) {
            keys = T->ext_l + a;
            vals = T->ext_micro + a;
            cnt = b - a;
        }
    } else {
        for (int32_t i = T->awave_off[t]; i < T->awave_off[t + 1]; ++i)
            if (T->awave_w[i] == w) {
                int32_t a = T->awave_aoff[i], b = T->awave_aoff[i + 1];
                if (b > a) {
                    keys = T->anchor_l + a;
                    vals = T->anchor_micro + a;
                    cnt = b - a;
                }
                break;
            }
    }
    if (!keys) {
        int32_t best_w = 0, best_i = -1;
        int best_dist = INT_MAX;
        int32_t target = extrap ? T->W[t] : w;
        for (int32_t i = T->awave_off[t]; i < T->awave_off[t + 1]; ++i) {
            if (T->awave_aoff[i + 1] == T->awave_aoff[i]) continue;
            int dist = abs(T->awave_w[i] - target);
            if (dist < best_dist || (dist == best_dist && T->awave_w[i] < best_w)) {
                best_w = T->awave_w[i];
                best_dist = dist;
                best_i = i;
            }
        }
        if (best_dist == INT_MAX) return WTO_RUNTIME_ERROR;
        *fb_wave = best_w;
        keys = T->anchor_l + T->awave_aoff[best_i];
        vals = T->anchor_micro + T->awave_aoff[best_i];
        cnt = T->awave_aoff[best_i + 1] - T->awave_aoff[best_i];
    }
    int64_t chosen;
    int st = wto_nearest_anchor(keys, cnt, l, &chosen, comps);
    if (st) return st;
    for (int32_t i = 0; i < cnt; ++i)
        if (keys[i] == chosen) {
            *micro = vals[i];
            return WTO_OK;
        }
    return WTO_OUT_OF_RANGE;
}

static int tune_one(const wto_tables* T, const int32_t* ord, int32_t n_sm, int32_t bps,
                    int64_t M, int64_t N, int64_t K, int32_t* macro, int32_t* micro, double* lat,
                    int64_t* g_out, int64_t* l_out, int32_t* w_out, int32_t* ex_out,
                    int32_t* comps, int32_t* n_missing, int32_t* anchor_fb) {
    if (T->n_tables == 0) return WTO_INVALID_ARGUMENT;               /* :120 */
    double best = INFINITY;                                          /* :124 */
    int32_t best_t = -1, bw = 0, bex = 0;
    int64_t bg = 0, bl = 0;
    int32_t missing = 0;
    for (int32_t j = 0; j < T->n_tables; ++j) {                     /* :135-149 */
        int32_t t = ord[j];
        int64_t g, l;
        int st = wto_map_dense(M, N, K, T->t_m[t], T->t_n[t], T->t_k[t], &g, &l);
        if (st) return st;
        double v;
        int32_t ex, w, used;
        st = wto_predict(T, t, g, l, n_sm, bps, &v, &ex, &w, &used);
        if (st) return st;
        if (used >= 0) ++missing;
        if (v < best) {                                              /* :140 strict */
            best = v;
            best_t = t;
            bg = g;
            bl = l;
            bw = w;
            bex = ex;
        }
    }
    if (best_t < 0) return WTO_RUNTIME_ERROR; /* reference dereferences null here (:151) */
    int st = retrieve_micro(T, best_t, bex, bw, bl, micro, comps, anchor_fb);
    if (st) return st;
    *macro = T->macro_id[best_t];
    *lat = best;
    *g_out = bg;
    *l_out = bl;
    *w_out = bw;
    *ex_out = bex;
    *n_missing = missing;
    return WTO_OK;
}

void wto_tune(const wto_tables* T, int32_t n_sm, int32_t bps, const int64_t* M, const int64_t* N,
              const int64_t* K, int64_t n, int32_t* macro, int32_t* micro, double* lat, int64_t* g,
              int64_t* l, int32_t* w, int32_t* extrap, int32_t* comps, int32_t* n_missing,
              int32_t* anchor_fb, int32_t* status) {
    int32_t* ord = sorted_order(T);
    for (int64_t i = 0; i < n; ++i)
        status[i] = tune_one(T, ord, n_sm, bps, M[i], N[i], K[i], &macro[i], &micro[i], &lat[i],
                             &g[i], &l[i], &w[i], &extrap[i], &comps[i], &n_missing[i],
                             &anchor_fb[i]);
    free(ord);
}

int wto_topk(const wto_tables* T, int32_t n_sm, int32_t bps, int64_t M, int64_t N, int64_t K,
             int32_t k, int32_t* macro, double* lat) {
    for (int32_t i = 0; i < k; ++i) {
        macro[i] = -1;
        lat[i] = NAN;
    }
    int32_t* ord = sorted_order(T);
    int32_t filled = 0;
    for (int32_t j = 0; j < T->n_tables; ++j) {
        int32_t t = ord[j];
        int64_t g, l;
        int st = wto_map_dense(M, N, K, T->t_m[t], T->t_n[t], T->t_k[t], &g, &l);
        double v;
        int32_t ex, w, used;
        if (!st) st = wto_predict(T, t, g, l, n_sm, bps, &v, &ex, &w, &used);
        if (st) {
            free(ord);
            return st;
        }
        if (isnan(v) || v == INFINITY) continue;
        /* insertion: strictly smaller latency moves ahead (ascending macro
         * order already breaks ties toward the smaller id). */
        int32_t pos = filled;
        while (pos > 0 && v < lat[pos - 1]) --pos;
        if (pos >= k) continue;
        int32_t last = filled < k ? filled : k - 1;
        for (int32_t q = last; q > pos; --q) {
            lat[q] = lat[q - 1];
            macro[q] = macro[q - 1];
        }
        lat[pos] = v;
        macro[pos] = T->macro_id[t];
        if (filled < k) ++filled;
    }
    free(ord);
    return WTO_OK;
}

/* ---- L3: fit_bucket (model.cpp:20-77) ----------------------------------- */

int wto_fit_bucket(const double* g, const double* l, const double* t, int32_t n, double* coeffs,
                   double* r2, double* mape, int32_t* degenerate) {
    if (n <= 0) return WTO_INVALID_ARGUMENT;                           /* :21 */
    size_t N = (size_t)n;
    double* design = (double*)malloc(sizeof(double) * N * 4);
    double* scaled = (double*)malloc(sizeof(double) * N * 4);
    double* scratch = (double*)malloc(sizeof(double) * N);
    double* work = (double*)malloc(sizeof(double) * N);
    for (size_t i = 0; i < N; ++i) {                                   /* :24-32 */
        design[i] = g[i] * l[i];
        design[N + i] = g[i];
        design[2 * N + i] = l[i];
        design[3 * N + i] = 1.0;
    }
    double scale[4];
    for (int c = 0; c < 4; ++c) {                                     /* :36-41 */
        double m = fabs(design[c * N]);
        for (size_t i = 1; i < N; ++i)
            if (fabs(design[c * N + i]) > m) m = fabs(design[c * N + i]);
        scale[c] = (m > 0) ? m : 1.0;
        for (size_t i = 0; i < N; ++i) scaled[c * N + i] = design[c * N + i] / scale[c];
    }
    wtf_cpqr q;                                                       /* :43-45 */
    double* qa = (double*)malloc(sizeof(double) * N * 4);
    memcpy(qa, scaled, sizeof(double) * N * 4);
    q.n = n;
    q.nc = 4;
    q.a = qa;
    wtf_cpqr_compute(&q, scratch);
    int rank = wtf_cpqr_rank(&q, 1e-10);
    double x[4] = {0.0, 0.0, 0.0, 0.0};
    *degenerate = 0;
    if (rank >= 4 && n >= 4) {                                        /* :49-50 */
        wtf_cpqr_solve(&q, t, x, work, scratch);
    } else {                                                          /* :51-59 */
        *degenerate = 1;
        int keep = rank < n ? rank : n;
        if (keep < 1) keep = 1;
        double* sub = (double*)malloc(sizeof(double) * N * (size_t)keep);
        for (int c = 0; c < keep; ++c) memcpy(sub + (size_t)c * N, scaled + (size_t)q.perm[c] * N, sizeof(double) * N);
        double part[4];
        wtf_hhqr_solve(sub, n, keep, t, part, work, scratch);
        for (int c = 0; c < keep; ++c) x[q.perm[c]] = part[c];
        free(sub);
    }
    for (int c = 0; c < 4; ++c) x[c] = x[c] / scale[c];               /* :60 */
    for (int c = 0; c < 4; ++c) coeffs[c] = x[c];
    /* :64-68: fitted = design*coeffs (column-major gemv), residual norms */
    double* fitted = (double*)malloc(sizeof(double) * N);
    for (size_t i = 0; i < N; ++i) {
        double acc = design[i] * x[0];
        acc = acc + design[N + i] * x[1];
        acc = acc + design[2 * N + i] * x[2];
        acc = acc + design[3 * N + i] * x[3];
        fitted[i] = acc;
    }
    for (size_t i = 0; i < N; ++i) {
        double d = t[i] - fitted[i];
        work[i] = d * d;
    }
    double ss_res = wtf_sum(work, 0, n);
    double mean = wtf_sum(t, 0, n) / (double)n;
    for (size_t i = 0; i < N; ++i) {
        double d = t[i] - mean;
        work[i] = d * d;
    }
    double ss_tot = wtf_sum(work, 0, n);
    *r2 = ss_tot > 0 ? 1.0 - ss_res / ss_tot : (ss_res < 1e-18 ? 1.0 : 0.0);
    double mp = 0.0;                                                  /* :71-74 */
    for (size_t i = 0; i < N; ++i) mp += fabs(t[i] - fitted[i]) / fabs(t[i]);
    *mape = mp / (double)n;
    free(design);
    free(scaled);
    free(scratch);
    free(work);
    free(qa);
    free(fitted);
    return WTO_OK;
}

/* ---- select_shared_micro (model.cpp:81-120) ---------------------------- */

typedef struct {
    int32_t micro;
    int64_t g;
    int64_t idx;
    double t;
} sel_rec;

static int cmp_sel(const void* x, const void* y) {
    const sel_rec* a = (const sel_rec*)x;
    const sel_rec* b = (const sel_rec*)y;
    if (a->micro != b->micro) return a->micro < b->micro ? -1 : 1;
    if (a->g != b->g) return a->g < b->g ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}
static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return a < b ? -1 : (a > b);
}

/* Core on a pre-gathered group; records in record order. */
static int select_core(const int64_t* g, const int32_t* micro, const double* t, int32_t n,
                       int32_t* micro_out, int32_t* partial, int64_t* g_out, double* t_out,
                       int32_t* n_out) {
    if (n <= 0) return WTO_INVALID_ARGUMENT;                          /* :82-83 */
    sel_rec* r = (sel_rec*)malloc(sizeof(sel_rec) * (size_t)n);
    int64_t* gs = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        r[i].micro = micro[i];
        r[i].g = g[i];
        r[i].idx = i;
        r[i].t = t[i];
        gs[i] = g[i];
    }
    qsort(gs, (size_t)n, sizeof(int64_t), cmp_i64);
    int32_t n_g = 0;                                                  /* all_g (:85) */
    for (int32_t i = 0; i < n; ++i)
        if (i == 0 || gs[i] != gs[i - 1]) ++n_g;
    qsort(r, (size_t)n, sizeof(sel_rec), cmp_sel);
    /* by_micro[micro][g] = latency, last write (largest idx) wins (:88) */
    for (int pass = 0; pass < 2; ++pass) {                            /* :91-117 */
        int require_full = (pass == 0);
        int32_t best_micro = -1, best_cover = 0, best_lo = 0, best_hi = 0;
        double best_mean = 0.0;
        int32_t i = 0;
        while (i < n) {
            int32_t j = i;
            while (j < n && r[j].micro == r[i].micro) ++j;
            int32_t cover = 0;
            double mean = 0.0;
            for (int32_t k = i; k < j; ++k)
                if (k + 1 == j || r[k + 1].g != r[k].g) {
                    mean += r[k].t;
                    ++cover;
                }
            mean /= cover;
            int skip = require_full && cover != n_g;
            if (!skip) {
                int better = best_micro < 0 || (require_full ? mean < best_mean : cover > best_cover);
                if (better) {
                    best_micro = r[i].micro;
                    best_mean = mean;
                    best_cover = cover;
                    best_lo = i;
                    best_hi = j;
                }
            }
            i = j;
        }
        if (best_micro >= 0) {
            *micro_out = best_micro;
            *partial = !require_full;
            int32_t c = 0;
            for (int32_t k = best_lo; k < best_hi; ++k)
                if (k + 1 == best_hi || r[k + 1].g != r[k].g) {
                    g_out[c] = r[k].g;
                    t_out[c] = r[k].t;
                    ++c;
                }
            *n_out = c;
            break;
        }
    }
    free(r);
    free(gs);
    return WTO_OK;
}

int wto_select_shared_micro(const int64_t* g, const int32_t* micro, const double* t, int32_t n,
                            int32_t* micro_out, int32_t* partial, int64_t* g_out, double* t_out,
                            int32_t* n_out) {
    return select_core(g, micro, t, n, micro_out, partial, g_out, t_out, n_out);
}

/* ---- build_dual_table (model.cpp:194-253) + fit_extrapolation (:140-192) */

typedef struct {
    int32_t mpos, w;
    int64_t l;
    int64_t idx;
} grp_key;

static int cmp_grp(const void* x, const void* y) {
    const grp_key* a = (const grp_key*)x;
    const grp_key* b = (const grp_key*)y;
    if (a->mpos != b->mpos) return a->mpos < b->mpos ? -1 : 1;
    if (a->w != b->w) return a->w < b->w ? -1 : 1;
    if (a->l != b->l) return a->l < b->l ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

typedef struct {
    int32_t w;
    int64_t l;
    int32_t micro, partial, ns;
    int64_t* g;
    double* t;
} sel_group;

static int cmp_id(const void* x, const void* y) {
    const int32_t* a = (const int32_t*)x;
    const int32_t* b = (const int32_t*)y;
    return a[0] < b[0] ? -1 : (a[0] > b[0]);
}

int wto_build(const int64_t* g, const int64_t* l, const int32_t* w, const int32_t* macro,
              const int32_t* micro, const double* lat, int64_t n_records,
              const int32_t* reg_ids, int32_t n_macros, int32_t W, int32_t p,
              wto_build_out* out) {
    if (n_records <= 0) return WTO_INVALID_ARGUMENT;                  /* :198-199 */
    if (W <= 0)                                                       /* :201-203 */
        for (int64_t i = 0; i < n_records; ++i)
            if (w[i] > W) W = w[i];
    out->W = W;
    out->p = p;
    /* registry position of every macro id; records of unknown ids are never
     * visited by group_records (:131-136). */
    int32_t* sorted_ids = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)(n_macros + 1));
    for (int32_t i = 0; i < n_macros; ++i) {
        sorted_ids[2 * i] = reg_ids[i];
        sorted_ids[2 * i + 1] = i;
    }
    qsort(sorted_ids, (size_t)n_macros, 2 * sizeof(int32_t), cmp_id);
    grp_key* keys = (grp_key*)malloc(sizeof(grp_key) * (size_t)n_records);
    int64_t nk = 0;
    for (int64_t i = 0; i < n_records; ++i) {
        int32_t lo = 0, hi = n_macros;
        while (lo < hi) {
            int32_t mid = (lo + hi) / 2;
            if (sorted_ids[2 * mid] < macro[i]) lo = mid + 1; else hi = mid;
        }
        if (lo < n_macros && sorted_ids[2 * lo] == macro[i]) {
            /* a duplicated registry id maps to its first position */
            int32_t pos = sorted_ids[2 * lo + 1];
            for (int32_t q = lo; q < n_macros && sorted_ids[2 * q] == macro[i]; ++q)
                if (sorted_ids[2 * q + 1] < pos) pos = sorted_ids[2 * q + 1];
            keys[nk].mpos = pos;
            keys[nk].w = w[i];
            keys[nk].l = l[i];
            keys[nk].idx = i;
            ++nk;
        }
    }
    qsort(keys, (size_t)nk, sizeof(grp_key), cmp_grp);

    int64_t* gg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nk + 1));
    int32_t* mm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nk + 1));
    double* tt = (double*)malloc(sizeof(double) * (size_t)(nk + 1));
    sel_group* groups = (sel_group*)malloc(sizeof(sel_group) * (size_t)(nk + 1));
    double* bg = (double*)malloc(sizeof(double) * (size_t)(nk + 1));
    double* bl = (double*)malloc(sizeof(double) * (size_t)(nk + 1));
    double* bt = (double*)malloc(sizeof(double) * (size_t)(nk + 1));

    int32_t nt = 0, nc = 0, naw = 0, nan_ = 0, nea = 0;
    out->coeff_off[0] = 0;
    out->awave_off[0] = 0;
    out->awave_aoff[0] = 0;
    out->ext_aoff[0] = 0;
    int64_t a = 0;
    while (a < nk) { /* one macro (registry order) */
        int64_t b = a;
        while (b < nk && keys[b].mpos == keys[a].mpos) ++b;
        /* shared-micro selection per (w, l) group (:222-233) */
        int32_t ng = 0;
        int64_t x = a;
        while (x < b) {
            int64_t y = x;
            while (y < b && keys[y].w == keys[x].w && keys[y].l == keys[x].l) ++y;
            int32_t n = (int32_t)(y - x);
            for (int32_t q = 0; q < n; ++q) {
                int64_t r = keys[x + q].idx;
                gg[q] = g[r];
                mm[q] = micro[r];
                tt[q] = lat[r];
            }
            sel_group* G = &groups[ng++];
            G->w = keys[x].w;
            G->l = keys[x].l;
            G->g = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
            G->t = (double*)malloc(sizeof(double) * (size_t)n);
            select_core(gg, mm, tt, n, &G->micro, &G->partial, G->g, G->t, &G->ns);
            x = y;
        }
        out->macro_id[nt] = reg_ids[keys[a].mpos];
        /* per-wave buckets (:222-242) */
        int32_t gi = 0;
        while (gi < ng) {
            int32_t gj = gi;
            while (gj < ng && groups[gj].w == groups[gi].w) ++gj;
            int32_t ns = 0;
            out->awave_w[naw] = groups[gi].w;
            for (int32_t q = gi; q < gj; ++q) {
                out->anchor_l[nan_] = groups[q].l;
                out->anchor_micro[nan_] = groups[q].micro;
                out->anchor_partial[nan_] = groups[q].partial;
                ++nan_;
                for (int32_t s = 0; s < groups[q].ns; ++s) {
                    bg[ns] = (double)groups[q].g[s];
                    bl[ns] = (double)groups[q].l;
                    bt[ns] = groups[q].t[s];
                    ++ns;
                }
            }
            out->awave_aoff[naw + 1] = nan_;
            ++naw;
            int32_t degen;
            wto_fit_bucket(bg, bl, bt, ns, out->coeff_theta + 4 * (size_t)nc, &out->diag_r2[nc],
                           &out->diag_mape[nc], &degen);
            out->coeff_w[nc] = groups[gi].w;
            out->diag_samples[nc] = ns;
            out->diag_flags[nc] = (degen ? 1 : 0) | (ns < 4 ? 2 : 0);
            ++nc;
            gi = gj;
        }
        /* fit_extrapolation (:140-192) */
        int32_t w_lo = W - p + 1 > 1 ? W - p + 1 : 1;
        int32_t waves_used = 0, ns = 0;
        int32_t prev_w = INT_MIN;
        for (int32_t q = 0; q < ng; ++q) {
            if (groups[q].w < w_lo || groups[q].w > W) continue;
            if (groups[q].w != prev_w) {
                ++waves_used;
                prev_w = groups[q].w;
            }
            for (int32_t s = 0; s < groups[q].ns; ++s) {
                bg[ns] = (double)groups[q].g[s];
                bl[ns] = (double)groups[q].l;
                bt[ns] = groups[q].t[s];
                ++ns;
            }
        }
        int32_t flags = 0;
        if (waves_used >= 2) {
            double r2, mape;
            int32_t degen;
            wto_fit_bucket(bg, bl, bt, ns, out->theta_ext + 4 * (size_t)nt, &r2, &mape, &degen);
            if (degen) flags |= 1;
            /* majority vote per l, ties -> smaller micro (:171-181) */
            int64_t* ls = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ng + 1));
            int32_t nls = 0;
            for (int32_t q = 0; q < ng; ++q)
                if (groups[q].w >= w_lo && groups[q].w <= W) ls[nls++] = groups[q].l;
            qsort(ls, (size_t)nls, sizeof(int64_t), cmp_i64);
            for (int32_t u = 0; u < nls; ++u) {
                if (u > 0 && ls[u] == ls[u - 1]) continue;
                int32_t best_micro = -1, best_count = -1;
                /* O(ng^2) tally, candidate micros visited in ascending order */
                int32_t cur = INT_MIN;
                for (;;) {
                    int32_t next = INT_MAX;
                    for (int32_t q = 0; q < ng; ++q)
                        if (groups[q].w >= w_lo && groups[q].w <= W && groups[q].l == ls[u] &&
                            groups[q].micro > cur && groups[q].micro < next)
                            next = groups[q].micro;
                    if (next == INT_MAX) break;
                    int32_t count = 0;
                    for (int32_t q = 0; q < ng; ++q)
                        if (groups[q].w >= w_lo && groups[q].w <= W && groups[q].l == ls[u] &&
                            groups[q].micro == next)
                            ++count;
                    if (count > best_count) {
                        best_count = count;
                        best_micro = next;
                    }
                    cur = next;
                }
                out->ext_l[nea] = ls[u];
                out->ext_micro[nea] = best_micro;
                ++nea;
            }
            free(ls);
        } else {
            /* copy the highest wave present (:182-191) */
            int32_t top = groups[ng - 1].w;
            ns = 0;
            for (int32_t q = 0; q < ng; ++q) {
                if (groups[q].w != top) continue;
                out->ext_l[nea] = groups[q].l;
                out->ext_micro[nea] = groups[q].micro;
                ++nea;
                for (int32_t s = 0; s < groups[q].ns; ++s) {
                    bg[ns] = (double)groups[q].g[s];
                    bl[ns] = (double)groups[q].l;
                    bt[ns] = groups[q].t[s];
                    ++ns;
                }
            }
            double r2, mape;
            int32_t degen;
            wto_fit_bucket(bg, bl, bt, ns, out->theta_ext + 4 * (size_t)nt, &r2, &mape, &degen);
            flags |= 2;
        }
        out->ext_flags[nt] = flags;
        for (int32_t q = 0; q < ng; ++q) {
            free(groups[q].g);
            free(groups[q].t);
        }
        ++nt;
        out->coeff_off[nt] = nc;
        out->awave_off[nt] = naw;
        out->ext_aoff[nt] = nea;
        a = b;
    }
    out->n_tables = nt;
    free(sorted_ids);
    free(keys);
    free(gg);
    free(mm);
    free(tt);
    free(groups);
    free(bg);
    free(bl);
    free(bt);
    return nt == 0 ? WTO_RUNTIME_ERROR : WTO_OK;                      /* :250-251 */
}
