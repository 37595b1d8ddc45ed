/*
 * wt_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's decision path (the checker the
 * CUDA path is compared against).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load the built library
 * (oracle/_build/libwtoracle.so); the product never links it.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * reference compiled verbatim (oracle/_ref/libwtref.so, see Makefile) and
 * against the golden vectors transcribed from the proj/tests sources.
 *
 * Tables are passed in a flat "table set" form that mirrors
 * DualTable (proj/include/wavetune/model.hpp:64-77) map-for-map: every
 * std::map becomes a key-sorted CSR slice.  Resolution of the reference's
 * fallbacks (missing wave, empty anchor map) is done HERE at query time,
 * exactly as tuner.cpp does, not from a pre-resolved image.
 */
#ifndef WT_ORACLE_H
#define WT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { WTO_OK = 0, WTO_INVALID_ARGUMENT = 1, WTO_RUNTIME_ERROR = 2, WTO_OUT_OF_RANGE = 3 };

typedef struct {
    int32_t n_tables;
    const int32_t* macro_id;   /* [n_tables] */
    const int32_t* W;          /* [n_tables] */
    const int64_t* t_m;        /* [n_tables] tiles joined from the registry */
    const int64_t* t_n;
    const int64_t* t_k;
    const double* theta_ext;   /* [n_tables*4] alpha,beta,gamma,delta */
    const int32_t* coeff_off;  /* [n_tables+1] CSR into coeff_w / coeff_theta */
    const int32_t* coeff_w;    /* wave keys, ascending per table */
    const double* coeff_theta; /* [n_coeff*4] */
    const int32_t* awave_off;  /* [n_tables+1] CSR into awave_w / awave_aoff */
    const int32_t* awave_w;    /* anchor_table wave keys, ascending (maps may be empty) */
    const int32_t* awave_aoff; /* [n_awave+1] CSR into anchor_l / anchor_micro */
    const int64_t* anchor_l;   /* ascending per map */
    const int32_t* anchor_micro;
    const int32_t* ext_aoff;   /* [n_tables+1] CSR into ext_l / ext_micro */
    const int64_t* ext_l;
    const int32_t* ext_micro;
} wto_tables;

/* kernel_map.hpp:17 ceil_div; kernel_map.cpp:235-243 dense branch. */
int wto_map_dense(int64_t m, int64_t n, int64_t k, int64_t t_m, int64_t t_n, int64_t t_k,
                  int64_t* g, int64_t* l);
/* kernel_map.cpp:266-271; returns status, *w out. */
int wto_wave_count(int64_t g, int32_t n_sm, int32_t bps, int32_t* w);
/* tuner.cpp:11-42.  *used_w = fallback wave or -1. */
int wto_predict(const wto_tables* T, int32_t t, int64_t g, int64_t l, int32_t n_sm, int32_t bps,
                double* lat, int32_t* extrap, int32_t* w, int32_t* used_w);
/* tuner.cpp:44-70. */
int wto_nearest_anchor(const int64_t* anchors, int32_t n, int64_t l, int64_t* out, int32_t* comps);

/* tune() (tuner.cpp:115-166) over n dense_gemm queries.  Outputs per query:
 * macro, micro, lat, g, l, w, extrap, comps, n_missing (count of
 * missing_wave flags), anchor_fb (fallback wave or -1), status. */
void wto_tune(const wto_tables* T, int32_t n_sm, int32_t bps, const int64_t* M, const int64_t* N,
              const int64_t* K, int64_t n, int32_t* macro, int32_t* micro, double* lat, int64_t* g,
              int64_t* l, int32_t* w, int32_t* extrap, int32_t* comps, int32_t* n_missing,
              int32_t* anchor_fb, int32_t* status);

/* Extension (no reference symbol): first k of the (latency, macro_id)
 * ascending order over non-NaN, non-+inf candidates; top-1 == tune()'s
 * Stage-I winner.  Unfilled slots get macro -1, lat NaN. */
int wto_topk(const wto_tables* T, int32_t n_sm, int32_t bps, int64_t M, int64_t N, int64_t K,
             int32_t k, int32_t* macro, double* lat);

/* model.cpp:20-77 with Eigen restated in wt_fit_core.h. */
int wto_fit_bucket(const double* g, const double* l, const double* t, int32_t n, double* coeffs,
                   double* r2, double* mape, int32_t* degenerate);

/* model.cpp:81-120 on one group (records of one (macro,w,l)). */
int wto_select_shared_micro(const int64_t* g, const int32_t* micro, const double* t, int32_t n,
                            int32_t* micro_out, int32_t* partial, int64_t* g_out, double* t_out,
                            int32_t* n_out);

/* build_dual_table (model.cpp:194-253) output, caller-allocated with
 * capacities >= n_records (+1 for offsets). */
typedef struct {
    int32_t n_tables, W, p;
    int32_t* macro_id;
    double* theta_ext;
    int32_t* ext_flags;   /* bit0 ext_degenerate_fit, bit1 ext_insufficient_waves */
    int32_t* coeff_off;   /* [n_tables+1] */
    int32_t* coeff_w;
    double* coeff_theta;
    double* diag_r2;      /* per coeff entry (= per diagnostics wave) */
    double* diag_mape;
    int32_t* diag_samples;
    int32_t* diag_flags;  /* bit0 degenerate_fit, bit1 sparse_bucket */
    int32_t* awave_off;   /* [n_tables+1] */
    int32_t* awave_w;
    int32_t* awave_aoff;  /* [n_awave+1] */
    int64_t* anchor_l;
    int32_t* anchor_micro;
    int32_t* anchor_partial; /* partial_micro_coverage_l<l> */
    int32_t* ext_aoff;    /* [n_tables+1] */
    int64_t* ext_l;
    int32_t* ext_micro;
} wto_build_out;

int wto_build(const int64_t* g, const int64_t* l, const int32_t* w, const int32_t* macro,
              const int32_t* micro, const double* lat, int64_t n_records,
              const int32_t* registry_macro_ids, int32_t n_macros, int32_t W, int32_t p,
              wto_build_out* out);

#ifdef __cplusplus
}
#endif
#endif /* WT_ORACLE_H */
