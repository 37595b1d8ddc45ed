/*
 * wavetune_c.h -- C-ABI of the B200-native WaveTune decision path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch
 * types.  The C++ drop-in API (include/wavetune/*.hpp, namespace wavetune)
 * and the Python module are thin layers over these entry points; a
 * cgo/JNI/ctypes binding would bind exactly this header.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   wt_engine_create   -- the (tables, registry, hw) triple every query of
 *                         tune() takes (include/wavetune/tuner.hpp:51-52);
 *                         validated and resolved once, held on the device.
 *   wt_tune_batch      -- wavetune::tune() (tuner.hpp:51-52, tuner.cpp:159-166)
 *   wt_tune_one        -- the same for one query at minimum latency
 *                         for n queries at once (Stage I argmin + Stage II).
 *   wt_predict_batch   -- wavetune::predict_latency() (tuner.hpp:38-40,
 *                         tuner.cpp:11-42).
 *   wt_explain         -- the per-table loop inside two_stage_select
 *                         (tuner.cpp:135-149) for one query, so the host can
 *                         rebuild Tuned.flags text exactly.
 *   wt_nearest_anchor_batch -- wavetune::nearest_anchor() (tuner.hpp:44-45).
 *   wt_grid_* / wt_sweep / wt_gather_batch -- extension (no reference
 *                         symbol): tune() materialised over a shape grid
 *                         ("dual lookup tables ... answer online queries")
 *                         and a table-gather for online queries.
 *   wt_fit_build       -- wavetune::build_dual_table() (model.hpp:95-98,
 *                         model.cpp:194-253) incl. select_shared_micro,
 *                         fit_bucket and fit_extrapolation.
 *   wt_fit_bucket_batch -- wavetune::fit_bucket() (model.hpp:42).
 *
 * Conventions.
 *   - Every entry point returns wt_status; on failure wt_last_error() holds
 *     the reference's message text for the same condition (thread-local).
 *   - "device" pointers are CUDA device (or managed) memory; "host" pointers
 *     are host memory.  Batched calls are stream-ordered on the given
 *     cudaStream_t (passed as void*, NULL = legacy default stream) and never
 *     synchronise the device unless the name ends in _sync.
 *   - Handles are immutable after creation; any number of host threads may
 *     issue batched calls on different streams concurrently.
 *   - Per-query failures (the reference would throw for that query) do not
 *     fail the batch: they are reported in the query's status byte
 *     (bits 24..31 of flags, a wt_status value) and its macro_id is -1.
 */
#ifndef WAVETUNE_C_H
#define WAVETUNE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WT_ABI_VERSION 1

typedef enum {
    WT_OK = 0,
    WT_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    WT_RUNTIME_ERROR = 2,    /* std::runtime_error */
    WT_OUT_OF_RANGE = 3,     /* std::out_of_range */
    WT_CUDA_ERROR = 4,
    WT_UNSUPPORTED = 5       /* outside the device path's documented domain */
} wt_status;

/* Kernel families (kernel_map.hpp:19). */
enum { WT_FAMILY_DENSE_GEMM = 0, WT_FAMILY_GROUPED_GEMM = 1, WT_FAMILY_FLASH_ATTENTION = 2 };

/* Decision flag bits (wt_decisions.flags). */
enum {
    WT_FLAG_EXTRAPOLATED = 1u << 0,   /* Regime.extrapolated of the winner */
    WT_FLAG_MISSING_WAVE = 1u << 1,   /* some table used a missing_wave_<w>_used_<k> fallback */
    WT_FLAG_ANCHOR_FALLBACK = 1u << 2 /* winner used anchor_fallback_wave_<k> */
};
#define WT_FLAG_STATUS(f) ((int)(((uint32_t)(f)) >> 24))

const char* wt_last_error(void);
const char* wt_version(void);
int wt_abi_version(void);

/* ---- inputs ----------------------------------------------------------- */

/* HardwareSpec (kernel_map.hpp:67-73); slots = n_sm * blocks_per_sm. */
typedef struct {
    int32_t n_sm;
    int32_t blocks_per_sm;
} wt_hw;

/* ConfigRegistry macros (kernel_map.hpp:47-60,81-94), host arrays.  For
 * FlashAttention registries t_m = t_q, t_k = t_kv and t_n is ignored. */
typedef struct {
    int32_t family;
    int32_t n_macros;
    const int32_t* id;
    const int64_t* t_m;
    const int64_t* t_n;
    const int64_t* t_k;
} wt_registry_desc;

/* std::vector<DualTable> (model.hpp:64-77), host arrays.  Every std::map is
 * a key-ascending CSR slice; tables may be in any order (tune() sorts them
 * by macro_id, tuner.cpp:127-132). */
typedef struct {
    int32_t n_tables;
    const int32_t* macro_id;   /* [n_tables] */
    const int32_t* W;          /* [n_tables] */
    const double* theta_ext;   /* [n_tables*4] alpha, beta, gamma, delta */
    const int32_t* coeff_off;  /* [n_tables+1] -> coeff_w / coeff_theta */
    const int32_t* coeff_w;    /* coeff_table keys (wave), ascending per table */
    const double* coeff_theta; /* [4 per key] */
    const int32_t* awave_off;  /* [n_tables+1] -> awave_w / awave_aoff */
    const int32_t* awave_w;    /* anchor_table keys (wave), ascending per table */
    const int32_t* awave_aoff; /* [n_awave+1] -> anchor_l / anchor_micro */
    const int64_t* anchor_l;   /* loop anchors, ascending per map */
    const int32_t* anchor_micro;
    const int32_t* ext_aoff;   /* [n_tables+1] -> ext_l / ext_micro */
    const int64_t* ext_l;
    const int32_t* ext_micro;
} wt_tables_desc;

/* ---- engine: validated, fallback-resolved device image ------------------ */

typedef struct wt_engine wt_engine;

typedef struct {
    int32_t n_configs;   /* Stage-I candidates C (= tables) */
    int32_t n_rows;      /* coefficient rows per config (max W + 1) */
    int32_t slots;       /* n_sm * blocks_per_sm */
    int32_t family;
    int32_t has_fallback_rows; /* any resolved missing-wave / empty-table row */
    int32_t device;
    size_t device_bytes; /* bytes of the resident image */
} wt_engine_info;

/* Validates like the reference (duplicate ids -> INVALID_ARGUMENT, table id
 * absent from the registry -> OUT_OF_RANGE "no macro config with id N",
 * no tables -> INVALID_ARGUMENT "no dual tables provided") and uploads (the
 * host arrays may be released on return).  The device image is built
 * asynchronously; the first call that uses the engine waits for it. */
wt_status wt_engine_create(const wt_tables_desc* tables, const wt_registry_desc* registry,
                           const wt_hw* hw, int device, wt_engine** out);
wt_status wt_engine_destroy(wt_engine* e);
/* Counts and flags of the engine.  has_fallback_rows is resolved from the
 * device image, so this call is a first use: it waits for the image build
 * (call it after queueing the work that should overlap the build). */
wt_status wt_engine_info_get(const wt_engine* e, wt_engine_info* out);
/* Host-only (no device needed): the exact pruning plan an engine built from
 * (tables, registry, hw) would use -- for tests and inspection.  Segments
 * are runs of <= 32 configs of one tile class; cls_cfg[pos] = config index
 * (ascending macro_id order) at class position pos, segment s covers
 * positions [seg_pos[s], seg_pos[s] + seg_n[s]); bit i of
 * masks[(s * R + row) * 16 + lb] set = config seg_pos[s] + i may win in wave
 * row `row`, L bucket lb (L in [2^lb, 2^(lb+1)), last bucket unbounded).
 * Call with masks == NULL to get *n_seg, *R and *C; buffers are caller-owned
 * (cls_cfg [C], seg_pos / seg_n [n_seg], masks [n_seg * R * 16]). */
wt_status wt_prune_plan(const wt_tables_desc* tables, const wt_registry_desc* registry, const wt_hw* hw,
                        int32_t* n_seg, int32_t* R, int32_t* C, int32_t* cls_cfg, int32_t* seg_pos,
                        int32_t* seg_n, uint32_t* masks);

/* Inspection: copies the engine's pruning masks (built on the device) to
 * host memory, laid out as wt_prune_plan's masks; n = n_seg * R * 16 words.
 * Synchronous. */
wt_status wt_engine_prune_masks(const wt_engine* e, uint32_t* masks, int64_t n);

/* Instrumentation: while `counter` (a device uint64, caller-owned) is set,
 * the grid sweep (k_sweep2) and the list evaluation (k_eval4) add the number
 * of (shape | query, config) evaluations they physically execute -- per warp
 * and segment, surviving configs x 32 lanes x shapes per lane, idle lanes
 * included.  NULL turns it off.  Costs one atomic per warp and segment. */
wt_status wt_engine_count_evals(wt_engine* e, unsigned long long* counter);

/* Extension (A/B and second-witness runs): enable = 0 makes every kernel
 * evaluate all configs (the pruning masks are ignored); 1 (default, unless
 * the WT_PRUNE=0 environment variable was set) uses them.  Not thread-safe
 * against calls in flight on the same engine. */
wt_status wt_engine_set_prune(wt_engine* e, int32_t enable);

/* Position of macro_id in the engine's ascending config order, or -1. */
int32_t wt_engine_config_index(const wt_engine* e, int32_t macro_id);

/* ---- outputs ---------------------------------------------------------- */

/* Per-query decision arrays (device).  Required: macro_id, micro_id,
 * latency_us.  Optional (NULL to skip): g, l, wave, flags, comparisons,
 * tail_frac, and the top-k block (k >= 1, [n*k] each, extension). */
typedef struct {
    int32_t* macro_id;
    int32_t* micro_id;
    double* latency_us;
    int64_t* g;
    int64_t* l;
    int32_t* wave;        /* Regime.w */
    uint32_t* flags;      /* WT_FLAG_* | status << 24 */
    int32_t* comparisons; /* DecisionStats.anchor_comparisons */
    double* tail_frac;    /* (g - (w-1)*slots) / slots of the winner (extension) */
    int32_t topk;         /* 0 = off */
    int32_t* topk_macro;
    double* topk_latency;
} wt_decisions;

/* ---- one query, lowest latency ----------------------------------------- */

/* tune() for a single query, synchronously (tuner.cpp:159-166 with n = 1):
 * the query travels as kernel arguments, one warp evaluates every config,
 * and the decision is written straight into engine-owned pinned host memory
 * that the caller polls -- no copies and no stream synchronisation on the
 * happy path.  Calls on one engine are serialised.  The per-query status
 * (INVALID_ARGUMENT / RUNTIME_ERROR / UNSUPPORTED) is returned in
 * flags >> 24 exactly as in wt_tune_batch; the return value reports only
 * API and CUDA errors. */
typedef struct wt_decision_one {
    double latency_us;
    int64_t g, l;
    double tail_frac;
    int32_t macro_id, micro_id, wave;
    uint32_t flags;
    int32_t comparisons;
} wt_decision_one;

wt_status wt_tune_one(const wt_engine* e, int32_t M, int32_t N, int32_t K, wt_decision_one* out);

/* Resident mode for wt_tune_one.  idle_us > 0: the first call starts one
 * resident CTA that polls the engine's pinned mailbox and answers each query
 * without a kernel launch; it leaves by itself after idle_us microseconds
 * without a query and the next call restarts it.  While it is resident a
 * device-wide synchronisation waits for it to leave (at most idle_us).
 * idle_us = 0 stops it and returns to one launch per query (the default). */
wt_status wt_engine_set_resident(wt_engine* e, int32_t idle_us);

/* ---- ablation baselines (tuner.hpp:54-85, tuner.cpp:168-250) ----------- */

#define WT_BASELINE_STEP 0   /* T = t_wave[(macro, nearest anchor)] * wave_count(g) */
#define WT_BASELINE_LINEAR 1 /* T = one bilinear fit per macro, no wave regimes */

typedef struct wt_baseline wt_baseline;

/* A baseline predictor on the device.  Step: n entries (macro_id[i],
 * anchor_l[i], values[i] = t_wave) sorted by (macro_id, anchor_l) -- the
 * StepPredictor map order.  Linear: n entries macro_id[i] (ascending),
 * values[4i..4i+3] = (alpha, beta, gamma, delta); anchor_l unused.
 * e != NULL binds the baseline to that engine's configs (needed for
 * wt_baseline_tune_batch); an engine table without an entry makes every
 * valid query fail with OUT_OF_RANGE, as baseline_predict throws. */
wt_status wt_baseline_create(const wt_engine* e, int device, int32_t kind, const int32_t* macro_id,
                             const int64_t* anchor_l, const double* values, int64_t n, wt_baseline** out);
wt_status wt_baseline_destroy(wt_baseline* b);

/* baseline_tune() for dense/attention queries (device arrays): Stage I with
 * the baseline predictor, Stage II on the engine's dual tables.  Same output
 * contract as wt_tune_batch (no top-k). */
wt_status wt_baseline_tune_batch(const wt_engine* e, const wt_baseline* b, const int32_t* M, const int32_t* N,
                                 const int32_t* K, int64_t n, const wt_decisions* out, void* stream);

/* baseline_predict(bp, macro_id, g, l, hw) for n device-array triples;
 * status[i] = OK / OUT_OF_RANGE (no entry) / INVALID_ARGUMENT (step, g < 1). */
wt_status wt_baseline_predict_batch(const wt_baseline* b, const int32_t* macro_id, const int64_t* g,
                                    const int64_t* l, int64_t n, const wt_hw* hw, double* latency, int32_t* status,
                                    void* stream);

/* ---- batched tune (evaluate mode: every query runs full Stage I) -------- */

/* Dense GEMM (M,N,K) / FlashAttention (s_q,n_heads,s_kv) queries, int32
 * device arrays; dims must be >= 1 (else per-query INVALID_ARGUMENT). */
wt_status wt_tune_batch(const wt_engine* e, const int32_t* M, const int32_t* N, const int32_t* K,
                        int64_t n, const wt_decisions* out, void* stream);

/* Grouped GEMM queries: query i has group rows rows[row_off[i] .. row_off[i+1])
 * (device arrays) and dims (N[i], K[i]) (kernel_map.cpp:244-257). */
wt_status wt_tune_grouped_batch(const wt_engine* e, const int64_t* row_off, const int32_t* rows,
                                const int32_t* N, const int32_t* K, int64_t n,
                                const wt_decisions* out, void* stream);

/* predict_latency for n (config index, g, l) triples (device arrays).
 * used_w = fallback wave when missing_wave_<w>_used_<k> fired, else -1. */
wt_status wt_predict_batch(const wt_engine* e, const int32_t* config, const int64_t* g,
                           const int64_t* l, int64_t n, double* latency_us, int32_t* wave,
                           int32_t* extrapolated, int32_t* used_w, int32_t* status, void* stream);

/* For one dense query, every config in ascending macro_id order (device
 * arrays of length n_configs): g, l, wave, used_w, latency. */
wt_status wt_explain(const wt_engine* e, int64_t M, int64_t N, int64_t K, int64_t* g, int64_t* l,
                     int32_t* wave, int32_t* used_w, double* latency_us, int32_t* status,
                     void* stream);

/* Anchor map of (config, row) as resolved at upload: writes up to cap
 * anchors/micros (host) and returns the count, or -1. */
int32_t wt_engine_anchor_map(const wt_engine* e, int32_t config, int32_t wave, int32_t extrapolated,
                             int64_t* anchors, int32_t* micros, int32_t cap, int32_t* fallback_wave);

/* nearest_anchor over a sorted device list, n queries. */
wt_status wt_nearest_anchor_batch(const int64_t* anchors, int32_t n_anchors, const int64_t* l,
                                  int64_t n, int64_t* out, int32_t* comparisons, void* stream);

/* ---- decision grid (extension): tune() materialised over shapes --------- */

typedef struct wt_grid wt_grid;

/* Grid over n_pairs (N, K) pairs (host arrays) x M in [m_lo, m_hi].
 * Entry index = pair * (m_hi - m_lo + 1) + (M - m_lo). */
typedef struct {
    int32_t n_pairs;
    const int32_t* N;
    const int32_t* K;
    int32_t m_lo, m_hi;
    int32_t topk; /* 0 = argmin only */
} wt_grid_desc;

/* 32-byte grid entry (device layout). */
typedef struct {
    double latency_us;
    int32_t macro_id;
    int32_t micro_id;
    int32_t wave;
    uint32_t flags;
    int32_t comparisons;
    float tail_frac;
} wt_grid_entry;

wt_status wt_grid_create(const wt_engine* e, const wt_grid_desc* desc, wt_grid** out);
/* The same, stream-ordered on `stream`: storage from the library's memory
 * pool and every upload queued on the stream (no host synchronisation), so a
 * build chain fit -> engine -> grid -> sweep stays on one stream.  Use the
 * grid on other streams only after ordering them behind `stream`.  Its
 * storage is not IPC-exportable (wt_grid_ipc_handle: WT_UNSUPPORTED). */
wt_status wt_grid_create_async(const wt_engine* e, const wt_grid_desc* desc, void* stream, wt_grid** out);
wt_status wt_grid_destroy(wt_grid* g);
/* Raw device storage (for collectives / inspection).  Taking it invalidates
 * the grid's run index (gathers then read the entries from L2) until the next
 * full wt_sweep or wt_grid_finalize -- call finalize after writing entries
 * (e.g. an all-gather of sweep shards).  The invalidation is a host-side
 * generation bump (no device work): gathers launched after this call never
 * use an index built for earlier entries, whatever stream built it. */
wt_status wt_grid_storage(const wt_grid* g, wt_grid_entry** entries, int64_t* n_entries,
                          int32_t** topk_macro, double** topk_latency);
/* Shapes a full sweep of the grid actually evaluates: a grid entry depends
 * on M only through ceil(M / t_m) for the engine's tile heights, so the sweep
 * takes one representative M per interval of constant quotients and copies
 * its entry over the interval (n_pairs * intervals; equals n_entries when the
 * intervals do not cut the work at least 4x and every M is evaluated). */
int64_t wt_grid_representatives(const wt_grid* g);
/* Fills entries [begin, end) (flattened index) -- one shard of the sweep.
 * A full-range sweep also rebuilds the grid's run index (below); a partial
 * one invalidates it until wt_grid_finalize. */
wt_status wt_sweep(const wt_engine* e, wt_grid* g, int64_t begin, int64_t end, void* stream);
/* Fused multi-GPU sweep: fills entries [begin, end) and stores each entry
 * into every grid storage in dests[0..n_dests) (n_dests <= 8; this rank's
 * own wt_grid_storage and its peers' storages opened with wt_ipc_open:
 * stores travel over NVLink from the sweep's epilogue, no all-gather).  All
 * destinations must have this grid's shape.  Afterwards (all ranks done:
 * device sync + barrier) each rank calls wt_grid_finalize on its grid.
 * Grids with top-k are not supported. */
wt_status wt_sweep_to(const wt_engine* e, wt_grid* g, int64_t begin, int64_t end, wt_grid_entry* const* dests,
                      int n_dests, void* stream);
/* CUDA IPC handle (64 bytes) of the grid's storage and the entries' byte
 * offset in it, for peers to open with wt_ipc_open. */
wt_status wt_grid_ipc_handle(const wt_grid* g, void* handle, int64_t* offset);
wt_status wt_ipc_open(const void* handle, int64_t offset, int device, wt_grid_entry** entries, void** base);
wt_status wt_ipc_close(void* base);
/* Rebuilds the run-compressed copy of the entries' heads (latency, macro,
 * micro are piecewise constant along M) that wt_gather_batch serves from
 * shared memory when it fits.  Stream-ordered, no host sync. */
wt_status wt_grid_finalize(const wt_engine* e, wt_grid* g, void* stream);
/* Online queries: on-grid shapes are gathered; off-grid ones are compacted
 * and evaluated in full (wt_tune_batch semantics).  Needs no host sync. */
wt_status wt_gather_batch(const wt_engine* e, const wt_grid* g, const int32_t* M, const int32_t* N,
                          const int32_t* K, int64_t n, const wt_decisions* out, void* stream);

/* 64-bit dimensions (the reference's DenseGemm{i64 m, n, k},
 * kernel_map.hpp:25-27; attention (s_q, n_heads, s_kv) the same way): i64
 * device arrays, otherwise the contract of wt_tune_batch / wt_gather_batch.
 * Queries whose dims all fit int32 take the int32 kernels; the others are
 * evaluated in 64-bit integer arithmetic by a warp-per-query kernel.  A tile
 * product above 2^63 or >= 2^31 waves for the smallest tile ->
 * WT_UNSUPPORTED in that query's flags.  No top-k (topk must be 0). */
wt_status wt_tune_batch_i64(const wt_engine* e, const int64_t* M, const int64_t* N, const int64_t* K, int64_t n,
                            const wt_decisions* out, void* stream);
wt_status wt_gather_batch_i64(const wt_engine* e, const wt_grid* g, const int64_t* M, const int64_t* N,
                              const int64_t* K, int64_t n, const wt_decisions* out, void* stream);

/* End-to-end convenience over HOST buffers (the call an application makes):
 * queries M/N/K and the outputs macro/micro/latency live in host memory
 * (pinned for full overlap).  The batch is cut into chunks of `chunk`
 * queries and pipelined over two internal streams: H2D copy, gather (grid
 * != NULL) or full evaluation (grid == NULL), D2H copy.  Synchronous. */
wt_status wt_decide_host_sync(const wt_engine* e, const wt_grid* g, const int32_t* M,
                              const int32_t* N, const int32_t* K, int64_t n, int32_t* macro_id,
                              int32_t* micro_id, double* latency_us, int64_t chunk);
/* The same, ordered after all work already queued on `stream` (NULL = the
 * legacy default stream, which is what wt_decide_host_sync uses): a grid
 * still being swept / finalized on that stream is complete before the first
 * gather reads it.  Work on other non-blocking streams is not waited for. */
wt_status wt_decide_host_stream_sync(const wt_engine* e, const wt_grid* g, const int32_t* M, const int32_t* N,
                                     const int32_t* K, int64_t n, int32_t* macro_id, int32_t* micro_id,
                                     double* latency_us, int64_t chunk, void* stream);

/* Kernel launch counter (for bench accounting): total launches issued by
 * this library in this process. */
int64_t wt_launch_count(void);

/* Per-kernel timing for benchmarks.  While enabled, wt_gather_batch records
 * CUDA events on its stream around (0) the gather kernel and (1) the
 * off-grid evaluation that follows it; wt_kernel_time_ms returns the
 * elapsed time of the most recent call (waits for its events). */
wt_status wt_set_kernel_timing(int enable);
wt_status wt_kernel_time_ms(int which, float* ms);

/* ---- batched fit / dual-table build (K2) --------------------------------- */

/* ProfileRecord SoA (profiler.hpp:56-63), host arrays. */
typedef struct {
    int64_t n;
    const int64_t* g;
    const int64_t* l;
    const int32_t* w;
    const int32_t* macro_id;
    const int32_t* micro_id;
    const double* latency_us;
} wt_records_desc;

/* Built tables, library-owned host arrays (valid until wt_build_free). */
typedef struct {
    int32_t n_tables, W, p;
    const int32_t* macro_id;
    const double* theta_ext;
    const int32_t* ext_flags;    /* bit0 ext_degenerate_fit, bit1 ext_insufficient_waves */
    const int32_t* coeff_off;
    const int32_t* coeff_w;
    const double* coeff_theta;
    const double* diag_r2;
    const double* diag_mape;
    const int32_t* diag_samples;
    const int32_t* diag_flags;   /* bit0 degenerate_fit, bit1 sparse_bucket */
    const int32_t* awave_off;
    const int32_t* awave_w;
    const int32_t* awave_aoff;
    const int64_t* anchor_l;
    const int32_t* anchor_micro;
    const int32_t* anchor_partial; /* partial_micro_coverage_l<l> */
    const int32_t* ext_aoff;
    const int64_t* ext_l;
    const int32_t* ext_micro;
    double device_ms;            /* GPU time of the build (CUDA events) */
    /* Ablation baselines fitted from the same shared-micro-selected samples
     * (tuner.cpp:191-220), per table in the order above.  Step: t_wave of
     * anchors [step_off[i], step_off[i+1]) (ascending l).  Linear: one
     * bilinear fit of all the table's samples, theta [4 per table]. */
    const int32_t* step_off;
    const int64_t* step_l;
    const double* step_t;
    const double* lin_theta;
    const double* lin_r2;
    const double* lin_mape;
    const int32_t* lin_degenerate;
} wt_build_result;

typedef struct wt_build wt_build;

/* build_dual_table(records, registry, hw, {W, p}) on the GPU.  registry_ids
 * is the registry's macro order (tables come out in that order). */
wt_status wt_fit_build(const wt_records_desc* records, const int32_t* registry_ids,
                       int32_t n_macros, int32_t W, int32_t p, int device, wt_build** out,
                       wt_build_result* result);
wt_status wt_build_free(wt_build* b);

/* build_dual_table over records ALREADY IN DEVICE MEMORY (wt_records_desc
 * with device pointers), stream-ordered on `stream`; the built tables stay on
 * the device (no host CSR).  Three scalar read-backs size the allocations
 * (host syncs of the stream); the fit itself, the extrapolation and the CSR
 * assembly are queued without further syncs.  flags: WT_FIT_BASELINES also
 * fits the ablation baselines (not part of build_dual_table).  The tables
 * feed wt_engine_create_from_build directly; wt_build_result_get copies them
 * to the host on demand. */
#define WT_FIT_BASELINES 1
wt_status wt_fit_build_device(const wt_records_desc* records, const int32_t* registry_ids, int32_t n_macros,
                              int32_t W, int32_t p, int32_t flags, int device, void* stream, wt_build** out);
/* Host copies of a build's tables (synchronous; valid until wt_build_free). */
wt_status wt_build_result_get(wt_build* b, wt_build_result* result);
/* Engine from a build's device-resident tables (registry = the one the build
 * was fitted against): the image -- rows, tile classes, pruning masks -- is
 * resolved on the device, the tables never cross PCIe.  Work is queued on
 * `stream` (ordered after the build) and not waited for: the first call that
 * uses the engine waits for the image (so the host can meanwhile, e.g.,
 * create a grid).  wt_build_free waits for all device work. */
wt_status wt_engine_create_from_build(const wt_build* b, const wt_registry_desc* registry, const wt_hw* hw,
                                      void* stream, wt_engine** out);

/* ---- exchanging builds between ranks (multi-GPU build, dist.py) ----------
 * A build fitted on one GPU for a contiguous slice of the registry (its shard
 * of build_dual_table) is packed into one contiguous device blob; the blobs
 * of all ranks travel in one collective (NCCL all-gather of equal-stride
 * blobs) and every rank merges them, in registry order, into one build on
 * its own device -- the same tables the single-GPU build of the whole
 * registry produces (merge_tables on the device: CSR offsets rebased).
 *
 * wt_build_pack_info: counts[5] = {n_tables, n_buckets, n_groups, W, p} and
 *   the packed size in bytes.
 * wt_build_pack: packs into device memory dst (cap >= bytes), queued on
 *   `stream` after the build's own work.
 * wt_build_merge: parts are packed[r * stride], r < n_parts, with counts
 *   [n_parts * 5] as wt_build_pack_info reported them (parts with zero
 *   tables are skipped; W and p must agree).  The merged build has no
 *   ablation baselines.  One host sync (the merged macro ids). */
wt_status wt_build_pack_info(const wt_build* b, int64_t* counts, size_t* bytes);
wt_status wt_build_pack(const wt_build* b, void* dst, size_t cap, void* stream);
wt_status wt_build_merge(const void* packed, size_t stride, int32_t n_parts, const int64_t* counts, int device,
                         void* stream, wt_build** out);

/* fit_bucket over nb independent buckets in one launch: samples of bucket b
 * are [off[b], off[b+1]) of g/l/t (host arrays).  coeffs [nb*4]. */
wt_status wt_fit_bucket_batch(const double* g, const double* l, const double* t,
                              const int64_t* off, int64_t nb, double* coeffs, double* r2,
                              double* mape, int32_t* degenerate, int device);

/* ---- synthetic-profile generator (wave simulator) ----- */

/* simulate() (wave_sim.cpp:80-117) for n independent jobs on `slots` slots:
 * job i dispatches g[i] blocks of duration max(eps, mean + sigma*N(0,1)),
 * N drawn from SplitMix64(mix_seed(seed[i], block)); gap = dispatch gap.
 * Host arrays in and out (synchronous). */
wt_status wt_simulate_batch(const int64_t* g, const double* mean, const double* sigma, const double* eps,
                            const double* gap, const uint64_t* seed, int64_t n, int32_t slots,
                            double* makespan, int device);

/* SimulatorBackend sweep of run_profile (profiler.cpp:192-218, 286-329):
 * records in (point, anchor, feasible pair) order, pairs in (macro_id,
 * micro_id) ascending order with their ground-truth entry. */
typedef struct {
    int64_t n_points;
    const int64_t* point_g;
    int64_t n_anchors;
    const int64_t* anchor_l;
    int64_t n_pairs;
    const int32_t* pair_macro;
    const int32_t* pair_micro;
    const double* pair_base;     /* GroundEntry.base */
    const double* pair_per_iter; /* GroundEntry.per_iter */
    const double* pair_gap;      /* GroundEntry.dispatch_gap */
    double sigma;
    double floor_frac;           /* BlockLatencyModel.floor_frac (0.01) */
    uint64_t seed;
    int32_t warmup, measured;
    int32_t slots;               /* n_sm * blocks_per_sm */
} wt_sim_profile_desc;

/* latency_us / status: host arrays of n_points*n_anchors*n_pairs. */
wt_status wt_profile_sim(const wt_sim_profile_desc* desc, double* latency_us, int32_t* status, int device,
                         double* device_ms);

#ifdef __cplusplus
}
#endif
#endif /* WAVETUNE_C_H */
