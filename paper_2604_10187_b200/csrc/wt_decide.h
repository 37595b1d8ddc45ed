// wt_decide.h -- launch interface between the C-ABI layer and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "wt_internal.h"

namespace wtb {

constexpr int kSweepThreads = 256;
constexpr int kSweepRPT = 4;  // shapes per thread in the sweep
constexpr int kEvalThreads = 256;
constexpr int kGatherThreads = 256;

struct DecOut {
    int32_t* macro;
    int32_t* micro;
    double* lat;
    int64_t* g;
    int64_t* l;
    int32_t* wave;
    uint32_t* flags;
    int32_t* comps;
    double* tail;
    int32_t topk;
    int32_t* topk_macro;
    double* topk_lat;
};

struct SweepArgs {
    const int32_t* N;  // [n_pairs] device
    const int32_t* K;
    int32_t m_lo;
    int64_t mcount;    // M values per pair (representative sweep: intervals per pair)
    // representative sweep (wt_sweep over M intervals): shape i of a pair has
    // M = mrep[i] instead of m_lo + i; null = every M of [m_lo, m_lo + mcount)
    const int32_t* mrep;
    int64_t begin, end;
    int32_t chunk;     // configs per shared-memory chunk
    wt_grid_entry* entries;
    int32_t topk;
    int32_t* topk_macro;
    double* topk_lat;
    // fused multi-GPU sweep (wt_sweep_to): the epilogue stores every entry
    // into each of these grids (local or peer-mapped over NVLink) instead of
    // `entries`; ndst == 0 -> `entries` only
    wt_grid_entry* dst[8];
    int32_t ndst;
};

#ifdef __CUDACC__
// one grid entry into `entries` or into every destination of a fused sweep
__device__ __forceinline__ void store_entry(const SweepArgs& a, int64_t idx, int4 lo, int4 hi) {
    if (a.ndst == 0) {
        int4* e = reinterpret_cast<int4*>(a.entries + idx);
        e[0] = lo;
        e[1] = hi;
        return;
    }
    for (int d = 0; d < a.ndst; ++d) {
        int4* e = reinterpret_cast<int4*>(a.dst[d] + idx);
        e[0] = lo;
        e[1] = hi;
    }
}
#endif

struct EvalArgs {
    const int32_t* M;
    const int32_t* N;
    const int32_t* K;
    int64_t n;
    const int64_t* idx;    // optional compacted query indices
    const int64_t* count;  // optional device count of idx
    int32_t inputs_compact;  // M/N/K indexed by list slot (idx only scatters outputs)
    int32_t chunk;
    DecOut out;
};

struct GroupedArgs {
    const int64_t* row_off;
    const int32_t* rows;
    const int32_t* N;
    const int32_t* K;
    int64_t n;
    DecOut out;
};

// Run-compressed grid heads for k_gather_h.  Along M the 16-byte head
// (latency, macro, micro) of a grid entry is piecewise constant -- G changes
// only where ceil(M / t_m) does -- so each pair's row is cut into blocks of
// 2^kRunBlkShift M values: bhead[p * nblk + b] is the block's head when the
// block holds a single run, else {first run index, 0, INT32_MIN, 0} and the
// runs (rkey[r] = flat entry index where run r starts, rkey[nruns] =
// 0xffffffff, rval[r] = head) resolve it.  Built on the device after a full
// sweep (or by wt_grid_finalize); hdr = {generation the index was built for
// (0 = none), nruns, any multi-run block, a head used the INT32_MIN marker}.
// The host bumps the grid's generation whenever entries may change outside a
// full sweep (raw storage handed out, partial / fused sweeps); a gather uses
// the index only when hdr[0] equals the generation it was launched with, so
// no device write is needed to invalidate it (and none can race).  The gather stages it in shared memory
// when it fits `budget` bytes, else reads heads from L2.
constexpr int kRunBlkShift = 6;
struct RunIndex {
    int32_t* hdr;
    int4* bhead;
    uint32_t* rkey;
    int4* rval;
    int32_t nblk;    // blocks per pair
    int32_t nbtot;   // n_pairs * nblk
    int32_t budget;  // shared-memory bytes reserved for the index (0 = none)
    int32_t gen;     // generation at enqueue time (build: written to hdr[0]; gather: expected)
};

struct GatherArgs {
    const uint64_t* pair_keys;  // sorted (N << 32 | K)
    const int32_t* pair_ids;
    int32_t n_pairs;
    int32_t m_lo, m_hi;
    int64_t mcount;
    const wt_grid_entry* entries;
    const int32_t* topk_macro;
    const double* topk_lat;
    const int32_t* M;
    const int32_t* N;
    const int32_t* K;
    int64_t n;
    DecOut out;
    int64_t* off_count;
    int64_t* off_idx;
    int32_t* off_M;  // compacted copies of the off-grid queries' dims
    int32_t* off_N;
    int32_t* off_K;
    // open-addressing (N, K) -> pair table for k_gather_h: 2^hbits int4
    // slots {N, K, pair id, 0}, empty = pair id -1; null when not built
    const int4* htab;
    int32_t hbits;
    RunIndex runs;
    // optional: grouping key of every compacted off-grid query + its bucket
    // histogram, computed while compacting (k_gather_h), for launch_eval3
    uint32_t* off_key;
    uint32_t* key_hist;
    int32_t key_bits;
    int32_t key_mode;
};

// slot of (N, K) in a 2^bits table: multiplicative hash, high bits
__host__ __device__ __forceinline__ uint32_t pair_slot(uint32_t N, uint32_t K, int bits) {
    const uint32_t h = N * 0x9E3779B1u + K * 0x7FEB352Du;
    return (h ^ (h >> 16)) * 0x85EBCA6Bu >> (32 - bits);
}

struct PredictArgs {
    const int32_t* config;
    const int64_t* g;
    const int64_t* l;
    int64_t n;
    double* lat;
    int32_t* wave;
    int32_t* extrap;
    int32_t* used_w;
    int32_t* status;
};

struct ExplainArgs {
    int64_t M, N, K;
    int64_t* g;
    int64_t* l;
    int32_t* wave;
    int32_t* used_w;
    double* lat;
    int32_t* status;
};

struct NearestArgs {
    const int64_t* anchors;
    int32_t n_anchors;
    const int64_t* l;
    int64_t n;
    int64_t* out;
    int32_t* comps;
};

// 64-bit-dimension queries (wt_wide.cu): narrowed copies + the wide list
struct WideArgs {
    const int64_t* M;
    const int64_t* N;
    const int64_t* K;
    int64_t n;
    int32_t* M32;
    int32_t* N32;
    int32_t* K32;
    int64_t* list;                // indices of queries with a dim >= 2^31
    unsigned long long* count;    // wide list length (zeroed by the caller)
    DecOut out;
};
cudaError_t launch_narrow(const WideArgs& a, cudaStream_t st);
cudaError_t launch_wide(const DevImage& im, const WideArgs& a, cudaStream_t st);

// Library-owned stream-ordered memory pool of a device (wt_capi.cu).
cudaMemPool_t device_pool(int device);
// Launch helpers for the current device, safe for concurrent host threads
// and several devices per process: the dynamic shared-memory limit of a
// kernel is raised monotonically per (device, kernel) -- never lowered under
// a launch in flight -- and occupancy is cached per (device, kernel,
// threads, dynamic smem).
cudaError_t prepare_smem(const void* kernel, size_t dyn_smem);
int occupancy(const void* kernel, int threads, size_t dyn_smem);  // >= 1
int device_sms();

size_t sweep_smem_bytes(const DevImage& im, int chunk, bool special);
size_t eval_smem_bytes(const DevImage& im, int chunk, bool special);
cudaError_t launch_sweep(const DevImage& im, const SweepArgs& a, bool wide, cudaStream_t st);
cudaError_t launch_eval(const DevImage& im, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_grouped(const DevImage& im, const GroupedArgs& a, int grid, cudaStream_t st);
cudaError_t launch_gather(const DevImage& im, const GatherArgs& a, int grid, cudaStream_t st);
// run index of a filled grid (n < 2^32 - 1 entries); temp from runs_temp_bytes
size_t runs_temp_bytes(int64_t n);
cudaError_t launch_runs_build(const wt_grid_entry* entries, int64_t n, int64_t mcount, const RunIndex& ri,
                              void* temp, cudaStream_t st);
cudaError_t launch_predict(const DevImage& im, const PredictArgs& a, cudaStream_t st);
// one query, one warp; result + sequence number written to (pinned) `out`
struct OneOut {
    double lat;
    int64_t g, l;
    double tail;
    int32_t macro, micro, wave;
    uint32_t flags;
    int32_t comps;
    volatile uint32_t seq;
};
cudaError_t launch_one(const DevImage& im, int32_t M, int32_t N, int32_t K, OneOut* out, uint32_t seq,
                       cudaStream_t st);
// Ablation baselines (wt_baseline.cu, reference tuner.cpp:168-250).
struct BaseImage {
    int32_t kind;            // WT_BASELINE_STEP / WT_BASELINE_LINEAR
    int32_t C;               // configs (engine order, or the baseline's own macros)
    int32_t missing;         // some config has no entry: every valid query fails
    int32_t S;               // slots (predict: per call)
    const int32_t* macro;    // [C] ascending (predict lookup)
    const int32_t* has;      // [C] 1 if the config has an entry
    const double4* theta;    // linear: [C]
    const int32_t* off;      // step: [C+1] into al / tw
    const int64_t* al;       // step: anchors, ascending per config
    const double* tw;        // step: per-wave latency per anchor
};
cudaError_t launch_btune(const DevImage& im, const BaseImage& b, const EvalArgs& a, cudaStream_t st);
struct BPredictArgs {
    const int32_t* macro;
    const int64_t* g;
    const int64_t* l;
    int64_t n;
    double* lat;
    int32_t* status;
};
cudaError_t launch_bpredict(const BaseImage& b, const BPredictArgs& a, cudaStream_t st);
// Resident decision server (wt_serve.cu): one CTA polls a pinned mailbox.
struct alignas(64) Mailbox {
    // host -> device: one 16-byte record, read by the server in one load
    // (the host stores M, N, K before req; all four share a cache line)
    volatile int32_t M, N, K;
    volatile uint32_t req;    // request sequence number
    volatile uint32_t stop;   // host -> device: leave now
    volatile uint32_t alive;  // 1 from launch until the server has left
    uint32_t pad[10];
    // device -> host: the decision as four 16-byte stores, each carrying the
    // sequence number in .w, so no fence is needed before the host reads:
    //   {lat lo, lat hi, macro, seq} {g lo, g hi, micro, seq}
    //   {l lo, l hi, wave, seq}      {flags, comps, tail (f32 bits), seq}
    volatile int4 resp[4];
};
// `last` = the last request already answered; idle_ns = leave after this
// long without a request.  Stages the image in shared memory when it fits.
cudaError_t launch_serve(const DevImage& im, int64_t n_anchor, Mailbox* mb, uint32_t last, int64_t idle_ns,
                         cudaStream_t st);
size_t sweep2_scratch_bytes(const DevImage& im, const SweepArgs& a);
cudaError_t launch_sweep2(const DevImage& im, const SweepArgs& a, bool wide, void* scratch, cudaStream_t st);
// Exclusive prefix sum of n u32 (wt_scan.cu); scratch of scan_scratch_bytes(n).
size_t scan_scratch_bytes(int64_t n);
int scan_launches(int64_t n);
cudaError_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, int64_t n, void* scratch, cudaStream_t st);
// Warp-per-shape sweep (representative sweeps; no top-k).
cudaError_t launch_sweep_w(const DevImage& im, const SweepArgs& a, cudaStream_t st);
// Copies representative entries rep[r - rb], r in [rb, re), onto every grid
// entry of their M interval inside the flat range [begin, end): interval i
// of a pair covers M in [mrep[i], mrep[i + 1]) (the last up to m_lo + mcount).
struct ExpandDst {
    wt_grid_entry* d[8];
    int32_t n;
};
cudaError_t launch_expand(const ExpandDst& dst, const wt_grid_entry* rep, int64_t rb, int64_t re, int64_t begin,
                          int64_t end, int32_t m_lo, int64_t mcount, const int32_t* mrep, int32_t nrep,
                          cudaStream_t st);
cudaError_t launch_eval2(const DevImage& im, const EvalArgs& a, int grid, cudaStream_t st);
// row-grouped list evaluation (wt_eval3.cu): key + histogram, scan, scatter,
// evaluation; scratch of eval3_scratch_bytes(a.n) (a.n = host upper bound)
size_t eval3_scratch_bytes(int64_t n);
struct Eval3Bufs {
    uint32_t* hist;  // 2^(key_bits + spread) bucket counters
    uint32_t* keys;  // per list slot
    int32_t key_bits;
    int32_t key_mode;
    size_t hist_bytes;
};
Eval3Bufs eval3_bufs(void* scratch, int64_t n);
// keys_ready: hist / keys were filled by the gather's compaction
cudaError_t launch_eval3(const DevImage& im, const EvalArgs& a, void* scratch, bool keys_ready, cudaStream_t st);
constexpr int kEval3Launches = 6;  // key, scan (3: 2^20 buckets), scatter, eval
int eval2_tile();
cudaError_t launch_explain(const DevImage& im, const ExplainArgs& a, cudaStream_t st);
cudaError_t launch_nearest(const NearestArgs& a, cudaStream_t st);

}  // namespace wtb
