// wt_capi.cu -- the extern "C" boundary declared in include/wavetune_c.h.
// Owns device images (engines) and decision grids, validates inputs the way
// the reference does, and launches the sm_100a kernels of wt_decide.cu.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <chrono>
#include <map>
#include <tuple>
#include <mutex>
#include <vector>

#include "wavetune_c.h"
#include "wt_decide.h"
#include "wt_image_dev.h"
#include "wt_internal.h"

namespace {
// NVTX range around each C-ABI entry point (a no-op unless a tool -- nsys,
// ncu --nvtx -- is attached): the library's calls show up by name on timelines.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace


using namespace wtb;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

wt_status set_err(wt_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

wt_status cuda_err(cudaError_t e, const char* where) {
    return set_err(WT_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};


// Library-owned stream-ordered pool: scratch stays mapped between calls
// (release threshold = max), so per-call compaction buffers cost nothing
// after the first call and need no host synchronisation.
cudaMemPool_t lib_pool(int device) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lock(mu);
    auto it = pools.find(device);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaDeviceGetDefaultMemPool(&pool, device);
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[device] = pool;
    return pool;
}

int sm_count(int device) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

}  // namespace

void wtb::set_last_error(const std::string& msg) { g_err = msg; }

namespace {
std::mutex g_launch_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_attr;                  // (device, kernel) -> limit set
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;              // -> CTAs per SM
std::map<int, int> g_sms;
}  // namespace

cudaError_t wtb::prepare_smem(const void* kernel, size_t dyn_smem) {
    if (dyn_smem == 0) return cudaSuccess;
    // never below the 48 KB default (a lower limit would reject launches
    // that need no opt-in); opted in once per (device, kernel, high-water)
    const size_t want = std::max<size_t>(dyn_smem, 48 * 1024);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_launch_mu);
    size_t& cur = g_smem_attr[{dev, kernel}];
    if (want <= cur) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(want));
    if (e == cudaSuccess) cur = want;
    return e;
}

int wtb::occupancy(const void* kernel, int threads, size_t dyn_smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (prepare_smem(kernel, dyn_smem) != cudaSuccess) return 1;
    std::lock_guard<std::mutex> lock(g_launch_mu);
    auto key = std::make_tuple(dev, kernel, threads, dyn_smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, dyn_smem);
    occ = std::max(occ, 1);
    g_occ[key] = occ;
    return occ;
}

int wtb::device_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_launch_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n;
    return n;
}
cudaMemPool_t wtb::device_pool(int device) { return lib_pool(device); }

// Host-side facts about an engine (the image itself lives on the device).
struct EngineMeta {
    int32_t C = 0, R = 0, S = 0, family = 0;
    bool special = false;
    std::vector<int32_t> macro_id;  // ascending (config order)
    int32_t tm_min = 0, tn_min = 0;
    int64_t n_pool = 0;             // anchor pool entries
    std::vector<int32_t> tm_vals;   // distinct t_m (ascending): grid M intervals
};

struct wt_engine {
    int device = 0;
    EngineMeta host;
    // The device image.  Creation only queues its build (no host sync); the
    // first call that uses the engine waits for it (ready_ev) and reads the
    // one data-dependent host fact, the special-row flag -- so the host can
    // go on (e.g. create a grid) while the image kernels run.
    DevImage dev_{};
    mutable std::atomic<bool> ready{true};
    mutable std::mutex ready_mu;
    cudaEvent_t ready_ev = nullptr;
    const uint32_t* spec_d = nullptr;  // device word: OR of the rows' special bits
    const DevImage& dev() const {
        if (!ready.load(std::memory_order_acquire)) resolve();
        return dev_;
    }
    DevImage& dev_mut() {
        dev();
        return dev_;
    }
    void resolve() const {
        std::lock_guard<std::mutex> lk(ready_mu);
        if (ready.load(std::memory_order_relaxed)) return;
        auto* self = const_cast<wt_engine*>(this);
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        uint32_t special = 0;
        cudaEventSynchronize(ready_ev);
        cudaMemcpy(&special, spec_d, 4, cudaMemcpyDeviceToHost);
        cudaSetDevice(prev);
        self->host.special = special != 0;
        self->dev_.special = special != 0 ? 1 : 0;
        ready.store(true, std::memory_order_release);
    }
    void* mem = nullptr;
    size_t bytes = 0;
    int eval_chunk = 0;
    int eval_grid = 0;
    int eval_grid2 = 0;
    // wt_tune_one: private stream + pinned, device-mapped mailbox
    mutable std::mutex one_mu;
    mutable cudaStream_t one_st = nullptr;
    mutable OneOut* one_h = nullptr;
    mutable OneOut* one_d = nullptr;
    mutable uint32_t one_seq = 0;
    // resident server (wt_engine_set_resident): pinned mailbox, idle timeout
    mutable Mailbox* mb_h = nullptr;
    mutable Mailbox* mb_d = nullptr;
    int64_t idle_ns = 0;
};

namespace {
void stop_server(const wt_engine* e) {
    if (!e->mb_h || !e->mb_h->alive) return;
    e->mb_h->stop = 1;
    cudaStreamSynchronize(e->one_st);
    e->mb_h->stop = 0;
    e->mb_h->alive = 0;
}
}  // namespace

struct wt_grid {
    const wt_engine* eng = nullptr;
    int32_t n_pairs = 0;
    int32_t m_lo = 1, m_hi = 0;
    int64_t mcount = 0, n_entries = 0;
    int32_t topk = 0;
    bool wide = false;
    void* mem = nullptr;
    bool pooled = false;    // mem from the library pool (wt_grid_create_async): not IPC-exportable
    // M intervals on which every ceil(M / t_m) is constant: a grid entry
    // depends on M only through those quotients (G = ceil(M/t_m) ceil(N/t_n)),
    // so the sweep evaluates one representative M per interval and copies
    // its entry over the interval (nrep = 0: plain sweep)
    int32_t nrep = 0;
    int32_t* d_mrep = nullptr;
    std::vector<int32_t> h_mrep;
    int32_t* dN = nullptr;
    int32_t* dK = nullptr;
    uint64_t* dkeys = nullptr;
    int32_t* dpid = nullptr;
    wt_grid_entry* entries = nullptr;
    int32_t* tk_macro = nullptr;
    double* tk_lat = nullptr;
    int32_t n_keys = 0;
    int4* dhash = nullptr;  // (N, K) -> pair open-addressing table (k_gather_h)
    int32_t hbits = 0;
    RunIndex runs{};        // run-compressed heads (k_gather_h); budget 0 = none
    mutable std::atomic<int32_t> gen{1};  // run-index generation (wt_decide.h, RunIndex)
    RunIndex runs_now() const {  // the index as a launch sees it
        RunIndex r = runs;
        r.gen = gen.load();
        return r;
    }
    void invalidate_runs() const {  // entries may change: stale index never matches again
        int32_t v = gen.load();
        while (!gen.compare_exchange_weak(v, v == INT32_MAX ? 1 : v + 1)) {
        }
    }
};

namespace {
std::atomic<int> g_timing{0};
cudaEvent_t g_tev[4] = {};
bool g_tev_used = false;
void timing_mark(int i, cudaStream_t s) {
    if (!g_timing.load()) return;
    if (!g_tev[i]) cudaEventCreate(&g_tev[i]);
    cudaEventRecord(g_tev[i], s);
    g_tev_used = true;
}
}  // namespace

extern "C" {

wt_status wt_set_kernel_timing(int enable) {
    g_timing.store(enable ? 1 : 0);
    return WT_OK;
}

wt_status wt_kernel_time_ms(int which, float* ms) {
    if (!ms || which < 0 || which > 1) return set_err(WT_INVALID_ARGUMENT, "which must be 0 or 1");
    if (!g_tev_used || !g_tev[2 * which] || !g_tev[2 * which + 1])
        return set_err(WT_RUNTIME_ERROR, "no timed call recorded");
    cudaError_t ce = cudaEventSynchronize(g_tev[2 * which + 1]);
    if (ce == cudaSuccess) ce = cudaEventElapsedTime(ms, g_tev[2 * which], g_tev[2 * which + 1]);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_kernel_time_ms");
    return WT_OK;
}

const char* wt_last_error(void) { return g_err.c_str(); }
const char* wt_version(void) { return "wavetune-b200 0.1 (sm_100a)"; }
int wt_abi_version(void) { return WT_ABI_VERSION; }
int64_t wt_launch_count(void) { return g_launches.load(); }

wt_status wt_prune_plan(const wt_tables_desc* tables, const wt_registry_desc* registry, const wt_hw* hw,
                        int32_t* n_seg, int32_t* R, int32_t* C, int32_t* cls_cfg, int32_t* seg_pos,
                        int32_t* seg_n, uint32_t* masks) {
    if (!tables || !registry || !hw || !n_seg || !R || !C) return set_err(WT_INVALID_ARGUMENT, "null argument");
    ImagePlan P;
    std::vector<uint32_t> segmask;
    std::string err;
    const wt_status st = masks ? prune_plan_host(*tables, *registry, *hw, &P, &segmask, &err)
                               : plan_image(tables->macro_id, tables->W, tables->n_tables, *registry, *hw, &P, &err);
    if (st != WT_OK) return set_err(st, err);
    const int32_t ns = int32_t(P.seg_pos.size());
    *n_seg = ns;
    *R = P.R;
    *C = P.C;
    if (!masks) return WT_OK;
    if (!cls_cfg || !seg_pos || !seg_n) return set_err(WT_INVALID_ARGUMENT, "null output buffer");
    std::copy(P.cls_cfg.begin(), P.cls_cfg.end(), cls_cfg);
    for (int32_t k = 0; k < ns; ++k) {
        seg_pos[k] = P.seg_pos[k];
        seg_n[k] = P.seg_tiles[4 * k + 3];
    }
    std::copy(segmask.begin(), segmask.end(), masks);
    return WT_OK;
}

}  // extern "C"

namespace {

// Device copy of the tables' CSR (wt_tables_desc with device pointers) and
// the pool arrays, as the image builder reads them.
struct DevTables {
    TabView tv{};
    const int64_t* anchor_l = nullptr;
    const int32_t* anchor_micro = nullptr;
    int64_t n_anchor = 0;
    const int64_t* ext_l = nullptr;
    const int32_t* ext_micro = nullptr;
    int64_t n_ext = 0;
};

// Allocates the engine's arena, uploads the plan (one H2D copy), builds the
// rows, class views and pruning masks on the device from `T`, copies the
// anchor pool, and reads back the special-row flag (the only host sync).
// Pinned staging for the plan upload (one buffer per host thread): a
// pageable H2D of this size blocks the host until the stream reaches the
// copy, i.e. until the fit's tail has run, which serialised the host's image
// preparation behind it.  Before the buffer is rewritten, the previous copy
// out of it is waited for (its event; normally long complete).
struct PinnedStage {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;  // recorded after the last copy out of p
    int done_dev = -1;  // (kept for the thread's life, like the fit's pinned words)
};
static void* pinned_stage(PinnedStage& ps, size_t bytes) {
    if (ps.done) cudaEventSynchronize(ps.done);
    if (bytes > ps.cap) {
        if (ps.p) cudaFreeHost(ps.p);
        ps.p = nullptr;
        ps.cap = 0;
        const size_t want = std::max<size_t>(bytes, 256 << 10);
        if (cudaMallocHost(&ps.p, want) != cudaSuccess) return nullptr;
        ps.cap = want;
    }
    return ps.p;
}
static void pinned_stage_mark(PinnedStage& ps, int device, cudaStream_t s) {
    if (ps.done && ps.done_dev != device) {
        cudaEventDestroy(ps.done);
        ps.done = nullptr;
    }
    if (!ps.done && cudaEventCreateWithFlags(&ps.done, cudaEventDisableTiming) != cudaSuccess) {
        ps.done = nullptr;
        return;
    }
    ps.done_dev = device;
    cudaEventRecord(ps.done, s);
}

wt_status engine_build(wt_engine* e, const ImagePlan& P, const DevTables& T, cudaStream_t s) {
    const size_t C = P.C, R = P.R, NS = P.seg_pos.size(), NCLS = P.cls_seg.size() - 1;
    const int64_t n_pool = std::max<int64_t>(1, T.n_anchor + T.n_ext);
    if (T.n_anchor + T.n_ext >= (int64_t(1) << 31))
        return set_err(WT_UNSUPPORTED, "anchor pool above 2^31 entries is outside the device path's range");
    Arena ar;
    // plan region first (uploaded in one copy), then the device-built arrays
    const size_t o_mid = ar.take(C * 4), o_til = ar.take(C * 16), o_mag = ar.take(C * 16), o_st = ar.take(NS * 16),
                 o_sm = ar.take(NS * 16), o_sp = ar.take(NS * 4), o_cc = ar.take(C * 4), o_ord = ar.take(C * 4),
                 o_cp = ar.take(C * 4), o_cs = ar.take((NCLS + 1) * 4);
    const size_t plan_bytes = ar.used;
    const size_t o_th = ar.take(C * R * 32), o_meta = ar.take(C * R * 4), o_used = ar.take(C * R * 4),
                 o_amap = ar.take(C * R * 8), o_afb = ar.take(C * R * 4), o_al = ar.take(size_t(n_pool) * 8),
                 o_am = ar.take(size_t(n_pool) * 4), o_th2 = ar.take(C * R * 32), o_m2 = ar.take(C * R * 4),
                 o_th2t = ar.take(C * R * 32), o_m2t = ar.take(C * R * 4), o_smask = ar.take(NS * R * kLB * 4),
                 o_sor = ar.take(NS * R * 4), o_spec = ar.take(4);
    // stream-ordered from the library pool (retained across engines: a
    // rebuild costs no cudaMalloc); ordered before the image kernels on s
    cudaError_t ce = cudaMallocFromPoolAsync(&e->mem, ar.used, lib_pool(e->device), s);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_engine_create: allocation");
    e->bytes = ar.used;
    char* base = static_cast<char*>(e->mem);
    thread_local PinnedStage pstage;
    char* pin = static_cast<char*>(pinned_stage(pstage, plan_bytes));
    std::vector<char> stage(pin ? 0 : plan_bytes, 0);
    char* sbuf = pin ? pin : stage.data();
    if (pin) std::memset(pin, 0, plan_bytes);
    auto put = [&](size_t off, const void* src, size_t n) {
        if (n) std::memcpy(sbuf + off, src, n);
    };
    put(o_mid, P.macro_id.data(), C * 4);
    put(o_til, P.tiles.data(), C * 16);
    put(o_mag, P.magic.data(), C * 16);
    put(o_st, P.seg_tiles.data(), NS * 16);
    put(o_sm, P.seg_magic.data(), NS * 16);
    put(o_sp, P.seg_pos.data(), NS * 4);
    put(o_cc, P.cls_cfg.data(), C * 4);
    put(o_ord, P.order.data(), C * 4);
    put(o_cp, P.cfg_pos.data(), C * 4);
    put(o_cs, P.cls_seg.data(), (NCLS + 1) * 4);
    ce = cudaMemcpyAsync(base, sbuf, plan_bytes, cudaMemcpyHostToDevice, s);
    if (ce == cudaSuccess && pin) pinned_stage_mark(pstage, e->device, s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(base + o_spec, 0, 4, s);
    auto at = [&](size_t off) { return static_cast<void*>(base + off); };
    if (ce == cudaSuccess && T.n_anchor > 0) {
        ce = cudaMemcpyAsync(at(o_al), T.anchor_l, size_t(T.n_anchor) * 8, cudaMemcpyDeviceToDevice, s);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(at(o_am), T.anchor_micro, size_t(T.n_anchor) * 4, cudaMemcpyDeviceToDevice, s);
    }
    if (ce == cudaSuccess && T.n_ext > 0) {
        ce = cudaMemcpyAsync(base + o_al + size_t(T.n_anchor) * 8, T.ext_l, size_t(T.n_ext) * 8,
                             cudaMemcpyDeviceToDevice, s);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(base + o_am + size_t(T.n_anchor) * 4, T.ext_micro, size_t(T.n_ext) * 4,
                                 cudaMemcpyDeviceToDevice, s);
    }
    if (ce == cudaSuccess && T.n_anchor + T.n_ext == 0) {  // keep the pool non-empty for the device
        const int64_t z = 0;
        const int32_t m1 = -1;
        ce = cudaMemcpyAsync(at(o_al), &z, 8, cudaMemcpyHostToDevice, s);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(at(o_am), &m1, 4, cudaMemcpyHostToDevice, s);
    }
    if (ce != cudaSuccess) return cuda_err(ce, "wt_engine_create: upload");
    ImgRowsArgs ra{};
    ra.C = P.C;
    ra.R = P.R;
    ra.order = static_cast<const int32_t*>(at(o_ord));
    ra.cfg_pos = static_cast<const int32_t*>(at(o_cp));
    ra.theta = static_cast<double4*>(at(o_th));
    ra.rowmeta = static_cast<uint32_t*>(at(o_meta));
    ra.used_w = static_cast<int32_t*>(at(o_used));
    ra.amap = static_cast<int2*>(at(o_amap));
    ra.afb = static_cast<int32_t*>(at(o_afb));
    ra.theta2 = static_cast<double4*>(at(o_th2));
    ra.meta2 = static_cast<uint32_t*>(at(o_m2));
    ra.theta2t = static_cast<double4*>(at(o_th2t));
    ra.meta2t = static_cast<uint32_t*>(at(o_m2t));
    ra.special = static_cast<uint32_t*>(at(o_spec));
    ImgPruneArgs pa{};
    pa.C = P.C;
    pa.R = P.R;
    pa.S = P.S;
    pa.nseg = int32_t(NS);
    pa.ncells = int64_t(NCLS) * P.R * kLB;
    pa.cls_seg = static_cast<const int32_t*>(at(o_cs));
    pa.seg_pos = static_cast<const int32_t*>(at(o_sp));
    pa.seg_tiles = static_cast<const int4*>(at(o_st));
    pa.theta2 = ra.theta2;
    pa.meta2 = ra.meta2;
    pa.segmask = static_cast<uint32_t*>(at(o_smask));
    pa.segor = static_cast<uint32_t*>(at(o_sor));
    static const bool tr = std::getenv("WT_TRACE_ENGINE") != nullptr;
    const auto tq = std::chrono::steady_clock::now();
    ce = launch_image_build(T.tv, ra, pa, s);
    g_launches += 2;
    // no host sync: the first use of the engine waits on this event
    if (ce == cudaSuccess && !e->ready_ev) ce = cudaEventCreateWithFlags(&e->ready_ev, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventRecord(e->ready_ev, s);
    if (tr) {
        cudaStreamSynchronize(s);
        std::fprintf(stderr, "[engine]   image kernels done %.3f ms after queueing\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq).count());
    }
    if (ce != cudaSuccess) return cuda_err(ce, "wt_engine_create: image build");
    e->spec_d = static_cast<const uint32_t*>(at(o_spec));
    e->ready.store(false, std::memory_order_release);

    EngineMeta& h = e->host;
    h.C = P.C;
    h.R = P.R;
    h.S = P.S;
    h.family = P.family;
    h.special = false;  // resolved at first use (wt_engine::resolve)
    h.macro_id = P.macro_id;
    h.tm_min = P.tm_min;
    h.tm_vals.clear();
    for (size_t c = 0; c < C; ++c) h.tm_vals.push_back(P.tiles[4 * c]);
    std::sort(h.tm_vals.begin(), h.tm_vals.end());
    h.tm_vals.erase(std::unique(h.tm_vals.begin(), h.tm_vals.end()), h.tm_vals.end());
    h.tn_min = P.tn_min;
    h.n_pool = n_pool;
    DevImage& d = e->dev_;
    d.C = P.C;
    d.R = P.R;
    d.S = P.S;
    d.RS = uint32_t(P.R) * uint32_t(P.S);
    const Magic ms = make_magic(uint32_t(P.S));
    d.mS = ms.m;
    d.sS = ms.s;
    d.special = 0;  // resolved at first use
    d.macro_id = static_cast<const int32_t*>(at(o_mid));
    d.tiles = static_cast<const int4*>(at(o_til));
    d.magic = static_cast<const uint4*>(at(o_mag));
    d.theta = ra.theta;
    d.rowmeta = ra.rowmeta;
    d.used_w = ra.used_w;
    d.amap = ra.amap;
    d.afb = ra.afb;
    d.anchor_l = static_cast<const int64_t*>(at(o_al));
    d.anchor_micro = static_cast<const int32_t*>(at(o_am));
    d.tm_min = P.tm_min;
    d.tn_min = P.tn_min;
    d.nseg = int32_t(NS);
    d.seg_cfg = P.seg_cfg;
    d.seg_tiles = pa.seg_tiles;
    d.seg_magic = static_cast<const uint4*>(at(o_sm));
    d.seg_pos = pa.seg_pos;
    d.cls_cfg = static_cast<const int32_t*>(at(o_cc));
    d.theta2 = ra.theta2;
    d.meta2 = ra.meta2;
    d.theta2t = ra.theta2t;
    d.meta2t = ra.meta2t;
    d.segmask = pa.segmask;
    d.segor = pa.segor;
    static const int prune = [] {
        const char* v = std::getenv("WT_PRUNE");
        return v ? std::atoi(v) : 1;
    }();
    d.prune = prune;
    d.seg_maxcfg = P.seg_maxcfg;
    // list-mode chunk: keep the staged rows near 40 KB so several CTAs fit per SM
    e->eval_chunk = int(std::max<size_t>(1, std::min<size_t>(C, 40960 / (R * 36 + 32))));
    e->eval_grid = sm_count(e->device) * 4;
    e->eval_grid2 = sm_count(e->device) * 4;  // upper bound; launch_eval2 clamps to residency
    return WT_OK;
}

}  // namespace

extern "C" {

wt_status wt_engine_create(const wt_tables_desc* tables, const wt_registry_desc* registry,
                           const wt_hw* hw, int device, wt_engine** out) {
    NvtxRange nvtx_("wt_engine_create");
    if (!tables || !registry || !hw || !out) return set_err(WT_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    ImagePlan P;
    std::string err;
    const wt_status st = plan_image(tables->macro_id, tables->W, tables->n_tables, *registry, *hw, &P, &err);
    if (st != WT_OK) return set_err(st, err);
    const wt_tables_desc& t = *tables;
    const int64_t n = t.n_tables, n_coeff = t.coeff_off[n], n_awave = t.awave_off[n];
    const int64_t n_anchor = t.awave_aoff[n_awave], n_ext = t.ext_aoff[n];
    DeviceGuard guard(device);
    // the tables' CSR travels once (one packed H2D copy); everything else is
    // resolved on the device
    Arena ar;
    const size_t o_W = ar.take(n * 4), o_te = ar.take(n * 32), o_co = ar.take((n + 1) * 4),
                 o_cw = ar.take(n_coeff * 4), o_ct = ar.take(n_coeff * 32), o_ao = ar.take((n + 1) * 4),
                 o_aw = ar.take(n_awave * 4), o_aa = ar.take((n_awave + 1) * 4), o_eo = ar.take((n + 1) * 4),
                 o_al = ar.take(n_anchor * 8), o_am = ar.take(n_anchor * 4), o_el = ar.take(n_ext * 8),
                 o_em = ar.take(n_ext * 4);
    std::vector<char> stage(ar.used, 0);
    auto put = [&](size_t off, const void* src, size_t bytes) {
        if (bytes) std::memcpy(stage.data() + off, src, bytes);
    };
    put(o_W, t.W, n * 4);
    put(o_te, t.theta_ext, n * 32);
    put(o_co, t.coeff_off, (n + 1) * 4);
    put(o_cw, t.coeff_w, n_coeff * 4);
    put(o_ct, t.coeff_theta, n_coeff * 32);
    put(o_ao, t.awave_off, (n + 1) * 4);
    put(o_aw, t.awave_w, n_awave * 4);
    put(o_aa, t.awave_aoff, (n_awave + 1) * 4);
    put(o_eo, t.ext_aoff, (n + 1) * 4);
    put(o_al, t.anchor_l, n_anchor * 8);
    put(o_am, t.anchor_micro, n_anchor * 4);
    put(o_el, t.ext_l, n_ext * 8);
    put(o_em, t.ext_micro, n_ext * 4);
    cudaStream_t s = nullptr;
    cudaError_t ce = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_engine_create: stream");
    struct SD {
        cudaStream_t s;
        ~SD() { cudaStreamDestroy(s); }
    } sd{s};
    void* tmp = nullptr;
    ce = cudaMallocFromPoolAsync(&tmp, ar.used, lib_pool(device), s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(tmp, stage.data(), ar.used, cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_engine_create: table upload");
    char* b = static_cast<char*>(tmp);
    DevTables T;
    T.tv = TabView{reinterpret_cast<const int32_t*>(b + o_W), reinterpret_cast<const double*>(b + o_te),
                   reinterpret_cast<const int32_t*>(b + o_co), reinterpret_cast<const int32_t*>(b + o_cw),
                   reinterpret_cast<const double*>(b + o_ct), reinterpret_cast<const int32_t*>(b + o_ao),
                   reinterpret_cast<const int32_t*>(b + o_aw), reinterpret_cast<const int32_t*>(b + o_aa),
                   reinterpret_cast<const int32_t*>(b + o_eo), n_anchor, nullptr};
    T.anchor_l = reinterpret_cast<const int64_t*>(b + o_al);
    T.anchor_micro = reinterpret_cast<const int32_t*>(b + o_am);
    T.n_anchor = n_anchor;
    T.ext_l = reinterpret_cast<const int64_t*>(b + o_el);
    T.ext_micro = reinterpret_cast<const int32_t*>(b + o_em);
    T.n_ext = n_ext;
    auto* e = new wt_engine;
    e->device = device;
    const wt_status bs = engine_build(e, P, T, s);
    cudaFreeAsync(tmp, s);
    if (bs != WT_OK) {
        if (e->mem) {
            cudaStreamSynchronize(s);
            cudaFreeAsync(e->mem, s);
        }
        delete e;
        return bs;
    }
    *out = e;
    return WT_OK;
}

wt_status wt_engine_create_from_build(const wt_build* b, const wt_registry_desc* registry, const wt_hw* hw,
                                      void* stream, wt_engine** out) {
    NvtxRange nvtx_("wt_engine_create_from_build");
    if (!b || !registry || !hw || !out) return set_err(WT_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    static const bool tr = std::getenv("WT_TRACE_ENGINE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    BuildTables bt{};
    if (build_device_tables(b, &bt) != WT_OK) return set_err(WT_INVALID_ARGUMENT, "invalid build");
    std::vector<int32_t> W(bt.n_tables, bt.W);
    ImagePlan P;
    std::string err;
    const wt_status st = plan_image(bt.macro_id_host, W.data(), bt.n_tables, *registry, *hw, &P, &err);
    if (st != WT_OK) return set_err(st, err);
    if (tr)
        std::fprintf(stderr, "[engine] plan_image %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    DeviceGuard guard(bt.device);
    DevTables T;
    T.tv = bt.tv;
    T.anchor_l = bt.anchor_l;
    T.anchor_micro = bt.anchor_micro;
    T.n_anchor = bt.n_anchor;
    T.ext_l = bt.ext_l;
    T.ext_micro = bt.ext_micro;
    T.n_ext = bt.n_ext;
    auto* e = new wt_engine;
    e->device = bt.device;
    const wt_status bs = engine_build(e, P, T, static_cast<cudaStream_t>(stream));
    if (tr)
        std::fprintf(stderr, "[engine] + engine_build %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (bs != WT_OK) {
        if (e->mem) {
            cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
            cudaFreeAsync(e->mem, static_cast<cudaStream_t>(stream));
        }
        delete e;
        return bs;
    }
    *out = e;
    return WT_OK;
}

wt_status wt_engine_destroy(wt_engine* e) {
    if (!e) return WT_OK;
    DeviceGuard guard(e->device);
    stop_server(e);
    if (e->one_st) cudaStreamDestroy(e->one_st);
    if (e->ready_ev) cudaEventDestroy(e->ready_ev);
    if (e->one_h) cudaFreeHost(e->one_h);
    if (e->mb_h) cudaFreeHost(e->mb_h);
    // pool memory: free after every stream's use of the engine (the
    // cudaFree this replaces synchronised the device too)
    cudaDeviceSynchronize();
    cudaFreeAsync(e->mem, nullptr);
    cudaStreamSynchronize(nullptr);
    delete e;
    return WT_OK;
}

wt_status wt_engine_info_get(const wt_engine* e, wt_engine_info* out) {
    if (!e || !out) return set_err(WT_INVALID_ARGUMENT, "null argument");
    out->n_configs = e->host.C;
    out->n_rows = e->host.R;
    out->slots = e->host.S;
    out->family = e->host.family;
    out->has_fallback_rows = e->dev().special ? 1 : 0;
    out->device = e->device;
    out->device_bytes = e->bytes;
    return WT_OK;
}

wt_status wt_engine_prune_masks(const wt_engine* e, uint32_t* masks, int64_t n) {
    if (!e || !masks) return set_err(WT_INVALID_ARGUMENT, "null argument");
    const int64_t want = int64_t(e->dev().nseg) * e->dev().R * kLB;
    if (n != want) return set_err(WT_INVALID_ARGUMENT, "masks must hold n_seg * R * 16 words");
    DeviceGuard guard(e->device);
    const cudaError_t ce = cudaMemcpy(masks, e->dev().segmask, size_t(n) * 4, cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_engine_prune_masks");
    return WT_OK;
}

wt_status wt_engine_count_evals(wt_engine* e, unsigned long long* counter) {
    if (!e) return set_err(WT_INVALID_ARGUMENT, "null argument");
    e->dev_mut().eval_count = counter;
    return WT_OK;
}

wt_status wt_engine_set_prune(wt_engine* e, int32_t enable) {
    if (!e) return set_err(WT_INVALID_ARGUMENT, "null argument");
    e->dev_mut().prune = enable ? 1 : 0;
    return WT_OK;
}

int32_t wt_engine_config_index(const wt_engine* e, int32_t macro_id) {
    if (!e) return -1;
    auto it = std::lower_bound(e->host.macro_id.begin(), e->host.macro_id.end(), macro_id);
    if (it == e->host.macro_id.end() || *it != macro_id) return -1;
    return int32_t(it - e->host.macro_id.begin());
}

int32_t wt_engine_anchor_map(const wt_engine* e, int32_t config, int32_t wave, int32_t extrapolated,
                             int64_t* anchors, int32_t* micros, int32_t cap, int32_t* fallback_wave) {
    if (!e || config < 0 || config >= e->host.C) return -1;
    const EngineMeta& h = e->host;
    int32_t row;
    if (extrapolated) row = h.R - 1;
    else if (wave >= 1 && wave < h.R) row = wave - 1;
    else return -1;
    // inspection call: small synchronous reads of the device image
    DeviceGuard guard(e->device);
    const size_t rr = size_t(config) * h.R + row;
    uint32_t meta = 0;
    int2 am{0, 0};
    int32_t fb = -1;
    if (cudaMemcpy(&meta, e->dev().rowmeta + rr, 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&am, e->dev().amap + rr, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&fb, e->dev().afb + rr, 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    if (meta & ROW_NO_ANCHOR) return -1;
    const int32_t n = std::min(am.y, std::max(cap, 0));
    if (n > 0 && anchors &&
        cudaMemcpy(anchors, e->dev().anchor_l + am.x, size_t(n) * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    if (n > 0 && micros &&
        cudaMemcpy(micros, e->dev().anchor_micro + am.x, size_t(n) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    if (fallback_wave) fallback_wave[0] = fb;
    return am.y;
}

static DecOut to_out(const wt_decisions* o) {
    DecOut d{};
    d.macro = o->macro_id;
    d.micro = o->micro_id;
    d.lat = o->latency_us;
    d.g = o->g;
    d.l = o->l;
    d.wave = o->wave;
    d.flags = o->flags;
    d.comps = o->comparisons;
    d.tail = o->tail_frac;
    d.topk = o->topk;
    d.topk_macro = o->topk_macro;
    d.topk_lat = o->topk_latency;
    return d;
}

static wt_status check_out(const wt_decisions* o) {
    if (!o || !o->macro_id || !o->micro_id || !o->latency_us)
        return set_err(WT_INVALID_ARGUMENT, "decision outputs macro_id, micro_id, latency_us are required");
    if (o->topk < 0 || o->topk > 8) return set_err(WT_UNSUPPORTED, "topk must be in [0, 8]");
    if (o->topk > 0 && (!o->topk_macro || !o->topk_latency))
        return set_err(WT_INVALID_ARGUMENT, "topk outputs missing");
    return WT_OK;
}

// List evaluation without top-k: the row-grouped pipeline (wt_eval3.cu) by
// default, the shared-memory staged kernel with WT_EVAL_MODE=2 (A/B runs).
static int eval_mode() {
    static const int mode = [] {
        const char* v = std::getenv("WT_EVAL_MODE");
        return v ? std::atoi(v) : 3;
    }();
    return mode;
}

// scratch != null: allocated (and keyed) by the caller
static cudaError_t run_list_eval(const wt_engine* e, const EvalArgs& a, cudaStream_t s, void* scratch = nullptr) {
    if (eval_mode() == 2) {
        const int64_t tiles = (a.n + eval2_tile() - 1) / eval2_tile();
        g_launches++;
        return launch_eval2(e->dev(), a, int(std::min<int64_t>(tiles, e->eval_grid2)), s);
    }
    const bool own = scratch == nullptr;
    cudaError_t ce = cudaSuccess;
    if (own) ce = cudaMallocFromPoolAsync(&scratch, eval3_scratch_bytes(a.n), lib_pool(e->device), s);
    if (ce != cudaSuccess) return ce;
    ce = launch_eval3(e->dev(), a, scratch, !own, s);
    if (own) cudaFreeAsync(scratch, s);
    g_launches += own ? kEval3Launches : kEval3Launches - 1;
    return ce;
}

// the decisions of queries [i, ...) of a batch (pointer offsets)
static wt_decisions offset_decisions(const wt_decisions& o, int64_t i) {
    wt_decisions d = o;
    d.macro_id += i;
    d.micro_id += i;
    d.latency_us += i;
    if (d.g) d.g += i;
    if (d.l) d.l += i;
    if (d.wave) d.wave += i;
    if (d.flags) d.flags += i;
    if (d.comparisons) d.comparisons += i;
    if (d.tail_frac) d.tail_frac += i;
    if (d.topk_macro) d.topk_macro += i * d.topk;
    if (d.topk_latency) d.topk_latency += i * d.topk;
    return d;
}

// scratch-bounding slice of huge batches (WT_BATCH_SLICE overrides, for tests;
// multiples of 4 keep the 16-byte alignment of the sliced arrays)
static int64_t batch_slice() {
    static const int64_t v = [] {
        const char* x = std::getenv("WT_BATCH_SLICE");
        const int64_t d = int64_t(1) << 28;
        const int64_t s = x ? std::atoll(x) : d;
        return s >= 4 ? s & ~int64_t(3) : d;
    }();
    return v;
}

wt_status wt_tune_batch(const wt_engine* e, const int32_t* M, const int32_t* N, const int32_t* K,
                        int64_t n, const wt_decisions* out, void* stream) {
    NvtxRange nvtx_("wt_tune_batch");
    if (!e) return set_err(WT_INVALID_ARGUMENT, "null engine");
    if (n < 0) return set_err(WT_INVALID_ARGUMENT, "negative batch size");
    wt_status st = check_out(out);
    if (st) return st;
    if (n == 0) return WT_OK;
    if (e->host.family == WT_FAMILY_GROUPED_GEMM)
        return set_err(WT_INVALID_ARGUMENT, "dense_gemm workload needs gemm tiles");
    DeviceGuard guard(e->device);
    EvalArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.n = n;
    a.chunk = e->eval_chunk;
    a.out = to_out(out);
    cudaError_t ce;
    if (a.out.topk > 0) {  // per-config order kernel keeps the top-k list
        const int64_t tiles = (n + kEvalThreads - 1) / kEvalThreads;
        ce = launch_eval(e->dev(), a, int(std::min<int64_t>(tiles, e->eval_grid)), static_cast<cudaStream_t>(stream));
        g_launches++;
    } else {
        ce = cudaSuccess;
        const int64_t kBatchSlice = batch_slice();
        for (int64_t i = 0; i < n && ce == cudaSuccess; i += kBatchSlice) {
            const wt_decisions d = offset_decisions(*out, i);
            EvalArgs b = a;
            b.M = M + i;
            b.N = N + i;
            b.K = K + i;
            b.n = std::min(kBatchSlice, n - i);
            b.out = to_out(&d);
            ce = run_list_eval(e, b, static_cast<cudaStream_t>(stream));
        }
    }
    if (ce != cudaSuccess) return cuda_err(ce, "wt_tune_batch");
    return WT_OK;
}

wt_status wt_tune_one(const wt_engine* e, int32_t M, int32_t N, int32_t K, wt_decision_one* out) {
    if (!e || !out) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (e->host.family == WT_FAMILY_GROUPED_GEMM)
        return set_err(WT_INVALID_ARGUMENT, "dense_gemm workload needs gemm tiles");
    std::lock_guard<std::mutex> lk(e->one_mu);
    DeviceGuard guard(e->device);
    if (!e->one_h) {
        cudaError_t ce = cudaStreamCreateWithFlags(&e->one_st, cudaStreamNonBlocking);
        if (ce == cudaSuccess)
            ce = cudaHostAlloc(reinterpret_cast<void**>(&e->one_h), sizeof(OneOut), cudaHostAllocMapped);
        if (ce == cudaSuccess) ce = cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->one_d), e->one_h, 0);
        if (ce != cudaSuccess) {
            if (e->one_h) cudaFreeHost(e->one_h);
            e->one_h = nullptr;
            return cuda_err(ce, "wt_tune_one setup");
        }
        e->one_h->seq = 0;
    }
    const uint32_t seq = ++e->one_seq == 0 ? ++e->one_seq : e->one_seq;
    cudaError_t ce = cudaSuccess;
    if (e->idle_ns > 0) {  // resident server: post, (re)start if it left, poll
        Mailbox* mb = e->mb_h;
        if (!mb) {
            ce = cudaHostAlloc(reinterpret_cast<void**>(&e->mb_h), sizeof(Mailbox), cudaHostAllocMapped);
            if (ce == cudaSuccess) ce = cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->mb_d), e->mb_h, 0);
            if (ce != cudaSuccess) return cuda_err(ce, "wt_tune_one mailbox");
            mb = e->mb_h;
            std::memset(static_cast<void*>(mb), 0, sizeof(Mailbox));
        }
        const int64_t n_anchor = e->host.n_pool;
        mb->M = M;
        mb->N = N;
        mb->K = K;
        std::atomic_thread_fence(std::memory_order_release);
        mb->req = seq;
        auto answered = [&] {
            for (int c = 0; c < 4; ++c)
                if (uint32_t(mb->resp[c].w) != seq) return false;
            return true;
        };
        for (uint32_t spin = 0; !answered(); ++spin) {
            if (!mb->alive) {
                std::atomic_thread_fence(std::memory_order_acquire);
                if (answered()) break;
                mb->alive = 1;
                ce = launch_serve(e->dev(), n_anchor, e->mb_d, seq - 1, e->idle_ns, e->one_st);
                g_launches++;
                if (ce != cudaSuccess) {
                    mb->alive = 0;
                    return cuda_err(ce, "wt_tune_one server");
                }
            }
            if ((spin & 4095u) == 4095u) {
                ce = cudaStreamQuery(e->one_st);
                if (ce != cudaSuccess && ce != cudaErrorNotReady) {
                    mb->alive = 0;
                    return cuda_err(ce, "wt_tune_one server");
                }
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        const int4 r0 = {mb->resp[0].x, mb->resp[0].y, mb->resp[0].z, 0};
        const int4 r1 = {mb->resp[1].x, mb->resp[1].y, mb->resp[1].z, 0};
        const int4 r2 = {mb->resp[2].x, mb->resp[2].y, mb->resp[2].z, 0};
        const int4 r3 = {mb->resp[3].x, mb->resp[3].y, mb->resp[3].z, 0};
        const uint64_t latb = uint64_t(uint32_t(r0.x)) | (uint64_t(uint32_t(r0.y)) << 32);
        std::memcpy(&out->latency_us, &latb, 8);
        out->macro_id = r0.z;
        out->g = int64_t(uint64_t(uint32_t(r1.x)) | (uint64_t(uint32_t(r1.y)) << 32));
        out->micro_id = r1.z;
        out->l = int64_t(uint64_t(uint32_t(r2.x)) | (uint64_t(uint32_t(r2.y)) << 32));
        out->wave = r2.z;
        out->flags = uint32_t(r3.x);
        out->comparisons = r3.y;
        float tail;
        std::memcpy(&tail, &r3.z, 4);
        out->tail_frac = double(tail);
        return WT_OK;
    }
    ce = launch_one(e->dev(), M, N, K, e->one_d, seq, e->one_st);
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_tune_one");
    // poll the mailbox; every 4096 spins ask the stream whether the kernel
    // ended without writing (a fault), so a broken launch cannot hang here
    for (uint32_t spin = 1; e->one_h->seq != seq; ++spin) {
        if ((spin & 4095u) == 0) {
            ce = cudaStreamQuery(e->one_st);
            if (ce == cudaSuccess && e->one_h->seq != seq) return set_err(WT_CUDA_ERROR, "wt_tune_one: no result");
            if (ce != cudaSuccess && ce != cudaErrorNotReady) return cuda_err(ce, "wt_tune_one");
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const OneOut& o = *e->one_h;
    out->latency_us = o.lat;
    out->g = o.g;
    out->l = o.l;
    out->tail_frac = o.tail;
    out->macro_id = o.macro;
    out->micro_id = o.micro;
    out->wave = o.wave;
    out->flags = o.flags;
    out->comparisons = o.comps;
    return WT_OK;
}

wt_status wt_engine_set_resident(wt_engine* e, int32_t idle_us) {
    if (!e) return set_err(WT_INVALID_ARGUMENT, "null engine");
    if (idle_us < 0) return set_err(WT_INVALID_ARGUMENT, "negative idle time");
    std::lock_guard<std::mutex> lk(e->one_mu);
    DeviceGuard guard(e->device);
    if (idle_us == 0) stop_server(e);
    e->idle_ns = int64_t(idle_us) * 1000;
    return WT_OK;
}

// ------------------------------------------------------- ablation baselines
struct wt_baseline {
    int device = 0;
    const wt_engine* eng = nullptr;
    BaseImage img{};
    void* mem = nullptr;
};

wt_status wt_baseline_create(const wt_engine* e, int device, int32_t kind, const int32_t* macro_id,
                             const int64_t* anchor_l, const double* values, int64_t n, wt_baseline** out) {
    if (!out) return set_err(WT_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (kind != WT_BASELINE_STEP && kind != WT_BASELINE_LINEAR) return set_err(WT_INVALID_ARGUMENT, "unknown baseline kind");
    if (n < 0 || (n > 0 && (!macro_id || !values || (kind == WT_BASELINE_STEP && !anchor_l))))
        return set_err(WT_INVALID_ARGUMENT, "null or negative baseline arrays");
    for (int64_t i = 1; i < n; ++i) {
        const bool asc = kind == WT_BASELINE_STEP
                             ? (macro_id[i - 1] < macro_id[i] ||
                                (macro_id[i - 1] == macro_id[i] && anchor_l[i - 1] < anchor_l[i]))
                             : macro_id[i - 1] < macro_id[i];
        if (!asc) return set_err(WT_INVALID_ARGUMENT, "baseline entries must be strictly ascending");
    }
    if (e) device = e->device;
    std::vector<int32_t> cfg;  // config macro ids, ascending
    if (e) cfg = e->host.macro_id;
    else
        for (int64_t i = 0; i < n; ++i)
            if (cfg.empty() || cfg.back() != macro_id[i]) cfg.push_back(macro_id[i]);
    const int C = int(cfg.size());
    std::vector<int32_t> has(C, 0), off(C + 1, 0);
    std::vector<double> theta(size_t(C) * 4, 0.0), tw;
    std::vector<int64_t> al;
    int missing = 0;
    int64_t i = 0;
    for (int c = 0; c < C; ++c) {
        while (i < n && macro_id[i] < cfg[c]) ++i;
        off[c] = int32_t(al.size());
        int64_t j = i;
        while (j < n && macro_id[j] == cfg[c]) {
            if (kind == WT_BASELINE_STEP) {
                al.push_back(anchor_l[j]);
                tw.push_back(values[j]);
            } else {
                for (int q = 0; q < 4; ++q) theta[size_t(c) * 4 + q] = values[4 * j + q];
            }
            ++j;
        }
        has[c] = j > i ? 1 : 0;
        if (!has[c]) missing = 1;
        i = j;
    }
    off[C] = int32_t(al.size());
    DeviceGuard guard(device);
    Arena ar;
    const size_t o_mac = ar.take(size_t(C) * 4), o_has = ar.take(size_t(C) * 4), o_th = ar.take(theta.size() * 8),
                 o_off = ar.take(off.size() * 4), o_al = ar.take(al.size() * 8), o_tw = ar.take(tw.size() * 8);
    auto* b = new wt_baseline;
    b->device = device;
    b->eng = e;
    cudaError_t ce = cudaMalloc(&b->mem, std::max<size_t>(ar.used, 256));
    if (ce != cudaSuccess) {
        delete b;
        return cuda_err(ce, "wt_baseline_create");
    }
    char* base = static_cast<char*>(b->mem);
    auto up = [&](size_t o, const void* src, size_t bytes) {
        if (bytes && ce == cudaSuccess) ce = cudaMemcpy(base + o, src, bytes, cudaMemcpyHostToDevice);
    };
    up(o_mac, cfg.data(), size_t(C) * 4);
    up(o_has, has.data(), size_t(C) * 4);
    up(o_th, theta.data(), theta.size() * 8);
    up(o_off, off.data(), off.size() * 4);
    up(o_al, al.data(), al.size() * 8);
    up(o_tw, tw.data(), tw.size() * 8);
    if (ce != cudaSuccess) {
        cudaFree(b->mem);
        delete b;
        return cuda_err(ce, "wt_baseline_create upload");
    }
    BaseImage& im = b->img;
    im.kind = kind;
    im.C = C;
    im.missing = e ? missing : 0;
    im.S = e ? e->host.S : 0;
    im.macro = reinterpret_cast<const int32_t*>(base + o_mac);
    im.has = reinterpret_cast<const int32_t*>(base + o_has);
    im.theta = reinterpret_cast<const double4*>(base + o_th);
    im.off = reinterpret_cast<const int32_t*>(base + o_off);
    im.al = reinterpret_cast<const int64_t*>(base + o_al);
    im.tw = reinterpret_cast<const double*>(base + o_tw);
    *out = b;
    return WT_OK;
}

wt_status wt_baseline_destroy(wt_baseline* b) {
    if (!b) return WT_OK;
    DeviceGuard guard(b->device);
    cudaFree(b->mem);
    delete b;
    return WT_OK;
}

wt_status wt_baseline_tune_batch(const wt_engine* e, const wt_baseline* b, const int32_t* M, const int32_t* N,
                                 const int32_t* K, int64_t n, const wt_decisions* out, void* stream) {
    if (!e || !b) return set_err(WT_INVALID_ARGUMENT, "null engine or baseline");
    if (b->eng != e) return set_err(WT_INVALID_ARGUMENT, "baseline was not created for this engine");
    if (n < 0) return set_err(WT_INVALID_ARGUMENT, "negative batch size");
    wt_status st = check_out(out);
    if (st) return st;
    if (out->topk) return set_err(WT_UNSUPPORTED, "topk is not available for baseline queries");
    if (n == 0) return WT_OK;
    if (e->host.family == WT_FAMILY_GROUPED_GEMM)
        return set_err(WT_INVALID_ARGUMENT, "dense_gemm workload needs gemm tiles");
    DeviceGuard guard(e->device);
    EvalArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.n = n;
    a.out = to_out(out);
    const cudaError_t ce = launch_btune(e->dev(), b->img, a, static_cast<cudaStream_t>(stream));
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_baseline_tune_batch");
    return WT_OK;
}

wt_status wt_baseline_predict_batch(const wt_baseline* b, const int32_t* macro_id, const int64_t* g,
                                    const int64_t* l, int64_t n, const wt_hw* hw, double* latency, int32_t* status,
                                    void* stream) {
    if (!b || !hw) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (n < 0) return set_err(WT_INVALID_ARGUMENT, "negative batch size");
    if (n == 0) return WT_OK;
    if (!macro_id || !g || !l || !latency || !status) return set_err(WT_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(b->device);
    BaseImage im = b->img;
    const int64_t S = int64_t(hw->n_sm) * hw->blocks_per_sm;
    im.S = (hw->n_sm < 1 || hw->blocks_per_sm < 1 || S > INT32_MAX) ? 0 : int32_t(S);
    BPredictArgs a{macro_id, g, l, n, latency, status};
    const cudaError_t ce = launch_bpredict(im, a, static_cast<cudaStream_t>(stream));
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_baseline_predict_batch");
    return WT_OK;
}

wt_status wt_tune_grouped_batch(const wt_engine* e, const int64_t* row_off, const int32_t* rows,
                                const int32_t* N, const int32_t* K, int64_t n,
                                const wt_decisions* out, void* stream) {
    if (!e) return set_err(WT_INVALID_ARGUMENT, "null engine");
    wt_status st = check_out(out);
    if (st) return st;
    if (out->topk) return set_err(WT_UNSUPPORTED, "topk is not available for grouped queries");
    if (n <= 0) return n == 0 ? WT_OK : set_err(WT_INVALID_ARGUMENT, "negative batch size");
    if (e->host.family == WT_FAMILY_FLASH_ATTENTION)
        return set_err(WT_INVALID_ARGUMENT, "grouped_gemm workload needs gemm tiles");
    DeviceGuard guard(e->device);
    GroupedArgs a{};
    a.row_off = row_off;
    a.rows = rows;
    a.N = N;
    a.K = K;
    a.n = n;
    a.out = to_out(out);
    const int grid = int(std::min<int64_t>((n * 32 + 255) / 256, int64_t(sm_count(e->device)) * 8));
    cudaError_t ce = launch_grouped(e->dev(), a, grid, static_cast<cudaStream_t>(stream));
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_tune_grouped_batch");
    return WT_OK;
}

wt_status wt_predict_batch(const wt_engine* e, const int32_t* config, const int64_t* g,
                           const int64_t* l, int64_t n, double* latency_us, int32_t* wave,
                           int32_t* extrapolated, int32_t* used_w, int32_t* status, void* stream) {
    if (!e || !latency_us) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return WT_OK;
    DeviceGuard guard(e->device);
    PredictArgs a{config, g, l, n, latency_us, wave, extrapolated, used_w, status};
    cudaError_t ce = launch_predict(e->dev(), a, static_cast<cudaStream_t>(stream));
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_predict_batch");
    return WT_OK;
}

wt_status wt_explain(const wt_engine* e, int64_t M, int64_t N, int64_t K, int64_t* g, int64_t* l,
                     int32_t* wave, int32_t* used_w, double* latency_us, int32_t* status,
                     void* stream) {
    if (!e || !g || !l || !wave || !used_w || !latency_us || !status)
        return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        return set_err(WT_UNSUPPORTED, "dims above 2^31-1 are outside the device path's range");
    DeviceGuard guard(e->device);
    ExplainArgs a{M, N, K, g, l, wave, used_w, latency_us, status};
    cudaError_t ce = launch_explain(e->dev(), a, static_cast<cudaStream_t>(stream));
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_explain");
    return WT_OK;
}

wt_status wt_nearest_anchor_batch(const int64_t* anchors, int32_t n_anchors, const int64_t* l,
                                  int64_t n, int64_t* out, int32_t* comparisons, void* stream) {
    if (n_anchors <= 0) return set_err(WT_INVALID_ARGUMENT, "nearest_anchor: empty anchor list");
    if (n <= 0) return WT_OK;
    NearestArgs a{anchors, n_anchors, l, n, out, comparisons};
    cudaError_t ce = launch_nearest(a, static_cast<cudaStream_t>(stream));
    g_launches++;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_nearest_anchor_batch");
    return WT_OK;
}

// ------------------------------------------------------------------ grid
namespace {
// pooled: storage from the library pool and every upload queued on `st` (no
// host sync); otherwise cudaMalloc (IPC-exportable) and synchronous uploads.
wt_status grid_create_impl(const wt_engine* e, const wt_grid_desc* desc, bool pooled, cudaStream_t st,
                           wt_grid** out) {
    if (!e || !desc || !out) return set_err(WT_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (desc->n_pairs <= 0) return set_err(WT_INVALID_ARGUMENT, "grid needs at least one (N, K) pair");
    if (desc->m_lo < 1 || desc->m_hi < desc->m_lo)
        return set_err(WT_INVALID_ARGUMENT, "grid M range must satisfy 1 <= m_lo <= m_hi");
    if (desc->topk < 0 || desc->topk > 8) return set_err(WT_UNSUPPORTED, "topk must be in [0, 8]");
    if (e->host.family == WT_FAMILY_GROUPED_GEMM)
        return set_err(WT_UNSUPPORTED, "decision grids cover dense / attention shapes");
    for (int32_t p = 0; p < desc->n_pairs; ++p)
        if (desc->N[p] < 1 || desc->K[p] < 1)
            return set_err(WT_INVALID_ARGUMENT, "dense_gemm dims must be >= 1");
    DeviceGuard guard(e->device);
    auto* g = new wt_grid;
    g->eng = e;
    g->n_pairs = desc->n_pairs;
    g->m_lo = desc->m_lo;
    g->m_hi = desc->m_hi;
    g->mcount = int64_t(desc->m_hi) - desc->m_lo + 1;
    g->n_entries = g->mcount * desc->n_pairs;
    g->topk = desc->topk;
    // narrow (32-bit g) sweep whenever every g fits
    uint64_t nt_max = 0;
    for (int32_t p = 0; p < desc->n_pairs; ++p)
        nt_max = std::max<uint64_t>(nt_max, (uint64_t(desc->N[p]) + e->host.tn_min - 1) / e->host.tn_min);
    const uint64_t mt_max = (uint64_t(desc->m_hi) + e->host.tm_min - 1) / e->host.tm_min;
    g->wide = mt_max * nt_max >= (uint64_t(1) << 32);
    // sorted unique (N, K) keys for the gather; first occurrence wins
    std::vector<std::pair<uint64_t, int32_t>> keys;
    for (int32_t p = 0; p < desc->n_pairs; ++p)
        keys.push_back({(uint64_t(uint32_t(desc->N[p])) << 32) | uint32_t(desc->K[p]), p});
    std::stable_sort(keys.begin(), keys.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    keys.erase(std::unique(keys.begin(), keys.end(),
                           [](const auto& a, const auto& b) { return a.first == b.first; }),
               keys.end());
    g->n_keys = int32_t(keys.size());
    Arena ar;
    const size_t o_n = ar.take(size_t(g->n_pairs) * 4), o_k = ar.take(size_t(g->n_pairs) * 4),
                 o_keys = ar.take(keys.size() * 8), o_pid = ar.take(keys.size() * 4),
                 o_ent = ar.take(size_t(g->n_entries) * sizeof(wt_grid_entry)),
                 o_tkm = ar.take(size_t(g->n_entries) * g->topk * 4),
                 o_tkl = ar.take(size_t(g->n_entries) * g->topk * 8);
    // hash table: load factor <= 1/2, linear probing, inserted in key order
    // (deterministic); only for tables that fit shared memory comfortably
    std::vector<int4> htab;
    if (keys.size() <= 2048) {
        int bits = 3;
        while ((size_t(1) << bits) < 2 * keys.size()) ++bits;
        htab.assign(size_t(1) << bits, make_int4(0, 0, -1, 0));
        for (auto& k : keys) {
            const uint32_t N = uint32_t(k.first >> 32), K = uint32_t(k.first);
            uint32_t h = pair_slot(N, K, bits);
            while (htab[h].z >= 0) h = (h + 1) & ((1u << bits) - 1u);
            htab[h] = make_int4(int(N), int(K), k.second, 0);
        }
        g->hbits = bits;
    }
    const size_t o_hash = ar.take(htab.size() * sizeof(int4));
    // M intervals: breakpoints at k * t_m + 1 for every distinct t_m; used
    // when they cut the work by at least 4x
    {
        const int64_t mc = g->mcount;
        std::vector<uint8_t> brk;
        if (mc >= 64 && mc <= (int64_t(1) << 26) && !e->host.tm_vals.empty()) {
            brk.assign(size_t(mc), 0);
            brk[0] = 1;
            for (int32_t tm : e->host.tm_vals) {
                // M = k * tm + 1 >= m_lo + 1
                int64_t k = (int64_t(desc->m_lo) + tm - 1) / tm;
                for (int64_t M = k * tm + 1; M <= desc->m_hi; M += tm) brk[size_t(M - desc->m_lo)] = 1;
            }
            int64_t nb = 0;
            for (uint8_t b : brk) nb += b;
            if (nb * 4 <= mc && nb < INT32_MAX) {
                g->h_mrep.reserve(size_t(nb));
                for (int64_t i = 0; i < mc; ++i)
                    if (brk[size_t(i)]) g->h_mrep.push_back(int32_t(desc->m_lo + i));
                g->nrep = int32_t(nb);
            }
        }
    }
    const size_t o_mrep = ar.take(size_t(g->nrep) * 4);
    // run index storage (worst case: every entry its own run) when its block
    // table alone leaves room in the shared-memory budget
    static const int runs_kb = [] {
        const char* v = std::getenv("WT_GATHER_RUNS_KB");
        return v ? std::atoi(v) : 40;
    }();
    const int64_t nblk = (g->mcount + (1 << kRunBlkShift) - 1) >> kRunBlkShift;
    const bool want_runs = !htab.empty() && runs_kb > 0 && g->n_entries < int64_t(0xfffffff0u) &&
                           int64_t(g->n_pairs) * nblk * 16 <= int64_t(runs_kb) * 1024;
    const size_t o_rhdr = ar.take(want_runs ? 16 : 0),
                 o_rbidx = ar.take(want_runs ? size_t(g->n_pairs) * nblk * 16 : 0),
                 o_rkey = ar.take(want_runs ? size_t(g->n_entries + 1) * 4 : 0),
                 o_rval = ar.take(want_runs ? size_t(g->n_entries) * 16 : 0);
    cudaError_t ce = pooled ? cudaMallocFromPoolAsync(&g->mem, ar.used, lib_pool(e->device), st)
                            : cudaMalloc(&g->mem, ar.used);
    if (ce != cudaSuccess) {
        delete g;
        return cuda_err(ce, "wt_grid_create: cudaMalloc");
    }
    g->pooled = pooled;
    // uploads: synchronous, or queued on st (pageable sources are staged by
    // the driver when the call returns, so the host vectors may go)
    auto up = [&](void* dst, const void* src, size_t n) {
        return pooled ? cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st)
                      : cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    };
    char* base = static_cast<char*>(g->mem);
    g->dN = reinterpret_cast<int32_t*>(base + o_n);
    g->dK = reinterpret_cast<int32_t*>(base + o_k);
    g->dkeys = reinterpret_cast<uint64_t*>(base + o_keys);
    g->dpid = reinterpret_cast<int32_t*>(base + o_pid);
    g->entries = reinterpret_cast<wt_grid_entry*>(base + o_ent);
    g->tk_macro = g->topk ? reinterpret_cast<int32_t*>(base + o_tkm) : nullptr;
    g->tk_lat = g->topk ? reinterpret_cast<double*>(base + o_tkl) : nullptr;
    g->dhash = htab.empty() ? nullptr : reinterpret_cast<int4*>(base + o_hash);
    if (g->nrep) {
        g->d_mrep = reinterpret_cast<int32_t*>(base + o_mrep);
        up(g->d_mrep, g->h_mrep.data(), g->h_mrep.size() * 4);
    }
    if (g->dhash) up(g->dhash, htab.data(), htab.size() * sizeof(int4));
    if (want_runs) {
        g->runs.hdr = reinterpret_cast<int32_t*>(base + o_rhdr);
        g->runs.bhead = reinterpret_cast<int4*>(base + o_rbidx);
        g->runs.rkey = reinterpret_cast<uint32_t*>(base + o_rkey);
        g->runs.rval = reinterpret_cast<int4*>(base + o_rval);
        g->runs.nblk = int32_t(nblk);
        g->runs.nbtot = int32_t(int64_t(g->n_pairs) * nblk);
        g->runs.budget = runs_kb * 1024;
        if (pooled) cudaMemsetAsync(g->runs.hdr, 0, 16, st);
        else cudaMemset(g->runs.hdr, 0, 16);
    }
    std::vector<uint64_t> kk;
    std::vector<int32_t> pid;
    for (auto& k : keys) {
        kk.push_back(k.first);
        pid.push_back(k.second);
    }
    up(g->dN, desc->N, size_t(g->n_pairs) * 4);
    up(g->dK, desc->K, size_t(g->n_pairs) * 4);
    up(g->dkeys, kk.data(), kk.size() * 8);
    ce = up(g->dpid, pid.data(), pid.size() * 4);
    if (ce != cudaSuccess) {
        if (pooled) {
            cudaFreeAsync(g->mem, st);
            cudaStreamSynchronize(st);
        } else {
            cudaFree(g->mem);
        }
        delete g;
        return cuda_err(ce, "wt_grid_create: upload");
    }
    *out = g;
    return WT_OK;
}
}  // namespace

wt_status wt_grid_create(const wt_engine* e, const wt_grid_desc* desc, wt_grid** out) {
    NvtxRange nvtx_("wt_grid_create");
    return grid_create_impl(e, desc, false, nullptr, out);
}

wt_status wt_grid_create_async(const wt_engine* e, const wt_grid_desc* desc, void* stream, wt_grid** out) {
    NvtxRange nvtx_("wt_grid_create_async");
    return grid_create_impl(e, desc, true, static_cast<cudaStream_t>(stream), out);
}

wt_status wt_grid_destroy(wt_grid* g) {
    if (!g) return WT_OK;
    DeviceGuard guard(g->eng->device);
    if (g->pooled) {
        // pool memory: released after every stream's use of the grid
        cudaDeviceSynchronize();
        cudaFreeAsync(g->mem, nullptr);
        cudaStreamSynchronize(nullptr);
    } else {
        cudaFree(g->mem);
    }
    delete g;
    return WT_OK;
}

int64_t wt_grid_representatives(const wt_grid* g) {
    if (!g) return 0;
    return g->nrep > 0 ? int64_t(g->nrep) * g->n_pairs : g->n_entries;
}

wt_status wt_grid_storage(const wt_grid* g, wt_grid_entry** entries, int64_t* n_entries,
                          int32_t** topk_macro, double** topk_latency) {
    if (!g) return set_err(WT_INVALID_ARGUMENT, "null grid");
    // whoever takes the raw storage may write it: the run index is stale
    // until the next full sweep / wt_grid_finalize (gathers read L2 meanwhile);
    // host-side generation bump, no device write that could race a build
    g->invalidate_runs();
    if (entries) *entries = g->entries;
    if (n_entries) *n_entries = g->n_entries;
    if (topk_macro) *topk_macro = g->tk_macro;
    if (topk_latency) *topk_latency = g->tk_lat;
    return WT_OK;
}

namespace {
bool sweep_dedup() {
    static const bool d = [] {
        const char* v = std::getenv("WT_SWEEP_DEDUP");
        return !v || std::atoi(v) != 0;
    }();
    return d;
}

// The representative sweep of [a.begin, a.end): one M per interval of
// constant ceil(M / t_m) (k_sweep_w, or k_sweep2 with WT_SWEEP_W=0) into a
// scratch list, then k_expand copies every interval's entry over its M
// values in the range, into each destination grid.
cudaError_t rep_sweep(const wt_engine* e, const wt_grid* g, const SweepArgs& a, const ExpandDst& dst,
                      cudaStream_t s) {
    static const int sweep_w = [] {
        const char* v = std::getenv("WT_SWEEP_W");
        return v ? std::atoi(v) : 1;
    }();
    auto rep_of = [&](int64_t flat) {
        const int64_t p = flat / g->mcount;
        const int32_t M = int32_t(g->m_lo + (flat - p * g->mcount));
        const int64_t i = int64_t(std::upper_bound(g->h_mrep.begin(), g->h_mrep.end(), M) - g->h_mrep.begin()) - 1;
        return p * g->nrep + i;
    };
    const int64_t rb = rep_of(a.begin), re = rep_of(a.end - 1) + 1;
    SweepArgs ra = a;
    ra.mcount = g->nrep;
    ra.mrep = g->d_mrep;
    ra.begin = rb;
    ra.end = re;
    ra.ndst = 0;
    const size_t eb = (size_t(re - rb) * sizeof(wt_grid_entry) + 255) & ~size_t(255);
    const size_t sb = sweep_w ? 0 : sweep2_scratch_bytes(e->dev(), ra);
    void* scratch = nullptr;
    cudaError_t ce = cudaMallocFromPoolAsync(&scratch, eb + sb, lib_pool(e->device), s);
    if (ce != cudaSuccess) return ce;
    wt_grid_entry* rep = static_cast<wt_grid_entry*>(scratch);
    // the sweep writes representative r at ra.entries + r: offset the list by -rb
    ra.entries = rep - rb;
    ce = sweep_w ? launch_sweep_w(e->dev(), ra, s)
                 : launch_sweep2(e->dev(), ra, g->wide, sb ? static_cast<char*>(scratch) + eb : nullptr, s);
    if (ce == cudaSuccess)
        ce = launch_expand(dst, rep, rb, re, a.begin, a.end, g->m_lo, g->mcount, g->d_mrep, g->nrep, s);
    cudaFreeAsync(scratch, s);
    g_launches += sb ? 3 : 2;
    return ce;
}
}  // namespace

wt_status wt_sweep(const wt_engine* e, wt_grid* g, int64_t begin, int64_t end, void* stream) {
    NvtxRange nvtx_("wt_sweep");
    if (!e || !g) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (g->eng != e) return set_err(WT_INVALID_ARGUMENT, "grid was created for another engine");
    if (begin < 0 || end > g->n_entries || begin > end)
        return set_err(WT_OUT_OF_RANGE, "sweep range outside the grid");
    if (begin == end) return WT_OK;
    DeviceGuard guard(e->device);
    SweepArgs a{};
    a.N = g->dN;
    a.K = g->dK;
    a.m_lo = g->m_lo;
    a.mcount = g->mcount;
    a.begin = begin;
    a.end = end;
    {  // configs per shared-memory chunk of the top-k sweep
        const size_t per_cfg = size_t(e->host.R) * (32 + (e->dev().special ? 4 : 0)) + 24;
        a.chunk = int(std::max<size_t>(1, std::min<size_t>(e->host.C, 49152 / per_cfg)));
    }
    a.entries = g->entries;
    a.topk = g->topk;
    a.topk_macro = g->tk_macro;
    a.topk_lat = g->tk_lat;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t ce;
    const bool dedup = sweep_dedup();
    if (g->topk > 0) {
        ce = launch_sweep(e->dev(), a, g->wide, s);
        g_launches++;
    } else if (dedup && g->nrep > 0) {
        ExpandDst dst{};
        dst.d[0] = g->entries;
        dst.n = 1;
        ce = rep_sweep(e, g, a, dst, s);  // counts its launches
    } else {
        void* scratch = nullptr;
        const size_t sb = sweep2_scratch_bytes(e->dev(), a);
        if (sb) {
            ce = cudaMallocFromPoolAsync(&scratch, sb, lib_pool(e->device), s);
            if (ce != cudaSuccess) return cuda_err(ce, "wt_sweep: scratch");
        }
        ce = launch_sweep2(e->dev(), a, g->wide, scratch, s);
        if (scratch) cudaFreeAsync(scratch, s);
        g_launches += sb ? 2 : 1;  // (+ split merge)
    }
    if (ce != cudaSuccess) return cuda_err(ce, "wt_sweep");
    // the run index follows the entries: rebuilt after a full sweep,
    // invalidated by a partial one (wt_grid_finalize rebuilds it)
    if (g->runs.budget > 0) {
        if (begin == 0 && end == g->n_entries) return wt_grid_finalize(e, g, stream);
        g->invalidate_runs();
    }
    return WT_OK;
}

wt_status wt_sweep_to(const wt_engine* e, wt_grid* g, int64_t begin, int64_t end, wt_grid_entry* const* dests,
                      int n_dests, void* stream) {
    NvtxRange nvtx_("wt_sweep_to");
    if (!e || !g || !dests) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (g->eng != e) return set_err(WT_INVALID_ARGUMENT, "grid was created for another engine");
    if (n_dests < 1 || n_dests > 8) return set_err(WT_INVALID_ARGUMENT, "n_dests must be in [1, 8]");
    if (g->topk > 0) return set_err(WT_UNSUPPORTED, "fused sweeps cover grids without top-k");
    if (begin < 0 || end > g->n_entries || begin > end)
        return set_err(WT_OUT_OF_RANGE, "sweep range outside the grid");
    for (int d = 0; d < n_dests; ++d)
        if (!dests[d]) return set_err(WT_INVALID_ARGUMENT, "null destination grid");
    if (begin == end) return WT_OK;
    DeviceGuard guard(e->device);
    SweepArgs a{};
    a.N = g->dN;
    a.K = g->dK;
    a.m_lo = g->m_lo;
    a.mcount = g->mcount;
    a.begin = begin;
    a.end = end;
    a.entries = g->entries;
    for (int d = 0; d < n_dests; ++d) a.dst[d] = dests[d];
    a.ndst = n_dests;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t ce = cudaSuccess;
    if (sweep_dedup() && g->nrep > 0) {
        // representative sweep; the expansion stores into every destination
        ExpandDst dst{};
        for (int d = 0; d < n_dests; ++d) dst.d[d] = dests[d];
        dst.n = n_dests;
        ce = rep_sweep(e, g, a, dst, s);
    } else {
        void* scratch = nullptr;
        const size_t sb = sweep2_scratch_bytes(e->dev(), a);
        if (sb) ce = cudaMallocFromPoolAsync(&scratch, sb, lib_pool(e->device), s);
        if (ce != cudaSuccess) return cuda_err(ce, "wt_sweep_to: scratch");
        ce = launch_sweep2(e->dev(), a, g->wide, scratch, s);
        if (scratch) cudaFreeAsync(scratch, s);
        g_launches += sb ? 2 : 1;
    }
    if (ce != cudaSuccess) return cuda_err(ce, "wt_sweep_to");
    // this grid's own run index is stale until the caller finalizes it
    g->invalidate_runs();
    return WT_OK;
}

wt_status wt_grid_ipc_handle(const wt_grid* g, void* handle, int64_t* offset) {
    if (!g || !handle || !offset) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (g->pooled) return set_err(WT_UNSUPPORTED, "grid storage from wt_grid_create_async is not IPC-exportable");
    DeviceGuard guard(g->eng->device);
    cudaIpcMemHandle_t h;
    const cudaError_t ce = cudaIpcGetMemHandle(&h, g->mem);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_grid_ipc_handle");
    std::memcpy(handle, &h, sizeof(h));
    *offset = reinterpret_cast<char*>(g->entries) - static_cast<char*>(g->mem);
    return WT_OK;
}

wt_status wt_ipc_open(const void* handle, int64_t offset, int device, wt_grid_entry** entries, void** base) {
    if (!handle || !entries || !base) return set_err(WT_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    const cudaError_t ce = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_ipc_open");
    *base = p;
    *entries = reinterpret_cast<wt_grid_entry*>(static_cast<char*>(p) + offset);
    return WT_OK;
}

wt_status wt_ipc_close(void* base) {
    if (!base) return WT_OK;
    const cudaError_t ce = cudaIpcCloseMemHandle(base);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_ipc_close");
    return WT_OK;
}

wt_status wt_grid_finalize(const wt_engine* e, wt_grid* g, void* stream) {
    NvtxRange nvtx_("wt_grid_finalize");
    if (!e || !g) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (g->eng != e) return set_err(WT_INVALID_ARGUMENT, "grid was created for another engine");
    if (g->runs.budget <= 0) return WT_OK;
    DeviceGuard guard(e->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void* temp = nullptr;
    cudaError_t ce = cudaMallocFromPoolAsync(&temp, runs_temp_bytes(g->n_entries), lib_pool(e->device), s);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_grid_finalize: scratch");
    ce = launch_runs_build(g->entries, g->n_entries, g->mcount, g->runs_now(), temp, s);
    cudaFreeAsync(temp, s);
    g_launches += 3 + scan_launches(g->n_entries);  // flags, scan, scatter, heads
    if (ce != cudaSuccess) return cuda_err(ce, "wt_grid_finalize");
    return WT_OK;
}

}  // extern "C"

// [count | idx (n) | M (n) | N (n) | K (n)] -- the off-grid compaction list
static size_t gather_scratch_bytes(int64_t n) {
    return size_t(n + 2) * sizeof(int64_t) + 3 * size_t(n + 4) * sizeof(int32_t);
}

static bool gather_needs_eval3(const wt_grid* g, const wt_decisions* out) {
    return g->topk == 0 && out->topk == 0 && eval_mode() == 3;
}

// The gather + off-grid evaluation of one batch.  Scratch buffers are taken
// from the library pool unless the caller supplies them (the host pipeline
// keeps one set per slot: pool reuse across its streams would otherwise add
// cross-stream waits).
static wt_status gather_impl(const wt_engine* e, const wt_grid* g, const int32_t* M, const int32_t* N,
                             const int32_t* K, int64_t n, const wt_decisions* out, cudaStream_t s,
                             void* scratch_in, void* escratch_in) {
    void* scratch = scratch_in;
    cudaError_t ce = cudaSuccess;
    if (!scratch) ce = cudaMallocFromPoolAsync(&scratch, gather_scratch_bytes(n), lib_pool(e->device), s);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_gather_batch: scratch");
    int64_t* count = static_cast<int64_t*>(scratch);
    int64_t* idx = count + 2;
    int32_t* offM = reinterpret_cast<int32_t*>(idx + n);
    int32_t* offN = offM + (n + 4);
    int32_t* offK = offN + (n + 4);
    cudaMemsetAsync(count, 0, sizeof(int64_t), s);
    GatherArgs a{};
    a.pair_keys = g->dkeys;
    a.pair_ids = g->dpid;
    a.n_pairs = g->n_keys;
    a.m_lo = g->m_lo;
    a.m_hi = g->m_hi;
    a.mcount = g->mcount;
    a.entries = g->entries;
    a.topk_macro = g->tk_macro;
    a.topk_lat = g->tk_lat;
    a.M = M;
    a.N = N;
    a.K = K;
    a.n = n;
    a.out = to_out(out);
    a.off_count = count;
    a.off_idx = idx;
    a.off_M = offM;
    a.off_N = offN;
    a.off_K = offK;
    a.htab = g->dhash;
    a.hbits = g->hbits;
    a.runs = g->runs_now();
    // row-grouped evaluation of the off-grid list: keys counted while compacting
    void* escratch = escratch_in;
    if (gather_needs_eval3(g, out)) {
        if (!escratch) ce = cudaMallocFromPoolAsync(&escratch, eval3_scratch_bytes(n), lib_pool(e->device), s);
        if (ce != cudaSuccess) {
            if (!scratch_in) cudaFreeAsync(scratch, s);
            return cuda_err(ce, "wt_gather_batch: eval scratch");
        }
        const Eval3Bufs b = eval3_bufs(escratch, n);
        cudaMemsetAsync(b.hist, 0, b.hist_bytes, s);
        a.off_key = b.keys;
        a.key_hist = b.hist;
        a.key_bits = b.key_bits;
        a.key_mode = b.key_mode;
    }
    const int grid = int(std::min<int64_t>((n + kGatherThreads - 1) / kGatherThreads,
                                           int64_t(sm_count(e->device)) * 8));
    timing_mark(0, s);
    ce = launch_gather(e->dev(), a, grid, s);
    timing_mark(1, s);
    timing_mark(2, s);
    g_launches++;
    if (ce == cudaSuccess) {
        EvalArgs ea{};
        ea.M = M;
        ea.N = N;
        ea.K = K;
        ea.n = n;
        ea.idx = idx;
        ea.count = count;
        ea.chunk = e->eval_chunk;
        ea.out = to_out(out);
        if (g->topk == 0) ea.out.topk = 0;
        if (ea.out.topk == 0) {  // list kernel reads the compacted dims contiguously
            ea.M = offM;
            ea.N = offN;
            ea.K = offK;
            ea.inputs_compact = 1;
        }
        if (ea.out.topk > 0) {
            ce = launch_eval(e->dev(), ea, e->eval_grid, s);
            g_launches++;
        } else {
            ce = run_list_eval(e, ea, s, escratch);
        }
    }
    timing_mark(3, s);
    if (!scratch_in) cudaFreeAsync(scratch, s);
    if (escratch && !escratch_in) cudaFreeAsync(escratch, s);
    if (ce != cudaSuccess) return cuda_err(ce, "wt_gather_batch");
    return WT_OK;
}

extern "C" {

wt_status wt_gather_batch(const wt_engine* e, const wt_grid* g, const int32_t* M, const int32_t* N,
                          const int32_t* K, int64_t n, const wt_decisions* out, void* stream) {
    NvtxRange nvtx_("wt_gather_batch");
    if (!e || !g) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (g->eng != e) return set_err(WT_INVALID_ARGUMENT, "grid was created for another engine");
    wt_status st = check_out(out);
    if (st) return st;
    if (out->topk && out->topk != g->topk)
        return set_err(WT_INVALID_ARGUMENT, "topk must match the grid's topk");
    if (n <= 0) return n == 0 ? WT_OK : set_err(WT_INVALID_ARGUMENT, "negative batch size");
    DeviceGuard guard(e->device);
    // batches beyond 2^28 queries run in stream-ordered slices, bounding the
    // compaction / evaluation scratch (~44 B per query of a slice)
    const int64_t kBatchSlice = batch_slice();
    for (int64_t i = 0; i < n; i += kBatchSlice) {
        const int64_t m = std::min(kBatchSlice, n - i);
        const wt_decisions d = offset_decisions(*out, i);
        const wt_status st2 =
            gather_impl(e, g, M + i, N + i, K + i, m, &d, static_cast<cudaStream_t>(stream), nullptr, nullptr);
        if (st2 != WT_OK) return st2;
    }
    return WT_OK;
}

// i64 queries (wt_wide.cu): narrow -> the int32 path -> wide fix-up, all
// stream-ordered on the caller's stream; scratch from the library pool.
static wt_status i64_batch(const wt_engine* e, const wt_grid* g, const int64_t* M, const int64_t* N,
                           const int64_t* K, int64_t n, const wt_decisions* out, void* stream, const char* what) {
    NvtxRange nvtx_(what);
    if (!e || !M || !N || !K) return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (g && g->eng != e) return set_err(WT_INVALID_ARGUMENT, "grid was created for another engine");
    wt_status st = check_out(out);
    if (st) return st;
    if (out->topk) return set_err(WT_UNSUPPORTED, "top-k is not offered for i64 queries");
    if (n <= 0) return n == 0 ? WT_OK : set_err(WT_INVALID_ARGUMENT, "negative batch size");
    if (!g && e->host.family == WT_FAMILY_GROUPED_GEMM)
        return set_err(WT_INVALID_ARGUMENT, "dense_gemm workload needs gemm tiles");
    DeviceGuard guard(e->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t a4 = (size_t(n) * 4 + 255) & ~size_t(255);
    const size_t bytes = 3 * a4 + size_t(n) * 8 + 256;
    char* p = nullptr;
    cudaError_t ce = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), bytes, lib_pool(e->device), s);
    if (ce != cudaSuccess) return cuda_err(ce, what);
    WideArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.n = n;
    a.M32 = reinterpret_cast<int32_t*>(p);
    a.N32 = reinterpret_cast<int32_t*>(p + a4);
    a.K32 = reinterpret_cast<int32_t*>(p + 2 * a4);
    a.count = reinterpret_cast<unsigned long long*>(p + 3 * a4);
    a.list = reinterpret_cast<int64_t*>(p + 3 * a4 + 256);
    a.out = to_out(out);
    ce = cudaMemsetAsync(a.count, 0, 8, s);
    if (ce == cudaSuccess) ce = launch_narrow(a, s);
    g_launches++;
    if (ce == cudaSuccess) {
        st = g ? wt_gather_batch(e, g, a.M32, a.N32, a.K32, n, out, stream)
               : wt_tune_batch(e, a.M32, a.N32, a.K32, n, out, stream);
        if (st == WT_OK) {
            ce = launch_wide(e->dev(), a, s);
            g_launches++;
        }
    }
    cudaFreeAsync(p, s);
    if (st != WT_OK) return st;
    if (ce != cudaSuccess) return cuda_err(ce, what);
    return WT_OK;
}

wt_status wt_tune_batch_i64(const wt_engine* e, const int64_t* M, const int64_t* N, const int64_t* K, int64_t n,
                            const wt_decisions* out, void* stream) {
    return i64_batch(e, nullptr, M, N, K, n, out, stream, "wt_tune_batch_i64");
}

wt_status wt_gather_batch_i64(const wt_engine* e, const wt_grid* g, const int64_t* M, const int64_t* N,
                              const int64_t* K, int64_t n, const wt_decisions* out, void* stream) {
    if (!g) return set_err(WT_INVALID_ARGUMENT, "null grid");
    return i64_batch(e, g, M, N, K, n, out, stream, "wt_gather_batch_i64");
}

wt_status wt_decide_host_sync(const wt_engine* e, const wt_grid* g, const int32_t* M,
                              const int32_t* N, const int32_t* K, int64_t n, int32_t* macro_id,
                              int32_t* micro_id, double* latency_us, int64_t chunk) {
    return wt_decide_host_stream_sync(e, g, M, N, K, n, macro_id, micro_id, latency_us, chunk, nullptr);
}

wt_status wt_decide_host_stream_sync(const wt_engine* e, const wt_grid* g, const int32_t* M, const int32_t* N,
                                     const int32_t* K, int64_t n, int32_t* macro_id, int32_t* micro_id,
                                     double* latency_us, int64_t chunk, void* stream) {
    NvtxRange nvtx_("wt_decide_host_sync");
    if (!e || !M || !N || !K || !macro_id || !micro_id || !latency_us)
        return set_err(WT_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return n == 0 ? WT_OK : set_err(WT_INVALID_ARGUMENT, "negative batch size");
    if (chunk <= 0) chunk = int64_t(1) << 22;
    chunk = std::min(chunk, n);
    DeviceGuard guard(e->device);
    // 4 slots: the H2D copy of chunk k+1..k+3 never waits behind the D2H of
    // chunk k on the same stream, so both copy engines stay busy
    constexpr int kMaxSlots = 4;
    const int kSlots = int(std::min<int64_t>(kMaxSlots, (n + chunk - 1) / chunk));
    cudaStream_t st[kMaxSlots] = {};
    void* buf[kMaxSlots] = {};
    // per slot: I/O buffers, then the gather's and the evaluation's scratch
    // (owned by the slot for the whole call: no pool traffic between streams)
    wt_decisions probe{};
    const bool ev3 = g && gather_needs_eval3(g, &probe);
    const size_t io = (size_t(chunk) * (8 + 3 * 4 + 4 + 4) + 255) & ~size_t(255);
    const size_t gs = g ? (gather_scratch_bytes(chunk) + 255) & ~size_t(255) : 0;
    const size_t es = ev3 ? eval3_scratch_bytes(chunk) : 0;
    const size_t per = io + gs + es;
    // the internal streams start after everything already queued on the
    // caller's stream (e.g. a sweep / finalize still filling the grid)
    cudaEvent_t after = nullptr;
    cudaError_t ce = cudaEventCreateWithFlags(&after, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventRecord(after, static_cast<cudaStream_t>(stream));
    for (int s = 0; s < kSlots && ce == cudaSuccess; ++s) {
        ce = cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(st[s], after, 0);
        if (ce == cudaSuccess) ce = cudaMallocFromPoolAsync(&buf[s], per, lib_pool(e->device), st[s]);
    }
    wt_status rs = WT_OK;
    for (int64_t i = 0, k = 0; ce == cudaSuccess && rs == WT_OK && i < n; i += chunk, ++k) {
        const int s = int(k % kSlots);
        const int64_t m = std::min(chunk, n - i);
        // doubles first: every sub-array stays naturally aligned for any chunk
        double* dlat = static_cast<double*>(buf[s]);
        int32_t* dM = reinterpret_cast<int32_t*>(dlat + chunk);
        int32_t* dN = dM + chunk;
        int32_t* dK = dN + chunk;
        int32_t* dmac = dK + chunk;
        int32_t* dmic = dmac + chunk;
        cudaMemcpyAsync(dM, M + i, size_t(m) * 4, cudaMemcpyHostToDevice, st[s]);
        cudaMemcpyAsync(dN, N + i, size_t(m) * 4, cudaMemcpyHostToDevice, st[s]);
        cudaMemcpyAsync(dK, K + i, size_t(m) * 4, cudaMemcpyHostToDevice, st[s]);
        wt_decisions d{};
        d.macro_id = dmac;
        d.micro_id = dmic;
        d.latency_us = dlat;
        if (g) {
            char* sb = static_cast<char*>(buf[s]) + io;
            rs = gather_impl(e, g, dM, dN, dK, m, &d, st[s], sb, ev3 ? sb + gs : nullptr);
        } else {
            rs = wt_tune_batch(e, dM, dN, dK, m, &d, st[s]);
        }
        cudaMemcpyAsync(macro_id + i, dmac, size_t(m) * 4, cudaMemcpyDeviceToHost, st[s]);
        cudaMemcpyAsync(micro_id + i, dmic, size_t(m) * 4, cudaMemcpyDeviceToHost, st[s]);
        ce = cudaMemcpyAsync(latency_us + i, dlat, size_t(m) * 8, cudaMemcpyDeviceToHost, st[s]);
    }
    for (int s = 0; s < kSlots; ++s) {
        if (st[s]) {
            cudaError_t e2 = cudaStreamSynchronize(st[s]);
            if (ce == cudaSuccess) ce = e2;
        }
        if (buf[s]) {
            cudaFreeAsync(buf[s], st[s]);
            cudaStreamSynchronize(st[s]);
        }
        if (st[s]) cudaStreamDestroy(st[s]);
    }
    if (after) cudaEventDestroy(after);
    if (rs != WT_OK) return rs;
    if (ce != cudaSuccess) return cuda_err(ce, "wt_decide_host_sync");
    return WT_OK;
}

// K2 entry points live in wt_fit.cu.

}  // extern "C"
