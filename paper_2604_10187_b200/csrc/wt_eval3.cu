// wt_eval3.cu -- list-mode Stage I over a row-grouped query list.
//
// The evaluation of one (query, config) pair needs the config's 32-byte
// coefficient row for the query's wave; FP64 allows ~9 evaluations per clock
// per SM, a 32-byte row load only ~4 unless lanes share it.  Lanes share it
// when the queries of a warp fall in the same wave row for the tile class
// being evaluated, so the list is first grouped by its rows:
//
//   k_ekey     one thread per query: the wave row of every tile class (the
//              rows depend on (t_m, t_n) only), folded into a kEvalKeyBits key
//              = rows of the smallest and the largest class (prefix, so that
//              neighbouring groups are similar) + a hash of all rows; bucket
//              histogram.
//   scan       exclusive sum over the 2^bits buckets (host-known size).
//   k_escatter counting-sort scatter of (query index, M, N, K) into bucket
//              order (order inside a bucket is irrelevant: every query's
//              answer is independent of where it is evaluated).
//   k_eval3    thread = 4 consecutive grouped queries; per tile class the warp
//              checks whether its 128 queries share one row: then each
//              config's row is loaded once (a broadcast, L1-resident) and
//              reused for the 4 queries; otherwise per-query loads.  No shared
//              memory staging, no barriers.
//
// Arithmetic, Stage I order and the epilogue are those of k_eval2
// (wt_decide2.cu): bitwise-identical latencies, strict-< inside a segment
// (ascending macro_id), lexicographic (latency, config index) merge across
// segments = "first minimum in ascending macro_id" (tuner.cpp:135-149).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "wt_decide.h"
#include "wt_device.cuh"

namespace wtb {

namespace {

constexpr int kT3 = 256;
constexpr int kMaxSmemSeg = 256;  // segment headers staged in shared memory up to this count
constexpr double kInf3 = __builtin_huge_val();


}  // namespace

// ------------------------------------------------------------------ keys
__global__ void k_ekey(DevImage im, EvalArgs a, int bits, int mode, uint32_t* keys, uint32_t* hist) {
    const int64_t n = a.count ? *a.count : a.n;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t src = a.inputs_compact ? i : (a.idx ? a.idx[i] : i);
        const uint32_t key = eval_key(im, a.M[src], a.N[src], a.K[src], bits, i, mode);
        keys[i] = key;
        atomicAdd(hist + key, 1u);
    }
}

// Counting-sort scatter with CTA-level aggregation: a chunk of 2048 list
// slots is ranked per key in a shared-memory hash table, then one global
// atomicAdd per (chunk, key) reserves the chunk's positions -- large groups
// cost one global atomic per chunk instead of one per query.
constexpr int kScPer = 8;       // slots per thread
constexpr int kScTab = 4096;    // table slots (load <= 1/2)
constexpr uint32_t kEmpty = 0xffffffffu;  // keys are < 2^27

// Records are packed {query index (low 32 bits), M, N, K}: one 16-byte store
// per query (scattered 4-byte stores cost a partial sector each).  Batches of
// 2^31 queries or more also store the index's high half in `qhi`.
__global__ void __launch_bounds__(kT3) k_escatter(EvalArgs a, const uint32_t* keys, uint32_t* offs, int4* rec,
                                                  int32_t* qhi) {
    __shared__ uint32_t tkey[kScTab];
    __shared__ uint32_t tcnt[kScTab];
    const int64_t n = a.count ? *a.count : a.n;
    const int64_t chunk = int64_t(kT3) * kScPer;
    for (int64_t c0 = int64_t(blockIdx.x) * chunk; c0 < n; c0 += int64_t(gridDim.x) * chunk) {
        for (int i = threadIdx.x; i < kScTab; i += kT3) {
            tkey[i] = kEmpty;
            tcnt[i] = 0;
        }
        __syncthreads();
        uint32_t slot[kScPer], rank[kScPer];
#pragma unroll
        for (int k = 0; k < kScPer; ++k) {
            const int64_t i = c0 + int64_t(k) * kT3 + threadIdx.x;
            slot[k] = kEmpty;
            if (i < n) {
                const uint32_t key = keys[i];
                uint32_t h = (key * 0x9E3779B1u) >> 20;  // 12 bits = kScTab
                for (;;) {
                    const uint32_t old = atomicCAS(tkey + h, kEmpty, key);
                    if (old == kEmpty || old == key) break;
                    h = (h + 1u) & (kScTab - 1u);
                }
                slot[k] = h;
                rank[k] = atomicAdd(tcnt + h, 1u);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kScTab; i += kT3)
            if (tcnt[i]) tcnt[i] = atomicAdd(offs + tkey[i], tcnt[i]);  // count -> chunk's base
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kScPer; ++k) {
            if (slot[k] == kEmpty) continue;
            const int64_t i = c0 + int64_t(k) * kT3 + threadIdx.x;
            const uint32_t p = tcnt[slot[k]] + rank[k];
            const int64_t src = a.inputs_compact ? i : (a.idx ? a.idx[i] : i);
            const int64_t q = a.idx ? a.idx[i] : i;
            rec[p] = make_int4(int32_t(uint32_t(q)), a.M[src], a.N[src], a.K[src]);
            if (qhi) qhi[p] = int32_t(q >> 32);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ eval
template <bool SPECIAL, bool HS>
__global__ void __launch_bounds__(kT3, 2) k_eval3(DevImage im, EvalArgs a, const int4* rec, const int32_t* qhi) {
    // segment headers in shared memory (broadcast LDS instead of dependent
    // global loads at every segment start)
    __shared__ int4 h_tiles[kMaxSmemSeg];
    __shared__ uint4 h_magic[kMaxSmemSeg];
    __shared__ int32_t h_pos[kMaxSmemSeg];
    constexpr bool hs = HS;  // nseg <= kMaxSmemSeg: headers from shared memory
    if (hs) {
        for (int i = threadIdx.x; i < im.nseg; i += blockDim.x) {
            h_tiles[i] = im.seg_tiles[i];
            h_magic[i] = im.seg_magic[i];
            h_pos[i] = im.seg_pos[i];
        }
    }
    __syncthreads();
    const int4* Ts = hs ? h_tiles : im.seg_tiles;
    const uint4* Ms = hs ? h_magic : im.seg_magic;
    const int32_t* Ps = hs ? h_pos : im.seg_pos;
    const int64_t n = a.count ? *a.count : a.n;
    const int64_t nt = (n + 3) / 4;  // thread tiles of 4 consecutive grouped queries
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int C = im.C;
    // Per-warp two-stage row buffers: while segment s is evaluated from one
    // stage, the lanes' loads of segment s+1's rows (at lane 0's row of that
    // tile class) are in flight and land in the other stage.  A warp whose
    // 128 queries share that row (the uniform case) then reads broadcasts
    // from shared memory instead of waiting on L1/L2.
    __shared__ __align__(16) double4 wrows[kT3 / 32][2][kSegCfg];
    const int lane = threadIdx.x & 31;
    double4* myrows = wrows[threadIdx.x >> 5][0];
    auto issue = [&](int s2, uint32_t r, int4& R0, int4& R1) {
        const int n2 = 2 * Ts[s2].w;  // 16-byte halves of the segment's rows
        const int4* src = reinterpret_cast<const int4*>(im.theta2t + size_t(r) * C + Ps[s2]);
        R0 = lane < n2 ? __ldg(src + lane) : make_int4(0, 0, 0, 0);
        R1 = lane + 32 < n2 ? __ldg(src + lane + 32) : make_int4(0, 0, 0, 0);
    };
    auto commit = [&](int stage, int s2, const int4& R0, const int4& R1) {
        const int n2 = 2 * Ts[s2].w;
        int4* dst = reinterpret_cast<int4*>(myrows + stage * kSegCfg);
        __syncwarp();
        if (lane < n2) dst[lane] = R0;
        if (lane + 32 < n2) dst[lane + 32] = R1;
        __syncwarp();
    };
    // warp-uniform trip count: every lane of a warp stays in the loop
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nt; base += stride) {
        const int64_t t = base + threadIdx.x;
        uint32_t y2M[4], y2N[4], y2K[4], status[4], acc[4];
        int64_t q[4];
        double best[4];
        int bp[4];  // winner's class-order position (config index resolved at the end)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = t * 4 + j;
            const bool live = t < nt && i < n;
            uint32_t M = 1, N = 1, K = 1, st = 0;
            q[j] = -1;
            if (live) {
                const int4 r = rec[i];
                q[j] = int64_t(uint32_t(r.x)) | (qhi ? int64_t(qhi[i]) << 32 : 0);
                st = query_status(im, r.y, r.z, r.w, &M, &N, &K);
            }
            y2M[j] = 2u * (M - 1u);
            y2N[j] = 2u * (N - 1u);
            y2K[j] = 2u * (K - 1u);
            status[j] = st;
            best[j] = kInf3;
            bp[j] = -1;
            acc[j] = 0;
        }
        uint32_t pm = 0, pn = 0, ps = 0xffffffffu, pk = 0, psk = 0xffffffffu;
        uint32_t row[4] = {0, 0, 0, 0};
        double gd[4] = {0, 0, 0, 0}, ld[4] = {0, 0, 0, 0};
        uint32_t lbp = 0;  // the 4 queries' L buckets, 8 bits each
        bool uni = false;
        const int s_first = 0;
        {
            uint64_t g;
            const uint32_t r = __shfl_sync(0xffffffffu, row_for(im, y2M[0], y2N[0], Ms[s_first], &g), 0);
            int4 R0, R1;
            issue(s_first, r, R0, R1);
            commit(0, s_first, R0, R1);
        }
        for (int s = s_first, stage = 0; s < im.nseg; stage ^= 1) {
            const int s_next = s + 1;
            const uint4 mg = Ms[s];
            const int pos = Ps[s];
            const int ncfg = Ts[s].w;
            if (mg.x != pm || mg.y != pn || (mg.w & 0xffffu) != ps) {
                pm = mg.x;
                pn = mg.y;
                ps = mg.w & 0xffffu;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint64_t g;
                    row[j] = row_for(im, y2M[j], y2N[j], mg, &g);
                    gd[j] = u64_to_f64(g);
                }
                const uint32_t r0 = __shfl_sync(0xffffffffu, row[0], 0);
                uni = __all_sync(0xffffffffu, row[0] == r0 && row[1] == r0 && row[2] == r0 && row[3] == r0);
            }
            const uint32_t sk = (mg.w >> 16) & 0xffu;
            if (mg.z != pk || sk != psk) {
                pk = mg.z;
                psk = sk;
                lbp = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t L = mdiv2(y2K[j], mg.z, sk) + 1u;
                    ld[j] = u32_to_f64(L);
                    lbp |= uint32_t(min(31 - __clz(int(L)), kLB - 1)) << (8 * j);
                }
            }
            // configs that can still win for the warp's (row, L bucket) cells
            uint32_t live = 0xffffffffu;
            if (im.prune) {
                live = 0;
                const uint32_t* mk = im.segmask + size_t(s) * im.R * kLB;
#pragma unroll
                for (int j = 0; j < 4; ++j) live |= __ldg(mk + row[j] * kLB + ((lbp >> (8 * j)) & 0xffu));
                live = __reduce_or_sync(0xffffffffu, live);
            }
            live &= ncfg >= 32 ? 0xffffffffu : ((1u << ncfg) - 1u);
            if constexpr (SPECIAL) {  // flags of every config count, evaluated or not
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] |= __ldg(im.segor + size_t(s) * im.R + row[j]);
            }
            const bool ahead = s_next < im.nseg;
            int4 R0 = make_int4(0, 0, 0, 0), R1 = R0;
            if (ahead) {
                const uint4 mn = Ms[s_next];
                uint32_t rn = row[0];
                if (mn.x != pm || mn.y != pn || (mn.w & 0xffffu) != ps) {
                    uint64_t g;
                    rn = row_for(im, y2M[0], y2N[0], mn, &g);
                }
                issue(s_next, __shfl_sync(0xffffffffu, rn, 0), R0, R1);
            }
            double sb[4] = {kInf3, kInf3, kInf3, kInf3};
            int sj[4] = {-1, -1, -1, -1};
            if (uni) {
                // one broadcast row per config ([row][class position] layout:
                // the segment's configs are contiguous), reused by 4 queries
                auto eval1 = [&](const double4& th, int c) {
                    double tt[4], u[4], v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) tt[j] = __dmul_rn(th.x, gd[j]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) u[j] = __dmul_rn(th.y, gd[j]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = __dmul_rn(th.z, ld[j]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) tt[j] = __dmul_rn(tt[j], ld[j]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) tt[j] = __dadd_rn(tt[j], u[j]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) tt[j] = __dadd_rn(tt[j], v[j]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) tt[j] = __dadd_rn(tt[j], th.w);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (tt[j] < sb[j]) {
                            sb[j] = tt[j];
                            sj[j] = c;
                        }
                };
                const double4* sp = myrows + stage * kSegCfg;
                // ascending config order: the strict-< scan keeps its meaning
                for (uint32_t mm = live; mm; mm &= mm - 1u) {
                    const int c = __ffs(int(mm)) - 1;
                    eval1(sp[c], c);
                }
            } else {
                for (uint32_t mm = live; mm; mm &= mm - 1u) {
                    const int c = __ffs(int(mm)) - 1;
                    double4 th[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) th[j] = ldg_row(im.theta2t + size_t(row[j]) * C + pos + c);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        double tt = __dmul_rn(__dmul_rn(th[j].x, gd[j]), ld[j]);
                        tt = __dadd_rn(tt, __dmul_rn(th[j].y, gd[j]));
                        tt = __dadd_rn(tt, __dmul_rn(th[j].z, ld[j]));
                        tt = __dadd_rn(tt, th[j].w);
                        if (tt < sb[j]) {
                            sb[j] = tt;
                            sj[j] = c;
                        }
                    }
                }
            }
            // lexicographic (latency, config index) merge; the config indices
            // are only needed on an exact tie
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (sj[j] < 0) continue;
                const int cand = pos + sj[j];
                if (sb[j] < best[j]) {
                    best[j] = sb[j];
                    bp[j] = cand;
                } else if (sb[j] == best[j] && __ldg(im.cls_cfg + cand) < __ldg(im.cls_cfg + bp[j])) {
                    bp[j] = cand;
                }
            }
            if (ahead) commit(stage ^ 1, s_next, R0, R1);
            s = s_next;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (q[j] < 0) continue;
            Final f;
            uint64_t g = 0;
            int64_t l = 0;
            const int bc = bp[j] >= 0 ? __ldg(im.cls_cfg + bp[j]) : -1;
            if (status[j]) {
                f.flags = status[j] << 24;
                f.macro = f.micro = f.wave = -1;
                f.comps = 0;
                f.tail = 0.f;
            } else {
                if (bc >= 0) {
                    const int4 tl4 = __ldg(im.tiles + bc);
                    const uint32_t M = y2M[j] / 2u + 1u, N = y2N[j] / 2u + 1u, K = y2K[j] / 2u + 1u;
                    g = uint64_t((M + uint32_t(tl4.x) - 1) / uint32_t(tl4.x)) *
                        uint64_t((N + uint32_t(tl4.y) - 1) / uint32_t(tl4.y));
                    l = int64_t((K + uint32_t(tl4.z) - 1) / uint32_t(tl4.z));
                }
                f = finish(im, bc, 0.0, g, l, acc[j]);
            }
            write_decision(a.out, q[j], f, best[j], g, l);
        }
    }
}

// k_eval4: the pruned evaluation without per-segment staging or merges.
// With the dominance masks only ~1 config per segment survives for a warp,
// so what costs is the per-segment bookkeeping, not the fp64 work: rows are
// recomputed only when (t_m, t_n) changes, L only when t_k leaves a 2-entry
// cache, the surviving configs' rows are loaded directly (warp-uniform
// addresses in the common case: one broadcast request), and every evaluation
// updates the running (latency, config index) winner in place -- strict-<
// plus the index tie-break, i.e. the lexicographic order tune()'s ascending
// strict-< scan produces (tuner.cpp:135-149).
template <bool SPECIAL, bool HS, int RPT>
__global__ void __launch_bounds__(kT3, RPT == 4 ? 2 : (RPT == 2 ? 3 : 4)) k_eval4(DevImage im, EvalArgs a, const int4* rec, const int32_t* qhi) {
    __shared__ int4 h_tiles[kMaxSmemSeg];
    __shared__ uint4 h_magic[kMaxSmemSeg];
    __shared__ int32_t h_pos[kMaxSmemSeg];
    // HS: segment headers and the class-position -> config map (dynamic,
    // C ints) in shared memory
    extern __shared__ int32_t h_cls[];
    if (HS) {
        for (int i = threadIdx.x; i < im.nseg; i += blockDim.x) {
            h_tiles[i] = im.seg_tiles[i];
            h_magic[i] = im.seg_magic[i];
            h_pos[i] = im.seg_pos[i];
        }
        for (int i = threadIdx.x; i < im.C; i += blockDim.x) h_cls[i] = im.cls_cfg[i];
    }
    __syncthreads();
    const int4* Ts = HS ? h_tiles : im.seg_tiles;
    const uint4* Ms = HS ? h_magic : im.seg_magic;
    const int32_t* Ps = HS ? h_pos : im.seg_pos;
    auto cfg_at = [&](int pos) { return HS ? h_cls[pos] : __ldg(im.cls_cfg + pos); };
    const int64_t n = a.count ? *a.count : a.n;
    const int64_t nt = (n + RPT - 1) / RPT;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int C = im.C, R = im.R;
    // Per-warp plan of 32 segments, built lane-parallel (lane = segment) from
    // lane 0's first query: its wave row and L bucket, the pruning mask of
    // that cell and the rows of its first two surviving configs, all loaded
    // at once.  A segment whose queries all share that (row, L bucket) --
    // known per (t_m, t_n) group and per t_k, see inplan below -- then reads
    // mask and rows from shared memory instead of two dependent global round
    // trips.
    __shared__ __align__(16) double4 pth[kT3 / 32][32][2];
    __shared__ uint32_t pmask[kT3 / 32][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // this warp's plan slices, addressed once (not re-derived per segment)
    double4 (*const my_pth)[2] = pth[wid];
    uint32_t* const my_pmask = pmask[wid];
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nt; base += stride) {
        const int64_t t = base + threadIdx.x;
        uint32_t y2M[RPT], y2N[RPT], y2K[RPT], status[RPT], acc[RPT];
        int64_t q[RPT];
        double best[RPT];
        int bci[RPT];  // winner's config index (INT32_MAX: none yet)
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int64_t i = t * RPT + j;
            const bool live = t < nt && i < n;
            uint32_t M = 1, N = 1, K = 1, st = 0;
            q[j] = -1;
            if (live) {
                const int4 r = rec[i];
                q[j] = int64_t(uint32_t(r.x)) | (qhi ? int64_t(qhi[i]) << 32 : 0);
                st = query_status(im, r.y, r.z, r.w, &M, &N, &K);
            }
            y2M[j] = 2u * (M - 1u);
            y2N[j] = 2u * (N - 1u);
            y2K[j] = 2u * (K - 1u);
            status[j] = st;
            best[j] = kInf3;
            bci[j] = INT32_MAX;
            acc[j] = 0;
        }
        uint32_t pm = 0, pn = 0, ps = 0xffffffffu;
        uint32_t row[RPT] = {};
        double gd[RPT] = {};
        bool uni = false;
        // two-entry cache of L per t_k (tags = magic, shift)
        uint32_t tagA = 0xffffffffu, tagB = 0xffffffffu;
        double ldA[RPT] = {}, ldB[RPT] = {};
        uint32_t lbA = 0, lbB = 0;
        // per cache slot: every query of the warp in lane 0's L bucket (the
        // plan's), decided once when the slot fills
        bool luA = false, luB = false;
        bool nextA = true;
        const uint32_t y2M0 = __shfl_sync(0xffffffffu, y2M[0], 0), y2N0 = __shfl_sync(0xffffffffu, y2N[0], 0),
                       y2K0 = __shfl_sync(0xffffffffu, y2K[0], 0);
        for (int s = 0; s < im.nseg; ++s) {
            if ((s & 31) == 0) {  // plan segments [s, s + 32)
                __syncwarp();     // the previous plan is no longer read
                const int sg = s + lane;
                uint32_t m = 0;
                if (sg < im.nseg) {
                    const uint4 mq = Ms[sg];
                    uint64_t g;
                    const uint32_t r = row_for(im, y2M0, y2N0, mq, &g);
                    const uint32_t L = mdiv2(y2K0, mq.z, (mq.w >> 16) & 0xffu) + 1u;
                    const uint32_t lb = uint32_t(min(31 - __clz(int(L)), kLB - 1));
                    const int nq = Ts[sg].w;
                    m = im.prune ? __ldg(im.segmask + (size_t(sg) * R + r) * kLB + lb) : 0xffffffffu;
                    m &= nq >= 32 ? 0xffffffffu : ((1u << nq) - 1u);
                    const double4* tp = im.theta2t + size_t(r) * C + Ps[sg];
                    if (m) my_pth[lane][0] = ldg_row(tp + (__ffs(int(m)) - 1));
                    const uint32_t m2 = m & (m - 1u);
                    if (m2) my_pth[lane][1] = ldg_row(tp + (__ffs(int(m2)) - 1));
                }
                my_pmask[lane] = m;
                __syncwarp();
            }
            const uint4 mg = Ms[s];
            const int pos = Ps[s];
            const int ncfg = Ts[s].w;
            if (mg.x != pm || mg.y != pn || (mg.w & 0xffffu) != ps) {
                pm = mg.x;
                pn = mg.y;
                ps = mg.w & 0xffffu;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    uint64_t g;
                    row[j] = row_for(im, y2M[j], y2N[j], mg, &g);
                    gd[j] = u64_to_f64(g);
                }
                const uint32_t r0 = __shfl_sync(0xffffffffu, row[0], 0);
                bool same = true;
#pragma unroll
                for (int j = 0; j < RPT; ++j) same = same && row[j] == r0;
                uni = __all_sync(0xffffffffu, same);
            }
            const uint32_t sk = (mg.w >> 16) & 0xffu;
            const uint32_t tag = mg.z ^ (sk << 24);
            if (tag != tagA && tag != tagB) {
                double* ld = nextA ? ldA : ldB;
                uint32_t lb = 0;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    const uint32_t L = mdiv2(y2K[j], mg.z, sk) + 1u;
                    ld[j] = u32_to_f64(L);
                    lb |= uint32_t(min(31 - __clz(int(L)), kLB - 1)) << (8 * j);
                }
                const uint32_t lb0 = __shfl_sync(0xffffffffu, lb & 0xffu, 0);
                bool lsame = true;
#pragma unroll
                for (int j = 0; j < RPT; ++j) lsame = lsame && ((lb >> (8 * j)) & 0xffu) == lb0;
                const bool lu = __all_sync(0xffffffffu, lsame);
                if (nextA) {
                    tagA = tag;
                    lbA = lb;
                    luA = lu;
                } else {
                    tagB = tag;
                    lbB = lb;
                    luB = lu;
                }
                nextA = !nextA;
            }
            const bool useA = tag == tagA;
            double ld[RPT];
#pragma unroll
            for (int j = 0; j < RPT; ++j) ld[j] = useA ? ldA[j] : ldB[j];
            const uint32_t lbp = useA ? lbA : lbB;
            // does the whole warp sit in the planned (row, L bucket) cell?
            // The plan is lane 0's first query's cell, so: every query's row
            // equals lane 0's (uni, per (t_m, t_n)) and every L bucket equals
            // lane 0's (per t_k slot) -- both warp-uniform, decided when they
            // were computed, no per-segment vote
            const bool inplan = uni && (useA ? luA : luB);
            uint32_t live;
            if (inplan) {
                live = my_pmask[s & 31];
            } else {
                live = 0xffffffffu;
                if (im.prune) {
                    const uint32_t* mk = im.segmask + size_t(s) * R * kLB;
                    live = 0;
#pragma unroll
                    for (int j = 0; j < RPT; ++j) live |= __ldg(mk + row[j] * kLB + ((lbp >> (8 * j)) & 0xffu));
                    live = __reduce_or_sync(0xffffffffu, live);
                }
                live &= ncfg >= 32 ? 0xffffffffu : ((1u << ncfg) - 1u);
            }
            if (im.eval_count && lane == 0)
                atomicAdd(im.eval_count, (unsigned long long)__popc(live) * 32ull * RPT);
            int k_staged = 0;  // index of the next planned row in pth
            if constexpr (SPECIAL) {
#pragma unroll
                for (int j = 0; j < RPT; ++j) acc[j] |= __ldg(im.segor + size_t(s) * R + row[j]);
            }
            for (uint32_t mm = live; mm; mm &= mm - 1u) {
                const int c = __ffs(int(mm)) - 1;
                const int ci = cfg_at(pos + c);
                double4 th[RPT];
                if (inplan && k_staged < 2) {
                    th[0] = my_pth[s & 31][k_staged++];
#pragma unroll
                    for (int j = 1; j < RPT; ++j) th[j] = th[0];
                } else if (uni) {
                    th[0] = ldg_row(im.theta2t + size_t(row[0]) * C + pos + c);
#pragma unroll
                    for (int j = 1; j < RPT; ++j) th[j] = th[0];
                } else {
#pragma unroll
                    for (int j = 0; j < RPT; ++j) th[j] = ldg_row(im.theta2t + size_t(row[j]) * C + pos + c);
                }
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    double tt = __dmul_rn(__dmul_rn(th[j].x, gd[j]), ld[j]);
                    tt = __dadd_rn(tt, __dmul_rn(th[j].y, gd[j]));
                    tt = __dadd_rn(tt, __dmul_rn(th[j].z, ld[j]));
                    tt = __dadd_rn(tt, th[j].w);
                    // ties go to the smaller index only between real winners:
                    // +inf never wins (tune() starts from +inf with strict <)
                    if (tt < best[j] || (tt == best[j] && ci < bci[j] && bci[j] != INT32_MAX)) {
                        best[j] = tt;
                        bci[j] = ci;
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            if (q[j] < 0) continue;
            Final f;
            uint64_t g = 0;
            int64_t l = 0;
            const int bc = bci[j] != INT32_MAX ? bci[j] : -1;
            if (status[j]) {
                f.flags = status[j] << 24;
                f.macro = f.micro = f.wave = -1;
                f.comps = 0;
                f.tail = 0.f;
            } else {
                if (bc >= 0) {
                    const int4 tl4 = __ldg(im.tiles + bc);
                    const uint32_t M = y2M[j] / 2u + 1u, N = y2N[j] / 2u + 1u, K = y2K[j] / 2u + 1u;
                    g = uint64_t((M + uint32_t(tl4.x) - 1) / uint32_t(tl4.x)) *
                        uint64_t((N + uint32_t(tl4.y) - 1) / uint32_t(tl4.y));
                    l = int64_t((K + uint32_t(tl4.z) - 1) / uint32_t(tl4.z));
                }
                f = finish(im, bc, 0.0, g, l, acc[j]);
            }
            write_decision(a.out, q[j], f, best[j], g, l);
        }
    }
}

// ---------------------------------------------------------------- launcher
namespace {
int key_bits() {
    static const int b = [] {
        const char* v = std::getenv("WT_EVAL_KEY_BITS");
        const int x = v ? std::atoi(v) : 18;
        return std::min(24, std::max(8, x));
    }();
    return b;
}
size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
int key_mode() {
    static const int m = [] {
        const char* v = std::getenv("WT_EVAL_KEY_MODE");
        return v ? std::atoi(v) : 1;
    }();
    return m;
}
}  // namespace

size_t eval3_scratch_bytes(int64_t n) {
    const size_t nb = size_t(1) << (key_bits() + kSpreadBits);
    const size_t scan = scan_scratch_bytes(int64_t(nb));
    const size_t un = size_t(std::max<int64_t>(n, 1));
    return al256(nb * 4) * 2 + al256(un * 4) + al256(un * 16) + al256(un * 4) + al256(scan);
}

Eval3Bufs eval3_bufs(void* scratch, int64_t n) {
    Eval3Bufs b;
    const size_t nb = size_t(1) << (key_bits() + kSpreadBits);
    const size_t un = size_t(std::max<int64_t>(n, 1));
    char* p = static_cast<char*>(scratch);
    b.hist = reinterpret_cast<uint32_t*>(p);
    b.keys = reinterpret_cast<uint32_t*>(p + 2 * al256(nb * 4));
    (void)un;
    b.key_bits = key_bits();
    b.key_mode = key_mode();
    b.hist_bytes = nb * 4;
    return b;
}

cudaError_t launch_eval3(const DevImage& im, const EvalArgs& a, void* scratch, bool keys_ready, cudaStream_t st) {
    const int bits = key_bits();
    const size_t nb = size_t(1) << (bits + kSpreadBits);
    const size_t un = size_t(std::max<int64_t>(a.n, 1));
    char* p = static_cast<char*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(p);
    p += al256(nb * 4);
    uint32_t* offs = reinterpret_cast<uint32_t*>(p);
    p += al256(nb * 4);
    uint32_t* keys = reinterpret_cast<uint32_t*>(p);
    p += al256(un * 4);
    int4* rec = reinterpret_cast<int4*>(p);
    p += al256(un * 16);
    int32_t* qhi = a.n >= (int64_t(1) << 31) ? reinterpret_cast<int32_t*>(p) : nullptr;
    p += al256(un * 4);
    void* tmp = p;

    const int sms = device_sms();
    const int occ = occupancy(reinterpret_cast<const void*>(k_eval3<false, true>), kT3, 0);
    const int occs = occupancy(reinterpret_cast<const void*>(k_eval3<true, true>), kT3, 0);
    // grids: enough CTAs for n (host upper bound), capped at a few waves
    const int64_t want = (a.n + kT3 - 1) / kT3;
    const int gk = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * 8)));
    cudaError_t e = cudaSuccess;
    if (!keys_ready) {
        e = cudaMemsetAsync(hist, 0, nb * 4, st);
        if (e != cudaSuccess) return e;
        k_ekey<<<gk, kT3, 0, st>>>(im, a, bits, key_mode(), keys, hist);
    }
    e = scan_exclusive_u32(hist, offs, int64_t(nb), tmp, st);
    if (e != cudaSuccess) return e;
    const int gs = int(std::max<int64_t>(1, std::min<int64_t>((a.n + kT3 * kScPer - 1) / (kT3 * kScPer),
                                                              int64_t(sms) * 4)));
    k_escatter<<<gs, kT3, 0, st>>>(a, keys, offs, rec, qhi);
    const int64_t want3 = (a.n + 4 * kT3 - 1) / (4 * kT3);
    const bool hs = im.nseg <= kMaxSmemSeg;
    const int g3 = int(std::max<int64_t>(1, std::min<int64_t>(want3, int64_t(sms) * (im.special ? occs : occ))));
    static const int kern = [] {
        const char* v = std::getenv("WT_EVAL_KERNEL");
        return v ? std::atoi(v) : 4;
    }();
    if (kern == 4) {
        static const int rpt = [] {
            const char* v = std::getenv("WT_EVAL4_RPT");
            const int x = v ? std::atoi(v) : 2;  // measured best on B200 (r01e: 2 > 1 > 4)
            return x == 1 || x == 4 ? x : 2;
        }();
        const bool hs4 = hs && im.C <= 8192;
        const size_t dyn = hs4 ? size_t(im.C) * sizeof(int32_t) : 0;
        auto go = [&](auto fn, int r) {
            const int o = occupancy(reinterpret_cast<const void*>(fn), kT3, dyn);  // raises the smem limit too
            const int64_t w = (a.n + int64_t(r) * kT3 - 1) / (int64_t(r) * kT3);
            const int g = int(std::max<int64_t>(1, std::min<int64_t>(w, int64_t(sms) * std::max(o, 1))));
            fn<<<g, kT3, dyn, st>>>(im, a, rec, qhi);
        };
#define WT_GO4(SP, H)                                         \
    (rpt == 1   ? go(k_eval4<SP, H, 1>, 1)                    \
     : rpt == 2 ? go(k_eval4<SP, H, 2>, 2)                    \
                : go(k_eval4<SP, H, 4>, 4))
        if (im.special) {
            if (hs4) WT_GO4(true, true); else WT_GO4(true, false);
        } else {
            if (hs4) WT_GO4(false, true); else WT_GO4(false, false);
        }
#undef WT_GO4
        return cudaGetLastError();
    }
    if (im.special)
        hs ? k_eval3<true, true><<<g3, kT3, 0, st>>>(im, a, rec, qhi) : k_eval3<true, false><<<g3, kT3, 0, st>>>(im, a, rec, qhi);
    else
        hs ? k_eval3<false, true><<<g3, kT3, 0, st>>>(im, a, rec, qhi) : k_eval3<false, false><<<g3, kT3, 0, st>>>(im, a, rec, qhi);
    return cudaGetLastError();
}

}  // namespace wtb
