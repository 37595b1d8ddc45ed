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

#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "wt_decide.h"
#include "wt_device.cuh"

namespace wtb {

namespace {

constexpr int kT3 = 256;
constexpr int kSpreadBits = 3;
constexpr int kMaxSmemSeg = 256;  // segment headers staged in shared memory up to this count
constexpr double kInf3 = __builtin_huge_val();

__device__ __forceinline__ bool lex_less3(double a, int ia, double b, int ib) {
    return a < b || (a == b && ia < ib);
}

// Per-query validity exactly as k_eval2 (kernel_map.cpp:238-239 + the
// 32-bit wave guard); invalid queries evaluate as (1, 1, 1) and are flagged.
__device__ __forceinline__ uint32_t query_status(const DevImage& im, int32_t m, int32_t n, int32_t k, uint32_t* M,
                                                 uint32_t* N, uint32_t* K) {
    *M = *N = *K = 1u;
    if (m < 1 || n < 1 || k < 1) return WT_INVALID_ARGUMENT;
    const uint64_t gmax = uint64_t((uint32_t(m) + uint32_t(im.tm_min) - 1) / uint32_t(im.tm_min)) *
                          uint64_t((uint32_t(n) + uint32_t(im.tn_min) - 1) / uint32_t(im.tn_min));
    if ((gmax + uint64_t(im.S) - 1) / uint64_t(im.S) >= (uint64_t(1) << 31)) return WT_UNSUPPORTED;
    *M = uint32_t(m);
    *N = uint32_t(n);
    *K = uint32_t(k);
    return 0;
}

__device__ __forceinline__ uint32_t row_for(const DevImage& im, uint32_t y2M, uint32_t y2N, uint4 mg, uint64_t* g) {
    const uint32_t mt = mdiv2(y2M, mg.x, mg.w & 0xffu) + 1u;
    const uint32_t nt = mdiv2(y2N, mg.y, (mg.w >> 8) & 0xffu) + 1u;
    *g = uint64_t(mt) * nt;
    const uint32_t gc = *g > im.RS ? im.RS : uint32_t(*g);
    return row_of(gc, im.mS, im.sS);
}

}  // namespace

// ------------------------------------------------------------------ keys
__global__ void k_ekey(DevImage im, EvalArgs a, int bits, uint32_t* keys, uint32_t* hist) {
    const int64_t n = a.count ? *a.count : a.n;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int br = 1;
    while ((1 << br) < im.R) ++br;
    const int pre = (2 * br + 4 <= bits) ? 2 : (br + 4 <= bits ? 1 : 0);
    const int hb = bits - pre * br;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t src = a.inputs_compact ? i : (a.idx ? a.idx[i] : i);
        uint32_t M, N, K;
        uint32_t key = 0;
        if (!query_status(im, a.M[src], a.N[src], a.K[src], &M, &N, &K)) {
            const uint32_t y2M = 2u * (M - 1u), y2N = 2u * (N - 1u);
            uint32_t h = 0x811c9dc5u, first = 0, last = 0, pm = 0, pn = 0, ps = 0xffffffffu;
            for (int s = 0; s < im.nseg; ++s) {
                const uint4 mg = __ldg(im.seg_magic + s);
                if (mg.x == pm && mg.y == pn && (mg.w & 0xffffu) == ps) continue;  // same (t_m, t_n)
                pm = mg.x;
                pn = mg.y;
                ps = mg.w & 0xffffu;
                uint64_t g;
                const uint32_t r = row_for(im, y2M, y2N, mg, &g);
                if (s == 0) first = r;
                last = r;
                h = (h ^ r) * 0x01000193u;
            }
            h ^= h >> 15;
            h *= 0x2c1b3c6du;
            h ^= h >> 12;
            if (pre == 2)
                key = (first << (bits - br)) | (last << (bits - 2 * br)) | (h & ((1u << hb) - 1u));
            else if (pre == 1)
                key = (first << (bits - br)) | (h & ((1u << hb) - 1u));
            else
                key = h & ((1u << bits) - 1u);
        }
        // 8 adjacent sub-buckets per key (by query slot) spread the atomics of
        // large groups; sub-buckets of one key stay contiguous after the scan
        key = (key << kSpreadBits) | uint32_t(i & ((1 << kSpreadBits) - 1));
        keys[i] = key;
        atomicAdd(hist + key, 1u);
    }
}

__global__ void k_escatter(EvalArgs a, const uint32_t* keys, uint32_t* offs, int64_t* sq, int32_t* sM, int32_t* sN,
                           int32_t* sK) {
    const int64_t n = a.count ? *a.count : a.n;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t p = atomicAdd(offs + keys[i], 1u);
        const int64_t src = a.inputs_compact ? i : (a.idx ? a.idx[i] : i);
        sq[p] = a.idx ? a.idx[i] : i;
        sM[p] = a.M[src];
        sN[p] = a.N[src];
        sK[p] = a.K[src];
    }
}

// ------------------------------------------------------------------ eval
template <bool SPECIAL>
__global__ void __launch_bounds__(kT3, 2) k_eval3(DevImage im, EvalArgs a, const int64_t* sq, const int32_t* sM,
                                               const int32_t* sN, const int32_t* sK) {
    // segment headers in shared memory (broadcast LDS instead of dependent
    // global loads at every segment start)
    __shared__ int4 h_tiles[kMaxSmemSeg];
    __shared__ uint4 h_magic[kMaxSmemSeg];
    __shared__ int32_t h_pos[kMaxSmemSeg];
    const bool hs = im.nseg <= kMaxSmemSeg;
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
                q[j] = sq[i];
                st = query_status(im, sM[i], sN[i], sK[i], &M, &N, &K);
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
        bool uni = false;
        for (int s = 0; s < im.nseg; ++s) {
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
#pragma unroll
                for (int j = 0; j < 4; ++j) ld[j] = u32_to_f64(mdiv2(y2K[j], mg.z, sk) + 1u);
            }
            double sb[4] = {kInf3, kInf3, kInf3, kInf3};
            int sj[4] = {-1, -1, -1, -1};
            if (uni) {
                // one broadcast row per config ([row][class position] layout:
                // the segment's configs are contiguous), reused by 4 queries
                const double4* p = im.theta2t + size_t(row[0]) * C + pos;
                const uint32_t* pmeta = im.meta2t + size_t(row[0]) * C + pos;
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
                    if constexpr (SPECIAL) {
                        const uint32_t mm = __ldg(pmeta + c);
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[j] |= mm;
                    }
                };
                // ping-pong buffers: the next pair of rows is in flight while
                // the current pair is evaluated
                double4 a0 = ldg_row(p), a1 = ncfg > 1 ? ldg_row(p + 1) : a0;
                int c = 0;
                for (; c + 1 < ncfg; c += 2) {
                    double4 b0 = a0, b1 = a1;
                    if (c + 2 < ncfg) b0 = ldg_row(p + c + 2);
                    if (c + 3 < ncfg) b1 = ldg_row(p + c + 3);
                    eval1(a0, c);
                    eval1(a1, c + 1);
                    a0 = b0;
                    a1 = b1;
                }
                if (c < ncfg) eval1(a0, c);
            } else {
                for (int c = 0; c < ncfg; ++c) {
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
                        if constexpr (SPECIAL) acc[j] |= __ldg(im.meta2t + size_t(row[j]) * C + pos + c);
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
}  // namespace

size_t eval3_scratch_bytes(int64_t n) {
    const size_t nb = size_t(1) << (key_bits() + kSpreadBits);
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), int(nb));
    const size_t un = size_t(std::max<int64_t>(n, 1));
    return al256(nb * 4) * 2 + al256(un * 4) + al256(un * 8) + 3 * al256(un * 4) + al256(scan);
}

cudaError_t launch_eval3(const DevImage& im, const EvalArgs& a, void* scratch, cudaStream_t st) {
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
    int64_t* sq = reinterpret_cast<int64_t*>(p);
    p += al256(un * 8);
    int32_t* sM = reinterpret_cast<int32_t*>(p);
    p += al256(un * 4);
    int32_t* sN = reinterpret_cast<int32_t*>(p);
    p += al256(un * 4);
    int32_t* sK = reinterpret_cast<int32_t*>(p);
    p += al256(un * 4);
    void* tmp = p;

    static int sms = 0, occ = 0, occs = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval3<false>, kT3, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, k_eval3<true>, kT3, 0);
        occ = std::max(occ, 1);
        occs = std::max(occs, 1);
    }
    // grids: enough CTAs for n (host upper bound), capped at a few waves
    const int64_t want = (a.n + kT3 - 1) / kT3;
    const int gk = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * 8)));
    cudaError_t e = cudaMemsetAsync(hist, 0, nb * 4, st);
    if (e != cudaSuccess) return e;
    k_ekey<<<gk, kT3, 0, st>>>(im, a, bits, keys, hist);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, hist, offs, int(nb), st);
    e = cub::DeviceScan::ExclusiveSum(tmp, sb, hist, offs, int(nb), st);
    if (e != cudaSuccess) return e;
    k_escatter<<<gk, kT3, 0, st>>>(a, keys, offs, sq, sM, sN, sK);
    const int64_t want3 = (a.n + 4 * kT3 - 1) / (4 * kT3);
    if (im.special) {
        const int g3 = int(std::max<int64_t>(1, std::min<int64_t>(want3, int64_t(sms) * occs)));
        k_eval3<true><<<g3, kT3, 0, st>>>(im, a, sq, sM, sN, sK);
    } else {
        const int g3 = int(std::max<int64_t>(1, std::min<int64_t>(want3, int64_t(sms) * occ)));
        k_eval3<false><<<g3, kT3, 0, st>>>(im, a, sq, sM, sN, sK);
    }
    return cudaGetLastError();
}

}  // namespace wtb
