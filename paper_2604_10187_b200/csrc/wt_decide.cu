// wt_decide.cu -- sm_100a kernels of the WaveTune decision path.
//
//   k_sweep   (K1, grid mode)  tune() over every (pair, M) of a shape grid:
//             lanes = shapes, configs + coefficient rows staged per pair in
//             shared memory with gamma*l folded in, integer magic division
//             for tiles and waves, register argmin per lane.
//   k_eval    (K1, list mode)  tune() for arbitrary dense/attention queries
//             (optionally a device-compacted index list from k_gather).
//   k_grouped tune() for grouped-GEMM queries: one warp per query, lanes over
//             configs, warp-shuffle argmin.
//   k_gather  (K3) online queries against a filled grid; off-grid queries are
//             compacted (warp-aggregated atomics) for k_eval.
//   k_predict / k_explain / k_nearest  per-table helpers for the drop-in API.
//
// Arithmetic is binary64 with explicit _rn intrinsics (no contraction) and
// exact 32-bit magic division, so results are bit-identical to the
// reference's C++ (SURVEY.md Appendix A).
#include <cuda_runtime.h>


#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "wt_decide.h"
#include "wt_device.cuh"

namespace wtb {


// ------------------------------------------------------------- K1: sweep
// Shared-memory chunk of configs for one (N, K) pair.
struct SweepCfg {
    uint32_t mM, sM, nt, pad;
};

template <int RPT, bool SPECIAL, bool WIDE, int KM>
__global__ void __launch_bounds__(kSweepThreads) k_sweep(DevImage im, SweepArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int CC = a.chunk;
    SweepCfg* scfg = reinterpret_cast<SweepCfg*>(smem);
    double* sld = reinterpret_cast<double*>(scfg + CC);
    double4* sth = reinterpret_cast<double4*>(sld + CC);
    uint32_t* smeta = reinterpret_cast<uint32_t*>(sth + size_t(CC) * im.R);

    const int tid = threadIdx.x;
    const int64_t tile = int64_t(kSweepThreads) * RPT;
    const int64_t t0 = a.begin + int64_t(blockIdx.x) * tile;
    const int64_t t1 = min(t0 + tile, a.end);
    const uint32_t RS = im.RS, mS = im.mS, sS = im.sS;
    const int R = im.R;

    // A tile may straddle pair boundaries: process one pair segment at a time.
    for (int64_t seg = t0; seg < t1;) {
        const int32_t p = int32_t(seg / a.mcount);
        const int64_t seg_end = min(t1, int64_t(p + 1) * a.mcount);
        const uint32_t Np = uint32_t(a.N[p]), Kp = uint32_t(a.K[p]);

        double best[RPT];
        int bc[RPT];
        uint32_t acc[RPT];
        uint32_t y2[RPT];
        double tkL[KM > 0 ? KM : 1][RPT];
        int tkI[KM > 0 ? KM : 1][RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int64_t idx = seg + int64_t(j) * kSweepThreads + tid;
            const int64_t mi = (idx < seg_end) ? idx - int64_t(p) * a.mcount : 0;
            const uint32_t M = uint32_t(a.m_lo + mi);
            y2[j] = 2u * (M - 1u);
            best[j] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
            bc[j] = -1;
            acc[j] = 0;
            if constexpr (KM > 0) {
#pragma unroll
                for (int q = 0; q < KM; ++q) {
                    tkL[q][j] = __longlong_as_double(0x7ff0000000000000LL);
                    tkI[q][j] = -1;
                }
            }
        }

        for (int c0 = 0; c0 < im.C; c0 += CC) {
            const int cc = min(CC, im.C - c0);
            __syncthreads();
            // stage per-config scalars: ceil(N/t_n), ceil(K/t_k), magic for t_m
            for (int i = tid; i < cc; i += kSweepThreads) {
                const int c = c0 + i;
                const int4 tl = __ldg(im.tiles + c);
                const uint4 mg = __ldg(im.magic + c);
                SweepCfg s;
                s.mM = mg.x;
                s.sM = mg.w & 0xffu;
                s.nt = uint32_t((uint64_t(Np) + uint32_t(tl.y) - 1) / uint32_t(tl.y));
                s.pad = 0;
                scfg[i] = s;
                const uint32_t lk = uint32_t((uint64_t(Kp) + uint32_t(tl.z) - 1) / uint32_t(tl.z));
                sld[i] = u32_to_f64(lk);
            }
            __syncthreads();
            // stage coefficient rows with gamma*l folded in (bit-identical
            // product: the reference forms gamma*l as one rounded DMUL)
            const int nrow = cc * R;
            const double4* gth = im.theta + size_t(c0) * R;
            for (int i = tid; i < nrow; i += kSweepThreads) {
                double4 th = ldg_row(gth + i);
                th.z = __dmul_rn(th.z, sld[i / R]);
                sth[i] = th;
                if constexpr (SPECIAL) smeta[i] = __ldg(im.rowmeta + size_t(c0) * R + i);
            }
            __syncthreads();

#pragma unroll 2
            for (int i = 0; i < cc; ++i) {
                const SweepCfg s = scfg[i];
                const double ld = sld[i];
                const double4* rows = sth + size_t(i) * R;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    const uint32_t q = mdiv2(y2[j], s.mM, s.sM);
                    uint32_t gc;
                    double gd;
                    if constexpr (WIDE) {
                        const uint64_t g = uint64_t(q) * s.nt + s.nt;
                        gc = g > RS ? RS : uint32_t(g);
                        gd = u64_to_f64(g);
                    } else {
                        const uint32_t g = q * s.nt + s.nt;
                        gc = min(g, RS);
                        gd = u32_to_f64(g);
                    }
                    const uint32_t row = row_of(gc, mS, sS);
                    const double4 th = rows[row];
                    const double t = bilinear(th.x, th.y, th.z, th.w, gd, ld);
                    if (t < best[j]) {
                        best[j] = t;
                        bc[j] = c0 + i;
                    }
                    if constexpr (SPECIAL) acc[j] |= smeta[size_t(i) * R + row];
                    if constexpr (KM > 0) {
                        double L[KM];
                        int I[KM];
#pragma unroll
                        for (int z = 0; z < KM; ++z) {
                            L[z] = tkL[z][j];
                            I[z] = tkI[z][j];
                        }
                        topk_insert<KM>(L, I, t, c0 + i);
#pragma unroll
                        for (int z = 0; z < KM; ++z) {
                            tkL[z][j] = L[z];
                            tkI[z][j] = I[z];
                        }
                    }
                }
            }
        }

        // epilogue: Stage II for each winner, one 32-byte entry per shape
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int64_t idx = seg + int64_t(j) * kSweepThreads + tid;
            if (idx >= seg_end) continue;
            const int c = bc[j];
            uint64_t g = 0;
            int64_t l = 0;
            if (c >= 0) {
                const int4 tl = __ldg(im.tiles + c);
                const uint32_t M = y2[j] / 2u + 1u;
                g = uint64_t((M + uint32_t(tl.x) - 1) / uint32_t(tl.x)) *
                    uint64_t((uint64_t(Np) + uint32_t(tl.y) - 1) / uint32_t(tl.y));
                l = int64_t((uint64_t(Kp) + uint32_t(tl.z) - 1) / uint32_t(tl.z));
            }
            const Final f = finish(im, c, best[j], g, l, acc[j]);
            const bool ok = (f.flags >> 24) == 0;
            int4 lo, hi;
            const double lat = ok ? best[j] : __longlong_as_double(0x7ff8000000000000LL);
            lo.x = __double2loint(lat);
            lo.y = __double2hiint(lat);
            lo.z = f.macro;
            lo.w = f.micro;
            hi.x = f.wave;
            hi.y = int(f.flags);
            hi.z = f.comps;
            hi.w = __float_as_int(f.tail);
            int4* e = reinterpret_cast<int4*>(a.entries + idx);
            e[0] = lo;
            e[1] = hi;
            if constexpr (KM > 0) {
                for (int z = 0; z < a.topk; ++z) {
                    const int ci = ok ? tkI[z][j] : -1;
                    a.topk_macro[idx * a.topk + z] = ci >= 0 ? __ldg(im.macro_id + ci) : -1;
                    a.topk_lat[idx * a.topk + z] =
                        ci >= 0 ? tkL[z][j] : __longlong_as_double(0x7ff8000000000000LL);
                }
            }
        }
        seg = seg_end;
    }
}

// --------------------------------------------------------- K1: list mode
template <bool SPECIAL, int KM>
__global__ void __launch_bounds__(kEvalThreads) k_eval(DevImage im, EvalArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int CC = a.chunk;
    int4* stile = reinterpret_cast<int4*>(smem);
    uint4* smag = reinterpret_cast<uint4*>(stile + CC);
    double4* sth = reinterpret_cast<double4*>(smag + CC);
    uint32_t* smeta = reinterpret_cast<uint32_t*>(sth + size_t(CC) * im.R);

    const int64_t n = a.count ? *a.count : a.n;
    const int64_t ntiles = (n + kEvalThreads - 1) / kEvalThreads;
    const uint32_t RS = im.RS, mS = im.mS, sS = im.sS;
    const int R = im.R;
    const int tid = threadIdx.x;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t slot = tile * kEvalThreads + tid;
        const bool live = slot < n;
        const int64_t q = live ? (a.idx ? a.idx[slot] : slot) : 0;
        uint32_t M = 1, N = 1, K = 1;
        uint32_t status = 0;
        if (live) {
            const int32_t m = a.M[q], nn = a.N[q], k = a.K[q];
            if (m < 1 || nn < 1 || k < 1) status = WT_INVALID_ARGUMENT;  // kernel_map.cpp:238-239
            else {
                M = uint32_t(m);
                N = uint32_t(nn);
                K = uint32_t(k);
                // guard: every wave count must fit the reference's int
                const uint64_t gmax = uint64_t((M + uint32_t(im.tm_min) - 1) / uint32_t(im.tm_min)) *
                                      uint64_t((N + uint32_t(im.tn_min) - 1) / uint32_t(im.tn_min));
                if ((gmax + uint64_t(im.S) - 1) / uint64_t(im.S) >= (uint64_t(1) << 31))
                    status = WT_UNSUPPORTED;
            }
        }
        const uint32_t y2M = 2u * (M - 1u), y2N = 2u * (N - 1u), y2K = 2u * (K - 1u);
        double best = __longlong_as_double(0x7ff0000000000000LL);
        int bc = -1;
        uint32_t acc = 0;
        double tkL[KM > 0 ? KM : 1];
        int tkI[KM > 0 ? KM : 1];
        if constexpr (KM > 0) {
#pragma unroll
            for (int z = 0; z < KM; ++z) {
                tkL[z] = __longlong_as_double(0x7ff0000000000000LL);
                tkI[z] = -1;
            }
        }
        for (int c0 = 0; c0 < im.C; c0 += CC) {
            const int cc = min(CC, im.C - c0);
            __syncthreads();
            for (int i = tid; i < cc; i += kEvalThreads) {
                stile[i] = __ldg(im.tiles + c0 + i);
                smag[i] = __ldg(im.magic + c0 + i);
            }
            const int nrow = cc * R;
            for (int i = tid; i < nrow; i += kEvalThreads) {
                sth[i] = ldg_row(im.theta + size_t(c0) * R + i);
                if constexpr (SPECIAL) smeta[i] = __ldg(im.rowmeta + size_t(c0) * R + i);
            }
            __syncthreads();
            for (int i = 0; i < cc; ++i) {
                const uint4 mg = smag[i];
                const uint32_t mt = mdiv2(y2M, mg.x, mg.w & 0xffu) + 1u;
                const uint32_t nt = mdiv2(y2N, mg.y, (mg.w >> 8) & 0xffu) + 1u;
                const uint32_t lk = mdiv2(y2K, mg.z, (mg.w >> 16) & 0xffu) + 1u;
                const uint64_t g = uint64_t(mt) * nt;
                const uint32_t gc = g > RS ? RS : uint32_t(g);
                const uint32_t row = row_of(gc, mS, sS);
                const double4 th = sth[size_t(i) * R + row];
                const double gd = u64_to_f64(g), ld = u32_to_f64(lk);
                const double t = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
                if (t < best) {
                    best = t;
                    bc = c0 + i;
                }
                if constexpr (SPECIAL) acc |= smeta[size_t(i) * R + row];
                if constexpr (KM > 0) topk_insert<KM>(tkL, tkI, t, c0 + i);
            }
        }
        if (live) {
            if (status) {
                Final f;
                f.flags = status << 24;
                f.macro = f.micro = f.wave = -1;
                f.comps = 0;
                f.tail = 0.f;
                write_decision(a.out, q, f, 0.0, 0, 0);
                if constexpr (KM > 0)
                    for (int z = 0; z < a.out.topk; ++z) {
                        a.out.topk_macro[q * a.out.topk + z] = -1;
                        a.out.topk_lat[q * a.out.topk + z] = __longlong_as_double(0x7ff8000000000000LL);
                    }
            } else {
                uint64_t g = 0;
                int64_t l = 0;
                if (bc >= 0) {
                    const int4 tl = __ldg(im.tiles + bc);
                    g = uint64_t((M + uint32_t(tl.x) - 1) / uint32_t(tl.x)) *
                        uint64_t((N + uint32_t(tl.y) - 1) / uint32_t(tl.y));
                    l = int64_t((K + uint32_t(tl.z) - 1) / uint32_t(tl.z));
                }
                const Final f = finish(im, bc, best, g, l, acc);
                write_decision(a.out, q, f, best, g, l);
                if constexpr (KM > 0) {
                    const bool ok = (f.flags >> 24) == 0;
                    for (int z = 0; z < a.out.topk; ++z) {
                        const int ci = ok ? tkI[z] : -1;
                        a.out.topk_macro[q * a.out.topk + z] = ci >= 0 ? __ldg(im.macro_id + ci) : -1;
                        a.out.topk_lat[q * a.out.topk + z] =
                            ci >= 0 ? tkL[z] : __longlong_as_double(0x7ff8000000000000LL);
                    }
                }
            }
        }
    }
}

// ------------------------------------------------ grouped GEMM (warp/query)
__global__ void __launch_bounds__(256) k_grouped(DevImage im, GroupedArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = warp; q < a.n; q += nwarps) {
        const int64_t r0 = a.row_off[q], r1 = a.row_off[q + 1];
        const int32_t N = a.N[q], K = a.K[q];
        uint32_t status = 0;
        if (N < 1 || K < 1) status = WT_INVALID_ARGUMENT;  // kernel_map.cpp:247-248
        for (int64_t r = r0 + lane; r < r1 && !status; r += 32)
            if (a.rows[r] < 0) status = WT_INVALID_ARGUMENT;  // :251
        status = __reduce_max_sync(0xffffffffu, status);
        double best = __longlong_as_double(0x7ff0000000000000LL);
        int bc = -1;
        uint32_t acc = 0;
        uint64_t bg = 0;
        if (!status) {
            for (int c = lane; c < im.C; c += 32) {
                const int4 tl = __ldg(im.tiles + c);
                const uint4 mg = __ldg(im.magic + c);
                uint64_t sum = 0;  // sum_i ceil(rows_i / t_m) over non-empty groups
                for (int64_t r = r0; r < r1; ++r) {
                    const int32_t rows = a.rows[r];
                    if (rows > 0) sum += cdiv_m(uint32_t(rows), mg.x, mg.w & 0xffu);
                }
                const uint32_t nt = cdiv_m(uint32_t(N), mg.y, (mg.w >> 8) & 0xffu);
                const uint32_t lk = cdiv_m(uint32_t(K), mg.z, (mg.w >> 16) & 0xffu);
                const uint64_t g = sum * nt;
                if (g == 0) {  // kernel_map.cpp:254-255: empty grid
                    acc |= 0x80000000u;
                    continue;
                }
                const uint32_t gc = g > im.RS ? im.RS : uint32_t(g);
                const uint32_t row = row_of(gc, im.mS, im.sS);
                const double4 th = ldg_row(im.theta + size_t(c) * im.R + row);
                const double gd = u64_to_f64(g), ld = u32_to_f64(lk);
                const double t = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
                acc |= __ldg(im.rowmeta + size_t(c) * im.R + row);
                if (t < best) {  // lane-local scan is ascending in c
                    best = t;
                    bc = c;
                    bg = g;
                }
                (void)tl;
            }
            // warp-shuffle argmin: smaller latency, ties -> smaller config
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, off);
                const uint64_t og = __shfl_xor_sync(0xffffffffu, bg, off);
                const bool take = (ob < best) || (ob == best && oc >= 0 && (bc < 0 || oc < bc));
                if (take) {
                    best = ob;
                    bc = oc;
                    bg = og;
                }
            }
            acc = __reduce_or_sync(0xffffffffu, acc);
            if (acc & 0x80000000u) status = WT_INVALID_ARGUMENT;
        }
        if (lane == 0) {
            if (status) {
                Final f;
                f.flags = status << 24;
                f.macro = f.micro = f.wave = -1;
                f.comps = 0;
                f.tail = 0.f;
                write_decision(a.out, q, f, 0.0, 0, 0);
            } else {
                int64_t l = 0;
                if (bc >= 0) {
                    const int4 tl = __ldg(im.tiles + bc);
                    l = int64_t((uint32_t(K) + uint32_t(tl.z) - 1) / uint32_t(tl.z));
                }
                const Final f = finish(im, bc, best, bg, l, acc);
                write_decision(a.out, q, f, best, bg, l);
            }
        }
    }
}

// ------------------------------------------------------------ K3: gather
// config index of a macro id (im.macro_id is ascending).
__device__ __forceinline__ int config_of(const DevImage& im, int32_t macro) {
    int lo = 0, hi = im.C;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(im.macro_id + mid) < macro)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Off-grid compaction: each warp buffers its off-grid query indices in a
// shared-memory slice and appends them with one global atomicAdd per ~32
// entries -- no block-wide barrier and no per-warp atomic on a hot address.
constexpr int kWarpBuf = 64;

struct WarpBuf {  // one warp's pending off-grid queries (index + dims)
    int64_t q[kWarpBuf];
    int32_t m[kWarpBuf], n[kWarpBuf], k[kWarpBuf];
};

// With a.off_key set, the drain also computes each appended query's
// grouping key for the list evaluation (wt_eval3.cu) and counts it -- work
// the HBM-bound gather absorbs, instead of a separate pass over the list.
__device__ __forceinline__ void wbuf_drain(WarpBuf& b, int& wcnt, const GatherArgs& a, int lane,
                                           const DevImage* im = nullptr) {
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(reinterpret_cast<unsigned long long*>(a.off_count), (unsigned long long)wcnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane; i < wcnt; i += 32) {
        a.off_idx[base + i] = b.q[i];
        a.off_M[base + i] = b.m[i];
        a.off_N[base + i] = b.n[i];
        a.off_K[base + i] = b.k[i];
        if (im && a.off_key) {
            const uint32_t key = eval_key(*im, b.m[i], b.n[i], b.k[i], a.key_bits, int64_t(base + i), a.key_mode);
            a.off_key[base + i] = key;
            atomicAdd(a.key_hist + key, 1u);
        }
    }
    __syncwarp();
    wcnt = 0;
}

__device__ __forceinline__ void wbuf_push(bool off, int64_t q, int32_t M, int32_t N, int32_t K, WarpBuf& b,
                                          int& wcnt, const GatherArgs& a, int lane, const DevImage* im = nullptr) {
    const unsigned mask = __ballot_sync(0xffffffffu, off);
    if (off) {
        const int at = wcnt + __popc(mask & ((1u << lane) - 1u));
        b.q[at] = q;
        b.m[at] = M;
        b.n[at] = N;
        b.k[at] = K;
    }
    wcnt += __popc(mask);
    if (wcnt > 32) wbuf_drain(b, wcnt, a, lane, im);
}

__device__ __forceinline__ void wbuf_flush(WarpBuf& b, int& wcnt, const GatherArgs& a, int lane,
                                           const DevImage* im = nullptr) {
    if (wcnt > 0) wbuf_drain(b, wcnt, a, lane, im);
}

// One query: returns true when answered from the grid (writes optional
// outputs); the caller stores the required three.
__device__ __forceinline__ bool gather_one(const DevImage& im, const GatherArgs& a, const uint64_t* keys,
                                           const int32_t* pid, int64_t q, int32_t M, int32_t N, int32_t K,
                                           bool full, int4* lo_out) {
    const uint64_t key = (uint64_t(uint32_t(N)) << 32) | uint32_t(K);
    int lo = 0, hi = a.n_pairs;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    if (!(lo < a.n_pairs && keys[lo] == key && M >= a.m_lo && M <= a.m_hi)) return false;
    const int64_t e = int64_t(pid[lo]) * a.mcount + (M - a.m_lo);
    const int4* src = reinterpret_cast<const int4*>(a.entries + e);
    *lo_out = __ldg(src);
    const DecOut& o = a.out;
    if (full) {
        const int4 hi4 = __ldg(src + 1);
        if (o.wave) o.wave[q] = hi4.x;
        if (o.flags) o.flags[q] = uint32_t(hi4.y);
        if (o.comps) o.comps[q] = hi4.z;
        if (o.tail) o.tail[q] = double(__int_as_float(hi4.w));
    }
    if (o.g || o.l) {
        const int c = lo_out->z >= 0 ? config_of(im, lo_out->z) : -1;
        uint64_t g = 0;
        int64_t l = 0;
        if (c >= 0) {
            const int4 tl = __ldg(im.tiles + c);
            g = uint64_t((uint32_t(M) + uint32_t(tl.x) - 1) / uint32_t(tl.x)) *
                uint64_t((uint32_t(N) + uint32_t(tl.y) - 1) / uint32_t(tl.y));
            l = int64_t((uint32_t(K) + uint32_t(tl.z) - 1) / uint32_t(tl.z));
        }
        if (o.g) o.g[q] = int64_t(g);
        if (o.l) o.l[q] = l;
    }
    if (o.topk_macro)
        for (int z = 0; z < o.topk; ++z) {
            o.topk_macro[q * o.topk + z] = a.topk_macro[e * o.topk + z];
            o.topk_lat[q * o.topk + z] = a.topk_lat[e * o.topk + z];
        }
    return true;
}

// V = 4: four consecutive queries per thread with 16-byte loads/stores
// (requires 16-byte aligned arrays); V = 1: scalar.
// PF: software pipelining -- the next grid-stride iteration's M/N/K vectors
// are loaded before the current ones are looked up, so HBM reads overlap the
// dependent L2 grid reads and the stores.
template <int V, bool PF, int MINB>
__global__ void __launch_bounds__(kGatherThreads, MINB) k_gather(DevImage im, GatherArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    int32_t* pid = reinterpret_cast<int32_t*>(keys + a.n_pairs);
    __shared__ WarpBuf wbuf[kGatherThreads / 32];
    for (int i = threadIdx.x; i < a.n_pairs; i += blockDim.x) {
        keys[i] = a.pair_keys[i];
        pid[i] = a.pair_ids[i];
    }
    __syncthreads();
    const DecOut& o = a.out;
    const bool full = o.wave || o.flags || o.comps || o.tail;
    const int lane = threadIdx.x & 31;
    WarpBuf& slice = wbuf[threadIdx.x >> 5];
    int wcnt = 0;
    const int64_t n = a.n;
    const int64_t nv = n / V;  // full vectors
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int4 pm = make_int4(0, 0, 0, 0), pn = pm, pk = pm;  // prefetched vectors (PF)
    if constexpr (PF && V == 4) {
        const int64_t v0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
        if (v0 < nv) {
            pm = __ldcs(reinterpret_cast<const int4*>(a.M) + v0);
            pn = __ldcs(reinterpret_cast<const int4*>(a.N) + v0);
            pk = __ldcs(reinterpret_cast<const int4*>(a.K) + v0);
        }
    }
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nv; base += stride) {
        const int64_t v = base + threadIdx.x;
        const bool live = v < nv;
        int32_t M[V], N[V], K[V];
        if constexpr (V == 4) {
            int4 m4 = make_int4(0, 0, 0, 0), n4 = m4, k4 = m4;
            if constexpr (PF) {
                m4 = pm;
                n4 = pn;
                k4 = pk;
                const int64_t v2 = v + stride;
                if (v2 < nv) {
                    pm = __ldcs(reinterpret_cast<const int4*>(a.M) + v2);
                    pn = __ldcs(reinterpret_cast<const int4*>(a.N) + v2);
                    pk = __ldcs(reinterpret_cast<const int4*>(a.K) + v2);
                }
            } else if (live) {
                m4 = __ldcs(reinterpret_cast<const int4*>(a.M) + v);
                n4 = __ldcs(reinterpret_cast<const int4*>(a.N) + v);
                k4 = __ldcs(reinterpret_cast<const int4*>(a.K) + v);
            }
            M[0] = m4.x; M[1] = m4.y; M[2] = m4.z; M[3] = m4.w;
            N[0] = n4.x; N[1] = n4.y; N[2] = n4.z; N[3] = n4.w;
            K[0] = k4.x; K[1] = k4.y; K[2] = k4.z; K[3] = k4.w;
        } else {
            M[0] = live ? __ldcs(a.M + v) : 0;
            N[0] = live ? __ldcs(a.N + v) : 0;
            K[0] = live ? __ldcs(a.K + v) : 0;
        }
        int32_t mac[V], mic[V];
        double lat[V];
        bool on[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            int4 lo4 = make_int4(0, 0, -1, -1);
            on[j] = live && gather_one(im, a, keys, pid, v * V + j, M[j], N[j], K[j], full, &lo4);
            mac[j] = lo4.z;
            mic[j] = lo4.w;
            lat[j] = __hiloint2double(lo4.y, lo4.x);
        }
        if (live) {
            if constexpr (V == 4) {
                // off-grid lanes are overwritten later by the evaluation kernel
                __stcs(reinterpret_cast<int4*>(o.macro) + v, make_int4(mac[0], mac[1], mac[2], mac[3]));
                __stcs(reinterpret_cast<int4*>(o.micro) + v, make_int4(mic[0], mic[1], mic[2], mic[3]));
                __stcs(reinterpret_cast<double2*>(o.lat) + 2 * v, make_double2(lat[0], lat[1]));
                __stcs(reinterpret_cast<double2*>(o.lat) + 2 * v + 1, make_double2(lat[2], lat[3]));
            } else if (on[0]) {
                __stcs(o.macro + v, mac[0]);
                __stcs(o.micro + v, mic[0]);
                __stcs(o.lat + v, lat[0]);
            }
        }
#pragma unroll
        for (int j = 0; j < V; ++j)
            wbuf_push(live && !on[j], v * V + j, M[j], N[j], K[j], slice, wcnt, a, lane, &im);
    }
    // scalar tail (n % V queries), handled by the first warp of block 0
    if (V > 1 && blockIdx.x == 0 && threadIdx.x < 32) {
        const int64_t q = nv * V + threadIdx.x;
        const bool live = q < n;
        bool on = false;
        int32_t tM = 0, tN = 0, tK = 0;
        if (live) {
            tM = a.M[q];
            tN = a.N[q];
            tK = a.K[q];
            int4 lo4;
            on = gather_one(im, a, keys, pid, q, tM, tN, tK, full, &lo4);
            if (on) {
                o.macro[q] = lo4.z;
                o.micro[q] = lo4.w;
                o.lat[q] = __hiloint2double(lo4.y, lo4.x);
            }
        }
        wbuf_push(live && !on, q, tM, tN, tK, slice, wcnt, a, lane, &im);
    }
    wbuf_flush(slice, wcnt, a, lane, &im);
}

// Hashed gather: the common call (macro / micro / latency outputs only,
// 16-byte aligned arrays, pair table hashed at grid creation).  Per query one
// LDS.128 probe of the open-addressing (N, K) table (linear probing, load
// factor <= 1/2: almost always the only probe), an unsigned range check on M,
// then the 16-byte head of the grid entry: from the run-compressed copy in
// shared memory when it fits (RUNS; the scattered 16-byte L2 reads otherwise
// cost one L1 wavefront per lane and bound the kernel), else from L2.
// Off-grid queries take the same per-warp compaction as k_gather, but only
// in warps that hold one.
struct RunSmem {
    const int4* head;
    const int4* val;
    const uint32_t* key;
};

template <bool RUNS>
__device__ __forceinline__ bool hlookup(const int4* tab, uint32_t hmask, int bits, const GatherArgs& a,
                                        const RunSmem& rs, uint32_t mlo, uint32_t mcnt, int32_t M, int32_t N,
                                        int32_t K, int4* out) {
    uint32_t h = pair_slot(uint32_t(N), uint32_t(K), bits);
    int4 e = tab[h];
    while (e.z >= 0 && (e.x != N || e.y != K)) {
        h = (h + 1u) & hmask;
        e = tab[h];
    }
    const uint32_t dm = uint32_t(M) - mlo;
    const bool hit = e.z >= 0 && dm < mcnt;
    *out = make_int4(0, 0, -1, -1);
    if (hit) {
        if constexpr (RUNS) {
            int4 hd = rs.head[uint32_t(e.z) * uint32_t(a.runs.nblk) + (dm >> kRunBlkShift)];
            if (hd.z == INT32_MIN) {  // block with several runs
                const uint32_t flat = uint32_t(e.z) * mcnt + dm;
                uint32_t r = uint32_t(hd.x);
                while (rs.key[r + 1] <= flat) ++r;
                hd = rs.val[r];
            }
            *out = hd;
        } else {
            *out = __ldg(reinterpret_cast<const int4*>(a.entries + (int64_t(e.z) * mcnt + dm)));
        }
    }
    return hit;
}

template <bool RUNS>
__device__ __forceinline__ void gather_h_loop(const DevImage& im, const GatherArgs& a, const int4* tab,
                                              const RunSmem& rs, WarpBuf& slice) {
    const int bits = a.hbits;
    const uint32_t hmask = (1u << bits) - 1u;
    const uint32_t mlo = uint32_t(a.m_lo), mcnt = uint32_t(a.mcount);
    const int lane = threadIdx.x & 31;
    int wcnt = 0;
    const int64_t n = a.n, nv = n / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int4* M4 = reinterpret_cast<const int4*>(a.M);
    const int4* N4 = reinterpret_cast<const int4*>(a.N);
    const int4* K4 = reinterpret_cast<const int4*>(a.K);
    int4 pm = make_int4(0, 0, 0, 0), pn = pm, pk = pm;
    {
        const int64_t v0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
        if (v0 < nv) {
            pm = __ldcs(M4 + v0);
            pn = __ldcs(N4 + v0);
            pk = __ldcs(K4 + v0);
        }
    }
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nv; base += stride) {
        const int64_t v = base + threadIdx.x;
        const bool live = v < nv;
        const int32_t M[4] = {pm.x, pm.y, pm.z, pm.w}, N[4] = {pn.x, pn.y, pn.z, pn.w},
                      K[4] = {pk.x, pk.y, pk.z, pk.w};
        if (v + stride < nv) {
            pm = __ldcs(M4 + v + stride);
            pn = __ldcs(N4 + v + stride);
            pk = __ldcs(K4 + v + stride);
        }
        // phase 1: the four first probes, issued back to back
        uint32_t h[4];
        int4 e[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            h[j] = pair_slot(uint32_t(N[j]), uint32_t(K[j]), bits);
            e[j] = tab[h[j]];
        }
        // rare: collision chains
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            while (e[j].z >= 0 && (e[j].x != N[j] || e[j].y != K[j])) {
                h[j] = (h[j] + 1u) & hmask;
                e[j] = tab[h[j]];
            }
        }
        // phase 2: the four heads, issued back to back
        int4 r[4];
        uint32_t offm = 0;
        uint32_t dm[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            dm[j] = uint32_t(M[j]) - mlo;
            const bool hit = e[j].z >= 0 && dm[j] < mcnt;
            offm |= hit ? 0u : (1u << j);
            r[j] = make_int4(0, 0, -1, -1);
            if constexpr (RUNS) {
                if (hit) r[j] = rs.head[uint32_t(e[j].z) * uint32_t(a.runs.nblk) + (dm[j] >> kRunBlkShift)];
            } else {
                if (hit) r[j] = __ldg(reinterpret_cast<const int4*>(a.entries + (int64_t(e[j].z) * mcnt + dm[j])));
            }
        }
        if constexpr (RUNS) {  // rare: blocks holding several runs
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (r[j].z == INT32_MIN && !((offm >> j) & 1u)) {
                    const uint32_t flat = uint32_t(e[j].z) * mcnt + dm[j];
                    uint32_t q = uint32_t(r[j].x);
                    while (rs.key[q + 1] <= flat) ++q;
                    r[j] = rs.val[q];
                }
            }
        }
        if (live) {
            // off-grid lanes are overwritten later by the evaluation kernel
            __stcs(reinterpret_cast<int4*>(a.out.macro) + v, make_int4(r[0].z, r[1].z, r[2].z, r[3].z));
            __stcs(reinterpret_cast<int4*>(a.out.micro) + v, make_int4(r[0].w, r[1].w, r[2].w, r[3].w));
            __stcs(reinterpret_cast<double2*>(a.out.lat) + 2 * v,
                   make_double2(__hiloint2double(r[0].y, r[0].x), __hiloint2double(r[1].y, r[1].x)));
            __stcs(reinterpret_cast<double2*>(a.out.lat) + 2 * v + 1,
                   make_double2(__hiloint2double(r[2].y, r[2].x), __hiloint2double(r[3].y, r[3].x)));
        } else {
            offm = 0;
        }
        if (__any_sync(0xffffffffu, offm != 0)) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                wbuf_push((offm >> j) & 1u, v * 4 + j, M[j], N[j], K[j], slice, wcnt, a, lane, &im);
        }
    }
    // scalar tail (n % 4 queries), first warp of block 0
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const int64_t q = nv * 4 + threadIdx.x;
        const bool live = q < n;
        bool on = false;
        int32_t tM = 0, tN = 0, tK = 0;
        if (live) {
            tM = a.M[q];
            tN = a.N[q];
            tK = a.K[q];
            int4 lo4;
            on = hlookup<RUNS>(tab, hmask, bits, a, rs, mlo, mcnt, tM, tN, tK, &lo4);
            if (on) {
                a.out.macro[q] = lo4.z;
                a.out.micro[q] = lo4.w;
                a.out.lat[q] = __hiloint2double(lo4.y, lo4.x);
            }
        }
        wbuf_push(live && !on, q, tM, tN, tK, slice, wcnt, a, lane, &im);
    }
    wbuf_flush(slice, wcnt, a, lane, &im);
}

template <int MINB>
__global__ void __launch_bounds__(kGatherThreads, MINB) k_gather_h(DevImage im, GatherArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    int4* tab = reinterpret_cast<int4*>(smem);
    __shared__ WarpBuf wbuf[kGatherThreads / 32];
    const int H = 1 << a.hbits;
    for (int i = threadIdx.x; i < H; i += blockDim.x) tab[i] = a.htab[i];
    // run index: usable when built and within the reserved shared memory
    const RunIndex& ri = a.runs;
    int nr = 0;
    bool runs = false, multi = false;
    if (ri.budget > 0) {
        const int4 hd = *reinterpret_cast<const int4*>(ri.hdr);
        nr = hd.y;
        multi = hd.z != 0;
        const int64_t need = int64_t(ri.nbtot) * 16 + (multi ? int64_t(nr) * 20 + 4 : 0);
        runs = hd.x != 0 && hd.x == ri.gen && need <= ri.budget;
    }
    RunSmem rs{};
    if (runs) {
        int4* head = tab + H;
        int4* val = head + ri.nbtot;
        uint32_t* key = reinterpret_cast<uint32_t*>(val + (multi ? nr : 0));
        for (int i = threadIdx.x; i < ri.nbtot; i += blockDim.x) head[i] = ri.bhead[i];
        if (multi) {
            for (int i = threadIdx.x; i < nr; i += blockDim.x) val[i] = ri.rval[i];
            for (int i = threadIdx.x; i <= nr; i += blockDim.x) key[i] = ri.rkey[i];
        }
        rs = RunSmem{head, val, key};
    }
    __syncthreads();
    WarpBuf& slice = wbuf[threadIdx.x >> 5];
    if (runs)
        gather_h_loop<true>(im, a, tab, rs, slice);
    else
        gather_h_loop<false>(im, a, tab, rs, slice);
}

// ---- run index build (after a full sweep / wt_grid_finalize)
__device__ __forceinline__ int4 head_of(const wt_grid_entry* e, int64_t i) {
    return __ldg(reinterpret_cast<const int4*>(e + i));
}

__global__ void k_runflags(const wt_grid_entry* ent, int64_t n, int64_t mcount, uint32_t* flags, int32_t* hdr) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 a = head_of(ent, i);
    uint32_t f = 1;
    if (i % mcount != 0) {
        const int4 b = head_of(ent, i - 1);
        f = (a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w) ? 1u : 0u;
    }
    flags[i] = f;
    if (a.z == INT32_MIN) atomicOr(hdr + 3, 1);  // the block marker would be ambiguous
}

__global__ void k_runscatter(const wt_grid_entry* ent, int64_t n, const uint32_t* flags, const uint32_t* ids,
                             RunIndex ri) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t f = flags[i], id = ids[i];
    if (f) {
        ri.rkey[id] = uint32_t(i);
        ri.rval[id] = head_of(ent, i);
    }
    if (i == n - 1) {
        const uint32_t nr = id + f;
        ri.rkey[nr] = 0xffffffffu;
        ri.hdr[1] = int32_t(nr);
    }
}

// one thread per block of M values: its head, or the multi-run marker
__global__ void k_runheads(int64_t mcount, const uint32_t* flags, const uint32_t* ids, RunIndex ri) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b == 0) ri.hdr[0] = ri.hdr[3] ? 0 : ri.gen;
    if (b >= ri.nbtot) return;
    const int64_t p = b / ri.nblk, blk = b - p * ri.nblk;
    const int64_t i0 = p * mcount + (blk << kRunBlkShift);
    const int64_t i1 = p * mcount + min(mcount, (blk + 1) << kRunBlkShift);  // exclusive
    const uint32_t r = ids[i0] + flags[i0] - 1u;  // run holding the block's first entry
    const bool single = ri.rkey[r + 1] >= uint64_t(i1);
    if (single) {
        ri.bhead[b] = ri.rval[r];
    } else {
        ri.bhead[b] = make_int4(int(r), 0, INT32_MIN, 0);
        atomicOr(ri.hdr + 2, 1);
    }
}

size_t runs_temp_bytes(int64_t n) {
    return scan_scratch_bytes(n) + 2 * ((size_t(n) * 4 + 255) & ~size_t(255));
}

cudaError_t launch_runs_build(const wt_grid_entry* entries, int64_t n, int64_t mcount, const RunIndex& ri,
                              void* temp, cudaStream_t st) {
    char* t = static_cast<char*>(temp);
    const size_t arr = (size_t(n) * 4 + 255) & ~size_t(255);
    uint32_t* flags = reinterpret_cast<uint32_t*>(t);
    uint32_t* ids = reinterpret_cast<uint32_t*>(t + arr);
    const unsigned g = unsigned((n + 255) / 256);
    cudaError_t e = cudaMemsetAsync(ri.hdr, 0, 16, st);
    if (e != cudaSuccess) return e;
    k_runflags<<<g, 256, 0, st>>>(entries, n, mcount, flags, ri.hdr);
    e = scan_exclusive_u32(flags, ids, n, t + 2 * arr, st);
    if (e != cudaSuccess) return e;
    k_runscatter<<<g, 256, 0, st>>>(entries, n, flags, ids, ri);
    k_runheads<<<unsigned((ri.nbtot + 255) / 256), 256, 0, st>>>(mcount, flags, ids, ri);
    return cudaGetLastError();
}

// ------------------------------------------------- drop-in per-table helpers
__global__ void k_predict(DevImage im, PredictArgs a) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const int c = a.config[i];
    const int64_t g = a.g[i], l = a.l[i];
    int32_t st = 0;
    if (c < 0 || c >= im.C) st = WT_OUT_OF_RANGE;
    else if (g < 1 || l < 1) st = WT_INVALID_ARGUMENT;  // tuner.cpp:14-15
    double lat = __longlong_as_double(0x7ff8000000000000LL);
    int32_t w = 0, ex = 0, used = -1;
    if (!st) {
        const uint64_t S = uint64_t(im.S);
        const uint64_t w64 = (uint64_t(g) + S - 1) / S;
        const uint32_t row = uint32_t(w64 < uint64_t(im.R) ? w64 : uint64_t(im.R)) - 1u;
        const size_t rr = size_t(c) * im.R + row;
        const uint32_t meta = im.rowmeta[rr];
        w = int32_t(uint32_t(w64));
        if (meta & ROW_NO_COEFF) {
            st = WT_RUNTIME_ERROR;
        } else {
            const double4 th = im.theta[rr];
            const double gd = u64_to_f64(uint64_t(g)), ld = u64_to_f64(uint64_t(l));
            lat = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
            ex = (meta & ROW_EXTRAP) ? 1 : 0;
            used = im.used_w[rr];
        }
    }
    a.lat[i] = lat;
    if (a.wave) a.wave[i] = w;
    if (a.extrap) a.extrap[i] = ex;
    if (a.used_w) a.used_w[i] = used;
    if (a.status) a.status[i] = st;
}

// Per-config prediction for one dense query (the loop body of
// two_stage_select, tuner.cpp:135-149), for Tuned.flags reconstruction.
__global__ void k_explain(DevImage im, ExplainArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= im.C) return;
    int32_t st = 0;
    if (a.M < 1 || a.N < 1 || a.K < 1) st = WT_INVALID_ARGUMENT;
    const int4 tl = __ldg(im.tiles + c);
    uint64_t g = 0;
    int64_t l = 0;
    double lat = __longlong_as_double(0x7ff8000000000000LL);
    int32_t w = 0, used = -1;
    if (!st) {
        g = uint64_t((uint64_t(a.M) + tl.x - 1) / uint64_t(tl.x)) *
            uint64_t((uint64_t(a.N) + tl.y - 1) / uint64_t(tl.y));
        l = int64_t((uint64_t(a.K) + tl.z - 1) / uint64_t(tl.z));
        const uint64_t S = uint64_t(im.S);
        const uint64_t w64 = (g + S - 1) / S;
        const uint32_t row = uint32_t(w64 < uint64_t(im.R) ? w64 : uint64_t(im.R)) - 1u;
        const size_t rr = size_t(c) * im.R + row;
        const uint32_t meta = im.rowmeta[rr];
        w = int32_t(uint32_t(w64));
        if (meta & ROW_NO_COEFF) {
            st = WT_RUNTIME_ERROR;
        } else {
            const double4 th = im.theta[rr];
            const double gd = u64_to_f64(g), ld = u64_to_f64(uint64_t(l));
            lat = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
            used = im.used_w[rr];
        }
    }
    a.g[c] = int64_t(g);
    a.l[c] = l;
    a.wave[c] = w;
    a.used_w[c] = used;
    a.lat[c] = lat;
    a.status[c] = st;
}

__global__ void k_nearest(NearestArgs a) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    int comps = 0;
    const int k = nearest_anchor_idx(a.anchors, a.n_anchors, a.l[i], &comps);
    a.out[i] = a.anchors[k];
    if (a.comps) a.comps[i] = comps;
}

// ------------------------------------------------------------- launchers
template <int RPT, bool SPECIAL, bool WIDE, int KM>
static cudaError_t launch_sweep_t(const DevImage& im, const SweepArgs& a, int grid, size_t smem,
                                  cudaStream_t st) {
    auto fn = k_sweep<RPT, SPECIAL, WIDE, KM>;
    cudaError_t e = prepare_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kSweepThreads, smem, st>>>(im, a);
    return cudaGetLastError();
}

// ------------------------------------------ one query, one warp (latency)
// tune() for a single query: the lanes stride the configs (ascending index),
// each keeping its own strict-< winner; a shuffle reduction on (latency,
// index) then picks the smallest latency with the smallest index among ties
// -- the reference's ascending strict-< scan (tuner.cpp:114-124).  The
// result goes straight to pinned host memory, then the sequence number the
// host polls.
__global__ void __launch_bounds__(32) k_one(DevImage im, int32_t m, int32_t nn, int32_t k, OneOut* out,
                                            uint32_t seq) {
    const int lane = threadIdx.x;
    uint32_t status = 0;
    uint32_t M = 1, N = 1, K = 1;
    if (m < 1 || nn < 1 || k < 1) status = WT_INVALID_ARGUMENT;  // kernel_map.cpp:238-239
    else {
        M = uint32_t(m);
        N = uint32_t(nn);
        K = uint32_t(k);
        const uint64_t gmax = uint64_t((M + uint32_t(im.tm_min) - 1) / uint32_t(im.tm_min)) *
                              uint64_t((N + uint32_t(im.tn_min) - 1) / uint32_t(im.tn_min));
        if ((gmax + uint64_t(im.S) - 1) / uint64_t(im.S) >= (uint64_t(1) << 31)) status = WT_UNSUPPORTED;
    }
    const uint32_t y2M = 2u * (M - 1u), y2N = 2u * (N - 1u), y2K = 2u * (K - 1u);
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bc = -1;
    uint32_t acc = 0;
    if (!status) {
#pragma unroll 4
        for (int c = lane; c < im.C; c += 32) {
            const uint4 mg = __ldg(im.magic + c);
            const uint32_t mt = mdiv2(y2M, mg.x, mg.w & 0xffu) + 1u;
            const uint32_t nt = mdiv2(y2N, mg.y, (mg.w >> 8) & 0xffu) + 1u;
            const uint32_t lk = mdiv2(y2K, mg.z, (mg.w >> 16) & 0xffu) + 1u;
            const uint64_t g = uint64_t(mt) * nt;
            const uint32_t gc = g > im.RS ? im.RS : uint32_t(g);
            const uint32_t row = row_of(gc, im.mS, im.sS);
            const size_t rr = size_t(c) * im.R + row;
            const double4 th = ldg_row(im.theta + rr);
            const double gd = u64_to_f64(g), ld = u32_to_f64(lk);
            const double t = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
            if (t < best) {
                best = t;
                bc = c;
            }
            if (im.special) acc |= __ldg(im.rowmeta + rr);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, off);
        acc |= __shfl_xor_sync(0xffffffffu, acc, off);
        if (oc >= 0 && (bc < 0 || ob < best || (ob == best && oc < bc))) {
            best = ob;
            bc = oc;
        }
    }
    if (lane != 0) return;
    Final f;
    uint64_t g = 0;
    int64_t l = 0;
    if (status) {
        f.flags = status << 24;
        f.macro = f.micro = f.wave = -1;
        f.comps = 0;
        f.tail = 0.f;
    } else {
        if (bc >= 0) {
            const int4 tl = __ldg(im.tiles + bc);
            g = uint64_t((M + uint32_t(tl.x) - 1) / uint32_t(tl.x)) * uint64_t((N + uint32_t(tl.y) - 1) / uint32_t(tl.y));
            l = int64_t((K + uint32_t(tl.z) - 1) / uint32_t(tl.z));
        }
        f = finish(im, bc, best, g, l, acc);
    }
    const bool ok = (f.flags >> 24) == 0;
    out->lat = ok ? best : __longlong_as_double(0x7ff8000000000000LL);
    out->g = ok ? int64_t(g) : 0;
    out->l = ok ? l : 0;
    out->tail = ok ? double(f.tail) : 0.0;
    out->macro = ok ? f.macro : -1;
    out->micro = ok ? f.micro : -1;
    out->wave = ok ? f.wave : 0;
    out->flags = f.flags;
    out->comps = ok ? f.comps : 0;
    __threadfence_system();
    out->seq = seq;
}

cudaError_t launch_one(const DevImage& im, int32_t M, int32_t N, int32_t K, OneOut* out, uint32_t seq,
                       cudaStream_t st) {
    k_one<<<1, 32, 0, st>>>(im, M, N, K, out, seq);
    return cudaGetLastError();
}

size_t sweep_smem_bytes(const DevImage& im, int chunk, bool special) {
    size_t b = size_t(chunk) * (sizeof(SweepCfg) + sizeof(double)) + size_t(chunk) * im.R * sizeof(double4);
    if (special) b += size_t(chunk) * im.R * sizeof(uint32_t);
    return b;
}

cudaError_t launch_sweep(const DevImage& im, const SweepArgs& a, bool wide, cudaStream_t st) {
    const int64_t n = a.end - a.begin;
    if (n <= 0) return cudaSuccess;
    const bool sp = im.special != 0;
    const size_t smem = sweep_smem_bytes(im, a.chunk, sp);
    const bool tk = a.topk > 0;
    const int rpt = tk ? 1 : kSweepRPT;
    const int grid = int((n + int64_t(kSweepThreads) * rpt - 1) / (int64_t(kSweepThreads) * rpt));
    if (tk) {
        if (wide) return sp ? launch_sweep_t<1, true, true, 8>(im, a, grid, smem, st)
                            : launch_sweep_t<1, false, true, 8>(im, a, grid, smem, st);
        return sp ? launch_sweep_t<1, true, false, 8>(im, a, grid, smem, st)
                  : launch_sweep_t<1, false, false, 8>(im, a, grid, smem, st);
    }
    if (wide) return sp ? launch_sweep_t<kSweepRPT, true, true, 0>(im, a, grid, smem, st)
                        : launch_sweep_t<kSweepRPT, false, true, 0>(im, a, grid, smem, st);
    return sp ? launch_sweep_t<kSweepRPT, true, false, 0>(im, a, grid, smem, st)
              : launch_sweep_t<kSweepRPT, false, false, 0>(im, a, grid, smem, st);
}

size_t eval_smem_bytes(const DevImage& im, int chunk, bool special) {
    size_t b = size_t(chunk) * (sizeof(int4) + sizeof(uint4)) + size_t(chunk) * im.R * sizeof(double4);
    if (special) b += size_t(chunk) * im.R * sizeof(uint32_t);
    return b;
}

template <bool SPECIAL, int KM>
static cudaError_t launch_eval_t(const DevImage& im, const EvalArgs& a, int grid, size_t smem,
                                 cudaStream_t st) {
    auto fn = k_eval<SPECIAL, KM>;
    cudaError_t e = prepare_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kEvalThreads, smem, st>>>(im, a);
    return cudaGetLastError();
}

cudaError_t launch_eval(const DevImage& im, const EvalArgs& a, int grid, cudaStream_t st) {
    const bool sp = im.special != 0;
    const size_t smem = eval_smem_bytes(im, a.chunk, sp);
    if (a.out.topk > 0)
        return sp ? launch_eval_t<true, 8>(im, a, grid, smem, st) : launch_eval_t<false, 8>(im, a, grid, smem, st);
    return sp ? launch_eval_t<true, 0>(im, a, grid, smem, st) : launch_eval_t<false, 0>(im, a, grid, smem, st);
}

cudaError_t launch_grouped(const DevImage& im, const GroupedArgs& a, int grid, cudaStream_t st) {
    k_grouped<<<grid, 256, 0, st>>>(im, a);
    return cudaGetLastError();
}

// Persistent grid: exactly the CTAs that are co-resident (a grid-stride loop
// over a partly non-resident grid leaves a half-occupied second wave).
// WT_GATHER_VARIANT (A/B runs): 0 = hashed kernel when the call allows it
// (else prefetching binary-search kernel, 4 CTAs/SM); 1 = prefetch, 5
// CTAs/SM (register cap); 2 = no prefetch, 5 CTAs/SM (cap); 3 = no prefetch,
// no cap; 4 = never hashed; 5 = hashed, 4 CTAs/SM (register cap).
template <int V, bool PF, int MINB>
static cudaError_t go_gather(const DevImage& im, const GatherArgs& a, int grid, size_t smem, cudaStream_t st) {
    const void* fn = reinterpret_cast<const void*>(k_gather<V, PF, MINB>);
    grid = std::min(grid, device_sms() * occupancy(fn, kGatherThreads, 4096));
    k_gather<V, PF, MINB><<<grid, kGatherThreads, smem, st>>>(im, a);
    return cudaGetLastError();
}

// Hashed gather launch: persistent grid of co-resident CTAs; the hash table
// and the run-index budget are dynamic shared memory.
template <int MINB>
static cudaError_t go_gather_h(const DevImage& im, const GatherArgs& a, int grid, cudaStream_t st) {
    const size_t hs = (size_t(1) << a.hbits) * sizeof(int4) + size_t(a.runs.budget);
    const void* fn = reinterpret_cast<const void*>(k_gather_h<MINB>);
    const int occ = occupancy(fn, kGatherThreads, hs);  // also raises the smem limit (static + dynamic > 48 KB)
    cudaError_t e = prepare_smem(fn, hs);
    if (e != cudaSuccess) return e;
    k_gather_h<MINB><<<std::min(grid, device_sms() * occ), kGatherThreads, hs, st>>>(im, a);
    return cudaGetLastError();
}

cudaError_t launch_gather(const DevImage& im, const GatherArgs& a, int grid, cudaStream_t st) {
    const size_t smem = size_t(a.n_pairs) * (sizeof(uint64_t) + sizeof(int32_t)) + 16;
    const auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    static const int variant = [] {
        const char* v = std::getenv("WT_GATHER_VARIANT");
        return v ? std::atoi(v) : 0;
    }();
    const bool aligned =
        al16(a.M) && al16(a.N) && al16(a.K) && al16(a.out.macro) && al16(a.out.micro) && al16(a.out.lat);
    const DecOut& o = a.out;
    const bool plain = !(o.wave || o.flags || o.comps || o.tail || o.g || o.l || o.topk_macro);
    if (aligned && plain && a.htab && variant != 4)
        return variant == 5 ? go_gather_h<4>(im, a, grid, st) : go_gather_h<0>(im, a, grid, st);
    if (aligned) {
        if (variant == 1) return go_gather<4, true, 5>(im, a, grid, smem, st);
        if (variant == 2) return go_gather<4, false, 5>(im, a, grid, smem, st);
        if (variant == 3) return go_gather<4, false, 0>(im, a, grid, smem, st);
        return go_gather<4, true, 0>(im, a, grid, smem, st);
    }
    return go_gather<1, false, 0>(im, a, grid, smem, st);
}

cudaError_t launch_predict(const DevImage& im, const PredictArgs& a, cudaStream_t st) {
    const int grid = int((a.n + 255) / 256);
    if (grid > 0) k_predict<<<grid, 256, 0, st>>>(im, a);
    return cudaGetLastError();
}

cudaError_t launch_explain(const DevImage& im, const ExplainArgs& a, cudaStream_t st) {
    k_explain<<<(im.C + 127) / 128, 128, 0, st>>>(im, a);
    return cudaGetLastError();
}

cudaError_t launch_nearest(const NearestArgs& a, cudaStream_t st) {
    const int grid = int((a.n + 255) / 256);
    if (grid > 0) k_nearest<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace wtb
