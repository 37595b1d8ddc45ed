// wt_baseline.cu -- the reference's ablation baselines on the GPU
// (reference tuner.cpp:168-250).
//
// baseline_tune() is two_stage_select with another Stage I predictor:
//   step:   T = t_wave[(macro, nearest step anchor of l)] * wave_count(g)
//   linear: T = theta_macro.predict(g, l)  (one bilinear fit, no regimes)
// Regime = {w > W, w} and Stage II (retrieve_micro on the dual tables) are
// unchanged, so the winner goes through the same finish() as tune().  The
// step product is one rounded DMUL of t and (double)w, as in the reference.
#include <cuda_runtime.h>

#include "wavetune_c.h"
#include "wt_decide.h"
#include "wt_device.cuh"

namespace wtb {
namespace {

constexpr int kBThreads = 256;

// baseline latency of config c (entry present) for (g, w, l)
__device__ __forceinline__ double bvalue(const BaseImage& b, int c, uint64_t g, double gd, uint64_t w, int64_t l,
                                         double ld) {
    if (b.kind == WT_BASELINE_LINEAR) {
        const double4 th = b.theta[c];
        return bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
    }
    const int o = b.off[c], n = b.off[c + 1] - o;
    int comps;
    const int k = nearest_anchor_idx(b.al + o, n, l, &comps);
    (void)g;
    return __dmul_rn(b.tw[o + k], u64_to_f64(w));
}

__global__ void __launch_bounds__(kBThreads) k_btune(DevImage im, BaseImage b, EvalArgs a) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < a.n; q += stride) {
        const int32_t m = a.M[q], nn = a.N[q], k = a.K[q];
        uint32_t status = 0, M = 1, N = 1, K = 1;
        if (m < 1 || nn < 1 || k < 1) status = WT_INVALID_ARGUMENT;  // kernel_map.cpp:238-239
        else {
            M = uint32_t(m);
            N = uint32_t(nn);
            K = uint32_t(k);
            const uint64_t gmax = uint64_t((M + uint32_t(im.tm_min) - 1) / uint32_t(im.tm_min)) *
                                  uint64_t((N + uint32_t(im.tn_min) - 1) / uint32_t(im.tn_min));
            if ((gmax + uint64_t(im.S) - 1) / uint64_t(im.S) >= (uint64_t(1) << 31)) status = WT_UNSUPPORTED;
            else if (b.missing) status = WT_OUT_OF_RANGE;  // baseline_predict throws (tuner.cpp:226-238)
        }
        Final f;
        double best = __longlong_as_double(0x7ff0000000000000LL);
        uint64_t bg = 0;
        int64_t bl = 0;
        if (status) {
            f.flags = status << 24;
            f.macro = f.micro = f.wave = -1;
            f.comps = 0;
            f.tail = 0.f;
        } else {
            const uint32_t y2M = 2u * (M - 1u), y2N = 2u * (N - 1u), y2K = 2u * (K - 1u);
            const uint64_t S = uint64_t(im.S);
            int bc = -1;
            for (int c = 0; c < im.C; ++c) {
                const uint4 mg = __ldg(im.magic + c);
                const uint32_t mt = mdiv2(y2M, mg.x, mg.w & 0xffu) + 1u;
                const uint32_t nt = mdiv2(y2N, mg.y, (mg.w >> 8) & 0xffu) + 1u;
                const uint32_t lk = mdiv2(y2K, mg.z, (mg.w >> 16) & 0xffu) + 1u;
                const uint64_t g = uint64_t(mt) * nt;
                const double t = bvalue(b, c, g, u64_to_f64(g), (g + S - 1) / S, int64_t(lk), u32_to_f64(lk));
                if (t < best) {
                    best = t;
                    bc = c;
                    bg = g;
                    bl = int64_t(lk);
                }
            }
            f = finish(im, bc, best, bg, bl, 0u);
        }
        write_decision(a.out, q, f, best, bg, bl);
    }
}

// baseline_predict (tuner.cpp:222-239): out_of_range when the macro has no
// entry, then (step) invalid_argument from wave_count for g < 1.
__global__ void k_bpredict(BaseImage b, BPredictArgs a) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= a.n) return;
    const int32_t mac = a.macro[q];
    int lo = 0, hi = b.C;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (b.macro[mid] < mac) lo = mid + 1;
        else hi = mid;
    }
    const int64_t g = a.g[q], l = a.l[q];
    if (lo == b.C || b.macro[lo] != mac || !b.has[lo]) {
        a.status[q] = WT_OUT_OF_RANGE;
        a.lat[q] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    if (b.kind == WT_BASELINE_LINEAR) {
        const double4 th = b.theta[lo];
        const double gd = __ll2double_rn(g), ld = __ll2double_rn(l);
        a.lat[q] = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
        a.status[q] = WT_OK;
        return;
    }
    if (g < 1 || b.S < 1) {
        a.status[q] = WT_INVALID_ARGUMENT;
        a.lat[q] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    const uint64_t w = (uint64_t(g) + uint64_t(b.S) - 1) / uint64_t(b.S);
    a.lat[q] = bvalue(b, lo, uint64_t(g), 0.0, w, l, 0.0);
    a.status[q] = WT_OK;
}

}  // namespace

cudaError_t launch_btune(const DevImage& im, const BaseImage& b, const EvalArgs& a, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    const int64_t blocks = (a.n + kBThreads - 1) / kBThreads;
    k_btune<<<int(blocks < 148 * 16 ? blocks : 148 * 16), kBThreads, 0, st>>>(im, b, a);
    return cudaGetLastError();
}

cudaError_t launch_bpredict(const BaseImage& b, const BPredictArgs& a, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    k_bpredict<<<int((a.n + 255) / 256), 256, 0, st>>>(b, a);
    return cudaGetLastError();
}

}  // namespace wtb
