// wt_wide.cu -- queries with 64-bit dimensions.
//
// The reference's workloads carry i64 dims (DenseGemm{i64 m, n, k},
// kernel_map.hpp:25-27; map_workload's i64 products, kernel_map.cpp:235-264).
// The batched kernels take int32 dims (half the query bytes on the HBM-bound
// gather), so the i64 entry points (wt_tune_batch_i64 / wt_gather_batch_i64)
// run in three stream-ordered steps with no host synchronisation:
//   k_narrow  dims that fit int32 are copied down; a query with any dim
//             >= 2^31 gets the placeholder (1, 1, 1) and its index is
//             appended to a wide list (one atomic per query, rare);
//   the int32 path (list evaluation / grid gather) on the narrowed arrays;
//   k_wide    warp per wide query, every config in 64-bit integer
//             arithmetic: G = ceil(m/t_m) * ceil(n/t_n), L = ceil(k/t_k),
//             wave row = min(ceil(G/S), R) - 1, the same bilinear in the
//             reference's association, warp-shuffle (latency, config) argmin,
//             Stage II -- overwriting the placeholder's answer.
// Guards mirror the int32 path: any dim < 1 -> INVALID_ARGUMENT
// (kernel_map.cpp:238-239); a tile product above 2^63 or ceil(G/S) >= 2^31
// for the smallest tile (wave_count's int, kernel_map.cpp:267-272) ->
// UNSUPPORTED.
#include <cuda_runtime.h>

#include <climits>

#include "wt_decide.h"
#include "wt_device.cuh"

namespace wtb {

__global__ void k_narrow(WideArgs a) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < a.n; q += stride) {
        const int64_t m = a.M[q], n = a.N[q], k = a.K[q];
        int32_t m32, n32, k32;
        if (m < 1 || n < 1 || k < 1) {
            m32 = 0;  // invalid either way: the int32 path flags it
            n32 = k32 = 1;
        } else if (m > INT_MAX || n > INT_MAX || k > INT_MAX) {
            m32 = n32 = k32 = 1;
            a.list[atomicAdd(a.count, 1ull)] = q;
        } else {
            m32 = int32_t(m);
            n32 = int32_t(n);
            k32 = int32_t(k);
        }
        a.M32[q] = m32;
        a.N32[q] = n32;
        a.K32[q] = k32;
    }
}

__device__ __forceinline__ uint64_t cdiv64(uint64_t x, uint64_t d) { return x / d + (x % d != 0); }

__global__ void __launch_bounds__(256) k_wide(DevImage im, WideArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t cnt = int64_t(*a.count);
    const uint64_t S = uint64_t(im.S);
    for (int64_t w = warp; w < cnt; w += nwarps) {
        const int64_t q = a.list[w];
        const uint64_t M = uint64_t(a.M[q]), N = uint64_t(a.N[q]), K = uint64_t(a.K[q]);
        uint32_t status = 0;
        {  // the smallest tile gives the largest grid
            const uint64_t mt = cdiv64(M, uint64_t(im.tm_min)), nt = cdiv64(N, uint64_t(im.tn_min));
            const uint64_t gmax = mt * nt;
            if (__umul64hi(mt, nt) != 0 || (gmax >> 63) != 0 || cdiv64(gmax, S) >= (uint64_t(1) << 31))
                status = WT_UNSUPPORTED;
        }
        double best = __longlong_as_double(0x7ff0000000000000LL);
        int bc = -1;
        uint32_t acc = 0;
        uint64_t bg = 0, bl = 0;
        if (!status) {
            for (int c = lane; c < im.C; c += 32) {
                const int4 tl = __ldg(im.tiles + c);
                const uint64_t g = cdiv64(M, uint64_t(tl.x)) * cdiv64(N, uint64_t(tl.y));
                const uint64_t lk = cdiv64(K, uint64_t(tl.z));
                const uint64_t wv = cdiv64(g, S);
                const uint32_t row = uint32_t(wv < uint64_t(im.R) ? wv : uint64_t(im.R)) - 1u;
                const double4 th = ldg_row(im.theta + size_t(c) * im.R + row);
                const double gd = u64_to_f64(g), ld = u64_to_f64(lk);
                const double t = bilinear(th.x, th.y, __dmul_rn(th.z, ld), th.w, gd, ld);
                acc |= __ldg(im.rowmeta + size_t(c) * im.R + row);
                if (t < best) {  // lane-local scan is ascending in c
                    best = t;
                    bc = c;
                    bg = g;
                    bl = lk;
                }
            }
            // warp-shuffle argmin: smaller latency, ties -> smaller config
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, off);
                const uint64_t og = __shfl_xor_sync(0xffffffffu, bg, off);
                const uint64_t ol = __shfl_xor_sync(0xffffffffu, bl, off);
                const bool take = (ob < best) || (ob == best && oc >= 0 && (bc < 0 || oc < bc));
                if (take) {
                    best = ob;
                    bc = oc;
                    bg = og;
                    bl = ol;
                }
            }
            acc = __reduce_or_sync(0xffffffffu, acc);
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
                const Final f = finish(im, bc, best, bg, int64_t(bl), acc);
                write_decision(a.out, q, f, best, bg, int64_t(bl));
            }
        }
    }
}

cudaError_t launch_narrow(const WideArgs& a, cudaStream_t st) {
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>((a.n + 255) / 256, int64_t(device_sms()) * 8)));
    k_narrow<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_wide(const DevImage& im, const WideArgs& a, cudaStream_t st) {
    // the wide count is on the device: size for the worst case, idle warps exit
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>((a.n + 7) / 8, int64_t(device_sms()) * 8)));
    k_wide<<<grid, 256, 0, st>>>(im, a);
    return cudaGetLastError();
}

}  // namespace wtb
