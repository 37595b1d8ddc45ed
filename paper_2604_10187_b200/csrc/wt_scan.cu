// wt_scan.cu -- exclusive prefix sum of u32 counts (the off-grid grouping
// histogram, 2^20 buckets, and the run-index flags of a grid), hand-written
// in place of a library scan on the decision path.
//
// Reduce-then-scan over tiles of 4096 elements (256 threads x 16 consecutive
// elements, 16-byte loads when aligned):
//   k_scan_reduce   tile sums -> partials
//   (recursion)     exclusive scan of the partials (one tile when <= 4096)
//   k_scan_tiles    each tile scanned with its partial as the carry-in
// Two streaming passes over the input (L2-resident at the sizes used here),
// no look-back chains, deterministic; sums wrap modulo 2^32 like any u32 scan.
#include <cuda_runtime.h>

#include <cstdint>

#include "wt_decide.h"

namespace wtb {
namespace {

constexpr int kScanT = 256;
constexpr int kScanItems = 16;
constexpr int64_t kScanTile = int64_t(kScanT) * kScanItems;

__device__ __forceinline__ void load16(const uint32_t* in, int64_t i0, int64_t n, uint32_t (&v)[kScanItems]) {
    const bool vec = i0 + kScanItems <= n && (reinterpret_cast<uintptr_t>(in + i0) & 15u) == 0;
    if (vec) {
        const uint4* p = reinterpret_cast<const uint4*>(in + i0);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            const uint4 x = __ldg(p + q);
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = i0 + k < n ? __ldg(in + i0 + k) : 0u;
    }
}

// exclusive scan of one value per thread across the block; returns the total
__device__ __forceinline__ uint32_t block_exclusive(uint32_t x, uint32_t* ex) {
    __shared__ uint32_t warp_tot[kScanT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanT / 32; ++w) {
        const uint32_t t = warp_tot[w];
        if (w < wid) wpre += t;
        tot += t;
    }
    *ex = wpre + inc - x;
    __syncthreads();  // warp_tot is reused by the next call
    return tot;
}

__global__ void __launch_bounds__(kScanT) k_scan_reduce(const uint32_t* in, int64_t n, uint32_t* part) {
    const int64_t i0 = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems];
    load16(in, i0, n, v);
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += v[k];
    uint32_t ex;
    const uint32_t tot = block_exclusive(s, &ex);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// carry = exclusive prefix of this tile (null: 0)
__global__ void __launch_bounds__(kScanT) k_scan_tiles(const uint32_t* in, uint32_t* out, int64_t n,
                                                       const uint32_t* carry) {
    const int64_t i0 = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems];
    load16(in, i0, n, v);
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += v[k];
    uint32_t ex;
    block_exclusive(s, &ex);
    uint32_t run = ex + (carry ? carry[blockIdx.x] : 0u);
    uint32_t o[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        o[k] = run;
        run += v[k];
    }
    const bool vec = i0 + kScanItems <= n && (reinterpret_cast<uintptr_t>(out + i0) & 15u) == 0;
    if (vec) {
        uint4* p = reinterpret_cast<uint4*>(out + i0);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) p[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (i0 + k < n) out[i0 + k] = o[k];
    }
}

int64_t tiles_of(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

}  // namespace

size_t scan_scratch_bytes(int64_t n) {
    size_t b = 0;
    for (int64_t t = tiles_of(n); t > 1; t = tiles_of(t)) b += 2 * ((size_t(t) * 4 + 255) & ~size_t(255));
    return b + 256;
}

int scan_launches(int64_t n) {
    if (n <= 0) return 0;
    const int64_t t = tiles_of(n);
    return t == 1 ? 1 : 2 + scan_launches(t);
}

cudaError_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, int64_t n, void* scratch, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t t = tiles_of(n);
    if (t == 1) {
        k_scan_tiles<<<1, kScanT, 0, st>>>(in, out, n, nullptr);
        return cudaGetLastError();
    }
    char* p = static_cast<char*>(scratch);
    const size_t tb = (size_t(t) * 4 + 255) & ~size_t(255);
    uint32_t* part = reinterpret_cast<uint32_t*>(p);
    uint32_t* carry = reinterpret_cast<uint32_t*>(p + tb);
    k_scan_reduce<<<unsigned(t), kScanT, 0, st>>>(in, n, part);
    cudaError_t e = scan_exclusive_u32(part, carry, t, p + 2 * tb, st);
    if (e != cudaSuccess) return e;
    k_scan_tiles<<<unsigned(t), kScanT, 0, st>>>(in, out, n, carry);
    return cudaGetLastError();
}

}  // namespace wtb
