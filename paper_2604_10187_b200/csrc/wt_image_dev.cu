// wt_image_dev.cu -- the device image built on the device.
//
// Input: dual tables as CSR already resident in HBM (uploaded by
// wt_engine_create, or produced there by the K2 fit) plus the host plan of
// wt_image.cpp (sorted order, registry join, tile classes / segments).
// Two kernels resolve what the host used to (612 ms single-threaded for
// config 3 in round 1):
//   k_img_rows   thread / (config, wave row): wt_rows.h resolve_row -- the
//                W horizon, missing-wave and anchor fallbacks -- written to
//                the config-ordered, class-ordered and row-major copies;
//   k_img_prune  warp / (tile class, wave row, L bucket) cell: the four
//                per-corner leaders by a lexicographic (value, position)
//                warp argmin, then one lane per config of each segment runs
//                the fp64 dominance test (wt_rows.h dominated) against them;
//                the ballot is the segment's mask word.  segor (OR of the
//                segment's row flags) comes from the same warp.
// Roofline: the rows are ~C * R * 80 B of writes (config 3: 15 MB, ~3 us at
// HBM speed); the prune cells do O(class size) fp64 work each and are
// latency-bound -- both are a few microseconds against the sweep they feed.
#include <cuda_runtime.h>

#include "wt_decide.h"
#include "wt_image_dev.h"
#include "wt_rows.h"

namespace wtb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__global__ void k_img_rows(TabView T, ImgRowsArgs a) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= int64_t(a.C) * a.R) return;
    const int32_t c = int32_t(i / a.R), r = int32_t(i - int64_t(c) * a.R);
    RowOut ro;
    resolve_row(T, a.order[c], r, a.R, &ro);
    double4 th = make_double4(0.0, 0.0, 0.0, 0.0);
    if (ro.theta) th = make_double4(ro.theta[0], ro.theta[1], ro.theta[2], ro.theta[3]);
    const size_t row = size_t(c) * a.R + r;
    a.theta[row] = th;
    a.rowmeta[row] = ro.meta;
    a.used_w[row] = ro.used_w;
    a.amap[row] = make_int2(ro.a_off, ro.a_cnt);
    a.afb[row] = ro.afb;
    const int32_t pos = a.cfg_pos[c];
    a.theta2[size_t(pos) * a.R + r] = th;
    a.meta2[size_t(pos) * a.R + r] = ro.meta;
    a.theta2t[size_t(r) * a.C + pos] = th;
    a.meta2t[size_t(r) * a.C + pos] = ro.meta;
    if (ro.meta & ROW_SPECIAL) atomicOr(a.special, 1u);
}

__device__ __forceinline__ bool lex_less(double v, int32_t p, double w, int32_t q) {
    // (value, position) order; p < 0 = none (never less)
    if (p < 0) return false;
    if (q < 0) return true;
    return v < w || (v == w && p < q);
}

__global__ void __launch_bounds__(256) k_img_prune(ImgPruneArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t cell = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (cell >= a.ncells) return;
    const int32_t lb = int32_t(cell % kLB);
    const int32_t r = int32_t((cell / kLB) % a.R);
    const int32_t k = int32_t(cell / (int64_t(kLB) * a.R));
    const int32_t s0 = a.cls_seg[k], s1 = a.cls_seg[k + 1];
    const int32_t p0 = a.seg_pos[s0], p1 = s1 < a.nseg ? a.seg_pos[s1] : a.C;
    const Cell cl = cell_of(r, lb, a.R, a.S);
    const int R = a.R;
    auto row = [&](int32_t pos) { return a.theta2 + (size_t(pos) * R + r); };
    // per-corner leaders: each lane scans its positions in ascending order
    // (strict < keeps the first), then a lexicographic warp argmin
    double bv[4] = {0.0, 0.0, 0.0, 0.0};
    int32_t bp[4] = {-1, -1, -1, -1};
    for (int32_t pos = p0 + lane; pos < p1; pos += 32) {
        const double4 t4 = *row(pos);
        const double t[4] = {t4.x, t4.y, t4.z, t4.w};
        if (!prunable(t, a.meta2[size_t(pos) * R + r])) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double v = corner_value(t, cl.Gs[q >> 1], cl.Ls[q & 1]);
            if (!isfinite(v)) continue;
            if (bp[q] < 0 || v < bv[q]) {
                bv[q] = v;
                bp[q] = pos;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const double ov = __shfl_xor_sync(FULL, bv[q], off);
            const int32_t op = __shfl_xor_sync(FULL, bp[q], off);
            if (lex_less(ov, op, bv[q], bp[q])) {
                bv[q] = ov;
                bp[q] = op;
            }
        }
    // the four leaders' rows in shared memory (warp-uniform, read as
    // broadcasts): 32 registers fewer per lane, more resident warps
    __shared__ double slt[8][4][4];
    double(*const lt)[4] = slt[threadIdx.x >> 5];
    if (lane < 4) {
        int32_t pq = bp[0];
#pragma unroll
        for (int q = 1; q < 4; ++q)
            if (lane == q) pq = bp[q];
        const double4 t4 = pq >= 0 ? *row(pq) : make_double4(0.0, 0.0, 0.0, 0.0);
        lt[lane][0] = t4.x;
        lt[lane][1] = t4.y;
        lt[lane][2] = t4.z;
        lt[lane][3] = t4.w;
    }
    __syncwarp();
    for (int32_t s = s0; s < s1; ++s) {
        const int32_t ps = a.seg_pos[s], cnt = a.seg_tiles[s].w;
        bool keep = false;
        uint32_t meta = 0;
        if (lane < cnt) {
            const int32_t v = ps + lane;
            const double4 t4 = *row(v);
            const double t[4] = {t4.x, t4.y, t4.z, t4.w};
            meta = a.meta2[size_t(v) * R + r];
            bool drop = false;
            if (prunable(t, meta))
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (!drop && bp[q] >= 0 && bp[q] != v)
                        drop = dominated(t, lt[q], cl.G0, cl.G1, cl.ginf, cl.L0, cl.L1, cl.linf);
            keep = !drop;
        }
        const uint32_t m = __ballot_sync(FULL, keep);
        if (lane == 0) a.segmask[(size_t(s) * R + r) * kLB + lb] = m;
        if (lb == 0) {
            const uint32_t o = __reduce_or_sync(FULL, meta);
            if (lane == 0) a.segor[size_t(s) * R + r] = o;
        }
    }
}

}  // namespace

cudaError_t launch_image_build(const TabView& T, const ImgRowsArgs& rows, const ImgPruneArgs& prune, cudaStream_t st) {
    const int64_t nrows = int64_t(rows.C) * rows.R;
    k_img_rows<<<unsigned((nrows + 255) / 256), 256, 0, st>>>(T, rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (prune.ncells > 0) k_img_prune<<<unsigned((prune.ncells * 32 + 255) / 256), 256, 0, st>>>(prune);
    return cudaGetLastError();
}

}  // namespace wtb
