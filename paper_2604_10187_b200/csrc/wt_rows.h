// wt_rows.h -- the per-(config, wave row) resolution of the reference's
// query-time rules and the per-cell dominance test of the pruning masks,
// written once as __host__ __device__ functions.  The device image builder
// (wt_image_dev.cu, one thread per row / one warp per cell) and the host-only
// inspection plan (wt_image.cpp, wt_prune_plan) call the same code, so the
// device masks are bit-identical to the host plan the CPU tests check.
#pragma once

#include <cmath>
#include <cstdint>

#include "wt_internal.h"

#if defined(__CUDACC__)
#define WT_HD __host__ __device__ __forceinline__
#else
#define WT_HD inline
#endif

namespace wtb {

// std::vector<DualTable> as key-ascending CSR (wt_tables_desc), host or
// device pointers.  Anchor pool = anchor_l[0 .. n_anchor) followed by
// ext_l[0 .. n_ext): a wave map i sits at awave_aoff[i], table t's
// extrapolation anchors at ext_base + ext_aoff[t].  ext_cnt == null: CSR
// (count = ext_aoff[t+1] - ext_aoff[t]); else count = ext_cnt[t] (the fit's
// uncompacted per-macro slices).
struct TabView {
    const int32_t* W;
    const double* theta_ext;
    const int32_t* coeff_off;
    const int32_t* coeff_w;
    const double* coeff_theta;
    const int32_t* awave_off;
    const int32_t* awave_w;
    const int32_t* awave_aoff;
    const int32_t* ext_aoff;
    int64_t ext_base;
    const int32_t* ext_cnt;
};

struct RowOut {
    const double* theta;  // 4 coefficients, or null (ROW_NO_COEFF)
    uint32_t meta;
    int32_t used_w;       // coefficient fallback source wave or -1
    int32_t a_off, a_cnt; // Stage-II map in the pool
    int32_t afb;          // anchor fallback wave or -1
};

// Row r (wave r + 1; the last row R-1 stands for every w >= R > W_c) of
// table t, following tuner.cpp:
//   * W horizon (tuner.cpp:17-18): w > W_c -> theta_ext, extrapolated;
//   * missing wave (tuner.cpp:20-39): nearest key over ALL keys, ties to the
//     smaller key (flag missing_wave_<w>_used_<k>); empty table -> error;
//   * Stage-II map (tuner.cpp:80-103): ext anchors when extrapolated and
//     non-empty, else anchor_table[w] when non-empty, else the nearest
//     non-empty wave map to (W_c if extrapolated else w), ties to the
//     smaller wave (anchor_fallback_wave_<k>); none -> error.
WT_HD void resolve_row(const TabView& T, int32_t t, int32_t r, int32_t R, RowOut* o) {
    const int32_t w = r + 1, Wc = T.W[t];
    uint32_t meta = 0;
    const double* th = nullptr;
    int32_t used = -1;
    const bool extrap = (r == R - 1) || (w > Wc);
    if (extrap) {
        meta |= ROW_EXTRAP;
        th = T.theta_ext + 4 * int64_t(t);
    } else {
        const int32_t lo = T.coeff_off[t], hi = T.coeff_off[t + 1];
        for (int32_t i = lo; i < hi; ++i)
            if (T.coeff_w[i] == w) th = T.coeff_theta + 4 * int64_t(i);
        if (!th) {
            if (hi == lo) {
                meta |= ROW_NO_COEFF;
            } else {
                int32_t best = INT32_MAX, best_w = 0, best_i = lo;
                for (int32_t i = lo; i < hi; ++i) {
                    const int32_t d = T.coeff_w[i] > w ? T.coeff_w[i] - w : w - T.coeff_w[i];
                    if (d < best || (d == best && T.coeff_w[i] < best_w)) {
                        best = d;
                        best_w = T.coeff_w[i];
                        best_i = i;
                    }
                }
                meta |= ROW_MISSING;
                used = best_w;
                th = T.coeff_theta + 4 * int64_t(best_i);
            }
        }
    }
    int32_t off = 0, cnt = 0, fbw = -1;
    bool have = false;
    const int32_t aw0 = T.awave_off[t], aw1 = T.awave_off[t + 1];
    if (extrap) {
        const int32_t e0 = T.ext_aoff[t], e1 = T.ext_cnt ? e0 + T.ext_cnt[t] : T.ext_aoff[t + 1];
        if (e1 > e0) {
            off = int32_t(T.ext_base + e0);
            cnt = e1 - e0;
            have = true;
        }
    } else {
        for (int32_t i = aw0; i < aw1; ++i)
            if (T.awave_w[i] == w && T.awave_aoff[i + 1] > T.awave_aoff[i]) {
                off = T.awave_aoff[i];
                cnt = T.awave_aoff[i + 1] - T.awave_aoff[i];
                have = true;
            }
    }
    if (!have) {
        const int32_t target = extrap ? Wc : w;
        int32_t best = INT32_MAX, best_w = 0;
        bool found = false;
        for (int32_t i = aw0; i < aw1; ++i) {
            if (T.awave_aoff[i + 1] <= T.awave_aoff[i]) continue;  // empty maps never serve
            const int32_t d = T.awave_w[i] > target ? T.awave_w[i] - target : target - T.awave_w[i];
            if (d < best || (d == best && T.awave_w[i] < best_w)) {
                best = d;
                best_w = T.awave_w[i];
                off = T.awave_aoff[i];
                cnt = T.awave_aoff[i + 1] - T.awave_aoff[i];
                found = true;
            }
        }
        if (found) {
            meta |= ROW_ANCHOR_FB;
            fbw = best_w;
        } else {
            meta |= ROW_NO_ANCHOR;
        }
    }
    o->theta = th;
    o->meta = meta;
    o->used_w = used;
    o->a_off = off;
    o->a_cnt = cnt;
    o->afb = fbw;
}

// ---- exact pruning ------------------------------------------
// A row takes part in pruning (as victim or dominator) only when it has
// coefficients and each is 0 or of magnitude in [1e-250, 1e250]: within that
// range every fp64 product / sum below is free of overflow and underflow, so
// the relative rounding bounds of the soundness argument hold.
WT_HD bool prunable(const double* t, uint32_t meta) {
    if (meta & ROW_NO_COEFF) return false;
    for (int q = 0; q < 4; ++q) {
        const double a = fabs(t[q]);
        if (!(a == 0.0 || (a >= 1e-250 && a <= 1e250))) return false;  // also rejects NaN / inf
    }
    return true;
}

// Value of a row at a sample point, for choosing the per-corner leaders
// (any choice of dominator is sound; this only sets how much is pruned).
WT_HD double corner_value(const double* t, double G, double L) {
    return t[0] * G * L + t[1] * G + t[2] * L + t[3];
}

// Is victim v strictly slower than d, after fp64 rounding of the reference's
// evaluation, for every integer (G, L) of the cell G in [G0, G1] (G1 = inf
// when ginf), L in [L0, L1] (inf when linf)?
//
// With S_x = |a_x| G L + |b_x| G + |c_x| L + |d_x|, the reference's 7-op
// evaluation errs by at most 5.6e-16 S_x, so
//   D(G, L) = f_v - f_d - eps (S_v + S_d) > 0,  eps = 1e-9,
// implies fl(f_v) > fl(f_d).  D is bilinear with coefficients
// k_q = v_q - d_q - eps (|v_q| + |d_q|), so D > 0 on the cell iff it holds at
// the finite corners and the slopes along unbounded sides are >= 0.  Here the
// k_q and corner values are themselves fp64: they are formed with
// eps' = eps + 1e-13, whose extra margin 1e-13 (|v_q| + |d_q|) exceeds the
// rounding of both the k_q (<= 4.5e-16 (|v_q| + |d_q|)) and the corner /
// slope evaluations (<= 5.6e-16 sum |k_q| m_q): a test that passes in fp64
// passes for the exact D at eps.
WT_HD bool dominated(const double* v, const double* d, double G0, double G1, bool ginf, double L0, double L1,
                     bool linf) {
    const double eps = 1.0001e-9;
    double k[4];
    for (int q = 0; q < 4; ++q) k[q] = (v[q] - d[q]) - eps * (fabs(v[q]) + fabs(d[q]));
    const double a = k[0], b = k[1], c = k[2], e = k[3];
    if (!(((a * G0) * L0 + b * G0) + c * L0 + e > 0.0)) return false;
    if (linf ? !(a * G0 + c >= 0.0) : !(((a * G0) * L1 + b * G0) + c * L1 + e > 0.0)) return false;
    if (ginf) {
        if (!(a * L0 + b >= 0.0)) return false;
        if (linf ? !(a >= 0.0) : !(a * L1 + b >= 0.0)) return false;
    } else {
        if (!(((a * G1) * L0 + b * G1) + c * L0 + e > 0.0)) return false;
        if (linf ? !(a * G1 + c >= 0.0) : !(((a * G1) * L1 + b * G1) + c * L1 + e > 0.0)) return false;
    }
    return true;
}

// Geometry of cell (row r, L bucket lb): G in [rS+1, (r+1)S] (last row
// unbounded), L in [2^lb, 2^(lb+1)-1] (last bucket unbounded); the leader
// sample points put the unbounded sides far out.
struct Cell {
    double G0, G1, L0, L1;
    bool ginf, linf;
    double Gs[2], Ls[2];
};
WT_HD Cell cell_of(int32_t r, int32_t lb, int32_t R, int32_t S) {
    Cell c;
    c.G0 = double(r) * S + 1;
    c.G1 = double(r + 1) * S;
    c.ginf = r == R - 1;
    c.L0 = ldexp(1.0, lb);
    c.L1 = ldexp(1.0, lb + 1) - 1;
    c.linf = lb == kLB - 1;
    c.Gs[0] = c.G0;
    c.Gs[1] = c.ginf ? c.G0 * 1e6 : c.G1;
    c.Ls[0] = c.L0;
    c.Ls[1] = c.linf ? 2147483647.0 : c.L1;
    return c;
}

}  // namespace wtb
