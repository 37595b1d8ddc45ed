// wt_fit.cu -- K2: build_dual_table on the GPU (model.cpp:194-253).
//
// Pipeline over the profile records resident in HBM:
//   1. registry position of every record (group_records visits registry
//      macros only, model.cpp:131-136); invalid records dropped (order kept)
//   2. two stable radix sorts (CUB, LSD over packed field keys):
//        order A by (macro_pos, w, l, micro, g, record index)
//        order B by (macro_pos, w, l, g, record index)
//      record index order is preserved by stability, so the last write of a
//      duplicated (micro, g) wins exactly like by_micro[micro][g] = t
//   3. k_select     thread / (macro, w, l) group: select_shared_micro
//                   (model.cpp:81-120) -- full-coverage argmin of the
//                   sequential mean, else widest coverage
//   4. k_samples    selected (g, l, t) samples laid out group after group, so
//                   every (macro, w) bucket and every extrapolation window is
//                   one contiguous slice in (w asc, l asc, g asc) order
//   5. k_qfit       4 lanes / bucket (8 buckets per warp): column-scaled
//                   ColPivHouseholderQR + reduced HouseholderQR, R^2, MAPE
//                   (model.cpp:20-77), each design column owned by one lane
//   6. k_ext_prep / k_qfit / k_ext_vote: fit_extrapolation
//                   (model.cpp:140-192), the pooled window fit on the same
//                   quad-lane solver
// The QR reproduces oracle/wt_fit_core.h's operation order exactly: every
// reduction is one lane's ascending accumulation, all binary64 _rn
// arithmetic, correctly rounded sqrt/div.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "wavetune_c.h"
#include "wt_decide.h"
#include "wt_image_dev.h"
#include "wt_internal.h"

namespace wtb {
namespace fit {

constexpr unsigned FULL = 0xffffffffu;

// --------------------------------------------------- quad-lane least squares
// fit_bucket (model.cpp:20-77) with 4 lanes per problem, 8 problems per warp.
// Lane q of a quad owns one design column at a time (column pivoting only
// re-maps logical columns to owning lanes, no data moves), so every dot
// product / norm is ONE lane's plain ascending accumulation -- the order of
// oracle/wt_fit_core.h, hence bit-identical results.  The owner of the
// pivot column builds the Householder reflector, then -- while the other
// owners apply it to their columns -- applies it to the right-hand side.
// Storage: element (row r, slot s) of the problem's 4 column slots at
// A[r * la + s], its right-hand side at rhs[r * lr]; shared memory (la = 32
// across the warp's 8 problems) when n <= rows, else the problem's own
// global scratch (5 doubles per sample, la = 4).
constexpr double kEps = DBL_EPSILON;

// Lane groups.  A problem is solved by 4*SUB lanes: column owner q (0..3)
// holds sub-lanes j = 0..SUB-1.  SUB = 1 (problems of <= kQRows rows: buckets):
// every row reduction is one lane's ascending accumulation.  SUB = 8 (larger
// problems: extrapolation windows, per-macro baselines): sub-lane j owns the
// rows r = j (mod 8), accumulates them in ascending order, and the eight
// partials combine as ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7)) (xor butterfly --
// exact, since each add is commutative).  oracle/wt_fit_core.h (wtf_dot /
// wtf_qsum) fixes the same two orders by problem size, so GPU and CPU agree
// bit for bit.  Elementwise row updates are split the same way.
template <int SUB>
struct Grp {
    int q, j;     // column owner, sub-lane
    unsigned m;   // the problem's lanes
    unsigned mo;  // the owner's sub-lanes (reductions)
    // broadcast from lane `src` of the group
    __device__ __forceinline__ double bc(double v, int src) const { return __shfl_sync(m, v, src, 4 * SUB); }
    __device__ __forceinline__ double own(double v, int col) const { return bc(v, col * SUB + j); }
    __device__ __forceinline__ double red(double p) const {
        if constexpr (SUB > 1) {
            p = __dadd_rn(p, __shfl_xor_sync(mo, p, 1));
            p = __dadd_rn(p, __shfl_xor_sync(mo, p, 2));
            p = __dadd_rn(p, __shfl_xor_sync(mo, p, 4));
        }
        return p;
    }
    __device__ __forceinline__ void sync() const { __syncwarp(m); }
    __device__ __forceinline__ void sync_own() const {
        if constexpr (SUB > 1) __syncwarp(mo);
    }
    // first row >= r0 of this sub-lane
    __device__ __forceinline__ int first(int r0) const {
        if constexpr (SUB == 1) return r0;
        return r0 + ((j - r0 % SUB) % SUB + SUB) % SUB;
    }
};

// dcol (below) through the read-only path, for the batched first pass
__device__ __forceinline__ double dcol_ldg(const double* g, const double* l, int c, int r) {
    return c == 0 ? __dmul_rn(__ldg(g + r), __ldg(l + r)) : c == 1 ? __ldg(g + r) : c == 2 ? __ldg(l + r) : 1.0;
}

// design column c of sample r (model.cpp:24-32): g*l, g, l, 1
__device__ __forceinline__ double dcol(const double* g, const double* l, int c, int r) {
    return c == 0 ? __dmul_rn(g[r], l[r]) : c == 1 ? g[r] : c == 2 ? l[r] : 1.0;
}

// Householder reflector on rows [k, n) of column `col` (stride la), by the
// column owner's sub-lanes: makeHouseholderInPlace (wtf_house).  Returns tau;
// *beta = new diagonal (written to col[k] by the caller).
template <int SUB>
__device__ double q_house(const Grp<SUB>& G, double* col, int la, int k, int n, double* beta) {
    const double c0 = col[k * la];
    double tailsq = 0.0;
    if (n - k != 1) {
        double p = 0.0;
        for (int r = G.first(k + 1); r < n; r += SUB) p = __dadd_rn(p, __dmul_rn(col[r * la], col[r * la]));
        tailsq = G.red(p);
    }
    if (tailsq <= DBL_MIN) {
        *beta = c0;
        for (int r = G.first(k + 1); r < n; r += SUB) col[r * la] = 0.0;
        return 0.0;
    }
    double b = __dsqrt_rn(__dadd_rn(__dmul_rn(c0, c0), tailsq));
    if (c0 >= 0.0) b = -b;
    const double d = __dadd_rn(c0, -b);
    for (int r = G.first(k + 1); r < n; r += SUB) col[r * la] = __ddiv_rn(col[r * la], d);
    *beta = b;
    return __ddiv_rn(__dadd_rn(b, -c0), b);
}

// q_house's scalars for one lane (SUB = 1): tau, *beta, the divisor *d of
// the tail rows, *zero = the tail is zeroed instead (tailsq <= DBL_MIN).
// The caller divides (or zeroes) rows [k+1, n) and writes beta to col[k].
__device__ double q_house_scalars(const double* col, int la, int k, int n, double* beta, double* d, int* zero) {
    const double c0 = col[k * la];
    double tailsq = 0.0;
    if (n - k != 1) {
        double p = 0.0;
        for (int r = k + 1; r < n; ++r) p = __dadd_rn(p, __dmul_rn(col[r * la], col[r * la]));
        tailsq = p;
    }
    if (tailsq <= DBL_MIN) {
        *beta = c0;
        *d = 1.0;
        *zero = 1;
        return 0.0;
    }
    double b = __dsqrt_rn(__dadd_rn(__dmul_rn(c0, c0), tailsq));
    if (c0 >= 0.0) b = -b;
    *d = __dadd_rn(c0, -b);
    *zero = 0;
    *beta = b;
    return __ddiv_rn(__dadd_rn(b, -c0), b);
}

// y[k..n) -= tau v (v . y), v = [1; ess[k+1..n)] (wtf_apply), by one owner's sub-lanes
template <int SUB>
__device__ void q_apply(const Grp<SUB>& G, const double* ess, int le, double tau, double* y, int ly, int k, int n) {
    if (n - k == 1) {
        if (G.j == 0) y[k * ly] = __dmul_rn(y[k * ly], __dadd_rn(1.0, -tau));
        return;
    }
    if (tau == 0.0) return;
    double p = 0.0;
    for (int r = G.first(k + 1); r < n; r += SUB) p = __dadd_rn(p, __dmul_rn(ess[r * le], y[r * ly]));
    double tmp = G.red(p);
    tmp = __dadd_rn(tmp, y[k * ly]);
    G.sync_own();  // every sub-lane has read y[k]
    if (G.j == 0) y[k * ly] = __dadd_rn(y[k * ly], -__dmul_rn(tau, tmp));
    for (int r = G.first(k + 1); r < n; r += SUB)
        y[r * ly] = __dadd_rn(y[r * ly], -__dmul_rn(__dmul_rn(tau, ess[r * le]), tmp));
}

// upper back-substitution on rhs[0..m) with R column i at A + slot[i]
// (wtf_backsolve); one lane
__device__ void q_backsolve(const double* A, int la, const int* slot, int m, double* rhs, int lr) {
    for (int i = m - 1; i >= 0; --i) {
        double ci = rhs[i * lr];
        if (ci != 0.0) {
            ci = __ddiv_rn(ci, A[i * la + slot[i]]);
            rhs[i * lr] = ci;
            for (int j = 0; j < i; ++j) rhs[j * lr] = __dadd_rn(rhs[j * lr], -__dmul_rn(ci, A[j * la + slot[i]]));
        }
    }
}

struct FitOut {
    double c[4];
    double r2, mape;
    int degenerate;
};

// One problem per group (4*SUB lanes; lane = q*SUB + j).
template <int SUB>
__device__ FitOut group_fit(const double* g, const double* l, const double* t, int n, double* A, int la,
                            double* rhs, int lr, const Grp<SUB>& G, bool diag) {
    const int q = G.q, j = G.j;
    // 1. scaled design (model.cpp:36-41), right-hand side = t
    double mxa = 0.0;
    bool have = false;
    // rows in batches of 8: the batch's global loads are issued together
    // (one memory latency per batch, not per row), then stored / maxed in
    // row order
    constexpr int kB = SUB == 1 ? 16 : 8;  // rows per batch and lane
    for (int r0 = G.first(0); r0 < n; r0 += kB * SUB) {
        double dv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int r = r0 + u * SUB;
            dv[u] = r < n ? dcol_ldg(g, l, q, r) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int r = r0 + u * SUB;
            if (r < n) {
                A[r * la + q] = dv[u];  // the raw column, scaled in place below (one read of g / l per row)
                const double v = fabs(dv[u]);
                if (!have || v > mxa) mxa = v;
                have = true;
            }
        }
    }
    if constexpr (SUB > 1) {  // max is order-free; design columns are finite
#pragma unroll
        for (int o = 1; o < SUB; o <<= 1) {
            const double u = __shfl_xor_sync(G.mo, mxa, o);
            const bool uh = __shfl_xor_sync(G.mo, int(have), o) != 0;
            if (uh && (!have || u > mxa)) mxa = u;
            have = have || uh;
        }
    }
    const double sc = mxa > 0 ? mxa : 1.0;
    double nrm = 0.0;
    for (int r = G.first(0); r < n; r += SUB) {
        const double v = __ddiv_rn(A[r * la + q], sc);
        A[r * la + q] = v;
        nrm = __dadd_rn(nrm, __dmul_rn(v, v));
    }
    nrm = G.red(nrm);
    if (q == 0)
        for (int r0 = G.first(0); r0 < n; r0 += 8 * SUB) {
            double tv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) tv[u] = r0 + u * SUB < n ? __ldg(t + r0 + u * SUB) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (r0 + u * SUB < n) rhs[(r0 + u * SUB) * lr] = tv[u];
        }
    double scale[4], upd[4], direct[4];
    const double dn = __dsqrt_rn(nrm);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        scale[c] = G.own(sc, c);
        direct[c] = upd[c] = G.own(dn, c);
    }
    G.sync();
    // 2. ColPivHouseholderQR (model.cpp:43-45): own[c] = slot of logical column c
    int own[4] = {0, 1, 2, 3};
    double mx = upd[0];
#pragma unroll
    for (int c = 1; c < 4; ++c)
        if (upd[c] > mx) mx = upd[c];
    const double th_help = __ddiv_rn(__dmul_rn(__dmul_rn(mx, kEps), __dmul_rn(mx, kEps)), double(n));
    const double downdate_th = __dsqrt_rn(kEps);
    const int size = n < 4 ? n : 4;
    int nz = size, trans[4] = {0, 1, 2, 3};
    double maxpiv = 0.0;
    for (int k = 0; k < size; ++k) {
        int big = k;
        double bigv = upd[k];
        for (int c = k + 1; c < 4; ++c)
            if (upd[c] > bigv) {
                bigv = upd[c];
                big = c;
            }
        if (nz == size && __dmul_rn(bigv, bigv) < __dmul_rn(th_help, double(n - k))) nz = k;
        trans[k] = big;
        if (big != k) {
            int ti = own[k];
            own[k] = own[big];
            own[big] = ti;
            double tv = upd[k];
            upd[k] = upd[big];
            upd[big] = tv;
            tv = direct[k];
            direct[k] = direct[big];
            direct[big] = tv;
        }
        int lj = 0;  // logical column this lane owns
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (own[c] == q) lj = c;
        double tk = 0.0, bk = 0.0;
        if constexpr (SUB == 1) {
            // the owner forms the reflector's scalars; the quad's four lanes
            // divide the tail rows (k+1+q, step 4) -- elementwise, so the
            // same correctly rounded quotients as one lane's loop
            double dk = 0.0;
            int zero = 0;
            if (lj == k) tk = q_house_scalars(A + q, la, k, n, &bk, &dk, &zero);
            dk = G.own(dk, own[k]);
            zero = __shfl_sync(G.m, zero, own[k], 4);
            G.sync();
            double* ck = A + own[k];
            for (int r = k + 1 + q; r < n; r += 4) ck[r * la] = zero ? 0.0 : __ddiv_rn(ck[r * la], dk);
            if (lj == k) A[k * la + q] = bk;  // row k: disjoint from the tail rows
        } else {
            if (lj == k) {
                tk = q_house(G, A + q, la, k, n, &bk);
                G.sync_own();  // every sub-lane has read col[k] (c0) before it is overwritten
                if (j == 0) A[k * la + q] = bk;
            }
        }
        tk = G.own(tk, own[k]);
        bk = G.own(bk, own[k]);
        if (fabs(bk) > maxpiv) maxpiv = fabs(bk);
        G.sync();
        if (lj > k)
            q_apply(G, A + own[k], la, tk, A + q, la, k, n);
        else if (lj == k)
            q_apply(G, A + q, la, tk, rhs, lr, k, n);  // H_k on the right-hand side, in step
        G.sync();
        double nu = upd[lj], nd = direct[lj];
        if (lj > k && nu != 0.0) {
            double tq = __ddiv_rn(fabs(A[k * la + q]), nu);
            tq = __dmul_rn(__dadd_rn(1.0, tq), __dadd_rn(1.0, -tq));
            if (tq < 0.0) tq = 0.0;
            const double ratio = __ddiv_rn(nu, nd);
            const double t2 = __dmul_rn(tq, __dmul_rn(ratio, ratio));
            if (t2 <= downdate_th) {
                double sp = 0.0;
                for (int r = G.first(k + 1); r < n; r += SUB) sp = __dadd_rn(sp, __dmul_rn(A[r * la + q], A[r * la + q]));
                nd = __dsqrt_rn(G.red(sp));
                nu = nd;
            } else {
                nu = __dmul_rn(nu, __dsqrt_rn(tq));
            }
        }
        for (int c = k + 1; c < 4; ++c) {
            upd[c] = G.own(nu, own[c]);
            direct[c] = G.own(nd, own[c]);
        }
    }
    int perm[4] = {0, 1, 2, 3};
    for (int k = 0; k < size; ++k) {
        const int tv = perm[k];
        perm[k] = perm[trans[k]];
        perm[trans[k]] = tv;
    }
    const double pre = __dmul_rn(fabs(maxpiv), 1e-10);
    int rank = 0;
    for (int i = 0; i < nz; ++i) rank += fabs(A[i * la + own[i]]) > pre;

    FitOut o;
    double x[4] = {0.0, 0.0, 0.0, 0.0};
    o.degenerate = 0;
    if (rank >= 4 && n >= 4) {
        // the right-hand side already carries H_0..H_3 (nz = 4 here)
        if (q == 0 && j == 0) {
            q_backsolve(A, la, own, nz, rhs, lr);
            for (int i = 0; i < nz; ++i) x[perm[i]] = rhs[i * lr];
        }
    } else {
        // reduced fit (model.cpp:51-59): unpivoted HouseholderQR of the first
        // `keep` pivot columns of the scaled design
        o.degenerate = 1;
        int keep = rank < n ? rank : n;
        if (keep < 1) keep = 1;
        const int hs = n < keep ? n : keep;
        G.sync();  // every lane is done reading the pivoted QR
        if (q < keep)
            for (int r = G.first(0); r < n; r += SUB) A[r * la + q] = __ddiv_rn(dcol(g, l, perm[q], r), scale[perm[q]]);
        if (q == 0)
            for (int r = G.first(0); r < n; r += SUB) rhs[r * lr] = t[r];
        G.sync();
        for (int k = 0; k < hs; ++k) {
            double tk = 0.0, bk = 0.0;
            if (q == k) {
                tk = q_house(G, A + q, la, k, n, &bk);
                G.sync_own();  // every sub-lane has read col[k] before it is overwritten
                if (j == 0) A[k * la + q] = bk;
            }
            tk = G.own(tk, k);
            G.sync();
            if (q > k && q < keep)
                q_apply(G, A + k, la, tk, A + q, la, k, n);
            else if (q == k)
                q_apply(G, A + q, la, tk, rhs, lr, k, n);
            G.sync();
        }
        if (q == 0 && j == 0) {
            const int id[4] = {0, 1, 2, 3};
            q_backsolve(A, la, id, hs, rhs, lr);
            for (int c = 0; c < hs; ++c) x[perm[c]] = rhs[c * lr];
        }
    }
    {  // coefficient c = x[c] / scale[c], divided once by column c's owner
        double xq = 0.0, sq = 1.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const double xc = G.bc(x[c], 0);
            if (c == q) {
                xq = xc;
                sq = scale[c];
            }
        }
        const double cq = __ddiv_rn(xq, sq);
#pragma unroll
        for (int c = 0; c < 4; ++c) o.c[c] = G.own(cq, c);
    }
    // 3. diagnostics (model.cpp:64-75): lane (0,0) SS_res, (1,0) mean + SS_tot,
    //    (2,0) MAPE -- each a sequential pass in sample order (skipped when
    //    the caller keeps none: extrapolation windows)
    double acc = 0.0;
    o.r2 = o.mape = 0.0;
    if (!diag) return o;
    if (j == 0) {
        // rows in batches (8 / 4) whose loads issue together; sums stay in
        // ascending row order
        if (q == 1) {
            for (int r0 = 0; r0 < n; r0 += 8) {
                double tv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) tv[u] = r0 + u < n ? __ldg(t + r0 + u) : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (r0 + u < n) acc = __dadd_rn(acc, tv[u]);
            }
            const double mean = __ddiv_rn(acc, double(n));
            acc = 0.0;
            for (int r0 = 0; r0 < n; r0 += 8) {
                double tv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) tv[u] = r0 + u < n ? __ldg(t + r0 + u) : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (r0 + u < n) {
                        const double d = __dadd_rn(tv[u], -mean);
                        acc = __dadd_rn(acc, __dmul_rn(d, d));
                    }
            }
        } else if (q != 3) {
            for (int r0 = 0; r0 < n; r0 += 4) {
                double gv[4], lv[4], tv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool in = r0 + u < n;
                    gv[u] = in ? __ldg(g + r0 + u) : 0.0;
                    lv[u] = in ? __ldg(l + r0 + u) : 0.0;
                    tv[u] = in ? __ldg(t + r0 + u) : 1.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (r0 + u < n) {
                        double f = __dmul_rn(__dmul_rn(gv[u], lv[u]), o.c[0]);
                        f = __dadd_rn(f, __dmul_rn(gv[u], o.c[1]));
                        f = __dadd_rn(f, __dmul_rn(lv[u], o.c[2]));
                        f = __dadd_rn(f, __dmul_rn(1.0, o.c[3]));
                        const double d = __dadd_rn(tv[u], -f);
                        acc = q == 0 ? __dadd_rn(acc, __dmul_rn(d, d))
                                     : __dadd_rn(acc, __ddiv_rn(fabs(d), fabs(tv[u])));
                    }
            }
        }
    }
    const double ss_res = G.bc(acc, 0), ss_tot = G.bc(acc, SUB), mp = G.bc(acc, 2 * SUB);
    o.r2 = ss_tot > 0 ? __dadd_rn(1.0, -__ddiv_rn(ss_res, ss_tot)) : (ss_res < 1e-18 ? 1.0 : 0.0);
    o.mape = __ddiv_rn(mp, double(n));
    return o;
}

// --------------------------------------------------------- build pipeline
struct Rec {
    const int64_t* g;
    const int64_t* l;
    const int32_t* w;
    const int32_t* macro;
    const int32_t* micro;
    const double* lat;
};

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// registry position of each record; per-macro smallest micro id (the sort
// key carries micro - that, usually 0 bits wide)
__global__ void k_mpos(Rec rc, int64_t n, const int32_t* ids_sorted, const int32_t* pos_sorted, int nm,
                       int32_t* mpos, int32_t* valid, int32_t* has_rec, int32_t* umin_m) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t id = rc.macro[i];
    int lo = 0, hi = nm;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ids_sorted[mid] < id)
            lo = mid + 1;
        else
            hi = mid;
    }
    const bool ok = lo < nm && ids_sorted[lo] == id;
    mpos[i] = ok ? pos_sorted[lo] : INT_MAX;
    valid[i] = ok ? 1 : 0;
    if (ok) {
        has_rec[pos_sorted[lo]] = 1;  // group_records finds this macro
        atomicMin(umin_m + pos_sorted[lo], rc.micro[i]);
    }
}

// The same with a dense id -> registry position table (ids in [0, nt)):
// one load per record instead of a binary search.
__global__ void k_mpos_dense(Rec rc, int64_t n, const int32_t* table, int nt, int32_t* mpos, int32_t* valid,
                             int32_t* has_rec, int32_t* umin_m) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t id = rc.macro[i];
    const int32_t p = (id >= 0 && id < nt) ? table[id] : -1;
    const bool ok = p >= 0;
    mpos[i] = ok ? p : INT_MAX;
    valid[i] = ok ? 1 : 0;
    if (ok) {
        has_rec[p] = 1;  // group_records finds this macro
        atomicMin(umin_m + p, rc.micro[i]);
    }
}

struct Ranges {
    unsigned long long gmin, gmax, lmin, lmax;
    int wmin, wmax, umin, umax;
};

// Field ranges for the sort-key packing: a full-occupancy grid, four
// records per thread per trip (independent loads in flight), warp then
// block reductions, one set of atomics per block (a per-record atomic on 8
// hot words serialises).  The micro field is micro - (smallest micro of the
// record's macro): umin = 0, umax = its largest value over valid records.
__global__ void __launch_bounds__(256) k_ranges(Rec rc, const int64_t* idx, int64_t n, const int32_t* mpos,
                                                const int32_t* umin_m, Ranges* out) {
    unsigned long long gmin = ~0ULL, gmax = 0, lmin = ~0ULL, lmax = 0;
    int wmin = INT_MAX, wmax = INT_MIN, umin = INT_MAX, umax = INT_MIN;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    auto take = [&](int64_t r) {
        // offset by 2^63 so signed order becomes unsigned order
        const unsigned long long g = (unsigned long long)rc.g[r] ^ 0x8000000000000000ULL;
        const unsigned long long l = (unsigned long long)rc.l[r] ^ 0x8000000000000000ULL;
        const int w = rc.w[r];
        const int32_t mp = mpos[r];
        const int32_t mu = rc.micro[r];
        gmin = min(gmin, g);
        gmax = max(gmax, g);
        lmin = min(lmin, l);
        lmax = max(lmax, l);
        wmin = min(wmin, w);
        wmax = max(wmax, w);
        if (mp != INT_MAX) {
            umin = 0;
            const long long ur = (long long)mu - umin_m[mp];
            umax = max(umax, int(ur < INT_MAX ? ur : INT_MAX));
        }
    };
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        int64_t r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = idx ? idx[i + k * stride] : i + k * stride;  // idx == null: every record
#pragma unroll
        for (int k = 0; k < 4; ++k) take(r[k]);
    }
    for (; i < n; i += stride) take(idx ? idx[i] : i);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        gmin = min(gmin, __shfl_xor_sync(FULL, gmin, off));
        gmax = max(gmax, __shfl_xor_sync(FULL, gmax, off));
        lmin = min(lmin, __shfl_xor_sync(FULL, lmin, off));
        lmax = max(lmax, __shfl_xor_sync(FULL, lmax, off));
    }
    wmin = __reduce_min_sync(FULL, wmin);
    wmax = __reduce_max_sync(FULL, wmax);
    umin = __reduce_min_sync(FULL, umin);
    umax = __reduce_max_sync(FULL, umax);
    __shared__ Ranges part[8];
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) part[wid] = Ranges{gmin, gmax, lmin, lmax, wmin, wmax, umin, umax};
    __syncthreads();
    if (threadIdx.x == 0) {
        Ranges t = part[0];
        for (int k = 1; k < int(blockDim.x >> 5); ++k) {
            t.gmin = min(t.gmin, part[k].gmin);
            t.gmax = max(t.gmax, part[k].gmax);
            t.lmin = min(t.lmin, part[k].lmin);
            t.lmax = max(t.lmax, part[k].lmax);
            t.wmin = min(t.wmin, part[k].wmin);
            t.wmax = max(t.wmax, part[k].wmax);
            t.umin = min(t.umin, part[k].umin);
            t.umax = max(t.umax, part[k].umax);
        }
        atomicMin(&out->gmin, t.gmin);
        atomicMax(&out->gmax, t.gmax);
        atomicMin(&out->lmin, t.lmin);
        atomicMax(&out->lmax, t.lmax);
        atomicMin(&out->wmin, t.wmin);
        atomicMax(&out->wmax, t.wmax);
        atomicMin(&out->umin, t.umin);
        atomicMax(&out->umax, t.umax);
    }
}

struct Field {
    int which;  // 0 g, 1 micro, 2 l, 3 w, 4 mpos
    unsigned long long base;
    int bits, shift;
};
struct Pass {
    Field f[5];
    int nf, bits;
};

__global__ void k_pack(Rec rc, const int32_t* mpos, const int32_t* umin_m, const uint32_t* perm, int64_t n, Pass ps,
                       unsigned long long* key) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = perm ? int64_t(perm[i]) : i;
    // the record's fields, loaded together (the field loop below only shifts)
    const unsigned long long g = (unsigned long long)rc.g[r] ^ 0x8000000000000000ULL;
    const unsigned long long l = (unsigned long long)rc.l[r] ^ 0x8000000000000000ULL;
    const int32_t w = rc.w[r];
    const int32_t mp = mpos[r];
    unsigned long long k = 0;
    for (int q = 0; q < ps.nf; ++q) {
        const Field& f = ps.f[q];
        unsigned long long v;
        switch (f.which) {
            case 0: v = g - f.base; break;
            case 1: v = (unsigned long long)((long long)rc.micro[r] - umin_m[mp]) - f.base; break;
            case 2: v = l - f.base; break;
            case 3: v = (unsigned long long)(long long)(w) - f.base; break;
            default: v = (unsigned long long)mp; break;
        }
        k |= v << f.shift;
    }
    key[i] = k;
}

__device__ __forceinline__ bool same_group(const Rec& rc, const int32_t* mpos, int64_t a, int64_t b) {
    return mpos[a] == mpos[b] && rc.w[a] == rc.w[b] && rc.l[a] == rc.l[b];
}

__global__ void k_group_flags(Rec rc, const int32_t* mpos, const uint32_t* ordA, int64_t n, int32_t* gflag) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    gflag[i] = (i == 0 || !same_group(rc, mpos, ordA[i], ordA[i - 1])) ? 1 : 0;
}

struct KeyFields {  // order A's single packing pass: shift / width / base of g, micro, l, w, macro position
    int sg, bg, su, bu, sl, bl, sw, bw, sm, bm;
    unsigned long long base_g, base_l, base_w;
};
__device__ __forceinline__ unsigned long long kfield(unsigned long long k, int shift, int bits) {
    return bits >= 64 ? k >> shift : (k >> shift) & ((1ULL << bits) - 1ULL);
}
__device__ __forceinline__ int64_t key_g(unsigned long long k, const KeyFields& f) {
    return (long long)((kfield(k, f.sg, f.bg) + f.base_g) ^ 0x8000000000000000ULL);
}
__device__ __forceinline__ int64_t key_l(unsigned long long k, const KeyFields& f) {
    return (long long)((kfield(k, f.sl, f.bl) + f.base_l) ^ 0x8000000000000000ULL);
}
// micro id: the key holds micro - (smallest micro of the record's macro)
__device__ __forceinline__ int32_t key_micro(unsigned long long k, const KeyFields& f, const int32_t* umin_m) {
    return int32_t(kfield(k, f.su, f.bu)) + umin_m[kfield(k, f.sm, f.bm)];
}

// The same from order A's sorted packed keys (one packing pass): records
// are in one group iff their keys agree above the l field's shift.
__global__ void k_group_flags_k(const unsigned long long* keys, int64_t n, int shift_grp, int32_t* gflag) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // shift_grp = bits of the (g, micro) fields below (l, w, macro); 64: one group
    const bool same = i > 0 && (shift_grp >= 64 || (keys[i] >> shift_grp) == (keys[i - 1] >> shift_grp));
    gflag[i] = same ? 0 : 1;
}

__global__ void k_group_starts(const int32_t* gflag, const int32_t* gid, int64_t n, int64_t* gstart) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (gflag[i]) gstart[gid[i]] = i;
}

struct Groups {
    const int64_t* start;  // [G+1]
    int32_t* micro;
    int32_t* partial;
    int64_t* sel_lo;
    int64_t* sel_hi;
    int32_t* nsamp;
};

// select_shared_micro (model.cpp:81-120) on group q = [start[q], start[q+1])
__global__ void k_select(Rec rc, const uint32_t* ordA, const uint32_t* ordB, int64_t G, Groups gr) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    const int64_t s = gr.start[q], e = gr.start[q + 1];
    int32_t n_g = 0;  // |all_g|
    for (int64_t i = s; i < e; ++i)
        if (i == s || rc.g[ordB[i]] != rc.g[ordB[i - 1]]) ++n_g;
    int32_t best_micro = -1, best_cover = 0, part = 0;
    int64_t blo = s, bhi = s;
    for (int pass = 0; pass < 2 && best_micro < 0; ++pass) {
        const bool full = pass == 0;
        double best_mean = 0.0;
        for (int64_t i = s; i < e;) {
            const int32_t mu = rc.micro[ordA[i]];
            int64_t j = i;
            while (j < e && rc.micro[ordA[j]] == mu) ++j;
            int32_t cover = 0;
            double mean = 0.0;
            for (int64_t k = i; k < j; ++k)
                if (k + 1 == j || rc.g[ordA[k + 1]] != rc.g[ordA[k]]) {  // last write of this g
                    mean = __dadd_rn(mean, rc.lat[ordA[k]]);
                    ++cover;
                }
            mean = __ddiv_rn(mean, double(cover));
            if (!(full && cover != n_g)) {
                const bool better = best_micro < 0 || (full ? mean < best_mean : cover > best_cover);
                if (better) {
                    best_micro = mu;
                    best_mean = mean;
                    best_cover = cover;
                    blo = i;
                    bhi = j;
                }
            }
            i = j;
        }
        part = full ? 0 : 1;
    }
    gr.micro[q] = best_micro;
    gr.partial[q] = part;
    gr.sel_lo[q] = blo;
    gr.sel_hi[q] = bhi;
    gr.nsamp[q] = best_cover;
}

__global__ void k_samples(Rec rc, const uint32_t* ordA, int64_t G, Groups gr, const int64_t* soff, double* sg,
                          double* sl, double* st) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    int64_t o = soff[q];
    const int64_t lo = gr.sel_lo[q], hi = gr.sel_hi[q];
    for (int64_t k = lo; k < hi; ++k)
        if (k + 1 == hi || rc.g[ordA[k + 1]] != rc.g[ordA[k]]) {
            const int64_t r = ordA[k];
            sg[o] = double(rc.g[r]);
            sl[o] = double(rc.l[r]);
            st[o] = rc.lat[r];
            ++o;
        }
}

// k_select / k_samples with g and micro read from order A's sorted keys
// (one packing pass, one micro id per macro: order B = order A): only the
// latencies are gathered through the permutation.  Same operations, same
// order -- bit-identical.
__global__ void k_select_k(Rec rc, const unsigned long long* keys, KeyFields kf, const int32_t* umin_m,
                           const uint32_t* ordA, int64_t G, Groups gr) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    const int64_t s = gr.start[q], e = gr.start[q + 1];
    int32_t n_g = 0;  // |all_g|
    for (int64_t i = s; i < e; ++i)
        if (i == s || key_g(keys[i], kf) != key_g(keys[i - 1], kf)) ++n_g;
    int32_t best_micro = -1, best_cover = 0, part = 0;
    int64_t blo = s, bhi = s;
    for (int pass = 0; pass < 2 && best_micro < 0; ++pass) {
        const bool full = pass == 0;
        double best_mean = 0.0;
        for (int64_t i = s; i < e;) {
            const int32_t mu = key_micro(keys[i], kf, umin_m);
            int64_t j = i;
            while (j < e && key_micro(keys[j], kf, umin_m) == mu) ++j;
            int32_t cover = 0;
            double mean = 0.0;
            // last write of each g, in batches of 8 whose latency gathers
            // issue together; the sum stays in ascending record order
            for (int64_t k0 = i; k0 < j; k0 += 8) {
                double lv[8];
                bool take[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int64_t k = k0 + u;
                    take[u] = k < j && (k + 1 == j || key_g(keys[k + 1], kf) != key_g(keys[k], kf));
                    lv[u] = take[u] ? __ldg(rc.lat + __ldg(ordA + k)) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (take[u]) {
                        mean = __dadd_rn(mean, lv[u]);
                        ++cover;
                    }
            }
            mean = __ddiv_rn(mean, double(cover));
            if (!(full && cover != n_g)) {
                const bool better = best_micro < 0 || (full ? mean < best_mean : cover > best_cover);
                if (better) {
                    best_micro = mu;
                    best_mean = mean;
                    best_cover = cover;
                    blo = i;
                    bhi = j;
                }
            }
            i = j;
        }
        part = full ? 0 : 1;
    }
    gr.micro[q] = best_micro;
    gr.partial[q] = part;
    gr.sel_lo[q] = blo;
    gr.sel_hi[q] = bhi;
    gr.nsamp[q] = best_cover;
}

__global__ void k_samples_k(Rec rc, const unsigned long long* keys, KeyFields kf, const uint32_t* ordA, int64_t G,
                            Groups gr, const int64_t* soff, double* sg, double* sl, double* st) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    int64_t o = soff[q];
    const int64_t lo = gr.sel_lo[q], hi = gr.sel_hi[q];
    // batches of 8 records: keys and the latency gathers issue together,
    // the samples are appended in record order
    for (int64_t k0 = lo; k0 < hi; k0 += 8) {
        unsigned long long kv[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) kv[u] = k0 + u < hi ? __ldg(keys + k0 + u) : 0ull;
        bool take[8];
        double lv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t k = k0 + u;
            take[u] = k < hi && (k + 1 == hi || key_g(kv[u + 1], kf) != key_g(kv[u], kf));
            lv[u] = take[u] ? __ldg(rc.lat + __ldg(ordA + k)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (take[u]) {
                sg[o] = double(key_g(kv[u], kf));
                sl[o] = double(key_l(kv[u], kf));
                st[o] = lv[u];
                ++o;
            }
    }
}

__global__ void k_group_meta(Rec rc, const int32_t* mpos, const uint32_t* ordA, int64_t G, Groups gr, int64_t* gm,
                             int64_t* gw, int64_t* gl, int32_t* bflag, int32_t* mflag) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    const int64_t r = ordA[gr.start[q]];
    gm[q] = mpos[r];
    gw[q] = rc.w[r];
    gl[q] = rc.l[r];
    int nb = 1, nm = 1;
    if (q > 0) {
        const int64_t r0 = ordA[gr.start[q - 1]];
        nm = mpos[r0] != mpos[r];
        nb = nm || rc.w[r0] != rc.w[r];
    }
    bflag[q] = nb;
    mflag[q] = nm;
}

// k_group_meta from the sorted keys (the group's first record's key)
__global__ void k_group_meta_k(const unsigned long long* keys, KeyFields kf, int64_t G, Groups gr, int64_t* gm,
                               int64_t* gw, int64_t* gl, int32_t* bflag, int32_t* mflag) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    const unsigned long long k = keys[gr.start[q]];
    const int64_t m = int64_t(kfield(k, kf.sm, kf.bm));
    const int64_t w = (long long)(kfield(k, kf.sw, kf.bw) + kf.base_w);
    gm[q] = m;
    gw[q] = w;
    gl[q] = (long long)((kfield(k, kf.sl, kf.bl) + kf.base_l) ^ 0x8000000000000000ULL);
    int nb = 1, nm = 1;
    if (q > 0) {
        const unsigned long long k0 = keys[gr.start[q - 1]];
        nm = int64_t(kfield(k0, kf.sm, kf.bm)) != m;
        nb = nm || (long long)(kfield(k0, kf.sw, kf.bw) + kf.base_w) != w;
    }
    bflag[q] = nb;
    mflag[q] = nm;
}

__global__ void k_bucket_meta(int64_t G, const int64_t* gm, const int64_t* gw, const int64_t* soff,
                              const int32_t* bflag, const int32_t* bid, const int32_t* mflag, const int32_t* mid,
                              int64_t* b_gstart, int64_t* b_w, int64_t* b_slo, int64_t* m_bstart, int64_t* m_pos) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= G) return;
    if (bflag[q]) {
        const int b = bid[q];
        b_gstart[b] = q;
        b_w[b] = gw[q];
        b_slo[b] = soff[q];
    }
    if (mflag[q]) {
        m_bstart[mid[q]] = bid[q];
        m_pos[mid[q]] = gm[q];
    }
}

__global__ void k_bucket_tail(int64_t NB, int64_t NM, int64_t G, int64_t S_total, const int64_t* soff,
                              int64_t* b_gstart, int64_t* b_shi, int64_t* m_bstart) {
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b == 0) {
        b_gstart[NB] = G;
        m_bstart[NM] = NB;
    }
    if (b >= NB) return;
    b_shi[b] = b + 1 < NB ? soff[b_gstart[b + 1]] : S_total;
}

struct Buckets {
    int64_t nb;
    const int64_t* slo;  // sample range per bucket
    const int64_t* shi;
    double* coeff;       // [nb*4]
    double* r2;
    double* mape;
    int32_t* degen;
};

constexpr int kQWarps = 4;      // warps per CTA of the small-problem fit (128 threads)
constexpr int kQRows = 24;      // problems of <= 24 samples: 4 lanes each, shared memory, sequential sums
                                // (= WTF_QROWS of oracle/wt_fit_core.h: the two orders switch there)
constexpr int kORows = 256;     // larger problems: a warp each (octet order), shared memory up to this size
constexpr int kOWarps = 4;
constexpr int kQScr = 5;        // global scratch doubles per sample (problems above kORows)

// Problems of <= kQRows samples: quad p of warp w takes problem 8w + p
// (grid-stride).  Shared slab per warp: [kQRows][32] column slots +
// [kQRows][8] right-hand sides.  Larger problems are k_ofit's.
__global__ void __launch_bounds__(32 * kQWarps, 6) k_qfit(const double* sg, const double* sl, const double* st,
                                                       Buckets b) {
    __shared__ double slab[kQWarps][kQRows * 40];
    const int lane = threadIdx.x & 31, q = lane & 3, pq = lane >> 2;
    Grp<1> G{q, 0, 0xFu << (lane & ~3), 0u};
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    double* sA = slab[threadIdx.x >> 5];
    double* sR = sA + kQRows * 32;
    for (int64_t base = warp * 8; base < b.nb; base += nw * 8) {
        const int64_t pi = base + pq;
        if (pi >= b.nb) continue;
        const int64_t lo = b.slo[pi], n = b.shi[pi] - lo;
        if (n <= 0 || n > kQRows) continue;
        const FitOut o =
            group_fit<1>(sg + lo, sl + lo, st + lo, int(n), sA + pq * 4, 32, sR + pq, 8, G, b.r2 || b.mape);
        if (q == 0) {
            for (int c = 0; c < 4; ++c) b.coeff[4 * pi + c] = o.c[c];
            if (b.r2) b.r2[pi] = o.r2;
            if (b.mape) b.mape[pi] = o.mape;
            b.degen[pi] = o.degenerate;
        }
        __syncwarp(G.m);  // the slab is reused by the quad's next problem
    }
}

// Problems of more than kQRows samples: a warp each (8 lanes per design
// column, octet order), in a [kORows][5] shared slab or -- above kORows --
// the problem's own global scratch (5 doubles per sample).
__global__ void __launch_bounds__(32 * kOWarps) k_ofit(const double* sg, const double* sl, const double* st,
                                                       Buckets b, double* gscr, int span) {
    __shared__ double slab[kOWarps][kORows * 5];
    const int lane = threadIdx.x & 31;
    Grp<8> G{lane >> 3, lane & 7, 0xffffffffu, 0xFFu << (lane & 24)};
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    double* sA = slab[threadIdx.x >> 5];
    // the warp scans `span` (<= 32) problems at a time (one per lane) and
    // solves the large ones among them in ascending order: span 32 when few
    // problems are large (buckets), 1 when most are (pooled windows)
    for (int64_t base = warp * span; base < b.nb; base += nw * span) {
        const int64_t mine = base + lane;
        const bool big = lane < span && mine < b.nb && b.shi[mine] - b.slo[mine] > kQRows;
        for (unsigned todo = __ballot_sync(0xffffffffu, big); todo; todo &= todo - 1u) {
            const int64_t pi = base + (__ffs(int(todo)) - 1);
            const int64_t lo = b.slo[pi], n = b.shi[pi] - lo;
            // two call sites: the shared slab's loads compile to LDS (a
            // pointer that may be either space would take generic loads)
            FitOut o;
            if (n <= kORows) {
                o = group_fit<8>(sg + lo, sl + lo, st + lo, int(n), sA, 4, sA + 4 * n, 1, G, b.r2 || b.mape);
            } else {
                double* A = gscr + kQScr * lo;
                o = group_fit<8>(sg + lo, sl + lo, st + lo, int(n), A, 4, A + 4 * n, 1, G, b.r2 || b.mape);
            }
            if (lane == 0) {
                for (int c = 0; c < 4; ++c) b.coeff[4 * pi + c] = o.c[c];
                if (b.r2) b.r2[pi] = o.r2;
                if (b.mape) b.mape[pi] = o.mape;
                b.degen[pi] = o.degenerate;
            }
            __syncwarp();  // the slab is reused by the warp's next problem
        }
    }
}

// fit_bucket over every problem of b: small ones on quads, large ones on
// warps.  `pooled` = the list is mostly large problems (extrapolation
// windows, per-macro baselines): the quad kernel is sized for few problems.
cudaError_t launch_qfit(bool pooled, const double* sg, const double* sl, const double* st, const Buckets& b,
                        double* gscr, int nsm, cudaStream_t s) {
    if (b.nb <= 0) return cudaSuccess;
    const int64_t cap = int64_t(nsm) * 16;
    const int gq = int(std::max<int64_t>(1, std::min<int64_t>((b.nb + 8 * kQWarps - 1) / (8 * kQWarps),
                                                              pooled ? int64_t(nsm) : cap)));
    k_qfit<<<gq, 32 * kQWarps, 0, s>>>(sg, sl, st, b);
    const int span = pooled ? 1 : 32;
    const int go = int(std::max<int64_t>(1, std::min<int64_t>((b.nb + span * kOWarps - 1) / (span * kOWarps),
                                                              pooled ? cap : int64_t(nsm) * 2)));
    k_ofit<<<go, 32 * kOWarps, 0, s>>>(sg, sl, st, b, gscr, span);
    return cudaGetLastError();
}

// ---- ablation baselines (tuner.cpp:168-220) from the selected samples.
// Sample range of each macro: its groups are contiguous and in (w, l) order,
// exactly the order selected_samples() appends them (tuner.cpp:174-187).
__global__ void k_macro_samples(int64_t NM, const int64_t* mbs, const int64_t* bgs, const int64_t* soff,
                                int64_t G, int64_t S_total, int64_t* mslo, int64_t* mshi) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= NM) return;
    const int64_t g0 = bgs[mbs[q]], g1 = bgs[mbs[q + 1]];
    mslo[q] = soff[g0];
    mshi[q] = g1 < G ? soff[g1] : S_total;
}

// fit_step_baseline: per (macro, l), num += w*t, den += w*w in sample order,
// t_wave = num/den.  One thread per macro walks its groups sequentially (the
// reference's summation order); slots live at the macro's first group index
// and come out sorted by l (the std::map order).
__global__ void k_step(int64_t NM, const int64_t* mbs, const int64_t* bgs, const int64_t* gw, const int64_t* gl,
                       const int64_t* soff, const int32_t* nsamp, const double* st, int64_t* slot_l,
                       double* slot_num, double* slot_den, int32_t* nslot) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= NM) return;
    const int64_t g0 = bgs[mbs[q]], g1 = bgs[mbs[q + 1]];
    int n = 0;
    for (int64_t grp = g0; grp < g1; ++grp) {
        const int64_t l = gl[grp];
        int s = 0;
        while (s < n && slot_l[g0 + s] != l) ++s;
        if (s == n) {
            slot_l[g0 + n] = l;
            slot_num[g0 + n] = 0.0;
            slot_den[g0 + n] = 0.0;
            ++n;
        }
        const double w = __ll2double_rn(gw[grp]);
        double num = slot_num[g0 + s], den = slot_den[g0 + s];
        for (int64_t i = soff[grp], e = soff[grp] + nsamp[grp]; i < e; ++i) {
            num = __dadd_rn(num, __dmul_rn(w, st[i]));
            den = __dadd_rn(den, __dmul_rn(w, w));
        }
        slot_num[g0 + s] = num;
        slot_den[g0 + s] = den;
    }
    for (int a = 1; a < n; ++a)  // insertion sort by l (distinct keys)
        for (int b = a; b > 0 && slot_l[g0 + b - 1] > slot_l[g0 + b]; --b) {
            const int64_t tl = slot_l[g0 + b];
            slot_l[g0 + b] = slot_l[g0 + b - 1];
            slot_l[g0 + b - 1] = tl;
            const double tn = slot_num[g0 + b], td = slot_den[g0 + b];
            slot_num[g0 + b] = slot_num[g0 + b - 1];
            slot_den[g0 + b] = slot_den[g0 + b - 1];
            slot_num[g0 + b - 1] = tn;
            slot_den[g0 + b - 1] = td;
        }
    for (int a = 0; a < n; ++a) slot_num[g0 + a] = __ddiv_rn(slot_num[g0 + a], slot_den[g0 + a]);
    nslot[q] = n;
}

// The same step baseline, parallel over (macro, loop count): k_step_slots
// lists each macro's distinct l ascending (the order the final insertion sort
// of k_step produces), then one thread per (macro, slot) accumulates its
// slot over the macro's groups in group order -- the identical sequence of
// additions -- and divides.
constexpr int kStepMaxSlots = 16;

__global__ void k_step_slots(int64_t NM, const int64_t* mbs, const int64_t* bgs, const int64_t* gl, int64_t* slot_l,
                             int32_t* nslot) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= NM) return;
    const int64_t g0 = bgs[mbs[q]], g1 = bgs[mbs[q + 1]];
    int n = 0;
    for (int64_t grp = g0; grp < g1; ++grp) {
        const int64_t l = gl[grp];
        int s = 0;
        while (s < n && slot_l[g0 + s] != l) ++s;
        if (s == n) {
            slot_l[g0 + n] = l;
            ++n;
        }
    }
    for (int a = 1; a < n; ++a)
        for (int b = a; b > 0 && slot_l[g0 + b - 1] > slot_l[g0 + b]; --b) {
            const int64_t tl = slot_l[g0 + b];
            slot_l[g0 + b] = slot_l[g0 + b - 1];
            slot_l[g0 + b - 1] = tl;
        }
    nslot[q] = n;
}

__global__ void k_step_sum(int64_t NM, const int64_t* mbs, const int64_t* bgs, const int64_t* gw, const int64_t* gl,
                           const int64_t* soff, const int32_t* nsamp, const double* st, const int64_t* slot_l,
                           const int32_t* nslot, double* slot_num, double* slot_den) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t q = idx / kStepMaxSlots;
    if (q >= NM) return;
    const int64_t g0 = bgs[mbs[q]], g1 = bgs[mbs[q + 1]];
    for (int s = int(idx % kStepMaxSlots); s < nslot[q]; s += kStepMaxSlots) {  // > 16 slots: strided
        const int64_t l = slot_l[g0 + s];
        double num = 0.0, den = 0.0;
        for (int64_t grp = g0; grp < g1; ++grp) {
            if (gl[grp] != l) continue;
            const double w = __ll2double_rn(gw[grp]);
            for (int64_t i = soff[grp], e = soff[grp] + nsamp[grp]; i < e; ++i) {
                num = __dadd_rn(num, __dmul_rn(w, st[i]));
                den = __dadd_rn(den, __dmul_rn(w, w));
            }
        }
        slot_num[g0 + s] = __ddiv_rn(num, den);
        slot_den[g0 + s] = den;
    }
}

struct Macros {
    int64_t nmac;
    const int64_t* bstart;  // [nmac+1] bucket range per macro
    const int64_t* bw;      // wave of each bucket
    const int64_t* gstart_of_bucket;  // [nb+1] group range per bucket
    int32_t W, p;
    double* theta;          // [nmac*4]
    int32_t* flags;
    int32_t* next;          // ext anchor count per macro
    int64_t* el;            // [G] ext anchors, slice at the macro's first group
    int32_t* em;
};

// fit_extrapolation (model.cpp:140-192), split around the pooled fit:
// k_ext_prep (thread / macro) finds the window [max(1, W-p+1), W]; with >= 2
// waves of data it queues the pooled slice for k_qfit, else it copies the
// highest wave's fit and anchors (ext_insufficient_waves).  k_ext_vote
// (thread / macro) then takes the fit's degenerate flag and the per-l
// majority micro (ties -> smaller micro id).
// fallback = false: the window bounds only (fallback macros get elo = ehi =
// 0 and wait for k_ext_prep(fallback = true) after the bucket fits, whose
// coefficients they copy) -- so the window fits can run beside the bucket
// fits.  fallback = true: only macros with elo == ehi.
template <bool FALLBACK>
__global__ void k_ext_prep(Rec rc, Buckets b, Groups gr, const uint32_t* ordA, Macros m, int64_t* elo, int64_t* ehi) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= m.nmac) return;
    if (FALLBACK && ehi[q] > elo[q]) return;  // a window macro (done beside the bucket fits)
    const int64_t b0 = m.bstart[q], b1 = m.bstart[q + 1];
    const int w_lo = max(1, m.W - m.p + 1);
    int64_t wb0 = -1, wb1 = -1;
    int used = 0;
    for (int64_t k = b0; k < b1; ++k)
        if (m.bw[k] >= w_lo && m.bw[k] <= m.W) {
            if (wb0 < 0) wb0 = k;
            wb1 = k + 1;
            ++used;
        }
    if (used >= 2) {
        elo[q] = b.slo[wb0];
        ehi[q] = b.shi[wb1 - 1];
        return;
    }
    elo[q] = ehi[q] = 0;
    if (!FALLBACK) return;
    // fewer than two window waves: the highest wave's fit and anchors
    const int64_t top = b1 - 1, gslice = m.gstart_of_bucket[b0];
    for (int c = 0; c < 4; ++c) m.theta[4 * q + c] = b.coeff[4 * top + c];
    m.flags[q] = 2;
    const int64_t g0 = m.gstart_of_bucket[top], g1 = m.gstart_of_bucket[top + 1];
    int cnt = 0;
    for (int64_t k = g0; k < g1; ++k) {
        m.el[gslice + cnt] = rc.l[ordA[gr.start[k]]];
        m.em[gslice + cnt] = gr.micro[k];
        ++cnt;
    }
    m.next[q] = cnt;
}

// Warp per macro.  The window's groups (w asc, l asc) carry (l, selected
// micro); the per-l majority micro (ties -> smaller micro) is found with
// O(n^2) lane-parallel counting over the window staged in shared memory
// (n = groups in the window, <= kVoteCap; larger windows take the serial
// scan on lane 0), then each l's winner is written at the rank of l among
// the distinct l values.
constexpr int kVoteWarps = 4;
constexpr int kVoteCap = 256;
__global__ void __launch_bounds__(32 * kVoteWarps)
    k_ext_vote(Rec rc, Groups gr, const uint32_t* ordA, Macros m, const int64_t* elo, const int64_t* ehi,
               const int32_t* edeg) {
    __shared__ int64_t sl[kVoteWarps][kVoteCap];
    __shared__ int32_t sm[kVoteWarps][kVoteCap], sc[kVoteWarps][kVoteCap], sf[kVoteWarps][kVoteCap];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (q >= m.nmac || ehi[q] <= elo[q]) return;
    if (lane == 0) m.flags[q] = edeg[q] ? 1 : 0;
    const int64_t b0 = m.bstart[q], b1 = m.bstart[q + 1];
    const int w_lo = max(1, m.W - m.p + 1);
    long long wb0 = LLONG_MAX, wb1 = -1;
    for (int64_t k = b0 + lane; k < b1; k += 32)
        if (m.bw[k] >= w_lo && m.bw[k] <= m.W) {
            wb0 = min(wb0, (long long)k);
            wb1 = max(wb1, (long long)k + 1);
        }
    wb0 = __reduce_min_sync(FULL, int(min(wb0, (long long)INT_MAX)));
    wb1 = __reduce_max_sync(FULL, int(wb1));
    const int64_t gslice = m.gstart_of_bucket[b0];
    const int64_t g0 = m.gstart_of_bucket[wb0], g1 = m.gstart_of_bucket[wb1];
    const int n = int(g1 - g0);
    if (n > kVoteCap) {
        if (lane != 0) return;
        int cnt = 0;
        int64_t prev_l = 0;
        bool have_prev = false;
        for (;;) {  // distinct l ascending
            bool found = false;
            int64_t lv = 0;
            for (int64_t k = g0; k < g1; ++k) {
                const int64_t gl = rc.l[ordA[gr.start[k]]];
                if ((!have_prev || gl > prev_l) && (!found || gl < lv)) {
                    lv = gl;
                    found = true;
                }
            }
            if (!found) break;
            int32_t best_micro = -1, best_count = -1, cur = INT_MIN;
            for (;;) {
                int32_t nxt = INT_MAX;
                for (int64_t k = g0; k < g1; ++k) {
                    const int64_t gl = rc.l[ordA[gr.start[k]]];
                    if (gl == lv && gr.micro[k] > cur && gr.micro[k] < nxt) nxt = gr.micro[k];
                }
                if (nxt == INT_MAX) break;
                int32_t c = 0;
                for (int64_t k = g0; k < g1; ++k)
                    if (rc.l[ordA[gr.start[k]]] == lv && gr.micro[k] == nxt) ++c;
                if (c > best_count) {
                    best_count = c;
                    best_micro = nxt;
                }
                cur = nxt;
            }
            m.el[gslice + cnt] = lv;
            m.em[gslice + cnt] = best_micro;
            ++cnt;
            prev_l = lv;
            have_prev = true;
        }
        m.next[q] = cnt;
        return;
    }
    int64_t* L = sl[wi];
    int32_t* U = sm[wi];
    int32_t* Cn = sc[wi];
    int32_t* FL = sf[wi];
    for (int k = lane; k < n; k += 32) {
        L[k] = rc.l[ordA[gr.start[g0 + k]]];
        U[k] = gr.micro[g0 + k];
    }
    __syncwarp();
    // occurrences of (l, micro) (-1 marks a repeat of an earlier entry) and
    // first occurrence of each l
    for (int k = lane; k < n; k += 32) {
        int c = 0;
        bool first = true, firstl = true;
        for (int j = 0; j < n; ++j)
            if (L[j] == L[k]) {
                if (j < k) firstl = false;
                if (U[j] == U[k]) {
                    ++c;
                    if (j < k) first = false;
                }
            }
        Cn[k] = first ? c : -1;
        FL[k] = firstl;
    }
    __syncwarp();
    int distinct = 0;
    for (int k = lane; k < n; k += 32) {
        const int64_t lk = L[k];
        bool win = Cn[k] >= 0;
        int rank = 0;  // distinct l values below lk
        for (int j = 0; j < n; ++j) {
            const int64_t lj = L[j];
            if (lj == lk) {
                if (Cn[j] > Cn[k] || (Cn[j] == Cn[k] && Cn[j] >= 0 && U[j] < U[k])) win = false;
            } else if (lj < lk) {
                rank += FL[j];
            }
        }
        if (win) {
            m.el[gslice + rank] = lk;
            m.em[gslice + rank] = U[k];
        }
        distinct += FL[k];
    }
    distinct = __reduce_add_sync(FULL, distinct);
    if (lane == 0) m.next[q] = distinct;
}

// Device-resident table CSR (wt_tables_desc layout, int32) from the fit's
// bucket / group / macro boundaries -- the tables never leave HBM on their
// way to the engine (wt_engine_create_from_build).  One thread per index of
// the longest array (NB + 1).
struct Csr32 {
    int32_t* macro_id;    // [NM] registry id
    int32_t* W;           // [NM]
    int32_t* coeff_off;   // [NM+1] = awave_off (one wave map per bucket)
    int32_t* coeff_w;     // [NB]   = awave_w
    int32_t* awave_aoff;  // [NB+1] group range of each bucket (anchors = groups)
    int32_t* ext_off;     // [NM]   first group of the macro: its ext-anchor slice
    int32_t* nsamp;       // [NB]   diagnostics: samples per bucket
    int32_t* dflags;      // [NB]   bit0 degenerate_fit, bit1 sparse_bucket
};
__global__ void k_csr32(int64_t NM, int64_t NB, const int64_t* mbs, const int64_t* bw, const int64_t* bgs,
                        const int64_t* slo, const int64_t* shi, const int32_t* degen, const int64_t* mpos,
                        const int32_t* reg_ids, int32_t W, Csr32 o) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i <= NM) o.coeff_off[i] = int32_t(mbs[i]);
    if (i < NM) {
        o.macro_id[i] = reg_ids[mpos[i]];
        o.W[i] = W;
        o.ext_off[i] = int32_t(bgs[mbs[i]]);
    }
    if (i < NB) {
        o.coeff_w[i] = int32_t(bw[i]);
        const int32_t ns = int32_t(shi[i] - slo[i]);
        o.nsamp[i] = ns;
        o.dflags[i] = (degen[i] ? 1 : 0) | (ns < 4 ? 2 : 0);
    }
    if (i <= NB) o.awave_aoff[i] = int32_t(bgs[i]);
}

}  // namespace fit
}  // namespace wtb

// ------------------------------------------------------------------ C-ABI
using namespace wtb::fit;
using wtb::Arena;
using wtb::TabView;

namespace {
// errors surface through wt_last_error() (wt_capi.cu)
struct FitErr {
    FitErr& operator=(const std::string& m) {
        wtb::set_last_error(m);
        return *this;
    }
    FitErr& operator=(const char* m) {
        wtb::set_last_error(m);
        return *this;
    }
} g_fit_err;
}

// The build: tables (and diagnostics) resident on the device, in the
// wt_tables_desc CSR layout, until wt_build_free.  Host copies are made on
// demand (wt_build_result_get) -- the engine is built from the device arrays
// directly (wt_engine_create_from_build).
struct wt_build {
    int device = 0;
    int32_t NM = 0, W = 0, p = 0;
    int64_t NB = 0, G = 0;
    bool baselines = false;
    double device_ms = 0.0;
    std::vector<void*> mem;  // device blocks owned by the build
    // device outputs
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, done = nullptr;  // fit start / end (device_ms), all work queued
    int32_t* d_degen = nullptr;
    int32_t *t_macro = nullptr, *t_W = nullptr, *t_coeff_off = nullptr, *t_coeff_w = nullptr,
            *t_awave_aoff = nullptr, *t_ext_off = nullptr, *t_ext_cnt = nullptr, *t_anchor_micro = nullptr,
            *t_ext_micro = nullptr, *d_nsamp = nullptr, *d_dflags = nullptr, *d_partial = nullptr,
            *d_ext_flags = nullptr;
    double *t_theta_ext = nullptr, *t_coeff_theta = nullptr, *d_r2 = nullptr, *d_mape = nullptr;
    int64_t *t_anchor_l = nullptr, *t_ext_l = nullptr;
    // ablation baselines (when requested)
    double *b_lin = nullptr, *b_lin_r2 = nullptr, *b_lin_mape = nullptr, *b_step_t = nullptr;
    int32_t *b_lin_deg = nullptr, *b_nslot = nullptr;
    int64_t* b_step_l = nullptr;
    std::vector<int32_t> h_macro_id;  // registry order, known on the host at build time
    // host copies (wt_build_result_get)
    bool host_ready = false;
    std::vector<int32_t> macro_id, ext_flags, coeff_off, coeff_w, diag_samples, diag_flags, awave_off, awave_w,
        awave_aoff, anchor_micro, anchor_partial, ext_aoff, ext_micro, step_off, lin_degen;
    std::vector<double> theta_ext, coeff_theta, diag_r2, diag_mape, step_t, lin_theta, lin_r2, lin_mape;
    std::vector<int64_t> anchor_l, ext_l, step_l;
};


#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            g_fit_err = std::string(#x) + ": " + cudaGetErrorString(e_);              \
            return WT_CUDA_ERROR;                                                      \
        }                                                                              \
    } while (0)

namespace {

// Temporaries come from the library's stream-ordered pool (cudaMalloc of
// hundreds of MB per build costs milliseconds of host time).
thread_local cudaStream_t t_alloc_stream = nullptr;
thread_local cudaMemPool_t t_alloc_pool = nullptr;

// a second stream per device for work that overlaps within one build
cudaStream_t aux_stream(int device) {
    static std::mutex mu;
    static std::map<int, cudaStream_t> st;
    std::lock_guard<std::mutex> lk(mu);
    auto it = st.find(device);
    if (it != st.end()) return it->second;
    cudaStream_t x = nullptr;
    cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    st[device] = x;
    return x;
}

// Pinned host words for the build's scalar read-backs (one per host thread;
// a pageable D2H is staged and costs several times a pinned one).
void* pinned_words(size_t bytes) {
    thread_local void* p = nullptr;
    thread_local size_t cap = 0;
    if (bytes > cap) {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 64 << 10);
        if (cudaMallocHost(&p, want) != cudaSuccess) return nullptr;
        cap = want;
    }
    return p;
}

// last element of each of up to 6 device arrays into one small block (one
// read-back instead of six); w32[k] != 0: an int32 array, else int64
struct Tails {
    const void* a[6];
    int32_t w32[6];
    int32_t n;
};
__global__ void k_tails(Tails t, int64_t idx, int64_t* out) {
    const int k = threadIdx.x;
    if (k >= t.n) return;
    out[k] = t.w32[k] ? int64_t(static_cast<const int32_t*>(t.a[k])[idx])
                      : static_cast<const int64_t*>(t.a[k])[idx];
}

// cub temporaries: the library pool too (the default pool releases its
// memory at every synchronisation and re-maps it on the next allocation)
cudaError_t talloc(void** p, size_t bytes, cudaStream_t s) {
    return t_alloc_pool ? cudaMallocFromPoolAsync(p, bytes, t_alloc_pool, s) : cudaMallocAsync(p, bytes, s);
}

template <typename T>
T* dalloc(std::vector<void*>& owned, size_t n) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    const cudaError_t e = t_alloc_pool ? cudaMallocFromPoolAsync(&p, bytes, t_alloc_pool, t_alloc_stream)
                                       : cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return nullptr;
    owned.push_back(p);
    return static_cast<T*>(p);
}

// stream-ordered release of the temporaries at scope exit (no host sync)
struct OwnedFree {
    std::vector<void*>* v;
    cudaStream_t s;
    ~OwnedFree() {
        for (void* q : *v) cudaFreeAsync(q, s);
        t_alloc_pool = nullptr;
        t_alloc_stream = nullptr;
    }
};

int bits_for(unsigned long long range) {
    int b = 0;
    while (b < 64 && (range >> b) != 0) ++b;
    return b;
}

// Plan LSD passes over fields (least significant first), packing greedily.
std::vector<Pass> plan_passes(const std::vector<Field>& fields) {
    std::vector<Pass> out;
    Pass cur{};
    cur.nf = 0;
    cur.bits = 0;
    for (const Field& f0 : fields) {
        Field f = f0;
        if (f.bits == 0) continue;  // constant field: orders nothing, costs loads
        if (cur.bits + f.bits > 64 && cur.nf > 0) {
            out.push_back(cur);
            cur = Pass{};
        }
        f.shift = cur.bits;
        cur.f[cur.nf++] = f;
        cur.bits += f.bits;
    }
    if (cur.nf > 0) out.push_back(cur);
    return out;
}

// Stable LSD sort of `perm` by the packed fields; after each pass the
// permutation buffers swap (no copy back): on return `perm` holds the order
// and `keys_alt` the last pass's sorted keys.
// identity: perm starts as 0..n-1 (every record valid), so the first pass
// packs record i directly.
wt_status run_sort(const Rec& rc, const int32_t* mpos, const int32_t* umin_m, uint32_t*& perm, uint32_t*& perm_alt,
                   int64_t n, const std::vector<Pass>& passes, unsigned long long* keys, unsigned long long* keys_alt,
                   void*& tmp, size_t& tmp_bytes, cudaStream_t s, bool identity = false) {
    bool first = true;
    for (const Pass& ps : passes) {
        const int blocks = int((n + 255) / 256);
        k_pack<<<blocks, 256, 0, s>>>(rc, mpos, umin_m, first && identity ? nullptr : perm, n, ps, keys);
        first = false;
        size_t need = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys_alt, perm, perm_alt, n, 0,
                                        std::max(1, ps.bits), s);
        if (need > tmp_bytes) {
            if (tmp) cudaFreeAsync(tmp, s);
            CK(talloc(&tmp, need, s));
            tmp_bytes = need;
        }
        CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_alt, perm, perm_alt, n, 0,
                                           std::max(1, ps.bits), s));
        std::swap(perm, perm_alt);
    }
    return WT_OK;
}

// build_dual_table (model.cpp:194-253) over records resident on the device,
// stream-ordered on s.  Host synchronisations: three scalar read-backs that
// size the next allocations (valid-record count + key ranges + per-macro
// presence; group count; bucket / sample counts).  Outputs land in B.
wt_status fit_core(const Rec& rc, int64_t n_all, const int32_t* registry_ids, int32_t n_macros, int32_t W,
                   int32_t p, bool baselines, int device, cudaStream_t s, wt_build* B) {
    if (n_all >= (int64_t(1) << 31)) {  // the sorts permute 32-bit record indices
        g_fit_err = "build_dual_table: 2^31 or more records are outside the device path's range";
        return WT_UNSUPPORTED;
    }
    t_alloc_stream = s;
    t_alloc_pool = wtb::device_pool(device);
    std::vector<void*> owned;
    OwnedFree freer{&owned, s};  // temporaries released stream-ordered after the last kernel
    // WT_FIT_TRACE=1 prints a synchronised wall-clock breakdown of the stages
    const bool tr = std::getenv("WT_FIT_TRACE") != nullptr;
    auto t_start = std::chrono::steady_clock::now();
    // WT_FIT_TRACE=2: no syncs -- an event per stage and the host clock when
    // the stage was queued; printed at the end (device reached vs host queued)
    const bool tr2 = tr && std::getenv("WT_FIT_TRACE")[0] == '2';
    struct Mark {
        const char* what;
        cudaEvent_t ev;
        double host_ms;
    };
    std::vector<Mark> marks;
    auto trace = [&](const char* what) {
        if (!tr) return;
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        if (tr2) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s);
            marks.push_back({what, e, ms});
            return;
        }
        cudaStreamSynchronize(s);
        std::fprintf(stderr, "[wt_fit] %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };
    struct MarkDump {
        std::vector<Mark>* m;
        cudaStream_t s;
        ~MarkDump() {
            if (m->empty()) return;
            cudaStreamSynchronize(s);
            for (const Mark& k : *m) {
                float d = 0.f;
                cudaEventElapsedTime(&d, m->front().ev, k.ev);
                std::fprintf(stderr, "[wt_fit] %-28s queued %8.3f ms  device +%8.3f ms\n", k.what, k.host_ms,
                             double(d) + m->front().host_ms);
            }
            for (const Mark& k : *m) cudaEventDestroy(k.ev);
        }
    } mark_dump{&marks, s};
    trace("start");

    // 1. registry positions (first occurrence of a duplicated id wins)
    std::vector<std::pair<int32_t, int32_t>> ids(n_macros);
    for (int32_t i = 0; i < n_macros; ++i) ids[i] = {registry_ids[i], i};
    if (!std::is_sorted(registry_ids, registry_ids + n_macros))  // usual registries ascend already
        std::sort(ids.begin(), ids.end());  // (id, position): the stable order by id
    ids.erase(std::unique(ids.begin(), ids.end(), [](auto& a, auto& b) { return a.first == b.first; }), ids.end());
    const int nid = int(ids.size());
    // one upload: sorted ids | their registry positions | registry ids (order)
    std::vector<int32_t> hup(2 * size_t(nid) + size_t(n_macros));
    for (int i = 0; i < nid; ++i) {
        hup[i] = ids[i].first;
        hup[nid + i] = ids[i].second;
    }
    std::copy(registry_ids, registry_ids + n_macros, hup.begin() + 2 * nid);
    // small non-negative ids (the usual registry): a dense id -> position
    // table after the upload block replaces the per-record binary search
    const int32_t id_min = nid ? ids.front().first : 0, id_max = nid ? ids.back().first : -1;
    const bool dense = nid > 0 && id_min >= 0 && int64_t(id_max) < std::max<int64_t>(4096, 8 * int64_t(nid));
    const size_t dense_off = hup.size();
    if (dense) {
        hup.resize(dense_off + size_t(id_max) + 1, -1);
        for (int i = 0; i < nid; ++i) hup[dense_off + size_t(ids[i].first)] = ids[i].second;
    }
    int32_t* dup = dalloc<int32_t>(owned, hup.size());
    // read-back block: nvalid (i64) | ranges | has_rec[n_macros]
    struct Head {
        int64_t nvalid;
        Ranges r;
    };
    const size_t rb_bytes = sizeof(Head) + size_t(n_macros) * 4;
    char* drb = dalloc<char>(owned, rb_bytes);
    int32_t* mpos = dalloc<int32_t>(owned, n_all);
    int32_t* valid = dalloc<int32_t>(owned, n_all);
    uint32_t* idx = dalloc<uint32_t>(owned, n_all);  // record indices (< 2^31: 32-bit sort values)
    int32_t* umin_m = dalloc<int32_t>(owned, n_macros);
    if (!dup || !drb || !mpos || !valid || !idx || !umin_m) {
        g_fit_err = "cudaMalloc failed";
        return WT_CUDA_ERROR;
    }
    Head h0{};
    h0.r = Ranges{~0ULL, 0ULL, ~0ULL, 0ULL, INT_MAX, INT_MIN, INT_MAX, INT_MIN};
    {
        // both uploads from the pinned words (no staging copy); the first
        // read-back below syncs the stream before the words are reused
        const size_t hb = (hup.size() * 4 + 255) & ~size_t(255);
        char* pw = static_cast<char*>(pinned_words(hb + sizeof(Head)));
        if (pw) {
            std::memcpy(pw, hup.data(), hup.size() * 4);
            std::memcpy(pw + hb, &h0, sizeof(Head));
            CK(cudaMemcpyAsync(dup, pw, hup.size() * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(drb, pw + hb, sizeof(Head), cudaMemcpyHostToDevice, s));
        } else {
            CK(cudaMemcpyAsync(dup, hup.data(), hup.size() * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(drb, &h0, sizeof(Head), cudaMemcpyHostToDevice, s));
        }
    }
    CK(cudaMemsetAsync(drb + sizeof(Head), 0, size_t(n_macros) * 4, s));
    Head* dh = reinterpret_cast<Head*>(drb);
    int32_t* has_rec = reinterpret_cast<int32_t*>(drb + sizeof(Head));
    const int blocks_all = int((n_all + 255) / 256);
    k_fill_i32<<<(n_macros + 255) / 256, 256, 0, s>>>(umin_m, n_macros, INT_MAX);
    if (dense)
        k_mpos_dense<<<blocks_all, 256, 0, s>>>(rc, n_all, dup + dense_off, id_max + 1, mpos, valid, has_rec, umin_m);
    else
        k_mpos<<<blocks_all, 256, 0, s>>>(rc, n_all, dup, dup + nid, nid, mpos, valid, has_rec, umin_m);
    // key ranges over every record (a superset of the valid ones: packing
    // stays exact) and max w over ALL records (model.cpp:201-203)
    k_ranges<<<int(std::min<int64_t>((n_all + 255) / 256, int64_t(wtb::device_sms()) * 8)), 256, 0, s>>>(rc, nullptr, n_all, mpos, umin_m,
                                                                                  &dh->r);
    {  // compact valid record indices, order preserved
        cub::CountingInputIterator<uint32_t> it(0);
        size_t need = 0;
        cub::DeviceSelect::Flagged(nullptr, need, it, valid, idx, &dh->nvalid, n_all, s);
        void* t = nullptr;
        CK(talloc(&t, need, s));
        CK(cub::DeviceSelect::Flagged(t, need, it, valid, idx, &dh->nvalid, n_all, s));
        cudaFreeAsync(t, s);
    }
    trace("registry + ranges queued");
    char* hrbp = static_cast<char*>(pinned_words(rb_bytes));
    std::vector<char> hrb_fallback;
    if (!hrbp) {
        hrb_fallback.resize(rb_bytes);
        hrbp = hrb_fallback.data();
    }
    CK(cudaMemcpyAsync(hrbp, drb, rb_bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const std::vector<char> hrb(hrbp, hrbp + rb_bytes);  // the pinned words are reused below
    Head hh;
    std::memcpy(&hh, hrb.data(), sizeof(Head));
    const int64_t n = hh.nvalid;
    const Ranges hr = hh.r;
    if (W <= 0) W = std::max(0, hr.wmax);
    if (n == 0) {
        g_fit_err = "build_dual_table: no macro produced a table";
        return WT_RUNTIME_ERROR;
    }
    B->h_macro_id.clear();
    {
        const int32_t* hr_has = reinterpret_cast<const int32_t*>(hrb.data() + sizeof(Head));
        for (int32_t i = 0; i < n_macros; ++i)
            if (hr_has[i]) B->h_macro_id.push_back(registry_ids[i]);
    }
    // (the ranges' g / l / w / micro bounds cover every record)
    const int bits_g = bits_for(hr.gmax - hr.gmin), bits_l = bits_for(hr.lmax - hr.lmin);
    const int bits_w = bits_for((unsigned long long)((long long)hr.wmax - hr.wmin));
    const int bits_u = hr.umax > 0 ? bits_for((unsigned long long)hr.umax) : 0;
    const int bits_m = bits_for((unsigned long long)std::max(1, n_macros));
    Field fg{0, hr.gmin, bits_g, 0}, fu{1, 0ULL, bits_u, 0},
        fl{2, hr.lmin, bits_l, 0}, fw{3, (unsigned long long)(long long)hr.wmin, bits_w, 0},
        fm{4, 0, bits_m, 0};
    auto passA = plan_passes({fg, fu, fl, fw, fm});
    auto passB = plan_passes({fg, fl, fw, fm});

    CK(cudaEventCreate(&B->ev0));
    CK(cudaEventCreate(&B->ev1));
    CK(cudaEventCreateWithFlags(&B->done, cudaEventDisableTiming));
    CK(cudaEventRecord(B->ev0, s));
    trace("registry + ranges");
    // 2. stable sorts
    // the sorts permute 32-bit record indices (12 bytes per element and pass
    // with the key instead of 16); order A starts as the compacted index list
    // itself (the passes swap buffers); the later kernels index with it as is
    uint32_t* permA = idx;
    uint32_t* alt = dalloc<uint32_t>(owned, n);
    unsigned long long* keys = dalloc<unsigned long long>(owned, n);
    unsigned long long* keys2 = dalloc<unsigned long long>(owned, n);
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    uint32_t* ordB = nullptr;
    uint32_t* ordA = nullptr;
    {
        // order B's sort runs first from a copy of the index list, so that
        // order A's sorted keys (its single pass) survive for the group kernels
        if (bits_u != 0) {
            uint32_t* permB = dalloc<uint32_t>(owned, n);
            uint32_t* altB = dalloc<uint32_t>(owned, n);
            CK(cudaMemcpyAsync(permB, idx, n * 4, cudaMemcpyDeviceToDevice, s));
            wt_status sb = run_sort(rc, mpos, umin_m, permB, altB, n, passB, keys, keys2, tmp, tmp_bytes, s,
                                    n == n_all);
            if (sb) return sb;
            ordB = permB;
        }
        wt_status sa = run_sort(rc, mpos, umin_m, permA, alt, n, passA, keys, keys2, tmp, tmp_bytes, s, n == n_all);
        if (sa) return sa;
        ordA = permA;
        // one micro id per macro: order A (macro, w, l, micro, g) is order B
        // (macro, w, l, g) -- one sort
        if (bits_u == 0) ordB = ordA;
    }
    if (tmp) cudaFreeAsync(tmp, s);
    // with one packing pass, order A's sorted keys hold (macro, w, l, micro,
    // g) of every sorted record: group boundaries and group keys come from
    // them instead of gathers through the permutation
    const unsigned long long* keysA = passA.size() == 1 ? keys2 : nullptr;
    KeyFields kf{};
    if (keysA) {
        // bases from the field definitions (a constant field is not in the
        // pass: width 0, its value is the base); shifts from the pass
        kf.base_g = fg.base;
        kf.base_l = fl.base;
        kf.base_w = fw.base;
        for (int q = 0; q < passA[0].nf; ++q) {
            const Field& f = passA[0].f[q];
            if (f.which == 0) { kf.sg = f.shift; kf.bg = f.bits; }
            if (f.which == 1) { kf.su = f.shift; kf.bu = f.bits; }
            if (f.which == 2) { kf.sl = f.shift; kf.bl = f.bits; }
            if (f.which == 3) { kf.sw = f.shift; kf.bw = f.bits; }
            if (f.which == 4) { kf.sm = f.shift; kf.bm = f.bits; }
        }
    }

    trace("sorts");
    // 3. groups
    const int blocks = int((n + 255) / 256);
    int32_t* gflag = dalloc<int32_t>(owned, n);
    int32_t* gid = dalloc<int32_t>(owned, n);
    if (keysA)
        k_group_flags_k<<<blocks, 256, 0, s>>>(keysA, n, kf.bg + kf.bu, gflag);
    else
        k_group_flags<<<blocks, 256, 0, s>>>(rc, mpos, ordA, n, gflag);
    {
        size_t need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, gflag, gid, n, s);
        void* t = nullptr;
        CK(talloc(&t, need, s));
        CK(cub::DeviceScan::ExclusiveSum(t, need, gflag, gid, n, s));
        cudaFreeAsync(t, s);
    }
    int64_t* dtail = dalloc<int64_t>(owned, 8);
    int64_t* htail = static_cast<int64_t*>(pinned_words(64));
    int64_t htail_fb[8];
    if (!htail) htail = htail_fb;
    {
        Tails t{{gid, gflag}, {1, 1}, 2};
        k_tails<<<1, 32, 0, s>>>(t, n - 1, dtail);
        CK(cudaMemcpyAsync(htail, dtail, 2 * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    const int64_t G = htail[0] + htail[1];
    // G-sized outputs (anchors = groups; ext-anchor slices live at each
    // macro's first group) in one block owned by the build
    {
        Arena ar;
        const size_t o_gl = ar.take(G * 8), o_gm = ar.take(G * 4), o_gp = ar.take(G * 4), o_el = ar.take(G * 8),
                     o_em = ar.take(G * 4);
        char* blk = dalloc<char>(B->mem, ar.used);
        if (!blk) {
            g_fit_err = "cudaMalloc failed (build outputs)";
            return WT_CUDA_ERROR;
        }
        B->t_anchor_l = reinterpret_cast<int64_t*>(blk + o_gl);
        B->t_anchor_micro = reinterpret_cast<int32_t*>(blk + o_gm);
        B->d_partial = reinterpret_cast<int32_t*>(blk + o_gp);
        B->t_ext_l = reinterpret_cast<int64_t*>(blk + o_el);
        B->t_ext_micro = reinterpret_cast<int32_t*>(blk + o_em);
    }
    int64_t* gstart = dalloc<int64_t>(owned, G + 1);
    k_group_starts<<<blocks, 256, 0, s>>>(gflag, gid, n, gstart);
    CK(cudaMemcpyAsync(gstart + G, &n, 8, cudaMemcpyHostToDevice, s));
    Groups gr{gstart, B->t_anchor_micro, B->d_partial, dalloc<int64_t>(owned, G), dalloc<int64_t>(owned, G),
              dalloc<int32_t>(owned, G)};
    const int gblocks = int((G + 127) / 128);
    const bool sel_keys = keysA && ordB == ordA;  // g / micro from the sorted keys
    if (sel_keys)
        k_select_k<<<gblocks, 128, 0, s>>>(rc, keysA, kf, umin_m, ordA, G, gr);
    else
        k_select<<<gblocks, 128, 0, s>>>(rc, ordA, ordB, G, gr);
    // sample offsets
    int64_t* soff = dalloc<int64_t>(owned, G + 1);
    {
        // widen nsamp to int64 via a transform iterator
        auto wid = cub::TransformInputIterator<int64_t, cub::CastOp<int64_t>, const int32_t*>(gr.nsamp,
                                                                                                cub::CastOp<int64_t>());
        size_t need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, wid, soff, G, s);
        void* t = nullptr;
        CK(talloc(&t, need, s));
        CK(cub::DeviceScan::ExclusiveSum(t, need, wid, soff, G, s));
        cudaFreeAsync(t, s);
    }
    trace("groups + select");
    // group keys and bucket / macro boundaries, all on the device
    int64_t* gm = dalloc<int64_t>(owned, G);
    int64_t* gw = dalloc<int64_t>(owned, G);
    int64_t* gl = B->t_anchor_l;
    int32_t* bflag = dalloc<int32_t>(owned, G);
    int32_t* mflag = dalloc<int32_t>(owned, G);
    int32_t* bid = dalloc<int32_t>(owned, G);
    int32_t* mid = dalloc<int32_t>(owned, G);
    if (keysA)
        k_group_meta_k<<<gblocks, 128, 0, s>>>(keysA, kf, G, gr, gm, gw, gl, bflag, mflag);
    else
        k_group_meta<<<gblocks, 128, 0, s>>>(rc, mpos, ordA, G, gr, gm, gw, gl, bflag, mflag);
    for (auto [in, out] : {std::pair<int32_t*, int32_t*>{bflag, bid}, std::pair<int32_t*, int32_t*>{mflag, mid}}) {
        size_t need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, G, s);
        void* t = nullptr;
        CK(talloc(&t, need, s));
        CK(cub::DeviceScan::ExclusiveSum(t, need, in, out, G, s));
        cudaFreeAsync(t, s);
    }
    {
        Tails t{{bid, bflag, mid, mflag, soff, gr.nsamp}, {1, 1, 1, 1, 0, 1}, 6};
        k_tails<<<1, 32, 0, s>>>(t, G - 1, dtail);
        CK(cudaMemcpyAsync(htail, dtail, 6 * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    const int64_t NB = htail[0] + htail[1], NM = htail[2] + htail[3];
    const int64_t S_total = htail[4] + htail[5];
    if (NM != int64_t(B->h_macro_id.size())) {
        g_fit_err = "build_dual_table: macro count mismatch";
        return WT_RUNTIME_ERROR;
    }
    // NM / NB-sized outputs in one block owned by the build
    {
        Arena ar;
        const size_t o_mac = ar.take(NM * 4), o_W = ar.take(NM * 4), o_te = ar.take(NM * 32),
                     o_co = ar.take((NM + 1) * 4), o_cw = ar.take(NB * 4), o_ct = ar.take(NB * 32),
                     o_aa = ar.take((NB + 1) * 4), o_eo = ar.take(NM * 4), o_ec = ar.take(NM * 4),
                     o_ns = ar.take(NB * 4), o_df = ar.take(NB * 4), o_ef = ar.take(NM * 4), o_r2 = ar.take(NB * 8),
                     o_mp = ar.take(NB * 8), o_dg = ar.take(NB * 4);
        char* blk = dalloc<char>(B->mem, ar.used);
        if (!blk) {
            g_fit_err = "cudaMalloc failed (build outputs)";
            return WT_CUDA_ERROR;
        }
        B->t_macro = reinterpret_cast<int32_t*>(blk + o_mac);
        B->t_W = reinterpret_cast<int32_t*>(blk + o_W);
        B->t_theta_ext = reinterpret_cast<double*>(blk + o_te);
        B->t_coeff_off = reinterpret_cast<int32_t*>(blk + o_co);
        B->t_coeff_w = reinterpret_cast<int32_t*>(blk + o_cw);
        B->t_coeff_theta = reinterpret_cast<double*>(blk + o_ct);
        B->t_awave_aoff = reinterpret_cast<int32_t*>(blk + o_aa);
        B->t_ext_off = reinterpret_cast<int32_t*>(blk + o_eo);
        B->t_ext_cnt = reinterpret_cast<int32_t*>(blk + o_ec);
        B->d_nsamp = reinterpret_cast<int32_t*>(blk + o_ns);
        B->d_dflags = reinterpret_cast<int32_t*>(blk + o_df);
        B->d_ext_flags = reinterpret_cast<int32_t*>(blk + o_ef);
        B->d_r2 = reinterpret_cast<double*>(blk + o_r2);
        B->d_mape = reinterpret_cast<double*>(blk + o_mp);
        B->d_degen = reinterpret_cast<int32_t*>(blk + o_dg);
    }
    int32_t* bdegen = B->d_degen;
    double* sg = dalloc<double>(owned, S_total);
    double* sl = dalloc<double>(owned, S_total);
    double* stt = dalloc<double>(owned, S_total);
    // global scratch of problems above kQRows samples (extrapolation pools,
    // linear baseline); virtual until touched
    double* scratch = dalloc<double>(owned, kQScr * S_total);
    if (!scratch) {
        g_fit_err = "cudaMalloc failed (fit scratch)";
        return WT_CUDA_ERROR;
    }
    if (keysA)
        k_samples_k<<<gblocks, 128, 0, s>>>(rc, keysA, kf, ordA, G, gr, soff, sg, sl, stt);
    else
        k_samples<<<gblocks, 128, 0, s>>>(rc, ordA, G, gr, soff, sg, sl, stt);
    int64_t* d_bslo = dalloc<int64_t>(owned, NB);
    int64_t* d_bshi = dalloc<int64_t>(owned, NB);
    int64_t* d_bgs = dalloc<int64_t>(owned, NB + 1);
    int64_t* d_bw = dalloc<int64_t>(owned, NB);
    int64_t* d_mbs = dalloc<int64_t>(owned, NM + 1);
    int64_t* d_mpos = dalloc<int64_t>(owned, NM);
    k_bucket_meta<<<gblocks, 128, 0, s>>>(G, gm, gw, soff, bflag, bid, mflag, mid, d_bgs, d_bw, d_bslo, d_mbs,
                                          d_mpos);
    k_bucket_tail<<<int((NB + 127) / 128), 128, 0, s>>>(NB, NM, G, S_total, soff, d_bgs, d_bshi, d_mbs);
    Buckets bk{NB, d_bslo, d_bshi, B->t_coeff_theta, B->d_r2, B->d_mape, bdegen};
    const int nsm = wtb::device_sms();
    trace("samples + meta");
    Macros mc{NM, d_mbs, d_bw, d_bgs, W, p, B->t_theta_ext, B->d_ext_flags, B->t_ext_cnt, B->t_ext_l, B->t_ext_micro};
    {
        // the extrapolation windows (model.cpp:140-192) need the samples
        // only: their pooled fits and anchor votes run on a second stream
        // beside the bucket fits; macros without a two-wave window copy their
        // top bucket's fit after the join
        int64_t* elo = dalloc<int64_t>(owned, NM);
        int64_t* ehi = dalloc<int64_t>(owned, NM);
        int32_t* edeg = dalloc<int32_t>(owned, NM);
        double* scratch2 = dalloc<double>(owned, kQScr * S_total);  // the window fits' own scratch
        if (!elo || !ehi || !edeg || !scratch2) {
            g_fit_err = "cudaMalloc failed (extrapolation)";
            return WT_CUDA_ERROR;
        }
        const int mblocks = int((NM + 127) / 128);
        cudaStream_t ax = aux_stream(device);
        cudaEvent_t fork = nullptr, join = nullptr;
        CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
        struct Evs {
            cudaEvent_t a, b;
            ~Evs() {
                cudaEventDestroy(a);
                cudaEventDestroy(b);
            }
        } evs{fork, join};
        CK(cudaEventRecord(fork, s));
        CK(cudaStreamWaitEvent(ax, fork, 0));
        k_ext_prep<false><<<mblocks, 128, 0, ax>>>(rc, bk, gr, ordA, mc, elo, ehi);
        // pooled window fits (model.cpp:171-176): theta_ext straight into the table
        Buckets ext{NM, elo, ehi, B->t_theta_ext, nullptr, nullptr, edeg};
        CK(launch_qfit(true, sg, sl, stt, ext, scratch2, nsm, ax));
        k_ext_vote<<<int((NM + kVoteWarps - 1) / kVoteWarps), 32 * kVoteWarps, 0, ax>>>(rc, gr, ordA, mc, elo, ehi,
                                                                                        edeg);
        CK(cudaEventRecord(join, ax));
        CK(launch_qfit(false, sg, sl, stt, bk, scratch, nsm, s));
        trace("k_qfit buckets");
        CK(cudaStreamWaitEvent(s, join, 0));
        k_ext_prep<true><<<mblocks, 128, 0, s>>>(rc, bk, gr, ordA, mc, elo, ehi);
    }
    trace("extrapolation");
    {
        Csr32 o{B->t_macro, B->t_W, B->t_coeff_off, B->t_coeff_w, B->t_awave_aoff, B->t_ext_off, B->d_nsamp,
                B->d_dflags};
        k_csr32<<<int((NB + 1 + 255) / 256), 256, 0, s>>>(NM, NB, d_mbs, d_bw, d_bgs, d_bslo, d_bshi, bdegen, d_mpos,
                                                          dup + 2 * nid, W, o);
    }
    CK(cudaEventRecord(B->ev1, s));
    if (baselines) {
        // ablation baselines from the same selected samples (not part of
        // build_dual_table; outside the build's device time)
        int64_t* d_mslo = dalloc<int64_t>(owned, NM);
        int64_t* d_mshi = dalloc<int64_t>(owned, NM);
        k_macro_samples<<<int((NM + 127) / 128), 128, 0, s>>>(NM, d_mbs, d_bgs, soff, G, S_total, d_mslo, d_mshi);
        B->b_lin = dalloc<double>(B->mem, NM * 4);
        B->b_lin_r2 = dalloc<double>(B->mem, NM);
        B->b_lin_mape = dalloc<double>(B->mem, NM);
        B->b_lin_deg = dalloc<int32_t>(B->mem, NM);
        B->b_step_l = dalloc<int64_t>(B->mem, G);
        B->b_step_t = dalloc<double>(B->mem, G);
        B->b_nslot = dalloc<int32_t>(B->mem, NM);
        double* d_sden = dalloc<double>(owned, G);
        if (!B->b_lin || !B->b_step_t || !B->b_nslot || !d_sden) {
            g_fit_err = "cudaMalloc failed (baselines)";
            return WT_CUDA_ERROR;
        }
        Buckets lin{NM, d_mslo, d_mshi, B->b_lin, B->b_lin_r2, B->b_lin_mape, B->b_lin_deg};
        CK(launch_qfit(true, sg, sl, stt, lin, scratch, nsm, s));
        static const bool serial = std::getenv("WT_STEP_SERIAL") != nullptr;
        if (serial) {
            k_step<<<int((NM + 127) / 128), 128, 0, s>>>(NM, d_mbs, d_bgs, gw, gl, soff, gr.nsamp, stt, B->b_step_l,
                                                          B->b_step_t, d_sden, B->b_nslot);
        } else {
            k_step_slots<<<int((NM + 127) / 128), 128, 0, s>>>(NM, d_mbs, d_bgs, gl, B->b_step_l, B->b_nslot);
            const int64_t nt = NM * kStepMaxSlots;
            k_step_sum<<<int((nt + 127) / 128), 128, 0, s>>>(NM, d_mbs, d_bgs, gw, gl, soff, gr.nsamp, stt,
                                                              B->b_step_l, B->b_nslot, B->b_step_t, d_sden);
        }
        trace("baselines");
    }
    CK(cudaGetLastError());
    B->NM = int32_t(NM);
    B->NB = NB;
    B->G = G;
    B->W = W;
    B->p = p;
    B->baselines = baselines;
    CK(cudaEventRecord(B->done, s));
    return WT_OK;
}

void build_release(wt_build* b) {
    // engines made from this build read its tables from their own streams
    // until their first use (wt_engine_create_from_build does not wait):
    // all device work completes before the tables go back to the pool
    cudaDeviceSynchronize();
    for (void* q : b->mem) cudaFreeAsync(q, nullptr);
    if (!b->mem.empty()) cudaStreamSynchronize(nullptr);
    b->mem.clear();
    for (cudaEvent_t* e : {&b->ev0, &b->ev1, &b->done})
        if (*e) {
            cudaEventDestroy(*e);
            *e = nullptr;
        }
}

// Host copies of the device tables, assembled into the CSR layout of
// wt_build_result (registry order).
wt_status build_download(wt_build* B) {
    if (B->host_ready) return WT_OK;
    CK(cudaEventSynchronize(B->done));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, B->ev0, B->ev1));
    B->device_ms = ms;
    const int64_t NM = B->NM, NB = B->NB, G = B->G;
    std::vector<int32_t> coeff_off(NM + 1), coeff_w(NB), aoff(NB + 1), ext_off(NM), ext_cnt(NM), gmicro(G), gpart(G),
        nsamp(NB), dflags(NB), eflags(NM), ldeg, nslot;
    std::vector<double> theta_ext(NM * 4), coeff(NB * 4), r2(NB), mape(NB), lth, lr2, lmape, stept;
    std::vector<int64_t> gl(G), el(G), stepl;
    auto get = [](void* dst, const void* src, size_t n) { return cudaMemcpy(dst, src, n, cudaMemcpyDeviceToHost); };
    CK(get(coeff_off.data(), B->t_coeff_off, (NM + 1) * 4));
    CK(get(coeff_w.data(), B->t_coeff_w, NB * 4));
    CK(get(aoff.data(), B->t_awave_aoff, (NB + 1) * 4));
    CK(get(ext_off.data(), B->t_ext_off, NM * 4));
    CK(get(ext_cnt.data(), B->t_ext_cnt, NM * 4));
    CK(get(gmicro.data(), B->t_anchor_micro, G * 4));
    CK(get(gpart.data(), B->d_partial, G * 4));
    CK(get(nsamp.data(), B->d_nsamp, NB * 4));
    CK(get(dflags.data(), B->d_dflags, NB * 4));
    CK(get(eflags.data(), B->d_ext_flags, NM * 4));
    CK(get(theta_ext.data(), B->t_theta_ext, NM * 32));
    CK(get(coeff.data(), B->t_coeff_theta, NB * 32));
    CK(get(r2.data(), B->d_r2, NB * 8));
    CK(get(mape.data(), B->d_mape, NB * 8));
    CK(get(gl.data(), B->t_anchor_l, G * 8));
    std::vector<int32_t> em(G);
    CK(get(el.data(), B->t_ext_l, G * 8));
    CK(get(em.data(), B->t_ext_micro, G * 4));
    if (B->baselines) {
        ldeg.resize(NM);
        nslot.resize(NM);
        lth.resize(NM * 4);
        lr2.resize(NM);
        lmape.resize(NM);
        stept.resize(G);
        stepl.resize(G);
        CK(get(ldeg.data(), B->b_lin_deg, NM * 4));
        CK(get(nslot.data(), B->b_nslot, NM * 4));
        CK(get(lth.data(), B->b_lin, NM * 32));
        CK(get(lr2.data(), B->b_lin_r2, NM * 8));
        CK(get(lmape.data(), B->b_lin_mape, NM * 8));
        CK(get(stept.data(), B->b_step_t, G * 8));
        CK(get(stepl.data(), B->b_step_l, G * 8));
    }
    B->coeff_off.assign(1, 0);
    B->awave_off.assign(1, 0);
    B->awave_aoff.assign(1, 0);
    B->ext_aoff.assign(1, 0);
    B->step_off.assign(1, 0);
    for (int64_t mq = 0; mq < NM; ++mq) {
        B->macro_id.push_back(B->h_macro_id[mq]);
        for (int c = 0; c < 4; ++c) B->theta_ext.push_back(theta_ext[4 * mq + c]);
        B->ext_flags.push_back(eflags[mq]);
        for (int64_t k = coeff_off[mq]; k < coeff_off[mq + 1]; ++k) {
            B->coeff_w.push_back(coeff_w[k]);
            for (int c = 0; c < 4; ++c) B->coeff_theta.push_back(coeff[4 * k + c]);
            B->diag_r2.push_back(r2[k]);
            B->diag_mape.push_back(mape[k]);
            B->diag_samples.push_back(nsamp[k]);
            B->diag_flags.push_back(dflags[k]);
            B->awave_w.push_back(coeff_w[k]);
            for (int64_t q = aoff[k]; q < aoff[k + 1]; ++q) {
                B->anchor_l.push_back(gl[q]);
                B->anchor_micro.push_back(gmicro[q]);
                B->anchor_partial.push_back(gpart[q]);
            }
            B->awave_aoff.push_back(int32_t(B->anchor_l.size()));
        }
        B->coeff_off.push_back(int32_t(B->coeff_w.size()));
        B->awave_off.push_back(int32_t(B->awave_w.size()));
        for (int q = 0; q < ext_cnt[mq]; ++q) {
            B->ext_l.push_back(el[ext_off[mq] + q]);
            B->ext_micro.push_back(em[ext_off[mq] + q]);
        }
        B->ext_aoff.push_back(int32_t(B->ext_l.size()));
        if (B->baselines) {
            const int64_t gs = ext_off[mq];  // step slots live at the macro's first group too
            for (int q = 0; q < nslot[mq]; ++q) {
                B->step_l.push_back(stepl[gs + q]);
                B->step_t.push_back(stept[gs + q]);
            }
            B->step_off.push_back(int32_t(B->step_l.size()));
            for (int c = 0; c < 4; ++c) B->lin_theta.push_back(lth[4 * mq + c]);
            B->lin_r2.push_back(lr2[mq]);
            B->lin_mape.push_back(lmape[mq]);
            B->lin_degen.push_back(ldeg[mq]);
        }
    }
    B->host_ready = true;
    return WT_OK;
}

void fill_result(const wt_build* B, wt_build_result* result) {
    wt_build_result& R = *result;
    R = wt_build_result{};
    R.n_tables = B->NM;
    R.W = B->W;
    R.p = B->p;
    R.macro_id = B->macro_id.data();
    R.theta_ext = B->theta_ext.data();
    R.ext_flags = B->ext_flags.data();
    R.coeff_off = B->coeff_off.data();
    R.coeff_w = B->coeff_w.data();
    R.coeff_theta = B->coeff_theta.data();
    R.diag_r2 = B->diag_r2.data();
    R.diag_mape = B->diag_mape.data();
    R.diag_samples = B->diag_samples.data();
    R.diag_flags = B->diag_flags.data();
    R.awave_off = B->awave_off.data();
    R.awave_w = B->awave_w.data();
    R.awave_aoff = B->awave_aoff.data();
    R.anchor_l = B->anchor_l.data();
    R.anchor_micro = B->anchor_micro.data();
    R.anchor_partial = B->anchor_partial.data();
    R.ext_aoff = B->ext_aoff.data();
    R.ext_l = B->ext_l.data();
    R.ext_micro = B->ext_micro.data();
    R.device_ms = B->device_ms;
    if (B->baselines) {
        R.step_off = B->step_off.data();
        R.step_l = B->step_l.data();
        R.step_t = B->step_t.data();
        R.lin_theta = B->lin_theta.data();
        R.lin_r2 = B->lin_r2.data();
        R.lin_mape = B->lin_mape.data();
        R.lin_degenerate = B->lin_degen.data();
    }
}

struct DevRestore {
    int d;
    ~DevRestore() { cudaSetDevice(d); }
};

}  // namespace

// ------------------------------------------- build exchange between ranks
// A build's device tables packed into one contiguous blob (wt_build_pack) so
// that shards fitted on different GPUs travel in ONE collective (an NCCL
// all-gather of equal-stride blobs), then merged back into one build in
// registry order on every rank (wt_build_merge): the per-rank tables are
// concatenated and the CSR offsets rebased -- coeff_off by the bucket count
// of the ranks before, awave_aoff / ext_off by their group count.  This is
// merge_tables (dist.py) on the device: shards are contiguous registry slices
// and fit_core's outputs depend on a macro's own records only, so the merged
// build equals the single-GPU build of the whole registry.
namespace {

enum PackArr {
    PA_MACRO, PA_W, PA_COFF, PA_EOFF, PA_ECNT, PA_EFLAGS,         // per table (i32; COFF has NM + 1)
    PA_CW, PA_AAOFF, PA_NSAMP, PA_DFLAGS, PA_DEGEN,               // per bucket (i32; AAOFF has NB + 1)
    PA_AMICRO, PA_PART, PA_EMICRO,                                // per group (i32)
    PA_TEXT, PA_CTH, PA_R2, PA_MAPE,                              // f64: 4 / table, 4 / bucket, 1, 1
    PA_AL, PA_EL,                                                 // i64 per group
    PA_N
};
constexpr uint64_t kPackMagic = 0x31424b5041505457ull;  // "WTPAPKB1"
struct PackHead {
    uint64_t magic;
    int64_t NM, NB, G, W, p, bytes, pad;
};
struct PackLayout {
    size_t off[PA_N], bytes[PA_N], total;
};

PackLayout pack_layout(int64_t NM, int64_t NB, int64_t G) {
    const int64_t n[PA_N] = {NM, NM, NM + 1, NM, NM, NM, NB, NB + 1, NB, NB, NB, G, G, G,
                             4 * NM, 4 * NB, NB, NB, G, G};
    const int esz[PA_N] = {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 8, 8, 8, 8, 8, 8};
    PackLayout L{};
    Arena ar;
    ar.take(sizeof(PackHead));
    for (int a = 0; a < PA_N; ++a) {
        L.bytes[a] = size_t(n[a]) * esz[a];
        L.off[a] = ar.take(L.bytes[a]);
    }
    L.total = ar.used;
    return L;
}

void* pack_ptr(const wt_build* B, int a) {
    switch (a) {
        case PA_MACRO: return B->t_macro;
        case PA_W: return B->t_W;
        case PA_COFF: return B->t_coeff_off;
        case PA_EOFF: return B->t_ext_off;
        case PA_ECNT: return B->t_ext_cnt;
        case PA_EFLAGS: return B->d_ext_flags;
        case PA_CW: return B->t_coeff_w;
        case PA_AAOFF: return B->t_awave_aoff;
        case PA_NSAMP: return B->d_nsamp;
        case PA_DFLAGS: return B->d_dflags;
        case PA_DEGEN: return B->d_degen;
        case PA_AMICRO: return B->t_anchor_micro;
        case PA_PART: return B->d_partial;
        case PA_EMICRO: return B->t_ext_micro;
        case PA_TEXT: return B->t_theta_ext;
        case PA_CTH: return B->t_coeff_theta;
        case PA_R2: return B->d_r2;
        case PA_MAPE: return B->d_mape;
        case PA_AL: return B->t_anchor_l;
        case PA_EL: return B->t_ext_l;
    }
    return nullptr;
}

void set_pack_ptr(wt_build* B, int a, void* p) {
    switch (a) {
        case PA_MACRO: B->t_macro = static_cast<int32_t*>(p); break;
        case PA_W: B->t_W = static_cast<int32_t*>(p); break;
        case PA_COFF: B->t_coeff_off = static_cast<int32_t*>(p); break;
        case PA_EOFF: B->t_ext_off = static_cast<int32_t*>(p); break;
        case PA_ECNT: B->t_ext_cnt = static_cast<int32_t*>(p); break;
        case PA_EFLAGS: B->d_ext_flags = static_cast<int32_t*>(p); break;
        case PA_CW: B->t_coeff_w = static_cast<int32_t*>(p); break;
        case PA_AAOFF: B->t_awave_aoff = static_cast<int32_t*>(p); break;
        case PA_NSAMP: B->d_nsamp = static_cast<int32_t*>(p); break;
        case PA_DFLAGS: B->d_dflags = static_cast<int32_t*>(p); break;
        case PA_DEGEN: B->d_degen = static_cast<int32_t*>(p); break;
        case PA_AMICRO: B->t_anchor_micro = static_cast<int32_t*>(p); break;
        case PA_PART: B->d_partial = static_cast<int32_t*>(p); break;
        case PA_EMICRO: B->t_ext_micro = static_cast<int32_t*>(p); break;
        case PA_TEXT: B->t_theta_ext = static_cast<double*>(p); break;
        case PA_CTH: B->t_coeff_theta = static_cast<double*>(p); break;
        case PA_R2: B->d_r2 = static_cast<double*>(p); break;
        case PA_MAPE: B->d_mape = static_cast<double*>(p); break;
        case PA_AL: B->t_anchor_l = static_cast<int64_t*>(p); break;
        case PA_EL: B->t_ext_l = static_cast<int64_t*>(p); break;
    }
}

// One launch copies up to kMergeSegs (rank, array) segments as 32-bit words,
// adding the segment's base to offset arrays (0 elsewhere: identity on the
// bit pattern).  blockIdx.y = segment.
constexpr int kMergeSegs = 96;
struct MergeSeg {
    const uint32_t* src;
    uint32_t* dst;
    int64_t words;
    uint32_t add;
    uint32_t pad;
};
struct MergeArgs {
    int32_t nseg;
    MergeSeg seg[kMergeSegs];
};

__global__ void __launch_bounds__(256) k_build_merge(const __grid_constant__ MergeArgs a) {
    const MergeSeg sg = a.seg[blockIdx.y];
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < sg.words; i += stride)
        sg.dst[i] = __ldg(sg.src + i) + sg.add;
}

}  // namespace

// For wt_capi.cu: the device CSR of a build (engine creation without a
// host round trip).
namespace wtb {
wt_status build_device_tables(const wt_build* b, BuildTables* out) {
    if (!b || !out) return WT_INVALID_ARGUMENT;
    out->device = b->device;
    out->n_tables = b->NM;
    out->macro_id_host = b->h_macro_id.data();
    out->W = b->W;
    out->tv = TabView{b->t_W, b->t_theta_ext, b->t_coeff_off, b->t_coeff_w, b->t_coeff_theta, b->t_coeff_off,
                      b->t_coeff_w, b->t_awave_aoff, b->t_ext_off, b->G, b->t_ext_cnt};
    out->anchor_l = b->t_anchor_l;
    out->anchor_micro = b->t_anchor_micro;
    out->n_anchor = b->G;
    out->ext_l = b->t_ext_l;
    out->ext_micro = b->t_ext_micro;
    out->n_ext = b->G;
    return WT_OK;
}
}  // namespace wtb

extern "C" {

wt_status wt_fit_build(const wt_records_desc* records, const int32_t* registry_ids, int32_t n_macros,
                       int32_t W, int32_t p, int device, wt_build** out, wt_build_result* result) {
    if (!records || !out || !result || (n_macros > 0 && !registry_ids)) {
        g_fit_err = "null argument";
        return WT_INVALID_ARGUMENT;
    }
    *out = nullptr;
    const int64_t n_all = records->n;
    if (n_all <= 0) {
        g_fit_err = "build_dual_table: empty record set";
        return WT_INVALID_ARGUMENT;
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(device);
    DevRestore restore{prev_dev};
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SD {
        cudaStream_t s;
        ~SD() { cudaStreamDestroy(s); }
    } sd{s};
    // upload the host records (one block from the pool; released stream-ordered)
    Arena ar;
    const size_t o_g = ar.take(n_all * 8), o_l = ar.take(n_all * 8), o_w = ar.take(n_all * 4),
                 o_ma = ar.take(n_all * 4), o_mi = ar.take(n_all * 4), o_t = ar.take(n_all * 8);
    void* blk = nullptr;
    CK(cudaMallocFromPoolAsync(&blk, ar.used, wtb::device_pool(device), s));
    char* b = static_cast<char*>(blk);
    CK(cudaMemcpyAsync(b + o_g, records->g, n_all * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(b + o_l, records->l, n_all * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(b + o_w, records->w, n_all * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(b + o_ma, records->macro_id, n_all * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(b + o_mi, records->micro_id, n_all * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(b + o_t, records->latency_us, n_all * 8, cudaMemcpyHostToDevice, s));
    Rec rc{reinterpret_cast<const int64_t*>(b + o_g), reinterpret_cast<const int64_t*>(b + o_l),
           reinterpret_cast<const int32_t*>(b + o_w), reinterpret_cast<const int32_t*>(b + o_ma),
           reinterpret_cast<const int32_t*>(b + o_mi), reinterpret_cast<const double*>(b + o_t)};
    auto* B = new wt_build;
    B->device = device;
    const wt_status st = fit_core(rc, n_all, registry_ids, n_macros, W, p, true, device, s, B);
    cudaFreeAsync(blk, s);
    cudaStreamSynchronize(s);
    if (st != WT_OK) {
        build_release(B);
        delete B;
        return st;
    }
    const wt_status st2 = build_download(B);
    if (st2 != WT_OK) {
        build_release(B);
        delete B;
        return st2;
    }
    fill_result(B, result);
    *out = B;
    return WT_OK;
}

wt_status wt_fit_build_device(const wt_records_desc* records, const int32_t* registry_ids, int32_t n_macros,
                              int32_t W, int32_t p, int32_t flags, int device, void* stream, wt_build** out) {
    if (!records || !out || (n_macros > 0 && !registry_ids)) {
        g_fit_err = "null argument";
        return WT_INVALID_ARGUMENT;
    }
    *out = nullptr;
    if (records->n <= 0) {
        g_fit_err = "build_dual_table: empty record set";
        return WT_INVALID_ARGUMENT;
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(device);
    DevRestore restore{prev_dev};
    Rec rc{records->g, records->l, records->w, records->macro_id, records->micro_id, records->latency_us};
    auto* B = new wt_build;
    B->device = device;
    const wt_status st = fit_core(rc, records->n, registry_ids, n_macros, W, p, (flags & WT_FIT_BASELINES) != 0,
                                  device, static_cast<cudaStream_t>(stream), B);
    if (st != WT_OK) {
        cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        build_release(B);
        delete B;
        return st;
    }
    *out = B;
    return WT_OK;
}

wt_status wt_build_result_get(wt_build* b, wt_build_result* result) {
    if (!b || !result) {
        g_fit_err = "null argument";
        return WT_INVALID_ARGUMENT;
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(b->device);
    DevRestore restore{prev_dev};
    const wt_status st = build_download(b);
    if (st != WT_OK) return st;
    fill_result(b, result);
    return WT_OK;
}

wt_status wt_build_free(wt_build* b) {
    if (!b) return WT_OK;
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(b->device);
    DevRestore restore{prev_dev};
    build_release(b);
    delete b;
    return WT_OK;
}

wt_status wt_fit_bucket_batch(const double* g, const double* l, const double* t, const int64_t* off,
                              int64_t nb, double* coeffs, double* r2, double* mape, int32_t* degenerate,
                              int device) {
    if (nb <= 0) return WT_OK;
    for (int64_t b = 0; b < nb; ++b)
        if (off[b + 1] <= off[b]) {
            g_fit_err = "fit_bucket: no samples";
            return WT_INVALID_ARGUMENT;
        }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    std::vector<void*> owned;
    struct Free {
        std::vector<void*>* v;
        ~Free() {
            for (void* q : *v) cudaFree(q);
        }
    } freer{&owned};
    const int64_t S = off[nb] - off[0];
    double* dg = dalloc<double>(owned, S);
    double* dl = dalloc<double>(owned, S);
    double* dt = dalloc<double>(owned, S);
    double* scr = dalloc<double>(owned, kQScr * S);
    int64_t* lo = dalloc<int64_t>(owned, nb);
    int64_t* hi = dalloc<int64_t>(owned, nb);
    std::vector<int64_t> hlo(nb), hhi(nb);
    for (int64_t b = 0; b < nb; ++b) {
        hlo[b] = off[b] - off[0];
        hhi[b] = off[b + 1] - off[0];
    }
    CK(cudaMemcpy(dg, g + off[0], S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dl, l + off[0], S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dt, t + off[0], S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lo, hlo.data(), nb * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(hi, hhi.data(), nb * 8, cudaMemcpyHostToDevice));
    Buckets bk{nb, lo, hi, dalloc<double>(owned, nb * 4), dalloc<double>(owned, nb), dalloc<double>(owned, nb),
               dalloc<int32_t>(owned, nb)};
    launch_qfit(false, dg, dl, dt, bk, scr, wtb::device_sms(), nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(coeffs, bk.coeff, nb * 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r2, bk.r2, nb * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(mape, bk.mape, nb * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(degenerate, bk.degen, nb * 4, cudaMemcpyDeviceToHost));
    return WT_OK;
}


wt_status wt_build_pack_info(const wt_build* b, int64_t* counts, size_t* bytes) {
    if (!b || !counts || !bytes) {
        g_fit_err = "null argument";
        return WT_INVALID_ARGUMENT;
    }
    counts[0] = b->NM;
    counts[1] = b->NB;
    counts[2] = b->G;
    counts[3] = b->W;
    counts[4] = b->p;
    *bytes = pack_layout(b->NM, b->NB, b->G).total;
    return WT_OK;
}

wt_status wt_build_pack(const wt_build* b, void* dst, size_t cap, void* stream) {
    if (!b || !dst) {
        g_fit_err = "null argument";
        return WT_INVALID_ARGUMENT;
    }
    const PackLayout L = pack_layout(b->NM, b->NB, b->G);
    if (cap < L.total) {
        g_fit_err = "wt_build_pack: destination smaller than the packed build";
        return WT_INVALID_ARGUMENT;
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(b->device);
    DevRestore restore{prev_dev};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaStreamWaitEvent(s, b->done, 0));  // the build's stream may differ
    char* d = static_cast<char*>(dst);
    const PackHead h{kPackMagic, b->NM, b->NB, b->G, b->W, b->p, int64_t(L.total), 0};
    CK(cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, s));  // pageable: staged before return
    for (int a = 0; a < PA_N; ++a)
        if (L.bytes[a]) CK(cudaMemcpyAsync(d + L.off[a], pack_ptr(b, a), L.bytes[a], cudaMemcpyDeviceToDevice, s));
    return WT_OK;
}

wt_status wt_build_merge(const void* packed, size_t stride, int32_t n_parts, const int64_t* counts, int device,
                         void* stream, wt_build** out) {
    if (!packed || !counts || !out || n_parts <= 0) {
        g_fit_err = "null argument";
        return WT_INVALID_ARGUMENT;
    }
    *out = nullptr;
    int64_t NM = 0, NB = 0, G = 0, W = -1, p = -1;
    for (int r = 0; r < n_parts; ++r) {
        const int64_t* c = counts + 5 * r;
        if (c[0] < 0 || c[1] < 0 || c[2] < 0) {
            g_fit_err = "wt_build_merge: negative count";
            return WT_INVALID_ARGUMENT;
        }
        if (c[0] == 0) continue;  // a rank without macros
        if (pack_layout(c[0], c[1], c[2]).total > stride) {
            g_fit_err = "wt_build_merge: part larger than the stride";
            return WT_INVALID_ARGUMENT;
        }
        if ((W >= 0 && c[3] != W) || (p >= 0 && c[4] != p)) {
            g_fit_err = "wt_build_merge: parts fitted with different W / p";
            return WT_INVALID_ARGUMENT;
        }
        W = c[3];
        p = c[4];
        NM += c[0];
        NB += c[1];
        G += c[2];
    }
    if (NM == 0) {
        g_fit_err = "build_dual_table: no macro produced a table";
        return WT_RUNTIME_ERROR;
    }
    if (NB >= INT32_MAX || G >= INT32_MAX) {
        g_fit_err = "wt_build_merge: merged build exceeds 32-bit offsets";
        return WT_UNSUPPORTED;
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(device);
    DevRestore restore{prev_dev};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* B = new wt_build;
    B->device = device;
    struct Guard {
        wt_build*& b;
        cudaStream_t s;
        bool ok = false;
        ~Guard() {
            if (ok || !b) return;
            cudaStreamSynchronize(s);
            build_release(b);
            delete b;
        }
    } guard{B, s};
    const PackLayout M = pack_layout(NM, NB, G);
    {
        void* blk = nullptr;
        CK(cudaMallocFromPoolAsync(&blk, M.total, wtb::device_pool(device), s));
        B->mem.push_back(blk);
        for (int a = 0; a < PA_N; ++a) set_pack_ptr(B, a, static_cast<char*>(blk) + M.off[a]);
    }
    CK(cudaEventCreate(&B->ev0));
    CK(cudaEventCreate(&B->ev1));
    CK(cudaEventCreateWithFlags(&B->done, cudaEventDisableTiming));
    CK(cudaEventRecord(B->ev0, s));
    // segments: (part, array); offset arrays rebased, their closing entry
    // taken from the last non-empty part only
    int last = -1;
    for (int r = 0; r < n_parts; ++r)
        if (counts[5 * r] > 0) last = r;
    std::vector<MergeSeg> segs;
    int64_t bNM = 0, bNB = 0, bG = 0, max_words = 0;
    for (int r = 0; r < n_parts; ++r) {
        const int64_t* c = counts + 5 * r;
        if (c[0] == 0) continue;
        const PackLayout L = pack_layout(c[0], c[1], c[2]);
        const char* src = static_cast<const char*>(packed) + size_t(r) * stride;
        // destination element offsets of this part per array
        const int64_t dst_el[PA_N] = {bNM, bNM, bNM, bNM, bNM, bNM, bNB, bNB, bNB, bNB, bNB, bG, bG, bG,
                                      4 * bNM, 4 * bNB, bNB, bNB, bG, bG};
        const int esz[PA_N] = {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 8, 8, 8, 8, 8, 8};
        for (int a = 0; a < PA_N; ++a) {
            int64_t bytes = int64_t(L.bytes[a]);
            uint32_t add = 0;
            if (a == PA_COFF || a == PA_AAOFF) {
                if (r != last) bytes -= 4;  // the next part's first entry closes this part
                add = uint32_t(a == PA_COFF ? bNB : bG);
            } else if (a == PA_EOFF) {
                add = uint32_t(bG);
            }
            if (bytes <= 0) continue;
            MergeSeg sg{};
            sg.src = reinterpret_cast<const uint32_t*>(src + L.off[a]);
            sg.dst = reinterpret_cast<uint32_t*>(static_cast<char*>(B->mem[0]) + M.off[a] + dst_el[a] * esz[a]);
            sg.words = bytes / 4;
            sg.add = add;
            segs.push_back(sg);
            max_words = std::max(max_words, sg.words);
        }
        bNM += c[0];
        bNB += c[1];
        bG += c[2];
    }
    for (size_t i0 = 0; i0 < segs.size(); i0 += kMergeSegs) {
        MergeArgs ma{};
        ma.nseg = int32_t(std::min<size_t>(kMergeSegs, segs.size() - i0));
        for (int i = 0; i < ma.nseg; ++i) ma.seg[i] = segs[i0 + i];
        const int gx = int(std::min<int64_t>(64, std::max<int64_t>(1, (max_words + 255) / 256)));
        k_build_merge<<<dim3(gx, ma.nseg), 256, 0, s>>>(ma);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(B->ev1, s));
    B->h_macro_id.resize(NM);
    CK(cudaMemcpyAsync(B->h_macro_id.data(), B->t_macro, size_t(NM) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));  // host macro ids (the engine plan needs them)
    B->NM = int32_t(NM);
    B->NB = NB;
    B->G = G;
    B->W = int32_t(W);
    B->p = int32_t(p);
    B->baselines = false;
    CK(cudaEventRecord(B->done, s));
    guard.ok = true;
    *out = B;
    return WT_OK;
}

}  // extern "C"
