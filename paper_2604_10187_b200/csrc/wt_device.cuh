// wt_device.cuh -- exact integer / fp64 building blocks for the sm_100a
// decision kernels.  Every helper reproduces the reference's C++ arithmetic
// bit for bit.
#pragma once

#include <cstdint>

#include "wt_decide.h"
#include "wt_internal.h"

namespace wtb {

// floor(y2/2 / d) for y2 = 2*y, y < 2^31 (see make_magic): IMAD.HI + SHF.
__device__ __forceinline__ uint32_t mdiv2(uint32_t y2, uint32_t m, uint32_t s) {
    return __umulhi(y2, m) >> s;
}

// ceil_div(x, d) = (x + d - 1) / d for 1 <= x < 2^31 (kernel_map.hpp:17).
__device__ __forceinline__ uint32_t cdiv_m(uint32_t x, uint32_t m, uint32_t s) {
    return mdiv2(2u * (x - 1u), m, s) + 1u;
}

// Exact (double)x for x < 2^32: one DADD, no I2F (the conversion pipe runs
// at a quarter of the DADD rate).
__device__ __forceinline__ double u32_to_f64(uint32_t x) {
    return __dsub_rn(__hiloint2double(0x43300000, int(x)), 4503599627370496.0);
}

// (double)x for x < 2^63 with the reference's rounding (i64 -> double, RN).
__device__ __forceinline__ double u64_to_f64(uint64_t x) {
    if (x < (uint64_t(1) << 52))
        return __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ULL | x)),
                         4503599627370496.0);
    return __ull2double_rn(x);
}

// BilinearCoeffs::predict (model.hpp:20-23) as the reference evaluates it:
//   ((((alpha*g)*l) + (beta*g)) + (gamma*l)) + delta, binary64, no FMA.
// gl = gamma * l may be precomputed (same rounded product).
__device__ __forceinline__ double bilinear(double a, double b, double gl, double d, double gd,
                                           double ld) {
    double t = __dmul_rn(__dmul_rn(a, gd), ld);
    t = __dadd_rn(t, __dmul_rn(b, gd));
    t = __dadd_rn(t, gl);
    return __dadd_rn(t, d);
}

// Row of the dense image for grid size g (w = ceil(g/S), rows clamp at R-1).
__device__ __forceinline__ uint32_t row_of(uint32_t g_clamped, uint32_t mS, uint32_t sS) {
    return mdiv2(2u * g_clamped - 2u, mS, sS);
}

// Read-only 32-byte row load (two 16-byte LDG.E.128.CONSTANT).
__device__ __forceinline__ double4 ldg_row(const double4* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// nearest_anchor (tuner.cpp:44-70): lower_bound, then the closer neighbour,
// ties to the smaller anchor.  Returns the index; *comps = comparisons.
__device__ __forceinline__ int nearest_anchor_idx(const int64_t* a, int n, int64_t l, int* comps) {
    int c = 0, lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        ++c;
        if (a[mid] < l)
            lo = mid + 1;
        else
            hi = mid;
    }
    int r;
    if (lo == 0) {
        r = 0;
    } else if (lo == n) {
        r = n - 1;
    } else {
        ++c;
        r = (l - a[lo - 1] <= a[lo] - l) ? lo - 1 : lo;
    }
    *comps = c;
    return r;
}

// Top-k insertion into an ascending list; equal latencies keep the earlier
// (smaller macro_id) entry first; NaN and +inf never enter.
template <int KM>
__device__ __forceinline__ void topk_insert(double (&L)[KM], int (&I)[KM], double v, int c) {
    if (!(v < L[KM - 1])) return;
    bool placed = false;
#pragma unroll
    for (int q = KM - 1; q > 0; --q) {
        if (v < L[q - 1]) {
            L[q] = L[q - 1];
            I[q] = I[q - 1];
        } else if (!placed) {
            L[q] = v;
            I[q] = c;
            placed = true;
        }
    }
    if (!placed) {
        L[0] = v;
        I[0] = c;
    }
}

// Read-only load: the non-coherent path for global memory (G), a plain
// generic load for images staged into shared memory (!G).
template <bool G, class T>
__device__ __forceinline__ T rd(const T* p) {
    if constexpr (G) return __ldg(p);
    else return *p;
}

// ---------------------------------------------------------------- Stage II
struct Stage2 {
    int32_t micro;
    int32_t comps;
    uint32_t flags;  // WT_FLAG_* bits and status << 24
};

template <bool G = true>
__device__ __forceinline__ Stage2 stage2(const DevImage& im, int c, uint32_t row, int64_t l) {
    const size_t rr = size_t(c) * im.R + row;
    const uint32_t meta = rd<G>(im.rowmeta + rr);
    Stage2 s;
    s.flags = (meta & ROW_EXTRAP) ? WT_FLAG_EXTRAPOLATED : 0u;
    if (meta & ROW_ANCHOR_FB) s.flags |= WT_FLAG_ANCHOR_FALLBACK;
    if (meta & ROW_NO_ANCHOR) {
        s.micro = -1;
        s.comps = 0;
        s.flags |= uint32_t(WT_RUNTIME_ERROR) << 24;
        return s;
    }
    const int2 am = rd<G>(im.amap + rr);
    int comps;
    int k = nearest_anchor_idx(im.anchor_l + am.x, am.y, l, &comps);
    s.micro = rd<G>(im.anchor_micro + am.x + k);
    s.comps = comps;
    return s;
}

// Winner epilogue shared by every mode: w (true wave count), regime,
// Stage II, tail fraction.
struct Final {
    int32_t macro, micro, wave, comps;
    uint32_t flags;
    float tail;
};

template <bool G = true>
__device__ __forceinline__ Final finish(const DevImage& im, int c, double best, uint64_t g,
                                        int64_t l, uint32_t acc_meta) {
    Final f;
    f.tail = 0.f;
    if (c < 0) {  // every candidate NaN or +inf: the reference dereferences null
        f.macro = f.micro = f.wave = -1;
        f.comps = 0;
        f.flags = uint32_t(WT_RUNTIME_ERROR) << 24;
        return f;
    }
    if (acc_meta & ROW_NO_COEFF) {  // predict_latency threw for some table
        f.macro = f.micro = f.wave = -1;
        f.comps = 0;
        f.flags = uint32_t(WT_RUNTIME_ERROR) << 24;
        return f;
    }
    const uint64_t S = uint64_t(im.S);
    const uint64_t w64 = (g + S - 1) / S;
    const uint32_t row = uint32_t(w64 < uint64_t(im.R) ? w64 : uint64_t(im.R)) - 1u;
    Stage2 s = stage2<G>(im, c, row, l);
    f.macro = rd<G>(im.macro_id + c);
    f.micro = s.micro;
    f.wave = int32_t(uint32_t(w64));
    f.comps = s.comps;
    f.flags = s.flags | ((acc_meta & ROW_MISSING) ? WT_FLAG_MISSING_WAVE : 0u);
    f.tail = float(double(g - (w64 - 1) * S) / double(S));
    if (f.flags >> 24) f.macro = -1;
    (void)best;
    return f;
}

// One decision into the SoA outputs (failed queries: -1 / NaN / zeros).
__device__ __forceinline__ void write_decision(const DecOut& o, int64_t q, const Final& f,
                                               double lat, uint64_t g, int64_t l) {
    const bool ok = (f.flags >> 24) == 0;
    o.macro[q] = ok ? f.macro : -1;
    o.micro[q] = ok ? f.micro : -1;
    o.lat[q] = ok ? lat : __longlong_as_double(0x7ff8000000000000LL);
    if (o.g) o.g[q] = ok ? int64_t(g) : 0;
    if (o.l) o.l[q] = ok ? l : 0;
    if (o.wave) o.wave[q] = ok ? f.wave : 0;
    if (o.flags) o.flags[q] = f.flags;
    if (o.comps) o.comps[q] = ok ? f.comps : 0;
    if (o.tail) o.tail[q] = ok ? double(f.tail) : 0.0;
}

// ---- list-mode grouping key (wt_eval3.cu)
constexpr int kSpreadBits = 2;

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

// wave row of shape (M, N) under a tile class's magic numbers (g = tiles)
__device__ __forceinline__ uint32_t row_for(const DevImage& im, uint32_t y2M, uint32_t y2N, uint4 mg, uint64_t* g) {
    const uint32_t mt = mdiv2(y2M, mg.x, mg.w & 0xffu) + 1u;
    const uint32_t nt = mdiv2(y2N, mg.y, (mg.w >> 8) & 0xffu) + 1u;
    *g = uint64_t(mt) * nt;
    const uint32_t gc = *g > im.RS ? im.RS : uint32_t(*g);
    return row_of(gc, im.mS, im.sS);
}

// Grouping key of a query (list evaluation, wt_eval3.cu): the wave row of
// the last tile class (a prefix, so neighbouring groups are similar), the
// bucket floor(log2 K) (the pruning masks are per L bucket) and a hash of
// the rows of every distinct (t_m, t_n); `bits` wide, then kSpreadBits
// sub-bucket bits from the list slot (spreads the atomics of large groups;
// the sub-buckets of one key stay adjacent after the scan).
// mode 0: rows of the first and the last class + hash (no K bucket).
__device__ __forceinline__ uint32_t eval_key(const DevImage& im, int32_t m, int32_t n, int32_t k, int bits,
                                             int64_t slot, int mode = 1) {
    uint32_t M, N, K;
    uint32_t key = 0;
    if (mode == 3) {  // no grouping (A/B): one key, list order kept chunk by chunk
        key = 0;
    } else if (!query_status(im, m, n, k, &M, &N, &K)) {
        int br = 1;
        while ((1 << br) < im.R) ++br;
        const uint32_t y2M = 2u * (M - 1u), y2N = 2u * (N - 1u);
        uint32_t h = 0x811c9dc5u, first = 0, last = 0, pm = 0, pn = 0, ps = 0xffffffffu;
        for (int s = 0; s < im.nseg; ++s) {
            const uint4 mg = __ldg(im.seg_magic + s);
            if (mg.x == pm && mg.y == pn && (mg.w & 0xffffu) == ps) continue;  // same (t_m, t_n)
            pm = mg.x;
            pn = mg.y;
            ps = mg.w & 0xffffu;
            uint64_t g;
            last = row_for(im, y2M, y2N, mg, &g);
            if (s == 0) first = last;
            h = (h ^ last) * 0x01000193u;
        }
        h ^= h >> 15;
        h *= 0x2c1b3c6du;
        h ^= h >> 12;
        const uint32_t kb = uint32_t(31 - __clz(int(K)));  // 0..30
        const int hb = bits - br - 5;
        if (mode == 0 && bits - 2 * br >= 2)
            key = (first << (bits - br)) | (last << (bits - 2 * br)) | (h & ((1u << (bits - 2 * br)) - 1u));
        else if (hb >= 2)
            key = (last << (bits - br)) | (kb << hb) | (h & ((1u << hb) - 1u));
        else
            key = h & ((1u << bits) - 1u);
    }
    return (key << kSpreadBits) | uint32_t(slot & ((1 << kSpreadBits) - 1));
}

}  // namespace wtb
