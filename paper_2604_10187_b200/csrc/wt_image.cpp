// wt_image.cpp -- resolves a std::vector<DualTable> (flattened as
// wt_tables_desc) into the dense device image the kernels read.
//
// Every data-dependent rule of the reference's query path is decided here,
// once, instead of per query:
//   * tables sorted by macro_id (tuner.cpp:127-132); duplicate ids are
//     rejected because std::sort leaves their order unspecified;
//   * registry.macro(id) join (kernel_map.cpp:96-100), out_of_range text;
//   * the W-horizon switch (tuner.cpp:17-18): row w-1 for w <= W_c holds
//     coeff_table[w], rows for w > W_c hold theta_ext;
//   * the missing-wave fallback (tuner.cpp:20-39): nearest key over ALL
//     keys, ties to the smaller key, source wave kept for the flag text;
//   * the Stage-II map choice and its fallback (tuner.cpp:80-103): ext
//     anchors when extrapolated and non-empty, else anchor_table[w] when
//     non-empty, else the nearest non-empty wave map to (W_c if
//     extrapolated else w), ties to the smaller wave.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <map>
#include <numeric>
#include <tuple>

#include "wt_internal.h"

namespace wtb {

namespace {

wt_status fail(std::string* err, wt_status st, const std::string& msg) {
    *err = msg;
    return st;
}

}  // namespace

namespace {

// Dominance test for the pruning masks.  d(G, L) = f_v - f_d - eps * (S_v + S_d)
// with f = alpha*G*L + beta*G + gamma*L + delta and S the same with absolute
// coefficients (a bound on the magnitude every fp64 rounding error of the
// evaluation scales with): d is bilinear, so d > 0 on a rectangle (possibly
// unbounded in G and/or L) iff it holds at the finite corners and the slopes
// along the unbounded directions are >= 0.  eps = 1e-9 is ~10^6 times the
// worst-case relative rounding error of the 7-operation evaluation, so
// d > 0 implies fl(f_v) > fl(f_d): the victim can neither win nor tie.
bool dominated_by(const double* v, const double* d, long double G0, long double G1, bool ginf, long double L0,
                  long double L1, bool linf) {
    for (int q = 0; q < 4; ++q)
        if (!std::isfinite(v[q]) || !std::isfinite(d[q])) return false;
    const long double eps = 1e-9L;
    long double k[4];
    for (int q = 0; q < 4; ++q)
        k[q] = (long double)v[q] - (long double)d[q] - eps * (std::fabs((long double)v[q]) + std::fabs((long double)d[q]));
    const long double a = k[0], b = k[1], c = k[2], e = k[3];
    auto val = [&](long double G, long double L) { return a * G * L + b * G + c * L + e; };
    if (!(val(G0, L0) > 0)) return false;
    if (linf ? !(a * G0 + c >= 0) : !(val(G0, L1) > 0)) return false;
    if (ginf) {
        if (!(a * L0 + b >= 0)) return false;
        if (linf ? !(a >= 0) : !(a * L1 + b >= 0)) return false;
    } else {
        if (!(val(G1, L0) > 0)) return false;
        if (linf ? !(a * G1 + c >= 0) : !(val(G1, L1) > 0)) return false;
    }
    return true;
}

// Masks for every (segment, row, L bucket): a config is dropped when one of
// the class's per-corner leaders (the configs with the smallest value at the
// rectangle's four corners, unbounded sides sampled far out) dominates it.
void build_prune_masks(HostImage& im) {
    const int32_t R = im.R, NS = int32_t(im.seg_pos.size()), C = im.C;
    const uint32_t S = uint32_t(im.S);
    im.segmask.assign(size_t(NS) * R * kLB, 0u);
    im.segor.assign(size_t(NS) * R, 0u);
    // classes = runs of segments with equal (t_m, t_n, t_k)
    std::vector<int32_t> cls_of(NS);
    for (int32_t s = 0, k = -1; s < NS; ++s) {
        if (s == 0 || im.seg_tiles[4 * s] != im.seg_tiles[4 * (s - 1)] ||
            im.seg_tiles[4 * s + 1] != im.seg_tiles[4 * (s - 1) + 1] ||
            im.seg_tiles[4 * s + 2] != im.seg_tiles[4 * (s - 1) + 2])
            ++k;
        cls_of[s] = k;
    }
    for (int32_t s0 = 0; s0 < NS;) {
        int32_t s1 = s0;
        while (s1 < NS && cls_of[s1] == cls_of[s0]) ++s1;
        const int32_t p0 = im.seg_pos[s0];
        const int32_t p1 = s1 < NS ? im.seg_pos[s1] : C;  // class positions [p0, p1)
        for (int32_t r = 0; r < R; ++r) {
            auto th = [&](int32_t pos) { return &im.theta2[(size_t(pos) * R + r) * 4]; };
            auto usable = [&](int32_t pos) {
                return !(im.meta2[size_t(pos) * R + r] & ROW_NO_COEFF);
            };
            const long double G0 = (long double)r * S + 1, G1 = (long double)(r + 1) * S;
            const bool ginf = r == R - 1;
            for (int32_t lb = 0; lb < kLB; ++lb) {
                const long double L0 = std::ldexp(1.0L, lb), L1 = std::ldexp(1.0L, lb + 1) - 1;
                const bool linf = lb == kLB - 1;
                const long double Gs[2] = {G0, ginf ? G0 * 1e6L : G1}, Ls[2] = {L0, linf ? 2147483647.0L : L1};
                std::vector<int32_t> lead;
                for (int i = 0; i < 2; ++i)
                    for (int j = 0; j < 2; ++j) {
                        int32_t best = -1;
                        long double bv = 0;
                        for (int32_t pos = p0; pos < p1; ++pos) {
                            const double* t = th(pos);
                            if (!usable(pos) || !std::isfinite(t[0]) || !std::isfinite(t[1]) || !std::isfinite(t[2]) ||
                                !std::isfinite(t[3]))
                                continue;
                            const long double v = t[0] * Gs[i] * Ls[j] + t[1] * Gs[i] + t[2] * Ls[j] + t[3];
                            if (best < 0 || v < bv) {
                                best = pos;
                                bv = v;
                            }
                        }
                        if (best >= 0 && std::find(lead.begin(), lead.end(), best) == lead.end()) lead.push_back(best);
                    }
                for (int32_t s = s0; s < s1; ++s) {
                    const int32_t ps = im.seg_pos[s], n = im.seg_tiles[4 * s + 3];
                    uint32_t m = 0;
                    for (int32_t i = 0; i < n; ++i) {
                        bool drop = false;
                        for (int32_t d : lead)
                            if (d != ps + i && usable(d) && dominated_by(th(ps + i), th(d), G0, G1, ginf, L0, L1, linf)) {
                                drop = true;
                                break;
                            }
                        if (!drop) m |= 1u << i;
                    }
                    im.segmask[(size_t(s) * R + r) * kLB + lb] = m;
                }
            }
            for (int32_t s = s0; s < s1; ++s) {
                uint32_t o = 0;
                for (int32_t i = 0; i < im.seg_tiles[4 * s + 3]; ++i) o |= im.meta2[size_t(im.seg_pos[s] + i) * R + r];
                im.segor[size_t(s) * R + r] = o;
            }
        }
        s0 = s1;
    }
}

}  // namespace

wt_status build_image(const wt_tables_desc& T, const wt_registry_desc& reg, const wt_hw& hw,
                      HostImage* out, std::string* err) {
    if (hw.n_sm < 1 || hw.blocks_per_sm < 1)
        return fail(err, WT_INVALID_ARGUMENT, "hardware spec must have positive capacities");
    if (T.n_tables <= 0) return fail(err, WT_INVALID_ARGUMENT, "no dual tables provided");
    const int64_t S64 = int64_t(hw.n_sm) * hw.blocks_per_sm;
    if (S64 >= (int64_t(1) << 30))
        return fail(err, WT_UNSUPPORTED, "slots = n_sm * blocks_per_sm exceeds the device path's range");

    // registry.macro(id): first macro with that id wins (linear scan order).
    std::map<int32_t, int32_t> reg_pos;
    for (int32_t i = reg.n_macros - 1; i >= 0; --i) reg_pos[reg.id[i]] = i;

    std::vector<int32_t> order(T.n_tables);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return T.macro_id[a] < T.macro_id[b]; });
    for (int32_t i = 1; i < T.n_tables; ++i)
        if (T.macro_id[order[i]] == T.macro_id[order[i - 1]])
            return fail(err, WT_INVALID_ARGUMENT,
                        "duplicate macro_id " + std::to_string(T.macro_id[order[i]]) +
                            " in dual tables");

    HostImage& im = *out;
    im.C = T.n_tables;
    im.S = int32_t(S64);
    im.family = reg.family;
    int32_t wmax = 0;
    for (int32_t i = 0; i < T.n_tables; ++i) wmax = std::max(wmax, T.W[i]);
    if (wmax > 2048)
        return fail(err, WT_UNSUPPORTED, "table W above 2048 is outside the device path's range");
    im.R = wmax + 1;
    if (int64_t(im.R) * S64 >= (int64_t(1) << 31))
        return fail(err, WT_UNSUPPORTED, "W * slots exceeds the device path's range");

    const int32_t C = im.C, R = im.R;
    im.macro_id.resize(C);
    im.W.resize(C);
    im.tiles.assign(size_t(C) * 4, 0);
    im.magic.assign(size_t(C) * 4, 0);
    im.theta.assign(size_t(C) * R * 4, 0.0);
    im.rowmeta.assign(size_t(C) * R, 0);
    im.used_w.assign(size_t(C) * R, -1);
    im.amap.assign(size_t(C) * R * 2, 0);
    im.afb.assign(size_t(C) * R, -1);
    im.anchor_l.clear();
    im.anchor_micro.clear();
    im.tm_min = INT32_MAX;
    im.tn_min = INT32_MAX;

    for (int32_t c = 0; c < C; ++c) {
        const int32_t t = order[c];
        const int32_t id = T.macro_id[t];
        im.macro_id[c] = id;
        im.W[c] = T.W[t];
        auto it = reg_pos.find(id);
        if (it == reg_pos.end())
            return fail(err, WT_OUT_OF_RANGE, "no macro config with id " + std::to_string(id));
        int64_t tm = reg.t_m[it->second], tn = reg.t_n[it->second], tk = reg.t_k[it->second];
        if (reg.family == WT_FAMILY_FLASH_ATTENTION) tn = 1;  // g = n_heads * ceil(s_q / t_q)
        if (tm < 1 || tn < 1 || tk < 1) return fail(err, WT_INVALID_ARGUMENT, "tile dims must be >= 1");
        if (tm > INT32_MAX || tn > INT32_MAX || tk > INT32_MAX)
            return fail(err, WT_UNSUPPORTED, "tile dims above 2^31-1 are outside the device path's range");
        im.tiles[4 * c + 0] = int32_t(tm);
        im.tiles[4 * c + 1] = int32_t(tn);
        im.tiles[4 * c + 2] = int32_t(tk);
        Magic a = make_magic(uint32_t(tm)), b = make_magic(uint32_t(tn)), k = make_magic(uint32_t(tk));
        im.magic[4 * c + 0] = a.m;
        im.magic[4 * c + 1] = b.m;
        im.magic[4 * c + 2] = k.m;
        im.magic[4 * c + 3] = a.s | (b.s << 8) | (k.s << 16);
        im.tm_min = std::min<int32_t>(im.tm_min, int32_t(tm));
        im.tn_min = std::min<int32_t>(im.tn_min, int32_t(tn));

        // Anchor maps of this table, stored once in the pool.
        const int32_t aw_lo = T.awave_off[t], aw_hi = T.awave_off[t + 1];
        std::vector<std::pair<int32_t, int32_t>> wave_map;  // (wave, pool offset) non-empty only
        std::vector<int32_t> wave_cnt;
        for (int32_t i = aw_lo; i < aw_hi; ++i) {
            int32_t lo = T.awave_aoff[i], hi = T.awave_aoff[i + 1];
            if (hi <= lo) continue;
            wave_map.push_back({T.awave_w[i], int32_t(im.anchor_l.size())});
            wave_cnt.push_back(hi - lo);
            for (int32_t q = lo; q < hi; ++q) {
                im.anchor_l.push_back(T.anchor_l[q]);
                im.anchor_micro.push_back(T.anchor_micro[q]);
            }
        }
        int32_t ext_off = int32_t(im.anchor_l.size());
        int32_t ext_cnt = T.ext_aoff[t + 1] - T.ext_aoff[t];
        for (int32_t q = T.ext_aoff[t]; q < T.ext_aoff[t + 1]; ++q) {
            im.anchor_l.push_back(T.ext_l[q]);
            im.anchor_micro.push_back(T.ext_micro[q]);
        }
        // nearest non-empty wave map to target (ties -> smaller wave)
        auto nearest_map = [&](int32_t target, int32_t* off, int32_t* cnt, int32_t* wave) {
            int best = INT_MAX;
            int32_t best_w = 0;
            bool found = false;
            for (size_t i = 0; i < wave_map.size(); ++i) {
                int d = std::abs(wave_map[i].first - target);
                if (d < best || (d == best && wave_map[i].first < best_w)) {
                    best = d;
                    best_w = wave_map[i].first;
                    *off = wave_map[i].second;
                    *cnt = wave_cnt[i];
                    found = true;
                }
            }
            *wave = best_w;
            return found;
        };

        const int32_t co_lo = T.coeff_off[t], co_hi = T.coeff_off[t + 1];
        const int32_t Wc = T.W[t];
        for (int32_t r = 0; r < R; ++r) {
            const int32_t w = r + 1;  // last row stands for every w >= R > W_c
            const size_t row = size_t(c) * R + r;
            uint32_t meta = 0;
            const double* th = nullptr;
            bool extrap = (r == R - 1) || (w > Wc);
            if (extrap) {
                meta |= ROW_EXTRAP;
                th = T.theta_ext + 4 * size_t(t);
            } else {
                for (int32_t i = co_lo; i < co_hi; ++i)
                    if (T.coeff_w[i] == w) th = T.coeff_theta + 4 * size_t(i);
                if (!th) {
                    if (co_hi == co_lo) {
                        meta |= ROW_NO_COEFF;
                    } else {
                        int best = INT_MAX;
                        int32_t best_w = 0, best_i = -1;
                        for (int32_t i = co_lo; i < co_hi; ++i) {
                            int d = std::abs(T.coeff_w[i] - w);
                            if (d < best || (d == best && T.coeff_w[i] < best_w)) {
                                best = d;
                                best_w = T.coeff_w[i];
                                best_i = i;
                            }
                        }
                        meta |= ROW_MISSING;
                        im.used_w[row] = best_w;
                        th = T.coeff_theta + 4 * size_t(best_i);
                    }
                }
            }
            if (th)
                for (int q = 0; q < 4; ++q) im.theta[4 * row + q] = th[q];
            // Stage-II map
            int32_t off = 0, cnt = 0, fbw = -1;
            bool have = false;
            if (extrap) {
                if (ext_cnt > 0) {
                    off = ext_off;
                    cnt = ext_cnt;
                    have = true;
                }
            } else {
                for (size_t i = 0; i < wave_map.size(); ++i)
                    if (wave_map[i].first == w) {
                        off = wave_map[i].second;
                        cnt = wave_cnt[i];
                        have = true;
                    }
            }
            if (!have) {
                int32_t target = extrap ? Wc : w;
                if (nearest_map(target, &off, &cnt, &fbw)) {
                    meta |= ROW_ANCHOR_FB;
                    im.afb[row] = fbw;
                } else {
                    meta |= ROW_NO_ANCHOR;
                }
            }
            im.amap[2 * row] = off;
            im.amap[2 * row + 1] = cnt;
            im.rowmeta[row] = meta;
            if (meta & ROW_SPECIAL) im.special = true;
        }
    }
    // Tile classes (first-appearance order) cut into segments of <= kSegCfg.
    {
        std::map<std::tuple<int32_t, int32_t, int32_t>, std::vector<int32_t>> cls;
        std::vector<std::tuple<int32_t, int32_t, int32_t>> first;
        for (int32_t c = 0; c < C; ++c) {
            auto key = std::make_tuple(im.tiles[4 * c], im.tiles[4 * c + 1], im.tiles[4 * c + 2]);
            auto& v = cls[key];
            if (v.empty()) first.push_back(key);
            v.push_back(c);
        }
        im.cls_cfg.clear();
        im.seg_tiles.clear();
        im.seg_magic.clear();
        im.seg_pos.clear();
        // classes in (t_m, t_n, t_k) order: consecutive segments share t_m / t_n,
        // so the kernels recompute the per-shape G (and its wave row) only when
        // the tile footprint changes
        (void)first;
        // segment size: all R rows of one segment must fit a 48 KB staging
        // budget (list mode stages every row); classes split evenly
        im.seg_cfg = int32_t(std::clamp<int64_t>(48 * 1024 / (int64_t(R) * 36), 1, kSegCfg));
        for (const auto& [key, unused] : cls) {
            const auto& v = cls[key];
            const size_t nparts = (v.size() + im.seg_cfg - 1) / im.seg_cfg;
            for (size_t part = 0, s = 0; part < nparts; ++part) {
                const size_t e = v.size() * (part + 1) / nparts;
                const int32_t n = int32_t(e - s);
                const int32_t c0 = v[s];
                im.seg_pos.push_back(int32_t(im.cls_cfg.size()));
                for (int32_t q = 0; q < 3; ++q) im.seg_tiles.push_back(im.tiles[4 * c0 + q]);
                im.seg_tiles.push_back(n);
                for (int32_t q = 0; q < 4; ++q) im.seg_magic.push_back(im.magic[4 * c0 + q]);
                for (int32_t q = 0; q < n; ++q) im.cls_cfg.push_back(v[s + q]);
                s = e;
            }
        }
        im.theta2.resize(im.theta.size());
        im.meta2.resize(im.rowmeta.size());
        for (int32_t pos = 0; pos < C; ++pos) {
            const int32_t c = im.cls_cfg[pos];
            std::copy(im.theta.begin() + size_t(c) * R * 4, im.theta.begin() + size_t(c + 1) * R * 4,
                      im.theta2.begin() + size_t(pos) * R * 4);
            std::copy(im.rowmeta.begin() + size_t(c) * R, im.rowmeta.begin() + size_t(c + 1) * R,
                      im.meta2.begin() + size_t(pos) * R);
        }
        build_prune_masks(im);
        im.theta2t.resize(im.theta.size());
        im.meta2t.resize(im.rowmeta.size());
        for (int32_t pos = 0; pos < C; ++pos)
            for (int32_t r = 0; r < R; ++r) {
                std::copy(im.theta2.begin() + (size_t(pos) * R + r) * 4, im.theta2.begin() + (size_t(pos) * R + r + 1) * 4,
                          im.theta2t.begin() + (size_t(r) * C + pos) * 4);
                im.meta2t[size_t(r) * C + pos] = im.meta2[size_t(pos) * R + r];
            }
    }
    if (im.anchor_l.empty()) {  // keep the pool non-empty for the device
        im.anchor_l.push_back(0);
        im.anchor_micro.push_back(-1);
    }
    return WT_OK;
}

}  // namespace wtb
