// wt_image.cpp -- host side of the device image: validation and the
// O(C log C) structure plan (plan_image), plus the host-only pruning plan
// (prune_plan_host, for wt_prune_plan and the CPU tests).
//
// The plan decides, once per (tables, registry, hw):
//   * tables sorted by macro_id (tuner.cpp:127-132); duplicate ids are
//     rejected because std::sort leaves their order unspecified;
//   * registry.macro(id) join (kernel_map.cpp:96-100), out_of_range text;
//   * R = max W + 1 coefficient rows per config and the slot count S;
//   * tile classes (configs with identical (t_m, t_n, t_k) map every shape to
//     the same (G, L, w)) cut into segments of <= kSegCfg configs.
// The per-row rules (W horizon, missing-wave and anchor fallbacks) and the
// pruning masks are resolved by the shared functions of wt_rows.h -- on the
// device for engines (wt_image_dev.cu), on the host here for the plan.
#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <map>
#include <numeric>
#include <tuple>
#include <unordered_map>

#include "wt_internal.h"
#include "wt_rows.h"

namespace wtb {

namespace {

wt_status fail(std::string* err, wt_status st, const std::string& msg) {
    *err = msg;
    return st;
}

}  // namespace

wt_status plan_image(const int32_t* macro_id, const int32_t* W, int32_t n, const wt_registry_desc& reg,
                     const wt_hw& hw, ImagePlan* out, std::string* err) {
    if (hw.n_sm < 1 || hw.blocks_per_sm < 1)
        return fail(err, WT_INVALID_ARGUMENT, "hardware spec must have positive capacities");
    if (n <= 0) return fail(err, WT_INVALID_ARGUMENT, "no dual tables provided");
    const int64_t S64 = int64_t(hw.n_sm) * hw.blocks_per_sm;
    if (S64 >= (int64_t(1) << 30))
        return fail(err, WT_UNSUPPORTED, "slots = n_sm * blocks_per_sm exceeds the device path's range");

    ImagePlan& P = *out;
    // ascending macro_id (duplicates are rejected below, so any sort that
    // breaks ties by position is the stable order): one sort of packed keys
    P.order.resize(n);
    if (std::is_sorted(macro_id, macro_id + n)) {  // the usual case: tables in ascending id order
        std::iota(P.order.begin(), P.order.end(), 0);
    } else {
        std::vector<uint64_t> key(n);
        for (int32_t i = 0; i < n; ++i) key[i] = (uint64_t(uint32_t(macro_id[i]) ^ 0x80000000u) << 32) | uint32_t(i);
        std::sort(key.begin(), key.end());
        for (int32_t i = 0; i < n; ++i) P.order[i] = int32_t(uint32_t(key[i]));
    }
    for (int32_t i = 1; i < n; ++i)
        if (macro_id[P.order[i]] == macro_id[P.order[i - 1]])
            return fail(err, WT_INVALID_ARGUMENT,
                        "duplicate macro_id " + std::to_string(macro_id[P.order[i]]) + " in dual tables");
    P.C = n;
    P.S = int32_t(S64);
    P.family = reg.family;
    int32_t wmax = 0;
    for (int32_t i = 0; i < n; ++i) wmax = std::max(wmax, W[i]);
    if (wmax > 2048) return fail(err, WT_UNSUPPORTED, "table W above 2048 is outside the device path's range");
    P.R = wmax + 1;
    if (int64_t(P.R) * S64 >= (int64_t(1) << 31))
        return fail(err, WT_UNSUPPORTED, "W * slots exceeds the device path's range");

    // registry.macro(id): first macro with that id wins (linear scan order)
    std::vector<std::pair<int32_t, int32_t>> ids(reg.n_macros);
    for (int32_t i = 0; i < reg.n_macros; ++i) ids[i] = {reg.id[i], i};
    if (!std::is_sorted(reg.id, reg.id + reg.n_macros))
        std::sort(ids.begin(), ids.end());  // (id, position): the first occurrence of an id sorts first

    const int32_t C = n;
    P.macro_id.resize(C);
    P.tiles.assign(size_t(C) * 4, 0);
    P.magic.assign(size_t(C) * 4, 0);
    P.tm_min = INT32_MAX;
    P.tn_min = INT32_MAX;
    std::vector<std::pair<uint32_t, Magic>> mcache;
    size_t k = 0;  // merge walk: tables and registry ids both ascend
    for (int32_t c = 0; c < C; ++c) {
        const int32_t id = macro_id[P.order[c]];
        P.macro_id[c] = id;
        while (k < ids.size() && ids[k].first < id) ++k;
        if (k == ids.size() || ids[k].first != id)
            return fail(err, WT_OUT_OF_RANGE, "no macro config with id " + std::to_string(id));
        const int32_t rp = ids[k].second;  // first occurrence of the id
        int64_t tm = reg.t_m[rp], tn = reg.t_n[rp], tk = reg.t_k[rp];
        if (reg.family == WT_FAMILY_FLASH_ATTENTION) tn = 1;  // g = n_heads * ceil(s_q / t_q)
        if (tm < 1 || tn < 1 || tk < 1) return fail(err, WT_INVALID_ARGUMENT, "tile dims must be >= 1");
        if (tm > INT32_MAX || tn > INT32_MAX || tk > INT32_MAX)
            return fail(err, WT_UNSUPPORTED, "tile dims above 2^31-1 are outside the device path's range");
        P.tiles[4 * c + 0] = int32_t(tm);
        P.tiles[4 * c + 1] = int32_t(tn);
        P.tiles[4 * c + 2] = int32_t(tk);
        // tile dims take few distinct values: memoised magic numbers
        auto magic = [&](uint32_t d) {
            for (const auto& x : mcache)
                if (x.first == d) return x.second;
            const Magic mg = make_magic(d);
            mcache.push_back({d, mg});
            return mg;
        };
        const Magic a = magic(uint32_t(tm)), b = magic(uint32_t(tn)), k = magic(uint32_t(tk));
        P.magic[4 * c + 0] = a.m;
        P.magic[4 * c + 1] = b.m;
        P.magic[4 * c + 2] = k.m;
        P.magic[4 * c + 3] = a.s | (b.s << 8) | (k.s << 16);
        P.tm_min = std::min<int32_t>(P.tm_min, int32_t(tm));
        P.tn_min = std::min<int32_t>(P.tn_min, int32_t(tn));
    }

    // Tile classes in (t_m, t_n, t_k) order -- consecutive segments share
    // t_m / t_n, so the kernels recompute the per-shape G (and its wave row)
    // only when the tile footprint changes -- each cut into segments of at
    // most seg_cfg configs (all R rows of a segment fit a 48 KB staging
    // budget: list mode stages every row), ascending macro_id inside.
    std::vector<int32_t> byc(C);
    {
        // the stable order by tile: bucket the configs by their (t_m, t_n,
        // t_k) class (few distinct classes; consecutive configs usually share
        // one), order the classes, then a counting sort in config order
        bool packable = true;
        for (int32_t c = 0; c < C && packable; ++c)
            for (int q = 0; q < 3; ++q) packable = packable && P.tiles[4 * c + q] < (1 << 21);
        if (packable) {
            auto pack = [&](int32_t c) {
                return (uint64_t(P.tiles[4 * c]) << 42) | (uint64_t(P.tiles[4 * c + 1]) << 21) |
                       uint64_t(P.tiles[4 * c + 2]);
            };
            std::unordered_map<uint64_t, int32_t> cid;
            std::vector<uint64_t> ckey;
            std::vector<int32_t> cls(C);
            uint64_t lastk = ~uint64_t(0);
            int32_t lastc = -1;
            for (int32_t c = 0; c < C; ++c) {
                const uint64_t kk = pack(c);
                if (kk != lastk) {
                    auto it = cid.find(kk);
                    if (it == cid.end()) it = cid.emplace(kk, int32_t(ckey.size())).first, ckey.push_back(kk);
                    lastk = kk;
                    lastc = it->second;
                }
                cls[c] = lastc;
            }
            const int32_t K = int32_t(ckey.size());
            std::vector<int32_t> rank(K), cnt(K + 1, 0);
            {
                std::vector<int32_t> o(K);
                std::iota(o.begin(), o.end(), 0);
                std::sort(o.begin(), o.end(), [&](int32_t a, int32_t b) { return ckey[a] < ckey[b]; });
                for (int32_t r = 0; r < K; ++r) rank[o[r]] = r;
            }
            for (int32_t c = 0; c < C; ++c) ++cnt[rank[cls[c]] + 1];
            for (int32_t r = 0; r < K; ++r) cnt[r + 1] += cnt[r];
            for (int32_t c = 0; c < C; ++c) byc[cnt[rank[cls[c]]]++] = c;
        } else {
            std::vector<std::array<int32_t, 4>> key(C);
            for (int32_t c = 0; c < C; ++c) key[c] = {P.tiles[4 * c], P.tiles[4 * c + 1], P.tiles[4 * c + 2], c};
            std::sort(key.begin(), key.end());
            for (int32_t c = 0; c < C; ++c) byc[c] = key[c][3];
        }
    }
    P.seg_cfg = int32_t(std::clamp<int64_t>(48 * 1024 / (int64_t(P.R) * 36), 1, kSegCfg));
    P.cls_cfg.clear();
    P.seg_tiles.clear();
    P.seg_magic.clear();
    P.seg_pos.clear();
    P.cls_seg.clear();
    P.seg_maxcfg = 1;
    for (int32_t i = 0; i < C;) {
        int32_t j = i + 1;
        const int32_t c0 = byc[i];
        while (j < C && P.tiles[4 * byc[j]] == P.tiles[4 * c0] && P.tiles[4 * byc[j] + 1] == P.tiles[4 * c0 + 1] &&
               P.tiles[4 * byc[j] + 2] == P.tiles[4 * c0 + 2])
            ++j;
        const int64_t sz = j - i;
        const int64_t nparts = (sz + P.seg_cfg - 1) / P.seg_cfg;
        P.cls_seg.push_back(int32_t(P.seg_pos.size()));
        for (int64_t part = 0, s = 0; part < nparts; ++part) {
            const int64_t e = sz * (part + 1) / nparts;
            const int32_t cnt = int32_t(e - s);
            P.seg_pos.push_back(int32_t(P.cls_cfg.size()));
            for (int q = 0; q < 3; ++q) P.seg_tiles.push_back(P.tiles[4 * c0 + q]);
            P.seg_tiles.push_back(cnt);
            for (int q = 0; q < 4; ++q) P.seg_magic.push_back(P.magic[4 * c0 + q]);
            for (int32_t q = 0; q < cnt; ++q) P.cls_cfg.push_back(byc[i + s + q]);
            P.seg_maxcfg = std::max(P.seg_maxcfg, cnt);
            s = e;
        }
        i = j;
    }
    P.cls_seg.push_back(int32_t(P.seg_pos.size()));
    P.cfg_pos.assign(C, 0);
    for (int32_t pos = 0; pos < C; ++pos) P.cfg_pos[P.cls_cfg[pos]] = pos;
    return WT_OK;
}

wt_status prune_plan_host(const wt_tables_desc& T, const wt_registry_desc& reg, const wt_hw& hw, ImagePlan* plan,
                          std::vector<uint32_t>* segmask, std::string* err) {
    const wt_status st = plan_image(T.macro_id, T.W, T.n_tables, reg, hw, plan, err);
    if (st != WT_OK) return st;
    const ImagePlan& P = *plan;
    const int32_t C = P.C, R = P.R;
    const TabView tv{T.W, T.theta_ext, T.coeff_off, T.coeff_w, T.coeff_theta, T.awave_off, T.awave_w, T.awave_aoff,
                     T.ext_aoff, 0, nullptr};
    // rows in class order
    std::vector<double> th2(size_t(C) * R * 4, 0.0);
    std::vector<uint32_t> m2(size_t(C) * R, 0);
    for (int32_t pos = 0; pos < C; ++pos) {
        const int32_t t = P.order[P.cls_cfg[pos]];
        for (int32_t r = 0; r < R; ++r) {
            RowOut o;
            resolve_row(tv, t, r, R, &o);
            if (o.theta)
                for (int q = 0; q < 4; ++q) th2[(size_t(pos) * R + r) * 4 + q] = o.theta[q];
            m2[size_t(pos) * R + r] = o.meta;
        }
    }
    const int32_t NS = int32_t(P.seg_pos.size()), NCLS = int32_t(P.cls_seg.size()) - 1;
    segmask->assign(size_t(NS) * R * kLB, 0u);
    for (int32_t k = 0; k < NCLS; ++k) {
        const int32_t s0 = P.cls_seg[k], s1 = P.cls_seg[k + 1];
        const int32_t p0 = P.seg_pos[s0], p1 = s1 < NS ? P.seg_pos[s1] : C;
        for (int32_t r = 0; r < R; ++r) {
            auto th = [&](int32_t pos) { return &th2[(size_t(pos) * R + r) * 4]; };
            auto ok = [&](int32_t pos) { return prunable(th(pos), m2[size_t(pos) * R + r]); };
            for (int32_t lb = 0; lb < kLB; ++lb) {
                const Cell cl = cell_of(r, lb, R, P.S);
                int32_t lead[4];
                for (int i = 0; i < 2; ++i)
                    for (int j = 0; j < 2; ++j) {
                        int32_t best = -1;
                        double bv = 0;
                        for (int32_t pos = p0; pos < p1; ++pos) {
                            if (!ok(pos)) continue;
                            const double v = corner_value(th(pos), cl.Gs[i], cl.Ls[j]);
                            if (!std::isfinite(v)) continue;
                            if (best < 0 || v < bv) {
                                best = pos;
                                bv = v;
                            }
                        }
                        lead[2 * i + j] = best;
                    }
                for (int32_t s = s0; s < s1; ++s) {
                    const int32_t ps = P.seg_pos[s], cnt = P.seg_tiles[4 * s + 3];
                    uint32_t m = 0;
                    for (int32_t i = 0; i < cnt; ++i) {
                        const int32_t v = ps + i;
                        bool drop = false;
                        if (ok(v))
                            for (int q = 0; q < 4 && !drop; ++q)
                                drop = lead[q] >= 0 && lead[q] != v &&
                                       dominated(th(v), th(lead[q]), cl.G0, cl.G1, cl.ginf, cl.L0, cl.L1, cl.linf);
                        if (!drop) m |= 1u << i;
                    }
                    (*segmask)[(size_t(s) * R + r) * kLB + lb] = m;
                }
            }
        }
    }
    return WT_OK;
}

}  // namespace wtb
