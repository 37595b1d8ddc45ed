// wt_internal.h -- shared between the host image builder, the C-ABI layer
// and the sm_100a kernels.  Not part of the public boundary.
#pragma once

#include <vector_types.h>

#include <cstdint>
#include <string>
#include <vector>

#include "wavetune_c.h"

namespace wtb {

// Row metadata bits (one u32 per (config, row)).
enum : uint32_t {
    ROW_EXTRAP = 1u << 0,       // row serves w > W_c: theta_ext, ext anchors
    ROW_MISSING = 1u << 1,      // coefficient fallback (missing_wave_<w>_used_<k>)
    ROW_NO_COEFF = 1u << 2,     // coeff_table empty and w <= W_c: runtime_error
    ROW_ANCHOR_FB = 1u << 3,    // anchor_fallback_wave_<k>
    ROW_NO_ANCHOR = 1u << 4,    // no non-empty anchor map: runtime_error
};
constexpr uint32_t ROW_SPECIAL = ROW_MISSING | ROW_NO_COEFF;

// Exact floor(y / d) for 0 <= y < 2^31 and 1 <= d < 2^31:
//   floor(y / d) = umulhi(2y, m) >> s,  s = ceil(log2 d), m = ceil(2^(31+s) / d)
// (m < 2^32; error y * (m*d - 2^(31+s)) < 2^31 * d <= 2^(31+s)).
struct Magic {
    uint32_t m;
    uint32_t s;
};
inline Magic make_magic(uint32_t d) {
    uint32_t s = 0;
    while ((uint64_t(1) << s) < d) ++s;
    const uint64_t num = uint64_t(1) << (31 + s);  // s <= 31: fits 64 bits
    const uint64_t m = (num + d - 1) / d;
    return Magic{(uint32_t)m, s};
}

// POD image handed to kernels by value.
struct DevImage {
    int32_t C;          // configs (tables), ascending macro_id
    int32_t R;          // rows per config: waves 1..R-1 then row R-1 = every w >= R
    int32_t S;          // slots
    uint32_t RS;        // R * S  (< 2^31)
    uint32_t mS, sS;    // magic for / S
    int32_t special;    // any ROW_SPECIAL row exists
    const int32_t* macro_id;  // [C]
    const int4* tiles;        // [C] {t_m, t_n, t_k, 0} (attention: t_n = 1)
    const uint4* magic;       // [C] {m_m, m_n, m_k, s_m | s_n << 8 | s_k << 16}
    const double4* theta;     // [C*R]
    const uint32_t* rowmeta;  // [C*R]
    const int32_t* used_w;    // [C*R] coefficient fallback source wave or -1
    const int2* amap;         // [C*R] {offset, count} into the anchor pool
    const int32_t* afb;       // [C*R] anchor fallback wave or -1
    const int64_t* anchor_l;  // pool
    const int32_t* anchor_micro;
    int32_t tm_min, tn_min;   // for the per-query wide-range guard
    // Tile-class view: configs with identical (t_m, t_n, t_k) map every shape
    // to the same (G, L, w), so the integer work is done once per class.
    // Classes are cut into segments of <= kSegCfg configs; within a segment
    // configs keep ascending macro_id order.
    int32_t nseg;
    int32_t seg_cfg;          // max configs per segment
    const int4* seg_tiles;    // [nseg] {t_m, t_n, t_k, ncfg}
    const uint4* seg_magic;   // [nseg] as magic
    const int32_t* seg_pos;   // [nseg] first position in the class-ordered list
    const int32_t* cls_cfg;   // [C] class-ordered position -> config index
    const double4* theta2;    // [C*R] rows in class order
    const uint32_t* meta2;    // [C*R] rowmeta in class order
    const double4* theta2t;   // [R][C] rows by wave, class order inside (k_eval3:
    const uint32_t* meta2t;   //        a segment's configs are contiguous)
    // Exact pruning: bit i of segmask[(seg * R + row) * kLB + lb] is clear when
    // config i of the segment is strictly beaten -- with a margin far above
    // fp64 rounding -- by another config of its tile class for every (G, L)
    // of wave row `row` and L-bucket lb (L in [2^lb, 2^(lb+1)), last bucket
    // unbounded); such a config can neither win nor tie Stage I there.
    // segor[seg * R + row] = OR of the segment's rowmeta at that row (the
    // flags of skipped configs still count).  prune = 0: all bits set.
    int32_t prune;
    int32_t seg_maxcfg;       // largest segment (configs)
    // instrumentation (null = off): physically executed (shape|query, config)
    // evaluations of k_sweep2 / k_eval4, lane-evaluations incl. idle lanes
    unsigned long long* eval_count;
    const uint32_t* segmask;
    const uint32_t* segor;
};

constexpr int kSegCfg = 32;
constexpr int kLB = 16;  // L buckets of the pruning masks

// Host-side structure of an image (plan_image): everything that depends only
// on the table ids, their W, the registry and the hardware -- O(C log C) --
// so the O(C * R) row resolution and the pruning masks can be built on the
// device from tables that already live there (wt_image_dev.cu).
struct ImagePlan {
    int32_t C = 0, R = 0, S = 0, family = 0;
    int32_t tm_min = 0, tn_min = 0;
    int32_t seg_cfg = 32;
    std::vector<int32_t> order;      // [C] config (ascending macro_id) -> table index
    std::vector<int32_t> macro_id;   // [C]
    std::vector<int32_t> tiles;      // 4 per config {t_m, t_n, t_k, 0}
    std::vector<uint32_t> magic;     // 4 per config
    std::vector<int32_t> seg_tiles;  // 4 per segment {t_m, t_n, t_k, ncfg}
    std::vector<uint32_t> seg_magic; // 4 per segment
    std::vector<int32_t> seg_pos;    // [nseg] first class-ordered position
    std::vector<int32_t> cls_cfg;    // [C] class-ordered position -> config
    std::vector<int32_t> cfg_pos;    // [C] config -> class-ordered position
    std::vector<int32_t> cls_seg;    // [ncls + 1] first segment of each tile class
    int32_t seg_maxcfg = 1;
};

// Validates and plans (the reference's error texts for duplicate ids,
// unknown ids, empty table sets).  macro_id / W: host arrays of n tables.
wt_status plan_image(const int32_t* macro_id, const int32_t* W, int32_t n, const wt_registry_desc& reg,
                     const wt_hw& hw, ImagePlan* out, std::string* err);

// Host-only pruning plan (wt_prune_plan): the same rows and masks the device
// builder produces, computed on the host from host tables.
wt_status prune_plan_host(const wt_tables_desc& t, const wt_registry_desc& r, const wt_hw& hw, ImagePlan* plan,
                          std::vector<uint32_t>* segmask, std::string* err);

// One device allocation carved into 256-byte aligned pieces.
struct Arena {
    size_t used = 0;
    size_t take(size_t bytes) {
        size_t off = used;
        used += (bytes + 255) & ~size_t(255);
        return off;
    }
};

// Thread-local message returned by wt_last_error().
void set_last_error(const std::string& msg);


}  // namespace wtb
