// wt_image_dev.h -- launch interface of the device image builder.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "wt_internal.h"
#include "wt_rows.h"

namespace wtb {

struct ImgRowsArgs {
    int32_t C, R;
    const int32_t* order;    // [C] config -> table index
    const int32_t* cfg_pos;  // [C] config -> class-ordered position
    double4* theta;
    uint32_t* rowmeta;
    int32_t* used_w;
    int2* amap;
    int32_t* afb;
    double4* theta2;
    uint32_t* meta2;
    double4* theta2t;
    uint32_t* meta2t;
    uint32_t* special;       // OR of (meta & ROW_SPECIAL) != 0
};

struct ImgPruneArgs {
    int32_t C, R, S, nseg;
    int64_t ncells;          // tile classes * R * kLB
    const int32_t* cls_seg;  // [ncls + 1]
    const int32_t* seg_pos;  // [nseg]
    const int4* seg_tiles;   // [nseg] {t_m, t_n, t_k, configs}
    const double4* theta2;
    const uint32_t* meta2;
    uint32_t* segmask;
    uint32_t* segor;
};

// Device-resident tables of a K2 build (wt_fit.cu), for engine creation
// without a host round trip.
struct BuildTables {
    int device;
    int32_t n_tables;
    const int32_t* macro_id_host;  // [n_tables] registry order
    int32_t W;                     // every table's W
    TabView tv;                    // device pointers
    const int64_t* anchor_l;
    const int32_t* anchor_micro;
    int64_t n_anchor;
    const int64_t* ext_l;
    const int32_t* ext_micro;
    int64_t n_ext;
};
wt_status build_device_tables(const wt_build* b, BuildTables* out);

cudaError_t launch_image_build(const TabView& T, const ImgRowsArgs& rows, const ImgPruneArgs& prune,
                               cudaStream_t st);

}  // namespace wtb
