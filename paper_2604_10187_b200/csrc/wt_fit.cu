// wt_fit.cu -- K2 batched least-squares / dual-table build (in progress).
#include "wavetune_c.h"

extern "C" {
wt_status wt_fit_build(const wt_records_desc*, const int32_t*, int32_t, int32_t, int32_t, int,
                       wt_build**, wt_build_result*) {
    return WT_UNSUPPORTED;
}
wt_status wt_build_free(wt_build*) { return WT_OK; }
wt_status wt_fit_bucket_batch(const double*, const double*, const double*, const int64_t*, int64_t,
                              double*, double*, double*, int32_t*, int) {
    return WT_UNSUPPORTED;
}
}
