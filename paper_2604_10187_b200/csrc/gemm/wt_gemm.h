// wt_gemm.h -- validation GEMM family: shared declarations.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace wtb::gemm {

// workspace layout: split-K arrival counters (zeroed once at allocation, kept
// zero by the kernels) | fp32 partial tiles
constexpr size_t kCounterBytes = size_t(64) << 10;
constexpr size_t kWorkspaceBytes = size_t(32) << 20;

struct RunArgs {
    int M, N, K;
    const void* A;  // bf16 [M, K] row-major
    const void* B;  // bf16 [N, K] row-major (K x N column-major)
    void* C;        // bf16 [M, N] row-major
    int swizzle;
    void* workspace;
    size_t workspace_bytes;
    void* stream;
};

// run(): reps == 0 -> one launch; reps > 0 -> `warmup` untimed launches,
// then `reps` launches bracketed by e0 / e1 on r.stream.  Returns 0, or
// 1 = shape / alignment not supported, 2 = setup failed, 3 = launch failed.
struct Config {
    int bm, bn, bk, stages;
    int (*run)(const RunArgs&, int warmup, int reps, cudaEvent_t e0, cudaEvent_t e1);
};

// the family compiled into this library (wt_tc_family.cu: the hand-written
// tcgen05 kernels; tools/cutlass_xcheck: the CUTLASS cross-check build)
extern const Config kFamily[];
extern const int kFamilySize;


}  // namespace wtb::gemm
