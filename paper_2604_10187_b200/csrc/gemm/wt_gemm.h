// wt_gemm.h -- validation GEMM family: shared declarations.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace wtb::gemm {

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

struct Config {
    int bm, bn, bk, stages;
    int (*run)(const RunArgs&, int warmup, int reps, cudaEvent_t e0, cudaEvent_t e1);
};


}  // namespace wtb::gemm
