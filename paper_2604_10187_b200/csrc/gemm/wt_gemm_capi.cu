// wt_gemm_capi.cu -- C-ABI of the validation GEMM family (include/wavetune_gemm.h).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "wavetune_c.h"
#include "wavetune_gemm.h"
#include "wt_gemm.h"

namespace wtb::gemm {
namespace {

constexpr size_t kWorkspace = kWorkspaceBytes;

struct DeviceState {
    void* workspace = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};

std::mutex g_mu;
DeviceState g_dev[64];

int state(DeviceState** out) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return WT_CUDA_ERROR;
    DeviceState& s = g_dev[d];
    if (!s.workspace) {
        if (cudaMalloc(&s.workspace, kWorkspace) != cudaSuccess) return WT_CUDA_ERROR;
        if (cudaMemset(s.workspace, 0, kWorkspace) != cudaSuccess) return WT_CUDA_ERROR;
        if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess) return WT_CUDA_ERROR;
        if (cudaEventCreate(&s.e0) != cudaSuccess || cudaEventCreate(&s.e1) != cudaSuccess) return WT_CUDA_ERROR;
    }
    *out = &s;
    return WT_OK;
}

bool valid_swizzle(int s) { return s == 1 || s == 2 || s == 4 || s == 8; }

int status_of(int rc) {
    switch (rc) {
        case 0: return WT_OK;
        case 1: return WT_UNSUPPORTED;      // shape / alignment not supported by the kernel
        case 2: return WT_RUNTIME_ERROR;    // setup (tensor maps, attributes, workspace)
        case 4: return WT_RUNTIME_ERROR;
        default: return WT_CUDA_ERROR;
    }
}

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_fill(__nv_bfloat16* p, size_t n, uint64_t seed) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t h = splitmix(seed ^ (i * 0xD6E8FEB86659FD93ull));
        p[i] = __float2bfloat16(float(int64_t(h >> 40) - (int64_t(1) << 23)) * (1.0f / float(1 << 23)));
    }
}

int launch_fill(void* p, size_t n, uint64_t seed, cudaStream_t st) {
    if (n == 0) return WT_OK;
    const int blocks = int(std::min<size_t>((n + 255) / 256, size_t(148) * 16));
    k_fill<<<blocks, 256, 0, st>>>(static_cast<__nv_bfloat16*>(p), n, seed);
    return cudaGetLastError() == cudaSuccess ? WT_OK : WT_CUDA_ERROR;
}

int time_one(DeviceState* s, int cfg, int swz, int M, int N, int K, const void* A, const void* B, void* C,
             int warmup, int reps, double* us) {
    RunArgs r{M, N, K, A, B, C, swz, s->workspace, kWorkspace, s->stream};
    const int rc = kFamily[cfg].run(r, warmup, reps, s->e0, s->e1);
    if (rc) return status_of(rc);
    if (cudaEventSynchronize(s->e1) != cudaSuccess) return WT_CUDA_ERROR;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, s->e0, s->e1) != cudaSuccess) return WT_CUDA_ERROR;
    *us = double(ms) * 1000.0 / reps;
    return WT_OK;
}

}  // namespace
}  // namespace wtb::gemm

using namespace wtb::gemm;

extern "C" {

int wt_gemm_family_size(void) { return kFamilySize; }

int wt_gemm_config(int cfg, int* bm, int* bn, int* bk, int* stages) {
    if (cfg < 0 || cfg >= kFamilySize) return WT_OUT_OF_RANGE;
    if (bm) *bm = kFamily[cfg].bm;
    if (bn) *bn = kFamily[cfg].bn;
    if (bk) *bk = kFamily[cfg].bk;
    if (stages) *stages = kFamily[cfg].stages;
    return WT_OK;
}

int wt_gemm_run(int cfg, int swizzle, int M, int N, int K, const void* A, const void* B, void* C, void* stream) {
    if (cfg < 0 || cfg >= kFamilySize) return WT_OUT_OF_RANGE;
    if (!valid_swizzle(swizzle) || M <= 0 || N <= 0 || K <= 0 || !A || !B || !C) return WT_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(g_mu);  // the workspace is shared per device
    DeviceState* s = nullptr;
    if (int rc = state(&s)) return rc;
    RunArgs r{M, N, K, A, B, C, swizzle, s->workspace, kWorkspace, stream};
    return status_of(kFamily[cfg].run(r, 0, 0, nullptr, nullptr));
}

int wt_gemm_time(int cfg, int swizzle, int M, int N, int K, const void* A, const void* B, void* C, int warmup,
                 int reps, double* mean_us) {
    if (cfg < 0 || cfg >= kFamilySize) return WT_OUT_OF_RANGE;
    if (!valid_swizzle(swizzle) || M <= 0 || N <= 0 || K <= 0 || !A || !B || !C || warmup < 0 || reps <= 0 ||
        !mean_us)
        return WT_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState* s = nullptr;
    if (int rc = state(&s)) return rc;
    return time_one(s, cfg, swizzle, M, N, K, A, B, C, warmup, reps, mean_us);
}

int wt_gemm_measure_batch(int n, const int32_t* cfg, const int32_t* swizzle, const int32_t* M, const int32_t* N,
                          const int32_t* K, int warmup, int reps, uint64_t seed, double* latency_us) {
    if (n < 0 || (n > 0 && (!cfg || !swizzle || !M || !N || !K || !latency_us)) || warmup < 0 || reps <= 0)
        return WT_INVALID_ARGUMENT;
    size_t mk = 0, nk = 0, mn = 0;
    for (int i = 0; i < n; ++i) {
        if (cfg[i] < 0 || cfg[i] >= kFamilySize) return WT_OUT_OF_RANGE;
        if (!valid_swizzle(swizzle[i]) || M[i] <= 0 || N[i] <= 0 || K[i] <= 0) return WT_INVALID_ARGUMENT;
        mk = std::max(mk, size_t(M[i]) * K[i]);
        nk = std::max(nk, size_t(N[i]) * K[i]);
        mn = std::max(mn, size_t(M[i]) * N[i]);
    }
    if (n == 0) return WT_OK;
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState* s = nullptr;
    if (int rc = state(&s)) return rc;
    void *A = nullptr, *B = nullptr, *C = nullptr;
    int rc = WT_OK;
    if (cudaMalloc(&A, mk * 2) != cudaSuccess || cudaMalloc(&B, nk * 2) != cudaSuccess ||
        cudaMalloc(&C, mn * 2) != cudaSuccess)
        rc = WT_CUDA_ERROR;
    if (rc == WT_OK) rc = launch_fill(A, mk, seed, s->stream);
    if (rc == WT_OK) rc = launch_fill(B, nk, seed ^ 0x5bd1e995ull, s->stream);
    for (int i = 0; rc == WT_OK && i < n; ++i) {
        double us = -1.0;
        const int r = time_one(s, cfg[i], swizzle[i], M[i], N[i], K[i], A, B, C, warmup, reps, &us);
        if (r == WT_UNSUPPORTED) us = -1.0;
        else if (r != WT_OK) rc = r;
        latency_us[i] = us;
    }
    cudaStreamSynchronize(s->stream);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
    return rc;
}

int wt_gemm_fill_uniform(void* p, size_t n, uint64_t seed, void* stream) {
    if (!p && n) return WT_INVALID_ARGUMENT;
    return launch_fill(p, n, seed, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
