// wt_tc_family.cu -- instantiations + host launch of the hand-written
// tcgen05 GEMM family (wt_tc.cuh): TMA tensor maps, persistent grid sizing,
// cluster launch for the CTA-pair tiles.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "wt_gemm.h"
#include "wt_tc.cuh"

namespace wtb::gemm {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static std::once_flag once;
    static EncodeFn fn = nullptr;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

int device_sms() {
    static int sms[64] = {};
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= 64) return 148;
    if (!sms[d]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        sms[d] = v > 0 ? v : 148;
    }
    return sms[d];
}

// bf16 [rows, K] row-major, box {64 elements (128 B), box_rows}, 128-byte swizzle;
// out-of-range boxes are zero-filled (M / N / K tails)
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

bool make_map(CUtensorMap* m, const void* base, int rows, int K, int box_rows) {
    EncodeFn enc = encode_fn();
    static const int promo = env_int("WT_GEMM_L2PROMO", 256);
    const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                      : promo == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                      : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (!enc) return false;
    const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(K) * 2};
    const cuuint32_t box[2] = {64u, cuuint32_t(box_rows)};
    const cuuint32_t es[2] = {1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool splitk_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("WT_GEMM_SPLITK");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int BM, int BN, int BK, int ST, bool SWAP>
int run_tc(const RunArgs& r, int warmup, int reps, cudaEvent_t e0, cudaEvent_t e1) {
    using S = tc::Shape<BM, BN, BK, ST, SWAP>;
    // TMA: 16-byte row pitch; 16-byte vector stores of C rows
    if (r.K % 8 || r.N % 8 || r.M <= 0 || r.N <= 0 || r.K <= 0) return 1;
    if ((reinterpret_cast<uintptr_t>(r.A) | reinterpret_cast<uintptr_t>(r.B) | reinterpret_cast<uintptr_t>(r.C)) & 15)
        return 1;
    tc::Params p{};
    p.M = r.M;
    p.N = r.N;
    p.K = r.K;
    p.C = static_cast<__nv_bfloat16*>(r.C);
    p.m_blocks = (r.M + BM - 1) / BM;
    p.n_blocks = (r.N + BN - 1) / BN;
    p.k_blocks = (r.K + BK - 1) / BK;
    // multicast cluster of the single-CTA tiles (WT_GEMM_MC = 2 / 4): CTAs on
    // consecutive n-blocks share one load of the m-block's operand.  Off by
    // default: measured on B200 it does not pay here (r02 probe: 128x4096x4096
    // 25.1 -> 26.9 us, 4096^3 on 128x256 tiles 108 -> 156 us) -- L2 request
    // volume is not what bounds these tiles.
    p.mc = 1;
    if (S::CG == 1) {
        static const int mc_env = env_int("WT_GEMM_MC", 1);
        const int want = mc_env;
        p.mc = want >= 4 && p.n_blocks >= 4 ? 4 : want >= 2 && p.n_blocks >= 2 ? 2 : 1;
    }
    p.n_groups = (p.n_blocks + p.mc - 1) / p.mc;
    p.tiles = p.m_blocks * p.n_groups;
    p.swizzle = std::max(1, r.swizzle);
    CUtensorMap ta, tb;
    // A = activations (M slot; N slot when swapped); the shared operand's box
    // is the multicast slice
    const int a_rows = SWAP ? S::B_ROWS : S::A_ROWS / p.mc;
    const int b_rows = SWAP ? S::A_ROWS : S::B_ROWS;
    const int a_box = SWAP ? a_rows / p.mc : a_rows;
    if (!make_map(&ta, r.A, r.M, r.K, a_box) || !make_map(&tb, r.B, r.N, r.K, b_rows)) return 2;
    // split-K for the small-M (swap-AB) tiles when they leave more than half
    // of the SMs idle: slices of >= 4 k-blocks, at most one unit per SM, and
    // at most 64 KB of fp32 partials for the last slice to reduce (measured:
    // with 128-column accumulators the serial reduction costs more than the
    // extra SMs gain, so the wide tiles never split).  WT_GEMM_SPLITK=0: off.
    const int avail = device_sms() / (S::CG * p.mc);
    p.splits = 1;
    if (SWAP && splitk_enabled() && 2 * p.tiles <= avail)
        p.splits = std::max(1, std::min({avail / p.tiles, p.k_blocks / 4, (64 << 10) / (128 * S::UN * 4)}));
    if (p.splits > 1) {
        // partial slots / counters per CTA tile (cluster tiles x mc)
        const size_t ctas = size_t(p.tiles) * p.mc;
        const size_t need = kCounterBytes + ctas * p.splits * S::CG * 128 * S::UN * 4;
        if (!r.workspace || need > r.workspace_bytes || ctas * S::CG * 4 > kCounterBytes)
            p.splits = 1;
        else {
            p.cnt = static_cast<int*>(r.workspace);
            p.ws = reinterpret_cast<float*>(static_cast<char*>(r.workspace) + kCounterBytes);
        }
    }
    static long long* trace_buf = nullptr;
    if (env_int("WT_GEMM_TRACE", 0)) {
        if (!trace_buf) cudaMalloc(&trace_buf, 1024 * sizeof(long long));
        p.trace = trace_buf;
    }
    p.nomma = env_int("WT_GEMM_NOMMA", 0);
    auto kern = tc::k_tc_gemm<BM, BN, BK, ST, SWAP>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !attr_set[dev]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM) != cudaSuccess)
            return 2;
        attr_set[dev] = true;
    }
    static const bool nonpersist = env_int("WT_GEMM_NONPERSIST", 0) != 0;  // A/B: one tile per cluster
    const int clusters = nonpersist ? p.tiles * p.splits : std::min(p.tiles * p.splits, avail);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(clusters * S::CG * p.mc));
    cfg.blockDim = dim3(S::THREADS);
    cfg.dynamicSmemBytes = S::SMEM;
    cfg.stream = static_cast<cudaStream_t>(r.stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S::CG * p.mc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    static const bool nocluster = env_int("WT_GEMM_NOCLUSTER", 0) != 0;
    cfg.numAttrs = (S::CG == 1 && p.mc == 1 && nocluster) ? 0 : 1;
    auto launch = [&]() { return cudaLaunchKernelEx(&cfg, kern, ta, tb, p) == cudaSuccess; };
    if (reps == 0) {
        const bool ok = launch();
        if (p.trace) {  // debug: CTA 0's producer issue / MMA full-wait clocks per k-block
            long long h[1024];
            cudaMemcpy(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost);
            const int nk = std::min(p.k_blocks / p.splits, 512);
            for (int k = 0; k < nk; ++k)
                std::fprintf(stderr, "kb %3d issue %8lld full %8lld lat %6lld\n", k, h[k] - h[0], h[512 + k] - h[0],
                             h[512 + k] - h[k]);
        }
        return ok ? 0 : 3;
    }
    for (int i = 0; i < warmup; ++i)
        if (!launch()) return 3;
    cudaEventRecord(e0, cfg.stream);
    for (int i = 0; i < reps; ++i)
        if (!launch()) return 3;
    cudaEventRecord(e1, cfg.stream);
    return 0;
}

}  // namespace

// (BM, BN, BK, stages): BM <= 64 = swap-AB small-M tiles, BM = 256 = CTA pair
const Config kFamily[] = {
    {32, 128, 64, 8, run_tc<32, 128, 64, 8, true>},
    {64, 128, 64, 8, run_tc<64, 128, 64, 8, true>},
    {64, 128, 128, 4, run_tc<64, 128, 128, 4, true>},
    {128, 64, 64, 4, run_tc<128, 64, 64, 4, false>},
    {128, 64, 64, 8, run_tc<128, 64, 64, 8, false>},
    {128, 128, 64, 4, run_tc<128, 128, 64, 4, false>},
    {128, 128, 64, 6, run_tc<128, 128, 64, 6, false>},
    {128, 128, 128, 3, run_tc<128, 128, 128, 3, false>},
    {128, 256, 64, 3, run_tc<128, 256, 64, 3, false>},
    {128, 256, 64, 4, run_tc<128, 256, 64, 4, false>},
    {256, 128, 64, 4, run_tc<256, 128, 64, 4, false>},
    {256, 128, 64, 6, run_tc<256, 128, 64, 6, false>},
    {256, 256, 64, 3, run_tc<256, 256, 64, 3, false>},
    {256, 256, 64, 5, run_tc<256, 256, 64, 5, false>},
    {256, 256, 128, 3, run_tc<256, 256, 128, 3, false>},
};
const int kFamilySize = int(sizeof(kFamily) / sizeof(kFamily[0]));

}  // namespace wtb::gemm
