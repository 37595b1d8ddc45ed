// wt_gemm_impl.cuh -- the validation GEMM family:
// bf16 x bf16 -> bf16 (fp32 accumulate) on sm_100a tcgen05 tensor cores with
// TMA loads, TMEM accumulators and a persistent warp-specialised schedule,
// instantiated from CuTe/CUTLASS 4.5 templates (flashinfer's vendored headers).
// One instantiation per (BM, BN, BK, stages); BM = 256 uses the 2-SM
// (cta_group::2) MMA on a 2-CTA cluster.  The raster swizzle of the
// persistent tile scheduler is a runtime knob.  These are exactly the knobs
// the WaveTune decision path chooses between (macro = tile, micro = stages x
// swizzle).
#pragma once

#include <cuda_runtime.h>

#include <cute/tensor.hpp>
#include <cutlass/cutlass.h>
#include <cutlass/epilogue/collective/collective_builder.hpp>
#include <cutlass/gemm/collective/collective_builder.hpp>
#include <cutlass/gemm/device/gemm_universal_adapter.h>
#include <cutlass/gemm/kernel/gemm_universal.hpp>
#include <cutlass/util/packed_stride.hpp>

#include <type_traits>

#include "wt_gemm.h"  // paper_2604_10187_b200/csrc/gemm

namespace wtb::gemm {

using namespace cute;

template <int BM, int BN, int BK, int ST>
struct Family {
    using EA = cutlass::bfloat16_t;
    using EB = cutlass::bfloat16_t;
    using EC = cutlass::bfloat16_t;
    using LA = cutlass::layout::RowMajor;     // A [M, K]
    using LB = cutlass::layout::ColumnMajor;  // B [K, N] == nn.Linear weight [N, K]
    using LC = cutlass::layout::RowMajor;     // C [M, N]
    static constexpr bool k2sm = BM == 256;
    using Tile = Shape<Int<BM>, Int<BN>, Int<BK>>;
    using Cluster = Shape<Int<k2sm ? 2 : 1>, _1, _1>;
    using MainSchedule = std::conditional_t<k2sm, cutlass::gemm::KernelTmaWarpSpecialized2SmSm100,
                                            cutlass::gemm::KernelTmaWarpSpecialized1SmSm100>;
    using EpiSchedule = std::conditional_t<k2sm, cutlass::epilogue::TmaWarpSpecialized2Sm,
                                           cutlass::epilogue::TmaWarpSpecialized1Sm>;
    using Epi = typename cutlass::epilogue::collective::CollectiveBuilder<
        cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, Tile, Cluster,
        cutlass::epilogue::collective::EpilogueTileAuto, float, float, EC, LC, 8, EC, LC, 8, EpiSchedule>::CollectiveOp;
    using Main = typename cutlass::gemm::collective::CollectiveBuilder<
        cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, EA, LA, 8, EB, LB, 8, float, Tile, Cluster,
        cutlass::gemm::collective::StageCount<ST>, MainSchedule>::CollectiveOp;
    using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Main, Epi, void>;
    using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;

    static typename Gemm::Arguments make_args(const RunArgs& r) {
        typename Gemm::Arguments args{
            cutlass::gemm::GemmUniversalMode::kGemm,
            {r.M, r.N, r.K, 1},
            {static_cast<const EA*>(r.A),
             cutlass::make_cute_packed_stride(typename Kernel::StrideA{}, {r.M, r.K, 1}),
             static_cast<const EB*>(r.B),
             cutlass::make_cute_packed_stride(typename Kernel::StrideB{}, {r.N, r.K, 1})},
            {{1.0f, 0.0f},
             static_cast<const EC*>(r.C),
             cutlass::make_cute_packed_stride(typename Kernel::StrideC{}, {r.M, r.N, 1}),
             static_cast<EC*>(r.C),
             cutlass::make_cute_packed_stride(typename Kernel::StrideD{}, {r.M, r.N, 1})}};
        args.scheduler.max_swizzle_size = r.swizzle;
        return args;
    }

    // reps == 0: one launch.  reps > 0: initialise once, `warmup` untimed
    // launches, then `reps` launches bracketed by the two events (the
    // adapter's per-call host work stays outside the device timing).
    static int run(const RunArgs& r, int warmup, int reps, cudaEvent_t e0, cudaEvent_t e1) {
        auto args = make_args(r);
        Gemm gemm;
        if (gemm.can_implement(args) != cutlass::Status::kSuccess) return 1;
        const size_t ws = Gemm::get_workspace_size(args);
        if (ws > r.workspace_bytes) return 4;
        auto st = static_cast<cudaStream_t>(r.stream);
        if (gemm.initialize(args, r.workspace, st) != cutlass::Status::kSuccess) return 2;
        if (reps == 0) return gemm.run(st) == cutlass::Status::kSuccess ? 0 : 3;
        for (int i = 0; i < warmup; ++i)
            if (gemm.run(st) != cutlass::Status::kSuccess) return 3;
        cudaEventRecord(e0, st);
        for (int i = 0; i < reps; ++i)
            if (gemm.run(st) != cutlass::Status::kSuccess) return 3;
        cudaEventRecord(e1, st);
        return 0;
    }
};

}  // namespace wtb::gemm

#define WT_GEMM_INSTANTIATE(NAME, BM, BN, BK, ST)                                 \
    namespace wtb::gemm {                                                          \
    int NAME(const RunArgs& r, int warmup, int reps, cudaEvent_t e0, cudaEvent_t e1) {     \
        return Family<BM, BN, BK, ST>::run(r, warmup, reps, e0, e1);                \
    }          \
    }
