// gemm_backend.hpp -- the B200 validation GEMM family behind the reference's
// MeasurementBackend interface (reference proj/include/wavetune/profiler.hpp:70).
//
// The reference measures real kernels only through ExternalCommandBackend
// (profiler.hpp:114: one process per measurement).  On B200 the family lives
// in lib/libwtgemm.so (include/wavetune_gemm.h) and is measured in-process
// with CUDA events: run_profile(plan, gemm_registry(), backend) profiles it,
// build_dual_table fits it, tune() picks from it.
#pragma once

#include <cstdint>

#include "wavetune/wavetune.hpp"

namespace wavetune {

// Registry of the compiled family: macro = tile (t_m, t_n, t_k), micro =
// (n_stages, swizzle) with micro.extra = {{"swizzle", s}}; (macro, micro) is
// feasible iff an instantiation with that tile and depth exists.  n_warps is
// the kernel's fixed warp-role count (informational).
ConfigRegistry gemm_registry();

class B200GemmBackend : public MeasurementBackend {
public:
    // warmup untimed launches, then the mean of `measured` back-to-back
    // launches (device time, CUDA events) per call, on library-owned operands
    // (uniform [-1, 1) bf16 from `seed`) grown to the largest problem seen.
    explicit B200GemmBackend(int warmup = 3, int measured = 10, std::uint64_t seed = 0);
    ~B200GemmBackend() override;
    B200GemmBackend(const B200GemmBackend&) = delete;
    B200GemmBackend& operator=(const B200GemmBackend&) = delete;

    double measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) override;

    // family instantiation for (macro, micro), or -1
    static int family_config(const MacroConfig& macro, const MicroConfig& micro);

private:
    void reserve(std::size_t a_elems, std::size_t b_elems, std::size_t c_elems);
    int warmup_, measured_;
    std::uint64_t seed_;
    void *a_ = nullptr, *b_ = nullptr, *c_ = nullptr;
    std::size_t a_cap_ = 0, b_cap_ = 0, c_cap_ = 0;
};

}  // namespace wavetune
