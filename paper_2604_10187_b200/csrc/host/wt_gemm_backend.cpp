// wt_gemm_backend.cpp -- B200GemmBackend / gemm_registry (include/wavetune/gemm_backend.hpp).
#include "wavetune/gemm_backend.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "wavetune_c.h"
#include "wavetune_gemm.h"

namespace wavetune {
namespace {

constexpr int kSwizzles[] = {1, 2, 4, 8};
constexpr int kWarpRoles = 6;  // sm100 warp-specialised GEMM: 4 epilogue + MMA + TMA producer

int micro_id_of(int stages, int swz_idx) { return (stages - 1) * 4 + swz_idx; }

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

i64 swizzle_of(const MicroConfig& m) {
    for (const auto& kv : m.extra)
        if (kv.first == "swizzle") return kv.second;
    return 1;
}

}  // namespace

ConfigRegistry gemm_registry() {
    ConfigRegistry r;
    r.family = KernelFamily::DenseGemm;
    const int n = wt_gemm_family_size();
    int max_stages = 1;
    std::vector<std::tuple<int, int, int>> tiles;
    for (int c = 0; c < n; ++c) {
        int bm, bn, bk, st;
        wt_gemm_config(c, &bm, &bn, &bk, &st);
        max_stages = std::max(max_stages, st);
        if (std::find(tiles.begin(), tiles.end(), std::make_tuple(bm, bn, bk)) == tiles.end())
            tiles.emplace_back(bm, bn, bk);
    }
    for (size_t i = 0; i < tiles.size(); ++i) {
        const auto [bm, bn, bk] = tiles[i];
        r.macros.push_back({int(i), GemmTiles{bm, bn, bk}});
    }
    for (int st = 1; st <= max_stages; ++st)
        for (int s = 0; s < 4; ++s) {
            MicroConfig m;
            m.id = micro_id_of(st, s);
            m.n_stages = st;
            m.n_warps = kWarpRoles;
            m.extra = {{"swizzle", kSwizzles[s]}};
            r.micros.push_back(m);
        }
    for (int c = 0; c < n; ++c) {
        int bm, bn, bk, st;
        wt_gemm_config(c, &bm, &bn, &bk, &st);
        const int macro = int(std::find(tiles.begin(), tiles.end(), std::make_tuple(bm, bn, bk)) - tiles.begin());
        for (int s = 0; s < 4; ++s) r.feasible.insert({macro, micro_id_of(st, s)});
    }
    r.validate();
    return r;
}

int B200GemmBackend::family_config(const MacroConfig& macro, const MicroConfig& micro) {
    const auto* t = std::get_if<GemmTiles>(&macro.tiles);
    if (!t) return -1;
    for (int c = 0, n = wt_gemm_family_size(); c < n; ++c) {
        int bm, bn, bk, st;
        wt_gemm_config(c, &bm, &bn, &bk, &st);
        if (bm == t->t_m && bn == t->t_n && bk == t->t_k && st == micro.n_stages) return c;
    }
    return -1;
}

B200GemmBackend::B200GemmBackend(int warmup, int measured, std::uint64_t seed)
    : warmup_(warmup), measured_(measured), seed_(seed) {
    if (warmup < 0 || measured <= 0) throw std::invalid_argument("B200GemmBackend: need warmup >= 0, measured > 0");
}

B200GemmBackend::~B200GemmBackend() {
    cudaFree(a_);
    cudaFree(b_);
    cudaFree(c_);
}

void B200GemmBackend::reserve(std::size_t a, std::size_t b, std::size_t c) {
    auto grow = [&](void*& p, std::size_t& cap, std::size_t want, std::uint64_t seed) {
        if (want <= cap) return;
        cudaFree(p);
        p = nullptr;
        cap = 0;
        check_cuda(cudaMalloc(&p, want * 2), "B200GemmBackend operand allocation");
        cap = want;
        if (seed && wt_gemm_fill_uniform(p, want, seed, nullptr) != WT_OK)
            throw std::runtime_error("B200GemmBackend: operand fill failed");
    };
    grow(a_, a_cap_, a, seed_ * 2 + 1);
    grow(b_, b_cap_, b, seed_ * 2 + 2);
    grow(c_, c_cap_, c, 0);
    check_cuda(cudaDeviceSynchronize(), "B200GemmBackend operand fill");
}

double B200GemmBackend::measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) {
    const auto* d = std::get_if<DenseGemm>(&x);
    if (!d) throw std::invalid_argument("B200GemmBackend measures dense GEMM workloads only");
    const int cfg = family_config(macro, micro);
    if (cfg < 0)
        throw std::invalid_argument("no compiled GEMM instantiation for macro " + std::to_string(macro.id) +
                                    " / micro " + std::to_string(micro.id));
    if (d->m > INT32_MAX || d->n > INT32_MAX || d->k > INT32_MAX) throw std::out_of_range("GEMM extent exceeds int32");
    reserve(std::size_t(d->m) * d->k, std::size_t(d->n) * d->k, std::size_t(d->m) * d->n);
    double us = 0.0;
    const int rc = wt_gemm_time(cfg, int(swizzle_of(micro)), int(d->m), int(d->n), int(d->k), a_, b_, c_, warmup_,
                                measured_, &us);
    if (rc != WT_OK) throw std::runtime_error("wt_gemm_time failed with status " + std::to_string(rc));
    return us;
}

}  // namespace wavetune
