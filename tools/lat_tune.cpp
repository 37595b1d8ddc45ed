// lat_tune.cpp -- single-query decision latency of the C++ drop-in, host
// wall clock, steady state.  Usage: lat_tune tables.json registry.json n_sm M N K
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "wavetune/wavetune.hpp"
#include "wavetune_c.h"

using namespace wavetune;

template <class F>
static void report(const char* what, F&& f, int n = 20000) {
    for (int i = 0; i < 200; ++i) f();
    std::vector<double> t(n);
    for (int i = 0; i < n; ++i) {
        auto a = std::chrono::steady_clock::now();
        f();
        t[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
    }
    std::sort(t.begin(), t.end());
    std::printf("%-34s p10 %6.2f  p50 %6.2f  p90 %6.2f  p99 %6.2f us\n", what, t[n / 10], t[n / 2], t[9 * n / 10],
                t[99 * n / 100]);
}

int main(int argc, char** argv) {
    if (argc < 7) return 2;
    const TableArtifact art = load_tables(argv[1]);
    const ConfigRegistry reg = ConfigRegistry::load(argv[2]);
    const HardwareSpec hw{std::atoi(argv[3]), 1, "b200"};
    const DenseGemm x{std::atoll(argv[4]), std::atoll(argv[5]), std::atoll(argv[6])};
    Engine eng(art.tables, reg, hw);
    auto* e = static_cast<wt_engine*>(eng.handle());
    wt_decision_one one{};
    report("C-ABI wt_tune_one", [&] { wt_tune_one(e, int32_t(x.m), int32_t(x.n), int32_t(x.k), &one); });
    report("C++ Engine::tune_one", [&] { (void)eng.tune_one(x); });
    report("C++ tune() (cached engine)", [&] { (void)tune(x, art.tables, reg, hw); });
    eng.set_resident(20000);
    report("C-ABI wt_tune_one, resident", [&] { wt_tune_one(e, int32_t(x.m), int32_t(x.n), int32_t(x.k), &one); });
    report("C++ Engine::tune_one, resident", [&] { (void)eng.tune_one(x); });
    eng.set_resident(0);
    const Tuned t = tune(x, art.tables, reg, hw);
    std::printf("decision: macro %d micro %d predicted %.3f us (C-ABI macro %d)\n", t.macro_id, t.micro_id,
                t.predicted_latency_us, one.macro_id);
    return 0;
}
