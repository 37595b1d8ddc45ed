// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (oracle/).
//
// A C shim over the reference's OWN C++ API, compiled together with the
// reference sources (proj/src/*.cpp, unmodified, read in place from
// /root/reference) into oracle/_ref/libwtref.so.  It lets the Python tests
// and bench.py's reference/cpu_baseline legs drive the real reference code:
//   tune()                tuner.cpp:159-166
//   predict_latency()     tuner.cpp:11-42
//   nearest_anchor()      tuner.cpp:44-70
//   fit_bucket()          model.cpp:20-77   (Eigen via oracle/eigen_shim)
//   select_shared_micro() model.cpp:81-120
//   build_dual_table()    model.cpp:194-253 + save_tables model.cpp:255-302
//   build_plan()          profiler.cpp:53-95
//   run_profile()         profiler.cpp:286-329 with SimulatorBackend
// Inputs/outputs are files in the reference's own formats (registry JSON,
// records CSV, tables JSON) plus plain arrays, so the reference parses its
// own artefacts.  Queries are split across std::thread workers (static
// interleave): tune() is pure and reentrant.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "wavetune/eval.hpp"
#include "wavetune/kernel_map.hpp"
#include "wavetune/model.hpp"
#include "wavetune/profiler.hpp"
#include "wavetune/tuner.hpp"
#include "wavetune/wave_sim.hpp"
#include "helpers.hpp"  // proj/tests/helpers.hpp: small_gemm_registry, two_regime_ground

#define WTREF_API extern "C" __attribute__((visibility("default")))

using namespace wavetune;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
    return 2;  // runtime_error and everything else
}

struct Handle {
    TableArtifact artifact;
    ConfigRegistry registry;
    HardwareSpec hw;
};
}  // namespace

WTREF_API const char* wtref_last_error() { return g_err.c_str(); }

WTREF_API void* wtref_open(const char* tables_json, const char* registry_json, int n_sm,
                           int blocks_per_sm) {
    try {
        auto* h = new Handle;
        h->artifact = load_tables(tables_json);
        h->registry = ConfigRegistry::load(registry_json);
        h->hw = HardwareSpec{n_sm, blocks_per_sm, "ref"};
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

WTREF_API void wtref_close(void* h) { delete static_cast<Handle*>(h); }

WTREF_API int wtref_num_tables(void* hp) {
    return static_cast<int>(static_cast<Handle*>(hp)->artifact.tables.size());
}

// Batched tune() over dense_gemm queries.  status[i]: 0 ok, 1 invalid_argument,
// 2 runtime_error, 3 out_of_range.  flag_count[i] = Tuned.flags.size().
WTREF_API int wtref_tune(void* hp, const int64_t* M, const int64_t* N, const int64_t* K,
                         int64_t n, int32_t* macro, int32_t* micro, double* lat, int64_t* g,
                         int64_t* l, int32_t* w, int32_t* extrap, int32_t* evals,
                         int32_t* comps, int32_t* flag_count, int32_t* status, int nthreads) {
    const Handle& h = *static_cast<Handle*>(hp);
    if (nthreads < 1) nthreads = 1;
    auto work = [&](int tid) {
        for (int64_t i = tid; i < n; i += nthreads) {
            try {
                Tuned t = tune(DenseGemm{M[i], N[i], K[i]}, h.artifact.tables, h.registry, h.hw);
                macro[i] = t.macro_id;
                micro[i] = t.micro_id;
                lat[i] = t.predicted_latency_us;
                if (g) g[i] = t.g;
                if (l) l[i] = t.l;
                if (w) w[i] = t.regime.w;
                if (extrap) extrap[i] = t.regime.extrapolated ? 1 : 0;
                if (evals) evals[i] = t.stats.model_evals;
                if (comps) comps[i] = t.stats.anchor_comparisons;
                if (flag_count) flag_count[i] = static_cast<int32_t>(t.flags.size());
                status[i] = 0;
            } catch (const std::exception& e) {
                status[i] = fail(e);
            }
        }
    };
    if (nthreads == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    return 0;
}

// Single tune() with its flag strings joined by '\n' into buf.
WTREF_API int wtref_tune_flags(void* hp, int64_t M, int64_t N, int64_t K, char* buf, int buflen) {
    const Handle& h = *static_cast<Handle*>(hp);
    try {
        Tuned t = tune(DenseGemm{M, N, K}, h.artifact.tables, h.registry, h.hw);
        std::string s;
        for (const auto& f : t.flags) s += f + "\n";
        std::snprintf(buf, buflen, "%s", s.c_str());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

WTREF_API int wtref_predict(void* hp, int table_index, int64_t g, int64_t l, double* lat,
                            int32_t* extrap, int32_t* w, char* flags, int buflen) {
    const Handle& h = *static_cast<Handle*>(hp);
    try {
        std::vector<std::string> fl;
        auto [v, regime] = predict_latency(h.artifact.tables.at(table_index), g, l, h.hw, &fl);
        *lat = v;
        *extrap = regime.extrapolated;
        *w = regime.w;
        std::string s;
        for (const auto& f : fl) s += f + "\n";
        if (flags) std::snprintf(flags, buflen, "%s", s.c_str());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

WTREF_API int64_t wtref_nearest_anchor(const int64_t* anchors, int n, int64_t l, int32_t* comps) {
    try {
        int c = 0;
        int64_t r = nearest_anchor(std::vector<i64>(anchors, anchors + n), l, &c);
        *comps = c;
        return r;
    } catch (const std::exception& e) {
        fail(e);
        *comps = -1;
        return -1;
    }
}

WTREF_API int wtref_fit_bucket(const double* g, const double* l, const double* t, int n,
                               double* coeffs, double* r2, double* mape, int32_t* degenerate) {
    try {
        std::vector<FitSample> s;
        for (int i = 0; i < n; ++i) s.push_back({g[i], l[i], t[i]});
        FitResult f = fit_bucket(s);
        coeffs[0] = f.coeffs.alpha;
        coeffs[1] = f.coeffs.beta;
        coeffs[2] = f.coeffs.gamma;
        coeffs[3] = f.coeffs.delta;
        *r2 = f.r2;
        *mape = f.mape;
        *degenerate = f.degenerate;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// select_shared_micro on one (macro, w, l) group; writes the chosen micro,
// partial flag and the selected (g, latency) samples (capacity cap).
WTREF_API int wtref_select_shared_micro(const int64_t* g, const int64_t* l, const int32_t* micro,
                                        const double* t, int n, int32_t* micro_out,
                                        int32_t* partial, int64_t* g_out, double* t_out, int cap,
                                        int32_t* n_out) {
    try {
        std::vector<ProfileRecord> grp;
        for (int i = 0; i < n; ++i) grp.push_back({g[i], l[i], 1, 0, micro[i], t[i]});
        SharedMicroSelection s = select_shared_micro(grp);
        *micro_out = s.micro_id;
        *partial = s.partial_coverage;
        int k = 0;
        for (const auto& [gg, tt] : s.samples) {
            if (k < cap) {
                g_out[k] = gg;
                t_out[k] = tt;
            }
            ++k;
        }
        *n_out = k;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// build_dual_table from a records CSV + registry JSON, saved as a tables JSON.
WTREF_API int wtref_build(const char* records_csv, const char* registry_json, const char* hw_name,
                          int n_sm, int W, int p, const char* out_tables_json) {
    try {
        auto records = read_records(records_csv);
        auto registry = ConfigRegistry::load(registry_json);
        TableArtifact a;
        a.family = registry.family;
        a.tables = build_dual_table(records, registry, HardwareSpec{n_sm, 1, hw_name}, {W, p});
        save_tables(a, out_tables_json);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// CPU baseline of the build: the reference's own
// build_dual_table (model.cpp:194-253) over the FULL record set, timed on a
// sample of macros and parallelised only across macros -- thread t runs one
// build_dual_table call over a registry holding sample macros t, t + T, ...
// Records are converted to ProfileRecord once, outside the timed region.
// Returns the wall seconds of the parallel region (or -1 on error);
// *n_tables = tables built.
WTREF_API double wtref_build_timed(const int64_t* g, const int64_t* l, const int32_t* w, const int32_t* macro,
                                   const int32_t* micro, const double* lat, int64_t n, const int32_t* sample_ids,
                                   const int64_t* t_m, const int64_t* t_n, const int64_t* t_k, int n_sample, int W,
                                   int p, int n_sm, int nthreads, int32_t* n_tables) {
    try {
        std::vector<ProfileRecord> records(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) records[i] = ProfileRecord{g[i], l[i], w[i], macro[i], micro[i], lat[i]};
        if (nthreads < 1) nthreads = 1;
        std::vector<ConfigRegistry> regs(nthreads);
        for (int i = 0; i < n_sample; ++i)
            regs[i % nthreads].macros.push_back(MacroConfig{sample_ids[i], GemmTiles{t_m[i], t_n[i], t_k[i]}});
        std::vector<int> built(nthreads, 0);
        auto work = [&](int t) {
            if (regs[t].macros.empty()) return;
            built[t] = static_cast<int>(
                build_dual_table(records, regs[t], HardwareSpec{n_sm, 1, "b200"}, {W, p}).size());
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        int tot = 0;
        for (int b : built) tot += b;
        if (n_tables) *n_tables = tot;
        return sec;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

// tables JSON -> load -> save (artifact identity checks).
WTREF_API int wtref_resave_tables(const char* in_json, const char* out_json) {
    try {
        save_tables(load_tables(in_json), out_json);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

WTREF_API int wtref_build_plan(int n_sm, int blocks_per_sm, int W, int I, double tau,
                               const int64_t* anchors, int n_anchors, const char* out_json) {
    try {
        PlanParams pp;
        pp.W = W;
        pp.I = I;
        pp.tau = tau;
        pp.loop_anchors.assign(anchors, anchors + n_anchors);
        build_plan(HardwareSpec{n_sm, blocks_per_sm, "ref"}, KernelFamily::DenseGemm, pp)
            .save(out_json);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference test fixture (test_tuner.cpp:14-30 / acceptance.cpp:228-244):
// small_gemm_registry + two_regime_ground, plan, SimulatorBackend profile.
WTREF_API int wtref_fixture(int n_sm, int n_macros, int n_micros, int W, int I, double tau,
                            const int64_t* anchors, int n_anchors, double sigma, uint64_t seed,
                            const char* registry_out, const char* records_out) {
    try {
        HardwareSpec hw{n_sm, 1, "sim"};
        ConfigRegistry reg = testing::small_gemm_registry(n_macros, n_micros);
        SyntheticKernelGround ground = testing::two_regime_ground(reg);
        PlanParams pp;
        pp.W = W;
        pp.I = I;
        pp.tau = tau;
        pp.loop_anchors.assign(anchors, anchors + n_anchors);
        SamplingPlan plan = build_plan(hw, KernelFamily::DenseGemm, pp);
        SimulatorBackend backend(hw, ground, sigma, seed);
        auto records = run_profile(plan, reg, backend);
        reg.save(registry_out);
        write_records(records, records_out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Ground truth of the reference fixture (helpers.hpp:40-56), saved as JSON.
WTREF_API int wtref_ground(int n_macros, int n_micros, const char* out) {
    try {
        ConfigRegistry reg = testing::small_gemm_registry(n_macros, n_micros);
        testing::two_regime_ground(reg).save(out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// simulate() with a constant block model (bindings.cpp:119-128 semantics).
WTREF_API int wtref_simulate(int n_sm, int64_t g, int64_t l, double mu, double sigma, uint64_t seed, double* out) {
    try {
        *out = simulate(SimMachine{HardwareSpec{n_sm, 1, ""}, seed}, g, l, BlockLatencyModel::constant(mu, sigma));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// oracle_best (wave_sim.cpp:136-161) for one dense query on the fixture ground.
WTREF_API int wtref_oracle_best(const char* registry_json, const char* ground_json, int n_sm, uint64_t seed,
                                int64_t M, int64_t N, int64_t K, double sigma, int reps, int32_t* macro,
                                int32_t* micro, double* lat) {
    try {
        auto reg = ConfigRegistry::load(registry_json);
        auto ground = SyntheticKernelGround::load(ground_json);
        OracleResult r = oracle_best(SimMachine{HardwareSpec{n_sm, 1, ""}, seed}, DenseGemm{M, N, K}, reg, ground,
                                     sigma, reps);
        *macro = r.macro_id;
        *micro = r.micro_id;
        *lat = r.latency_us;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- ablation baselines (tuner.cpp:168-250) ---------------------------------

// fit_step_baseline + fit_linear_baseline from a records CSV.  Step entries in
// map order ((macro, l) ascending); linear thetas in macro order.
WTREF_API int wtref_fit_baselines(const char* records_csv, int64_t cap, int32_t* step_macro, int64_t* step_l,
                                  double* step_t, int64_t* n_step, int32_t* lin_macro, double* lin_theta,
                                  int64_t* n_lin) {
    try {
        auto recs = read_records(records_csv);
        BaselinePredictor s = fit_step_baseline(recs);
        BaselinePredictor l = fit_linear_baseline(recs);
        int64_t k = 0;
        for (const auto& [key, t] : s.step.t_wave) {
            if (k >= cap) throw std::runtime_error("wtref_fit_baselines: cap too small");
            step_macro[k] = key.first;
            step_l[k] = key.second;
            step_t[k] = t;
            ++k;
        }
        *n_step = k;
        k = 0;
        for (const auto& [m, th] : l.linear.theta) {
            if (k >= cap) throw std::runtime_error("wtref_fit_baselines: cap too small");
            lin_macro[k] = m;
            lin_theta[4 * k + 0] = th.alpha;
            lin_theta[4 * k + 1] = th.beta;
            lin_theta[4 * k + 2] = th.gamma;
            lin_theta[4 * k + 3] = th.delta;
            ++k;
        }
        *n_lin = k;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

namespace {
// kind 0 = step: entries (macro[i], l[i], t[i]); kind 1 = linear: macro[i], theta[4i..4i+3]
BaselinePredictor make_bp(int kind, const int32_t* macro, const int64_t* l, const double* t, int64_t n) {
    BaselinePredictor bp;
    bp.kind = kind == 0 ? BaselinePredictor::Kind::Step : BaselinePredictor::Kind::GlobalLinear;
    for (int64_t i = 0; i < n; ++i) {
        if (kind == 0) bp.step.t_wave[{macro[i], l[i]}] = t[i];
        else bp.linear.theta[macro[i]] = BilinearCoeffs{t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]};
    }
    return bp;
}
}  // namespace

WTREF_API int wtref_baseline_predict(int kind, const int32_t* macro, const int64_t* l, const double* t, int64_t n,
                                     int n_sm, int bps, int32_t qmacro, int64_t qg, int64_t ql, double* out) {
    try {
        *out = baseline_predict(make_bp(kind, macro, l, t, n), qmacro, qg, ql, HardwareSpec{n_sm, bps, ""});
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Batched baseline_tune() over dense queries against an opened handle's tables.
WTREF_API int wtref_baseline_tune(void* hp, int kind, const int32_t* bmacro, const int64_t* bl, const double* bt,
                                  int64_t nb, const int64_t* M, const int64_t* N, const int64_t* K, int64_t n,
                                  int32_t* macro, int32_t* micro, double* lat, int32_t* w, int32_t* extrap,
                                  int32_t* comps, int32_t* flag_count, int32_t* status, int nthreads) {
    const Handle& h = *static_cast<Handle*>(hp);
    const BaselinePredictor bp = make_bp(kind, bmacro, bl, bt, nb);
    if (nthreads < 1) nthreads = 1;
    auto work = [&](int tid) {
        for (int64_t i = tid; i < n; i += nthreads) {
            try {
                Tuned t = baseline_tune(DenseGemm{M[i], N[i], K[i]}, bp, h.artifact.tables, h.registry, h.hw);
                macro[i] = t.macro_id;
                micro[i] = t.micro_id;
                lat[i] = t.predicted_latency_us;
                w[i] = t.regime.w;
                extrap[i] = t.regime.extrapolated ? 1 : 0;
                comps[i] = t.stats.anchor_comparisons;
                flag_count[i] = static_cast<int32_t>(t.flags.size());
                status[i] = 0;
            } catch (const std::exception& e) {
                status[i] = fail(e);
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    return 0;
}
