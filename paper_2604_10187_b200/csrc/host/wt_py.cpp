// wt_py.cpp -- pybind11 module `_core`: the reference's Python surface
// (proj/src/bindings.cpp names and keyword arguments) over the C++ drop-in,
// plus batched entry points on numpy arrays.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "wavetune/gemm_backend.hpp"
#include "wavetune/wavetune.hpp"
#include "wavetune_c.h"

namespace py = pybind11;
using namespace wavetune;

PYBIND11_MODULE(_core, m) {
    m.doc() = "WaveTune decision path on B200 (sm_100a kernels behind a C-ABI)";

    py::class_<DenseGemm>(m, "DenseGemm")
        .def(py::init<i64, i64, i64>(), py::arg("m"), py::arg("n"), py::arg("k"))
        .def_readwrite("m", &DenseGemm::m)
        .def_readwrite("n", &DenseGemm::n)
        .def_readwrite("k", &DenseGemm::k);
    py::class_<GroupedGemm>(m, "GroupedGemm")
        .def(py::init<std::vector<i64>, i64, i64>(), py::arg("group_rows"), py::arg("n"), py::arg("k"))
        .def_readwrite("group_rows", &GroupedGemm::group_rows)
        .def_readwrite("n", &GroupedGemm::n)
        .def_readwrite("k", &GroupedGemm::k);
    py::class_<FlashAttention>(m, "FlashAttention")
        .def(py::init<i64, i64, i64>(), py::arg("n_heads"), py::arg("s_q"), py::arg("s_kv"))
        .def_readwrite("n_heads", &FlashAttention::n_heads)
        .def_readwrite("s_q", &FlashAttention::s_q)
        .def_readwrite("s_kv", &FlashAttention::s_kv);
    m.def("parse_workload", &workload_from_string, py::arg("text"));
    m.def("workload_to_string", &workload_to_string, py::arg("workload"));

    py::class_<GemmTiles>(m, "GemmTiles")
        .def(py::init<i64, i64, i64>(), py::arg("t_m"), py::arg("t_n"), py::arg("t_k"))
        .def_readwrite("t_m", &GemmTiles::t_m)
        .def_readwrite("t_n", &GemmTiles::t_n)
        .def_readwrite("t_k", &GemmTiles::t_k);
    py::class_<AttnTiles>(m, "AttnTiles")
        .def(py::init<i64, i64>(), py::arg("t_q"), py::arg("t_kv"))
        .def_readwrite("t_q", &AttnTiles::t_q)
        .def_readwrite("t_kv", &AttnTiles::t_kv);
    py::class_<MacroConfig>(m, "MacroConfig")
        .def(py::init([](int id, std::variant<GemmTiles, AttnTiles> t) { return MacroConfig{id, t}; }),
             py::arg("id"), py::arg("tiles"))
        .def_readwrite("id", &MacroConfig::id)
        .def_readwrite("tiles", &MacroConfig::tiles);
    py::class_<MicroConfig>(m, "MicroConfig")
        .def(py::init([](int id, i64 s, i64 w) { return MicroConfig{id, s, w, {}}; }), py::arg("id"),
             py::arg("n_stages"), py::arg("n_warps"))
        .def_readwrite("id", &MicroConfig::id)
        .def_readwrite("n_stages", &MicroConfig::n_stages)
        .def_readwrite("n_warps", &MicroConfig::n_warps)
        .def_readwrite("extra", &MicroConfig::extra);
    py::class_<HardwareSpec>(m, "HardwareSpec")
        .def(py::init([](int n_sm, int bps, std::string name) { return HardwareSpec{n_sm, bps, std::move(name)}; }),
             py::arg("n_sm"), py::arg("blocks_per_sm") = 1, py::arg("name") = "")
        .def_readwrite("n_sm", &HardwareSpec::n_sm)
        .def_readwrite("blocks_per_sm", &HardwareSpec::blocks_per_sm)
        .def_readwrite("name", &HardwareSpec::name)
        .def("slots", &HardwareSpec::slots);

    py::class_<ConfigRegistry>(m, "ConfigRegistry")
        .def(py::init<>())
        .def_property(
            "family", [](const ConfigRegistry& r) { return std::string(family_name(r.family)); },
            [](ConfigRegistry& r, const std::string& f) { r.family = family_from_name(f); })
        .def_readwrite("macros", &ConfigRegistry::macros)
        .def_readwrite("micros", &ConfigRegistry::micros)
        .def("add_feasible", [](ConfigRegistry& r, int a, int b) { r.feasible.emplace(a, b); })
        .def_property_readonly("feasible", [](const ConfigRegistry& r) {
            return std::vector<std::pair<int, int>>(r.feasible.begin(), r.feasible.end());
        })
        .def("macro", &ConfigRegistry::macro, py::return_value_policy::copy)
        .def("micro", &ConfigRegistry::micro, py::return_value_policy::copy)
        .def("feasible_micros", &ConfigRegistry::feasible_micros)
        .def("validate", &ConfigRegistry::validate)
        .def_static("load", &ConfigRegistry::load)
        .def("save", &ConfigRegistry::save);

    m.def("map_workload", &map_workload, py::arg("workload"), py::arg("macro"));
    m.def("wave_count", &wave_count, py::arg("g"), py::arg("hw"));
    m.def(
        "instantiate_workload",
        [](i64 mg, i64 ng, i64 l, const MacroConfig& c) { return instantiate_workload({mg, ng}, l, c); },
        py::arg("m_g"), py::arg("n_g"), py::arg("l"), py::arg("macro"));

    py::class_<ProfileRecord>(m, "ProfileRecord")
        .def(py::init([](i64 g, i64 l, int w, int ma, int mi, double t) { return ProfileRecord{g, l, w, ma, mi, t}; }),
             py::arg("g"), py::arg("l"), py::arg("w"), py::arg("macro_id"), py::arg("micro_id"),
             py::arg("latency_us"))
        .def_readonly("g", &ProfileRecord::g)
        .def_readonly("l", &ProfileRecord::l)
        .def_readonly("w", &ProfileRecord::w)
        .def_readonly("macro_id", &ProfileRecord::macro_id)
        .def_readonly("micro_id", &ProfileRecord::micro_id)
        .def_readonly("latency_us", &ProfileRecord::latency_us);
    py::class_<GridPoint>(m, "GridPoint")
        .def_readonly("w", &GridPoint::w)
        .def_readonly("i", &GridPoint::i)
        .def_readonly("g", &GridPoint::g);
    py::class_<SamplingPlan>(m, "SamplingPlan")
        .def_readonly("W", &SamplingPlan::W)
        .def_readonly("I", &SamplingPlan::I)
        .def_readonly("loop_anchors", &SamplingPlan::loop_anchors)
        .def_readonly("grid_points", &SamplingPlan::grid_points)
        .def_static("load", &SamplingPlan::load)
        .def("save", &SamplingPlan::save);
    m.def(
        "build_plan",
        [](const HardwareSpec& hw, const std::string& family, int W, int I, double tau, std::vector<i64> anchors,
           std::optional<i64> n_heads) {
            return build_plan(hw, family_from_name(family), PlanParams{W, I, tau, std::move(anchors), n_heads});
        },
        py::arg("hw"), py::arg("family"), py::arg("W"), py::arg("I"), py::arg("tau"), py::arg("loop_anchors"),
        py::arg("n_heads") = std::nullopt);
    // simulator (reference bindings.cpp:104-128, 165-174)
    py::class_<GroundEntry>(m, "GroundEntry")
        .def(py::init([](double base, double per_iter, double gap) { return GroundEntry{base, per_iter, gap}; }),
             py::arg("base"), py::arg("per_iter"), py::arg("dispatch_gap") = 0.0)
        .def_readwrite("base", &GroundEntry::base)
        .def_readwrite("per_iter", &GroundEntry::per_iter)
        .def_readwrite("dispatch_gap", &GroundEntry::dispatch_gap);
    py::class_<SyntheticKernelGround>(m, "SyntheticKernelGround")
        .def(py::init<>())
        .def("set_entry", [](SyntheticKernelGround& g, int a, int b, const GroundEntry& e) { g.entries[{a, b}] = e; })
        .def("mean", &SyntheticKernelGround::mean)
        .def_static("load", &SyntheticKernelGround::load)
        .def("save", &SyntheticKernelGround::save);
    m.def(
        "simulate",
        [](const HardwareSpec& hw, i64 g, i64 l, double mu, double sigma, std::uint64_t seed) {
            return simulate(SimMachine{hw, seed}, g, l, BlockLatencyModel::constant(mu, sigma));
        },
        py::arg("hw"), py::arg("g"), py::arg("l"), py::arg("mu"), py::arg("sigma") = 0.0, py::arg("seed") = 0,
        "makespan of g blocks with Normal(mu, sigma) durations (GPU wave simulator)");
    m.def(
        "run_profile_sim",
        [](const SamplingPlan& plan, const ConfigRegistry& reg, const SyntheticKernelGround& ground, double sigma,
           std::uint64_t seed) {
            SimulatorBackend b(plan.hw, ground, sigma, seed);
            return run_profile(plan, reg, b);
        },
        py::arg("plan"), py::arg("registry"), py::arg("ground"), py::arg("sigma") = 0.0, py::arg("seed") = 0);
    py::class_<OracleResult>(m, "OracleResult")
        .def_readonly("macro_id", &OracleResult::macro_id)
        .def_readonly("micro_id", &OracleResult::micro_id)
        .def_readonly("latency_us", &OracleResult::latency_us);
    m.def(
        "oracle_best",
        [](const HardwareSpec& hw, std::uint64_t seed, const KernelWorkload& x, const ConfigRegistry& reg,
           const SyntheticKernelGround& ground, double sigma, int reps) {
            return oracle_best(SimMachine{hw, seed}, x, reg, ground, sigma, reps);
        },
        py::arg("hw"), py::arg("seed"), py::arg("workload"), py::arg("registry"), py::arg("ground"),
        py::arg("sigma") = 0.0, py::arg("reps") = 3);
    m.def("write_records", &write_records);
    m.def("read_records", &read_records);
    m.def(
        "run_profile_replay",
        [](const SamplingPlan& plan, const ConfigRegistry& reg, const std::vector<ProfileRecord>& recs) {
            CsvReplayBackend b(recs);
            return run_profile(plan, reg, b);
        },
        py::arg("plan"), py::arg("registry"), py::arg("records"));
    m.def(
        "records_from_arrays",
        [](py::array_t<i64> g, py::array_t<i64> l, py::array_t<int32_t> w, py::array_t<int32_t> ma,
           py::array_t<int32_t> mi, py::array_t<double> t) {
            const auto n = g.size();
            std::vector<ProfileRecord> out(n);
            auto G = g.unchecked<1>();
            auto L = l.unchecked<1>();
            auto Wv = w.unchecked<1>();
            auto A = ma.unchecked<1>();
            auto B = mi.unchecked<1>();
            auto T = t.unchecked<1>();
            for (py::ssize_t i = 0; i < n; ++i) out[i] = {G(i), L(i), Wv(i), A(i), B(i), T(i)};
            return out;
        });

    py::class_<BilinearCoeffs>(m, "BilinearCoeffs")
        .def(py::init([](double a, double b, double c, double d) { return BilinearCoeffs{a, b, c, d}; }),
             py::arg("alpha") = 0.0, py::arg("beta") = 0.0, py::arg("gamma") = 0.0, py::arg("delta") = 0.0)
        .def_readwrite("alpha", &BilinearCoeffs::alpha)
        .def_readwrite("beta", &BilinearCoeffs::beta)
        .def_readwrite("gamma", &BilinearCoeffs::gamma)
        .def_readwrite("delta", &BilinearCoeffs::delta)
        .def("predict", &BilinearCoeffs::predict);
    py::class_<FitSample>(m, "FitSample")
        .def(py::init([](double g, double l, double t) { return FitSample{g, l, t}; }), py::arg("g"), py::arg("l"),
             py::arg("latency_us"));
    py::class_<FitResult>(m, "FitResult")
        .def_readonly("coeffs", &FitResult::coeffs)
        .def_readonly("r2", &FitResult::r2)
        .def_readonly("mape", &FitResult::mape)
        .def_readonly("degenerate", &FitResult::degenerate);
    py::class_<SharedMicroSelection>(m, "SharedMicroSelection")
        .def_readonly("micro_id", &SharedMicroSelection::micro_id)
        .def_readonly("samples", &SharedMicroSelection::samples)
        .def_readonly("partial_coverage", &SharedMicroSelection::partial_coverage);
    py::class_<ExtrapolationFit>(m, "ExtrapolationFit")
        .def_readonly("theta_ext", &ExtrapolationFit::theta_ext)
        .def_readonly("ext_anchors", &ExtrapolationFit::ext_anchors)
        .def_readonly("flags", &ExtrapolationFit::flags);
    py::class_<WaveDiagnostics>(m, "WaveDiagnostics")
        .def_readonly("r2", &WaveDiagnostics::r2)
        .def_readonly("mape", &WaveDiagnostics::mape)
        .def_readonly("samples", &WaveDiagnostics::samples)
        .def_readonly("flags", &WaveDiagnostics::flags);
    py::class_<DualTable>(m, "DualTable")
        .def(py::init<>())
        .def_readwrite("macro_id", &DualTable::macro_id)
        .def_readwrite("hardware", &DualTable::hardware)
        .def_readwrite("W", &DualTable::W)
        .def_readwrite("p", &DualTable::p)
        .def_readwrite("coeff_table", &DualTable::coeff_table)
        .def_readwrite("theta_ext", &DualTable::theta_ext)
        .def_readwrite("anchor_table", &DualTable::anchor_table)
        .def_readwrite("ext_anchors", &DualTable::ext_anchors)
        .def_readwrite("diagnostics", &DualTable::diagnostics)
        .def_readwrite("ext_flags", &DualTable::ext_flags)
        .def("__eq__", [](const DualTable& a, const DualTable& b) { return a == b; });
    py::class_<TableArtifact>(m, "TableArtifact")
        .def(py::init<>())
        .def_property(
            "family", [](const TableArtifact& a) { return std::string(family_name(a.family)); },
            [](TableArtifact& a, const std::string& f) { a.family = family_from_name(f); })
        .def_readwrite("tables", &TableArtifact::tables)
        .def("__eq__", [](const TableArtifact& a, const TableArtifact& b) { return a == b; });

    m.def("fit_bucket", &fit_bucket, py::arg("samples"));
    m.def("select_shared_micro", &select_shared_micro, py::arg("group"));
    m.def("fit_extrapolation", &fit_extrapolation, py::arg("records"), py::arg("W"), py::arg("p"));
    m.def(
        "build_dual_table",
        [](const std::vector<ProfileRecord>& r, const ConfigRegistry& reg, const HardwareSpec& hw, int W, int p) {
            return build_dual_table(r, reg, hw, {W, p});
        },
        py::arg("records"), py::arg("registry"), py::arg("hw"), py::arg("W") = 0, py::arg("p") = 10);
    m.def(
        "build_tables",
        [](const std::vector<ProfileRecord>& r, const ConfigRegistry& reg, const HardwareSpec& hw, int W, int p) {
            TableArtifact a;
            a.family = reg.family;
            a.tables = build_dual_table(r, reg, hw, {W, p});
            return a;
        },
        py::arg("records"), py::arg("registry"), py::arg("hw"), py::arg("W") = 0, py::arg("p") = 10);
    m.def("save_tables", &save_tables);
    m.def("load_tables", &load_tables);

    py::class_<DecisionStats>(m, "DecisionStats")
        .def_readonly("model_evals", &DecisionStats::model_evals)
        .def_readonly("anchor_comparisons", &DecisionStats::anchor_comparisons);
    py::class_<Regime>(m, "Regime")
        .def_readonly("extrapolated", &Regime::extrapolated)
        .def_readonly("w", &Regime::w);
    py::class_<Tuned>(m, "Tuned")
        .def_readonly("macro_id", &Tuned::macro_id)
        .def_readonly("micro_id", &Tuned::micro_id)
        .def_readonly("predicted_latency_us", &Tuned::predicted_latency_us)
        .def_readonly("g", &Tuned::g)
        .def_readonly("l", &Tuned::l)
        .def_readonly("regime", &Tuned::regime)
        .def_readonly("stats", &Tuned::stats)
        .def_readonly("flags", &Tuned::flags);

    m.def(
        "tune",
        [](const KernelWorkload& x, const TableArtifact& a, const ConfigRegistry& reg, const HardwareSpec& hw) {
            return tune(x, a.tables, reg, hw);
        },
        py::arg("workload"), py::arg("tables"), py::arg("registry"), py::arg("hw"));
    // ---- ablation baselines (tuner.hpp:54-85)
    py::class_<StepPredictor>(m, "StepPredictor")
        .def(py::init<>())
        .def_readwrite("t_wave", &StepPredictor::t_wave);
    py::class_<GlobalLinearPredictor>(m, "GlobalLinearPredictor")
        .def(py::init<>())
        .def_readwrite("theta", &GlobalLinearPredictor::theta);
    py::class_<BaselinePredictor>(m, "BaselinePredictor")
        .def(py::init<>())
        .def_property(
            "kind",
            [](const BaselinePredictor& b) {
                return std::string(b.kind == BaselinePredictor::Kind::Step ? "step" : "linear");
            },
            [](BaselinePredictor& b, const std::string& k) {
                if (k != "step" && k != "linear") throw std::invalid_argument("kind must be 'step' or 'linear'");
                b.kind = k == "step" ? BaselinePredictor::Kind::Step : BaselinePredictor::Kind::GlobalLinear;
            })
        .def_readwrite("step", &BaselinePredictor::step)
        .def_readwrite("linear", &BaselinePredictor::linear);
    m.def("fit_step_baseline", &fit_step_baseline, py::arg("records"));
    m.def("fit_linear_baseline", &fit_linear_baseline, py::arg("records"));
    m.def("baseline_predict", &baseline_predict, py::arg("bp"), py::arg("macro_id"), py::arg("g"), py::arg("l"),
          py::arg("hw"));
    m.def(
        "baseline_tune",
        [](const KernelWorkload& x, const BaselinePredictor& bp, const TableArtifact& a, const ConfigRegistry& reg,
           const HardwareSpec& hw) { return baseline_tune(x, bp, a.tables, reg, hw); },
        py::arg("workload"), py::arg("bp"), py::arg("tables"), py::arg("registry"), py::arg("hw"));
    m.def(
        "predict_latency",
        [](const DualTable& t, i64 g, i64 l, const HardwareSpec& hw) {
            std::vector<std::string> flags;
            auto [lat, reg] = predict_latency(t, g, l, hw, &flags);
            return py::make_tuple(lat, reg);
        },
        py::arg("table"), py::arg("g"), py::arg("l"), py::arg("hw"));
    m.def(
        "nearest_anchor",
        [](const std::vector<i64>& a, i64 l) {
            int c = 0;
            i64 r = nearest_anchor(a, l, &c);
            return py::make_tuple(r, c);
        },
        py::arg("sorted_anchors"), py::arg("l"));

    // ---- batched surface (new): a device-resident engine
    py::class_<Engine, std::shared_ptr<Engine>>(m, "Engine")
        .def(py::init([](const TableArtifact& a, const ConfigRegistry& reg, const HardwareSpec& hw, int device) {
                 return std::make_shared<Engine>(a.tables, reg, hw, device);
             }),
             py::arg("tables"), py::arg("registry"), py::arg("hw"), py::arg("device") = 0)
        .def_property_readonly("n_configs", &Engine::n_configs)
        .def_property_readonly("handle", [](const Engine& e) { return reinterpret_cast<uintptr_t>(e.handle()); })
        .def("tune", &Engine::tune_one, py::arg("workload"))
        .def("set_resident", &Engine::set_resident, py::arg("idle_us"))
        .def(
            "tune_batch",
            [](const Engine& e, py::array_t<int32_t> M, py::array_t<int32_t> N, py::array_t<int32_t> K) {
                std::vector<int32_t> m(M.data(), M.data() + M.size()), n(N.data(), N.data() + N.size()),
                    k(K.data(), K.data() + K.size());
                std::vector<int32_t> ma, mi;
                std::vector<double> lat;
                {
                    py::gil_scoped_release nogil;
                    e.tune_host(m, n, k, ma, mi, lat);
                }
                return py::make_tuple(py::array_t<int32_t>(ma.size(), ma.data()),
                                      py::array_t<int32_t>(mi.size(), mi.data()),
                                      py::array_t<double>(lat.size(), lat.data()));
            },
            py::arg("M"), py::arg("N"), py::arg("K"));
    // ---- B200 validation GEMM family behind MeasurementBackend (new)
    m.def("gemm_registry", &gemm_registry);
    py::class_<B200GemmBackend>(m, "B200GemmBackend")
        .def(py::init<int, int, std::uint64_t>(), py::arg("warmup") = 3, py::arg("measured") = 10,
             py::arg("seed") = 0)
        .def("measure", &B200GemmBackend::measure, py::arg("workload"), py::arg("macro"), py::arg("micro"),
             py::call_guard<py::gil_scoped_release>())
        .def_static("family_config", &B200GemmBackend::family_config, py::arg("macro"), py::arg("micro"))
        .def(
            "profile",
            [](B200GemmBackend& b, const SamplingPlan& plan, const ConfigRegistry& reg) {
                py::gil_scoped_release nogil;
                return run_profile(plan, reg, b);
            },
            py::arg("plan"), py::arg("registry"));
    m.def("abi_version", &wt_abi_version);
    m.def("version", []() { return std::string(wt_version()); });
}
