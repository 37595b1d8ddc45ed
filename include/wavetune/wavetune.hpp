// wavetune.hpp -- C++ drop-in API of the B200-native WaveTune decision path.
//
// Same namespace, type names, members and function signatures as the
// reference's public headers (proj/include/wavetune/{kernel_map,model,
// tuner,profiler}.hpp), so code written against the reference recompiles
// unchanged.  Underneath, every decision / fit runs in the sm_100a kernels of
// libwtb200.so through the C-ABI in include/wavetune_c.h; this layer only
// converts value types, caches device images and rebuilds flag strings.
// The per-module headers (kernel_map.hpp, model.hpp, ...) include this file.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <tuple>
#include <utility>
#include <variant>
#include <vector>

namespace wavetune {

using i64 = std::int64_t;

inline i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

// ============================================================ workloads
enum class KernelFamily { DenseGemm, GroupedGemm, FlashAttention };
const char* family_name(KernelFamily f);
KernelFamily family_from_name(std::string_view name);

struct DenseGemm {
    i64 m, n, k;
};
struct GroupedGemm {
    std::vector<i64> group_rows;
    i64 n, k;
};
struct FlashAttention {
    i64 n_heads, s_q, s_kv;
};
using KernelWorkload = std::variant<DenseGemm, GroupedGemm, FlashAttention>;

KernelFamily family_of(const KernelWorkload& x);
std::string workload_to_string(const KernelWorkload& x);
KernelWorkload workload_from_string(std::string_view text);

// ============================================================ configs
struct GemmTiles {
    i64 t_m, t_n, t_k;
};
struct AttnTiles {
    i64 t_q, t_kv;
};
struct MacroConfig {
    int id = 0;
    std::variant<GemmTiles, AttnTiles> tiles;
};
struct MicroConfig {
    int id = 0;
    i64 n_stages = 1;
    i64 n_warps = 1;
    std::vector<std::pair<std::string, i64>> extra;
};
struct HardwareSpec {
    int n_sm = 1;
    int blocks_per_sm = 1;
    std::string name;
    int slots() const { return n_sm * blocks_per_sm; }
};
struct PhysicalCoords {
    i64 g = 0;
    i64 l = 0;
    int w = 0;
};

struct ConfigRegistry {
    KernelFamily family = KernelFamily::DenseGemm;
    std::vector<MacroConfig> macros;
    std::vector<MicroConfig> micros;
    std::set<std::pair<int, int>> feasible;

    const MacroConfig& macro(int id) const;
    const MicroConfig& micro(int id) const;
    std::vector<int> feasible_micros(int macro_id) const;
    void validate() const;
    static ConfigRegistry load(const std::string& path);
    void save(const std::string& path) const;
};

std::pair<i64, i64> map_workload(const KernelWorkload& x, const MacroConfig& c);
int wave_count(i64 g, const HardwareSpec& hw);
PhysicalCoords physical_coords(const KernelWorkload& x, const MacroConfig& c, const HardwareSpec& hw);

struct GridFactoring {
    i64 m_g, n_g;
};
KernelWorkload instantiate_workload(GridFactoring f, i64 l, const MacroConfig& c);
KernelWorkload instantiate_workload_attention(i64 g, i64 l, const MacroConfig& c, i64 n_heads);

// ============================================================ wave simulator
// Synthetic ground truth + discrete-event wave simulator (reference
// wave_sim.hpp).  The latency-model callbacks are evaluated on the host to
// obtain (mean, gap) per (macro, micro, l); the dispatch simulation itself
// runs on the GPU (wt_simulate_batch / wt_profile_sim).
struct BlockLatencyModel {
    std::function<double(int macro_id, int micro_id, i64 l)> mean_fn;
    double sigma = 0.0;
    double floor_frac = 0.01;
    std::function<double(int, int)> dispatch_gap;
    static BlockLatencyModel constant(double mu, double sigma = 0.0);
};
struct GroundEntry {
    double base = 0.0;
    double per_iter = 0.0;
    double dispatch_gap = 0.0;
};
struct SyntheticKernelGround {
    std::map<std::pair<int, int>, GroundEntry> entries;
    const GroundEntry& at(int macro_id, int micro_id) const;
    double mean(int macro_id, int micro_id, i64 l) const;
    BlockLatencyModel latency_model(double sigma) const;
    static SyntheticKernelGround load(const std::string& path);
    void save(const std::string& path) const;
};
struct SimMachine {
    HardwareSpec hw;
    std::uint64_t seed = 0;
};
double simulate(const SimMachine& machine, i64 g, i64 l, const BlockLatencyModel& blm, int macro_id = 0,
                int micro_id = 0);
struct SweepPoint {
    i64 g;
    double latency_us;
};
std::vector<SweepPoint> sweep_profile(const SimMachine& machine, const std::vector<i64>& g_list, i64 l,
                                      const BlockLatencyModel& blm, int macro_id = 0, int micro_id = 0);
struct OracleResult {
    int macro_id;
    int micro_id;
    double latency_us;
};
OracleResult oracle_best(const SimMachine& machine, const KernelWorkload& x, const ConfigRegistry& registry,
                         const SyntheticKernelGround& ground, double sigma, int reps = 3);

// ============================================================ sampling
struct GridPoint {
    int w = 0;
    int i = 0;
    i64 g = 0;
    std::optional<GridFactoring> factoring;
};
struct SamplingPlan {
    KernelFamily family = KernelFamily::DenseGemm;
    HardwareSpec hw;
    int W = 1;
    int I = 1;
    double tau = 1.1;
    std::optional<i64> n_heads;
    std::vector<i64> loop_anchors;
    std::vector<GridPoint> grid_points;
    static SamplingPlan load(const std::string& path);
    void save(const std::string& path) const;
};
struct PlanParams {
    int W = 1;
    int I = 1;
    double tau = 1.1;
    std::vector<i64> loop_anchors;
    std::optional<i64> n_heads;
};
std::optional<GridPoint> select_grid_point(i64 a, i64 b, KernelFamily family, double tau,
                                           std::optional<i64> n_heads = {});
SamplingPlan build_plan(const HardwareSpec& hw, KernelFamily family, const PlanParams& params);

struct ProfileRecord {
    i64 g = 0;
    i64 l = 0;
    int w = 0;
    int macro_id = 0;
    int micro_id = 0;
    double latency_us = 0.0;
};
void write_records(const std::vector<ProfileRecord>& records, const std::string& path);
std::vector<ProfileRecord> read_records(const std::string& path);

class MeasurementBackend {
public:
    virtual ~MeasurementBackend() = default;
    virtual double measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) = 0;
    virtual bool concurrency_safe() const { return false; }
};
class SimulatorBackend : public MeasurementBackend {
public:
    SimulatorBackend(HardwareSpec hw, SyntheticKernelGround ground, double sigma, std::uint64_t seed,
                     int warmup = 3, int measured = 5);
    double measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) override;
    bool concurrency_safe() const override { return true; }
    // the whole run_profile sweep in one device launch (used by run_profile)
    std::vector<ProfileRecord> profile(const struct SamplingPlan& plan, const ConfigRegistry& registry) const;

private:
    HardwareSpec hw_;
    SyntheticKernelGround ground_;
    double sigma_;
    std::uint64_t seed_;
    int warmup_, measured_;
};
class CsvReplayBackend : public MeasurementBackend {
public:
    explicit CsvReplayBackend(const std::vector<ProfileRecord>& records);
    static CsvReplayBackend from_file(const std::string& path);
    double measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) override;
    bool concurrency_safe() const override { return true; }

private:
    std::map<std::tuple<i64, i64, int, int>, double> table_;
};
class ExternalCommandBackend : public MeasurementBackend {
public:
    explicit ExternalCommandBackend(std::string command);
    double measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) override;

private:
    std::string command_;
};
std::vector<ProfileRecord> run_profile(const SamplingPlan& plan, const ConfigRegistry& registry,
                                       MeasurementBackend& backend);

// ============================================================ model
struct BilinearCoeffs {
    double alpha = 0.0;
    double beta = 0.0;
    double gamma = 0.0;
    double delta = 0.0;
    // Host convenience with the reference's operation order; the decision
    // path itself evaluates on the device.
    double predict(i64 g, i64 l) const {
        const double gd = static_cast<double>(g), ld = static_cast<double>(l);
        return alpha * gd * ld + beta * gd + gamma * ld + delta;
    }
    bool operator==(const BilinearCoeffs&) const = default;
};
struct FitSample {
    double g, l, latency_us;
};
struct FitResult {
    BilinearCoeffs coeffs;
    double r2 = 0.0;
    double mape = 0.0;
    bool degenerate = false;
};
FitResult fit_bucket(const std::vector<FitSample>& samples);

struct SharedMicroSelection {
    int micro_id = -1;
    std::vector<std::pair<i64, double>> samples;
    bool partial_coverage = false;
};
SharedMicroSelection select_shared_micro(const std::vector<ProfileRecord>& group);

struct WaveDiagnostics {
    double r2 = 0.0;
    double mape = 0.0;
    int samples = 0;
    std::vector<std::string> flags;
    bool operator==(const WaveDiagnostics&) const = default;
};
struct DualTable {
    int macro_id = -1;
    std::string hardware;
    int W = 0;
    int p = 0;
    std::map<int, BilinearCoeffs> coeff_table;
    BilinearCoeffs theta_ext;
    std::map<int, std::map<i64, int>> anchor_table;
    std::map<i64, int> ext_anchors;
    std::map<int, WaveDiagnostics> diagnostics;
    std::vector<std::string> ext_flags;
    bool operator==(const DualTable&) const = default;
};
struct ExtrapolationFit {
    BilinearCoeffs theta_ext;
    std::map<i64, int> ext_anchors;
    std::vector<std::string> flags;
};
ExtrapolationFit fit_extrapolation(const std::vector<ProfileRecord>& records, int W, int p);

struct TableBuildParams {
    int W = 0;
    int p = 10;
};
std::vector<DualTable> build_dual_table(const std::vector<ProfileRecord>& records,
                                        const ConfigRegistry& registry, const HardwareSpec& hw,
                                        const TableBuildParams& params);

struct TableArtifact {
    KernelFamily family = KernelFamily::DenseGemm;
    std::vector<DualTable> tables;
    bool operator==(const TableArtifact&) const = default;
};
void save_tables(const TableArtifact& artifact, const std::string& path);
TableArtifact load_tables(const std::string& path);

// ============================================================ tuner
struct DecisionStats {
    int model_evals = 0;
    int anchor_comparisons = 0;
};
struct Regime {
    bool extrapolated = false;
    int w = 0;
    bool operator==(const Regime&) const = default;
};
struct Tuned {
    int macro_id = -1;
    int micro_id = -1;
    double predicted_latency_us = 0.0;
    i64 g = 0;
    i64 l = 0;
    Regime regime;
    DecisionStats stats;
    std::vector<std::string> flags;
};

std::pair<double, Regime> predict_latency(const DualTable& table, i64 g, i64 l, const HardwareSpec& hw,
                                          std::vector<std::string>* flags = nullptr);
i64 nearest_anchor(const std::vector<i64>& sorted_anchors, i64 l, int* comparisons = nullptr);
Tuned tune(const KernelWorkload& x, const std::vector<DualTable>& tables, const ConfigRegistry& registry,
           const HardwareSpec& hw);

// ---- ablation baselines (reference tuner.hpp:54-85): fitted by K2 on the
// GPU from the same selected samples, evaluated by the baseline kernels.
struct StepPredictor {
    std::map<std::pair<int, i64>, double> t_wave;  // (macro_id, loop anchor) -> per-wave latency
};
struct GlobalLinearPredictor {
    std::map<int, BilinearCoeffs> theta;  // macro_id -> single global fit
};
struct BaselinePredictor {
    enum class Kind { Step, GlobalLinear } kind = Kind::Step;
    StepPredictor step;
    GlobalLinearPredictor linear;
};
BaselinePredictor fit_step_baseline(const std::vector<ProfileRecord>& records);
BaselinePredictor fit_linear_baseline(const std::vector<ProfileRecord>& records);
double baseline_predict(const BaselinePredictor& bp, int macro_id, i64 g, i64 l, const HardwareSpec& hw);
Tuned baseline_tune(const KernelWorkload& x, const BaselinePredictor& bp, const std::vector<DualTable>& tables,
                    const ConfigRegistry& registry, const HardwareSpec& hw);

// ============================================================ batched (new)
// A device-resident engine: the (tables, registry, hw) triple validated and
// uploaded once; queries go straight to the kernels.
class Engine {
public:
    Engine(const std::vector<DualTable>& tables, const ConfigRegistry& registry, const HardwareSpec& hw,
           int device = 0);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void* handle() const { return handle_; }
    int device() const { return device_; }
    int n_configs() const { return n_configs_; }
    // One full tune() with flags (single query).
    Tuned tune_one(const KernelWorkload& x) const;
    // idle_us > 0: single queries are answered by a resident polling CTA
    // (no launch per query) that leaves after idle_us without queries.
    void set_resident(int idle_us);
    // Batched dense/attention decisions on host vectors (copies inside).
    void tune_host(const std::vector<int32_t>& M, const std::vector<int32_t>& N, const std::vector<int32_t>& K,
                   std::vector<int32_t>& macro, std::vector<int32_t>& micro, std::vector<double>& latency) const;

private:
    void* handle_ = nullptr;
    int device_ = 0;
    int n_configs_ = 0;
    std::vector<int> macro_sorted_;
    std::vector<std::tuple<int, int, int>> tiles_sorted_;
    std::vector<DualTable> tables_sorted_;
    KernelFamily family_;
    HardwareSpec hw_;
};

}  // namespace wavetune
