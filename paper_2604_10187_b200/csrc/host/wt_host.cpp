// wt_host.cpp -- the C++ drop-in API (include/wavetune/wavetune.hpp).
//
// Host-side plumbing only: value types, the reference's on-disk formats
// (registry / plan JSON, records CSV, tables JSON with %a hex floats), the
// sampling plan, and the measurement-backend plugin interface.  Every
// decision and every fit is delegated to the sm_100a kernels through the
// C-ABI (include/wavetune_c.h); there is no CPU evaluation of the latency
// model in this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <set>
#include <limits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <mutex>
#include <sstream>
#include <unordered_map>

#include <json.hpp>

#include "wavetune/wavetune.hpp"
#include "wavetune_c.h"

namespace wavetune {

using nlohmann::json;

// ---------------------------------------------------------------- errors
namespace {

[[noreturn]] void rethrow(wt_status st, const std::string& ctx = "") {
    std::string msg = wt_last_error();
    if (!ctx.empty()) msg = ctx;
    switch (st) {
        case WT_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case WT_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

void ok(wt_status st) {
    if (st != WT_OK) rethrow(st);
}

void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Small device scratch reused per host thread (single-query drop-in calls).
struct Scratch {
    void* p = nullptr;
    size_t n = 0;
    int dev = -1;
    ~Scratch() {
        if (p) cudaFree(p);
    }
    void* get(size_t bytes, int device) {
        if (bytes > n || dev != device) {
            if (p) cudaFree(p);
            cudaSetDevice(device);
            cu(cudaMalloc(&p, bytes), "scratch");
            n = bytes;
            dev = device;
        }
        return p;
    }
};
thread_local Scratch t_scratch;

}  // namespace

// ------------------------------------------------------------- families
const char* family_name(KernelFamily f) {
    switch (f) {
        case KernelFamily::DenseGemm: return "dense_gemm";
        case KernelFamily::GroupedGemm: return "grouped_gemm";
        case KernelFamily::FlashAttention: return "flash_attention";
    }
    return "unknown";
}

KernelFamily family_from_name(std::string_view s) {
    static const std::pair<const char*, KernelFamily> names[] = {
        {"dense_gemm", KernelFamily::DenseGemm},      {"gemm", KernelFamily::DenseGemm},
        {"grouped_gemm", KernelFamily::GroupedGemm},  {"moe", KernelFamily::GroupedGemm},
        {"flash_attention", KernelFamily::FlashAttention}, {"attention", KernelFamily::FlashAttention}};
    for (const auto& [n, f] : names)
        if (s == n) return f;
    throw std::invalid_argument("unknown kernel family: " + std::string(s));
}

KernelFamily family_of(const KernelWorkload& x) {
    return std::visit(
        [](const auto& w) {
            using T = std::decay_t<decltype(w)>;
            if constexpr (std::is_same_v<T, DenseGemm>) return KernelFamily::DenseGemm;
            else if constexpr (std::is_same_v<T, GroupedGemm>) return KernelFamily::GroupedGemm;
            else return KernelFamily::FlashAttention;
        },
        x);
}

// ------------------------------------------------------- workload text
std::string workload_to_string(const KernelWorkload& x) {
    std::ostringstream o;
    o << family_name(family_of(x)) << ',';
    if (auto* d = std::get_if<DenseGemm>(&x)) {
        o << d->m << ',' << d->n << ',' << d->k;
    } else if (auto* a = std::get_if<FlashAttention>(&x)) {
        o << a->n_heads << ',' << a->s_q << ',' << a->s_kv;
    } else {
        const auto& gg = std::get<GroupedGemm>(x);
        o << gg.n << ',' << gg.k << ',';
        for (size_t i = 0; i < gg.group_rows.size(); ++i) o << (i ? ";" : "") << gg.group_rows[i];
    }
    return o.str();
}

namespace {
i64 parse_i64(const std::string& s) {
    size_t used = 0;
    i64 v = std::stoll(s, &used);
    if (used != s.size()) throw std::invalid_argument("bad integer in workload: " + s);
    return v;
}
std::vector<std::string> split(std::string_view text, char sep) {
    std::vector<std::string> out(1);
    for (char c : text) {
        if (c == sep) out.emplace_back();
        else out.back().push_back(c);
    }
    return out;
}
}  // namespace

KernelWorkload workload_from_string(std::string_view text) {
    auto f = split(text, ',');
    if (f.size() != 4)
        throw std::invalid_argument("workload must have 4 comma-separated fields: " + std::string(text));
    if (f[0] == "dense_gemm") return DenseGemm{parse_i64(f[1]), parse_i64(f[2]), parse_i64(f[3])};
    if (f[0] == "flash_attention") return FlashAttention{parse_i64(f[1]), parse_i64(f[2]), parse_i64(f[3])};
    if (f[0] == "grouped_gemm") {
        GroupedGemm gg{{}, parse_i64(f[1]), parse_i64(f[2])};
        std::string rows = f[3];
        if (!rows.empty())
            for (auto& part : split(rows, ';')) gg.group_rows.push_back(parse_i64(part));
        if (gg.group_rows.empty()) throw std::invalid_argument("grouped_gemm needs at least one group");
        return gg;
    }
    throw std::invalid_argument("unknown workload tag: " + f[0]);
}

// ------------------------------------------------------------ registry
const MacroConfig& ConfigRegistry::macro(int id) const {
    auto it = std::find_if(macros.begin(), macros.end(), [&](const MacroConfig& m) { return m.id == id; });
    if (it == macros.end()) throw std::out_of_range("no macro config with id " + std::to_string(id));
    return *it;
}

const MicroConfig& ConfigRegistry::micro(int id) const {
    auto it = std::find_if(micros.begin(), micros.end(), [&](const MicroConfig& m) { return m.id == id; });
    if (it == micros.end()) throw std::out_of_range("no micro config with id " + std::to_string(id));
    return *it;
}

std::vector<int> ConfigRegistry::feasible_micros(int macro_id) const {
    std::vector<int> out;
    for (auto it = feasible.lower_bound({macro_id, INT32_MIN}); it != feasible.end() && it->first == macro_id; ++it)
        out.push_back(it->second);
    return out;  // std::set order: ascending micro id
}

void ConfigRegistry::validate() const {
    std::set<int> ma, mi;
    for (const auto& m : macros) {
        if (!ma.insert(m.id).second) throw std::invalid_argument("duplicate macro_id " + std::to_string(m.id));
        const bool attn_family = family == KernelFamily::FlashAttention;
        if (const auto* g = std::get_if<GemmTiles>(&m.tiles)) {
            if (g->t_m < 1 || g->t_n < 1 || g->t_k < 1) throw std::invalid_argument("tile dims must be >= 1");
            if (attn_family) throw std::invalid_argument("gemm tiles in attention registry");
        } else {
            const auto& a = std::get<AttnTiles>(m.tiles);
            if (a.t_q < 1 || a.t_kv < 1) throw std::invalid_argument("tile dims must be >= 1");
            if (!attn_family) throw std::invalid_argument("attention tiles in gemm registry");
        }
    }
    for (const auto& u : micros) {
        if (!mi.insert(u.id).second) throw std::invalid_argument("duplicate micro_id " + std::to_string(u.id));
        if (u.n_stages < 1 || u.n_warps < 1) throw std::invalid_argument("micro params must be >= 1");
    }
    for (const auto& [a, b] : feasible)
        if (!ma.count(a) || !mi.count(b)) throw std::invalid_argument("feasible pair references unknown id");
    for (int a : ma)
        if (feasible_micros(a).empty())
            throw std::invalid_argument("macro " + std::to_string(a) + " has no feasible micro");
}

void ConfigRegistry::save(const std::string& path) const {
    validate();
    json j;
    j["version"] = 1;
    j["family"] = family_name(family);
    j["macros"] = json::array();
    for (const auto& m : macros) {
        json jm = {{"id", m.id}};
        if (const auto* g = std::get_if<GemmTiles>(&m.tiles)) {
            jm["t_m"] = g->t_m;
            jm["t_n"] = g->t_n;
            jm["t_k"] = g->t_k;
        } else {
            const auto& a = std::get<AttnTiles>(m.tiles);
            jm["t_q"] = a.t_q;
            jm["t_kv"] = a.t_kv;
        }
        j["macros"].push_back(jm);
    }
    j["micros"] = json::array();
    for (const auto& u : micros) {
        json ju = {{"id", u.id}, {"n_stages", u.n_stages}, {"n_warps", u.n_warps}};
        if (!u.extra.empty()) {
            json e = json::object();
            for (const auto& [k, v] : u.extra) e[k] = v;
            ju["extra"] = e;
        }
        j["micros"].push_back(ju);
    }
    j["feasible"] = json::array();
    for (const auto& [a, b] : feasible) j["feasible"].push_back({a, b});
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write registry file: " + path);
    out << j.dump(2) << "\n";
}

ConfigRegistry ConfigRegistry::load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open registry file: " + path);
    json j;
    in >> j;
    if (!j.contains("version")) throw std::invalid_argument("registry file missing 'version' field");
    if (j.at("version").get<int>() != 1)
        throw std::invalid_argument("registry version mismatch: expected 1, found " + j.at("version").dump());
    ConfigRegistry r;
    r.family = family_from_name(j.at("family").get<std::string>());
    for (const auto& jm : j.at("macros")) {
        MacroConfig m;
        m.id = jm.at("id").get<int>();
        if (jm.contains("t_q")) m.tiles = AttnTiles{jm.at("t_q").get<i64>(), jm.at("t_kv").get<i64>()};
        else m.tiles = GemmTiles{jm.at("t_m").get<i64>(), jm.at("t_n").get<i64>(), jm.at("t_k").get<i64>()};
        r.macros.push_back(m);
    }
    for (const auto& ju : j.at("micros")) {
        MicroConfig u;
        u.id = ju.at("id").get<int>();
        u.n_stages = ju.at("n_stages").get<i64>();
        u.n_warps = ju.at("n_warps").get<i64>();
        if (ju.contains("extra"))
            for (const auto& [k, v] : ju.at("extra").items()) u.extra.emplace_back(k, v.get<i64>());
        r.micros.push_back(u);
    }
    for (const auto& p : j.at("feasible")) r.feasible.emplace(p.at(0).get<int>(), p.at(1).get<int>());
    r.validate();
    return r;
}

// ------------------------------------------------------------- mapping
std::pair<i64, i64> map_workload(const KernelWorkload& x, const MacroConfig& c) {
    if (const auto* d = std::get_if<DenseGemm>(&x)) {
        const auto* t = std::get_if<GemmTiles>(&c.tiles);
        if (!t) throw std::invalid_argument("dense_gemm workload needs gemm tiles");
        if (d->m < 1 || d->n < 1 || d->k < 1) throw std::invalid_argument("dense_gemm dims must be >= 1");
        return {ceil_div(d->m, t->t_m) * ceil_div(d->n, t->t_n), ceil_div(d->k, t->t_k)};
    }
    if (const auto* gg = std::get_if<GroupedGemm>(&x)) {
        const auto* t = std::get_if<GemmTiles>(&c.tiles);
        if (!t) throw std::invalid_argument("grouped_gemm workload needs gemm tiles");
        if (gg->n < 1 || gg->k < 1) throw std::invalid_argument("grouped_gemm dims must be >= 1");
        i64 tiles_m = 0;
        for (i64 r : gg->group_rows) {
            if (r < 0) throw std::invalid_argument("negative group row count");
            tiles_m += r > 0 ? ceil_div(r, t->t_m) : 0;
        }
        const i64 g = tiles_m * ceil_div(gg->n, t->t_n);
        if (g == 0) throw std::invalid_argument("grouped_gemm maps to an empty grid");
        return {g, ceil_div(gg->k, t->t_k)};
    }
    const auto& a = std::get<FlashAttention>(x);
    const auto* t = std::get_if<AttnTiles>(&c.tiles);
    if (!t) throw std::invalid_argument("attention workload needs attention tiles");
    if (a.n_heads < 1 || a.s_q < 1 || a.s_kv < 1) throw std::invalid_argument("attention dims must be >= 1");
    return {a.n_heads * ceil_div(a.s_q, t->t_q), ceil_div(a.s_kv, t->t_kv)};
}

int wave_count(i64 g, const HardwareSpec& hw) {
    if (g < 1) throw std::invalid_argument("grid size must be >= 1");
    if (hw.n_sm < 1 || hw.blocks_per_sm < 1)
        throw std::invalid_argument("hardware spec must have positive capacities");
    return static_cast<int>(ceil_div(g, hw.slots()));
}

PhysicalCoords physical_coords(const KernelWorkload& x, const MacroConfig& c, const HardwareSpec& hw) {
    const auto [g, l] = map_workload(x, c);
    return {g, l, wave_count(g, hw)};
}

KernelWorkload instantiate_workload(GridFactoring f, i64 l, const MacroConfig& c) {
    const auto* t = std::get_if<GemmTiles>(&c.tiles);
    if (!t) throw std::invalid_argument("grid factoring requires gemm tiles");
    if (f.m_g < 1 || f.n_g < 1 || l < 1) throw std::invalid_argument("factoring and loop count must be >= 1");
    return DenseGemm{f.m_g * t->t_m, f.n_g * t->t_n, l * t->t_k};
}

KernelWorkload instantiate_workload_attention(i64 g, i64 l, const MacroConfig& c, i64 n_heads) {
    const auto* t = std::get_if<AttnTiles>(&c.tiles);
    if (!t) throw std::invalid_argument("attention instantiation requires attention tiles");
    if (n_heads < 1 || g < 1 || l < 1) throw std::invalid_argument("grid, loop count, and heads must be >= 1");
    if (g % n_heads)
        throw std::invalid_argument("attention grid size " + std::to_string(g) + " not divisible by n_heads " +
                                    std::to_string(n_heads));
    return FlashAttention{n_heads, (g / n_heads) * t->t_q, l * t->t_kv};
}

// ---------------------------------------------------------- sampling plan
std::optional<GridPoint> select_grid_point(i64 a, i64 b, KernelFamily family, double tau,
                                           std::optional<i64> n_heads) {
    if (a < 1 || a > b) throw std::invalid_argument("invalid interval");
    if (family == KernelFamily::FlashAttention) {
        if (!n_heads || *n_heads < 1) throw std::invalid_argument("attention plans require n_heads");
        const i64 g = b - b % *n_heads;
        if (g < a) return std::nullopt;
        GridPoint p;
        p.g = g;
        return p;
    }
    // largest g in [a, b] with a squarest factoring m <= n <= tau*m
    for (i64 g = b; g >= a; --g) {
        i64 m = static_cast<i64>(std::sqrt(static_cast<double>(g)));
        while ((m + 1) * (m + 1) <= g) ++m;
        while (m * m > g) --m;
        for (; m >= 1; --m) {
            if (g % m) continue;
            const i64 n = g / m;
            if (n < m) continue;
            if (static_cast<double>(n) <= tau * static_cast<double>(m)) {
                GridPoint p;
                p.g = g;
                p.factoring = GridFactoring{m, n};
                return p;
            }
            break;  // the squarest divisor already violates tau
        }
    }
    return std::nullopt;
}

SamplingPlan build_plan(const HardwareSpec& hw, KernelFamily family, const PlanParams& pp) {
    if (pp.W < 1 || pp.I < 1) throw std::invalid_argument("W and I must be >= 1");
    if (pp.tau <= 1.0) throw std::invalid_argument("tau must be > 1");
    if (pp.loop_anchors.empty()) throw std::invalid_argument("loop_anchors must be non-empty");
    if (family == KernelFamily::FlashAttention && (!pp.n_heads || *pp.n_heads < 1))
        throw std::invalid_argument("attention plans require n_heads");
    SamplingPlan plan;
    plan.family = family;
    plan.hw = hw;
    plan.W = pp.W;
    plan.I = pp.I;
    plan.tau = pp.tau;
    plan.n_heads = pp.n_heads;
    plan.loop_anchors = pp.loop_anchors;
    std::sort(plan.loop_anchors.begin(), plan.loop_anchors.end());
    const i64 span = hw.slots(), width = span / pp.I, extra = span % pp.I;
    for (int w = 1; w <= pp.W; ++w) {
        i64 lo = static_cast<i64>(w - 1) * span + 1;
        for (int i = 1; i <= pp.I; ++i) {
            const i64 hi = lo + width + (i <= extra ? 1 : 0) - 1;
            if (auto p = select_grid_point(lo, hi, family, pp.tau, pp.n_heads)) {
                p->w = w;
                p->i = i;
                plan.grid_points.push_back(*p);
            } else {
                std::cerr << "plan: no admissible grid size in [" << lo << ", " << hi << "] (w=" << w
                          << ", i=" << i << "), dropped\n";
            }
            lo = hi + 1;
        }
    }
    return plan;
}

void SamplingPlan::save(const std::string& path) const {
    json j;
    j["version"] = 1;
    j["family"] = family_name(family);
    j["n_sm"] = hw.n_sm;
    j["blocks_per_sm"] = hw.blocks_per_sm;
    j["hardware"] = hw.name;
    j["W"] = W;
    j["I"] = I;
    j["tau"] = tau;
    if (n_heads) j["n_heads"] = *n_heads;
    j["loop_anchors"] = loop_anchors;
    j["grid_points"] = json::array();
    for (const auto& p : grid_points) {
        json jp = {{"w", p.w}, {"i", p.i}, {"g", p.g}};
        if (p.factoring) {
            jp["m_g"] = p.factoring->m_g;
            jp["n_g"] = p.factoring->n_g;
        }
        j["grid_points"].push_back(jp);
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write plan file: " + path);
    out << j.dump(2) << "\n";
}

SamplingPlan SamplingPlan::load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open plan file: " + path);
    json j;
    in >> j;
    if (j.value("version", 0) != 1)
        throw std::invalid_argument("plan version mismatch: expected 1, found " + j.value("version", json(0)).dump());
    SamplingPlan p;
    p.family = family_from_name(j.at("family").get<std::string>());
    p.hw.n_sm = j.at("n_sm").get<int>();
    p.hw.blocks_per_sm = j.value("blocks_per_sm", 1);
    p.hw.name = j.value("hardware", "");
    p.W = j.at("W").get<int>();
    p.I = j.at("I").get<int>();
    p.tau = j.at("tau").get<double>();
    if (j.contains("n_heads")) p.n_heads = j.at("n_heads").get<i64>();
    p.loop_anchors = j.at("loop_anchors").get<std::vector<i64>>();
    for (const auto& jp : j.at("grid_points")) {
        GridPoint g;
        g.w = jp.at("w").get<int>();
        g.i = jp.at("i").get<int>();
        g.g = jp.at("g").get<i64>();
        if (jp.contains("m_g")) g.factoring = GridFactoring{jp.at("m_g").get<i64>(), jp.at("n_g").get<i64>()};
        p.grid_points.push_back(g);
    }
    return p;
}

// ---------------------------------------------------------------- records
void write_records(const std::vector<ProfileRecord>& records, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write dataset file: " + path);
    out << "g,l,w,macro_id,micro_id,latency_us\n";
    char num[64];
    for (const auto& r : records) {
        std::snprintf(num, sizeof num, "%.17g", r.latency_us);
        out << r.g << ',' << r.l << ',' << r.w << ',' << r.macro_id << ',' << r.micro_id << ',' << num << '\n';
    }
}

std::vector<ProfileRecord> read_records(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open dataset file: " + path);
    std::string line;
    if (!std::getline(in, line) || line != "g,l,w,macro_id,micro_id,latency_us")
        throw std::runtime_error("bad dataset header in " + path);
    std::vector<ProfileRecord> out;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        ProfileRecord r;
        char c1, c2, c3, c4, c5;
        std::istringstream row(line);
        if (!(row >> r.g >> c1 >> r.l >> c2 >> r.w >> c3 >> r.macro_id >> c4 >> r.micro_id >> c5 >> r.latency_us))
            throw std::runtime_error("malformed dataset row: " + line);
        if (r.latency_us <= 0) throw std::runtime_error("non-positive latency in dataset row: " + line);
        out.push_back(r);
    }
    return out;
}

CsvReplayBackend::CsvReplayBackend(const std::vector<ProfileRecord>& records) {
    for (const auto& r : records) table_[{r.g, r.l, r.macro_id, r.micro_id}] = r.latency_us;
}
CsvReplayBackend CsvReplayBackend::from_file(const std::string& path) { return CsvReplayBackend(read_records(path)); }
double CsvReplayBackend::measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) {
    const auto [g, l] = map_workload(x, macro);
    auto it = table_.find({g, l, macro.id, micro.id});
    if (it == table_.end())
        throw std::runtime_error("replay dataset has no entry for g=" + std::to_string(g) + " l=" + std::to_string(l) +
                                 " macro=" + std::to_string(macro.id) + " micro=" + std::to_string(micro.id));
    return it->second;
}

ExternalCommandBackend::ExternalCommandBackend(std::string command) : command_(std::move(command)) {}
double ExternalCommandBackend::measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) {
    std::ostringstream cmd;
    cmd << command_ << ' ' << family_name(family_of(x));
    std::string fields = workload_to_string(x);
    auto parts = split(fields, ',');
    if (const auto* gg = std::get_if<GroupedGemm>(&x)) {
        cmd << ' ' << gg->n << ' ' << gg->k;
        for (i64 r : gg->group_rows) cmd << ' ' << r;
    } else {
        cmd << ' ' << parts[1] << ' ' << parts[2] << ' ' << parts[3];
    }
    if (const auto* t = std::get_if<GemmTiles>(&macro.tiles)) cmd << ' ' << t->t_m << ' ' << t->t_n << ' ' << t->t_k;
    else cmd << ' ' << std::get<AttnTiles>(macro.tiles).t_q << ' ' << std::get<AttnTiles>(macro.tiles).t_kv;
    cmd << ' ' << micro.n_stages << ' ' << micro.n_warps;
    for (const auto& kv : micro.extra) cmd << ' ' << kv.second;
    FILE* pipe = popen(cmd.str().c_str(), "r");
    if (!pipe) throw std::runtime_error("failed to launch: " + cmd.str());
    std::string text;
    char buf[256];
    while (std::fgets(buf, sizeof buf, pipe)) text += buf;
    const int status = pclose(pipe);
    if (status != 0) throw std::runtime_error("measurement command exited with status " + std::to_string(status));
    std::istringstream parse(text);
    double v;
    if (!(parse >> v) || v <= 0) throw std::runtime_error("measurement command printed no latency: '" + text + "'");
    return v;
}

std::vector<ProfileRecord> run_profile(const SamplingPlan& plan, const ConfigRegistry& registry,
                                       MeasurementBackend& backend) {
    registry.validate();
    if (registry.family != plan.family) throw std::invalid_argument("registry family does not match plan family");
    // the simulator backend runs the whole sweep in one device launch
    if (const auto* sim = dynamic_cast<const SimulatorBackend*>(&backend)) return sim->profile(plan, registry);
    std::vector<MacroConfig> macros = registry.macros;
    std::sort(macros.begin(), macros.end(), [](const MacroConfig& a, const MacroConfig& b) { return a.id < b.id; });
    std::vector<ProfileRecord> out;
    size_t tried = 0, failed = 0;
    for (const auto& pt : plan.grid_points)
        for (i64 l : plan.loop_anchors)
            for (const auto& mc : macros) {
                const KernelWorkload x = plan.family == KernelFamily::FlashAttention
                                             ? instantiate_workload_attention(pt.g, l, mc, *plan.n_heads)
                                             : instantiate_workload(*pt.factoring, l, mc);
                for (int mu : registry.feasible_micros(mc.id)) {
                    ++tried;
                    try {
                        const double t = backend.measure(x, mc, registry.micro(mu));
                        out.push_back({pt.g, l, wave_count(pt.g, plan.hw), mc.id, mu, t});
                    } catch (const std::exception& e) {
                        ++failed;
                        std::cerr << "profile: skipped g=" << pt.g << " l=" << l << " macro=" << mc.id
                                  << " micro=" << mu << ": " << e.what() << "\n";
                    }
                }
            }
    if (tried > 0 && failed * 10 > tried)
        throw std::runtime_error("profiling aborted: " + std::to_string(failed) + " of " + std::to_string(tried) +
                                 " measurements failed (>10%)");
    return out;
}

// --------------------------------------------------------------- simulator
BlockLatencyModel BlockLatencyModel::constant(double mu, double sigma) {
    if (mu <= 0) throw std::invalid_argument("mean block latency must be positive");
    BlockLatencyModel b;
    b.mean_fn = [mu](int, int, i64) { return mu; };
    b.sigma = sigma;
    return b;
}

const GroundEntry& SyntheticKernelGround::at(int macro_id, int micro_id) const {
    auto it = entries.find({macro_id, micro_id});
    if (it == entries.end())
        throw std::out_of_range("no ground-truth entry for (" + std::to_string(macro_id) + ", " +
                                std::to_string(micro_id) + ")");
    return it->second;
}

double SyntheticKernelGround::mean(int macro_id, int micro_id, i64 l) const {
    const GroundEntry& e = at(macro_id, micro_id);
    return e.base + e.per_iter * static_cast<double>(l);
}

BlockLatencyModel SyntheticKernelGround::latency_model(double sigma) const {
    BlockLatencyModel b;
    b.mean_fn = [this](int a, int m, i64 l) { return mean(a, m, l); };
    b.dispatch_gap = [this](int a, int m) { return at(a, m).dispatch_gap; };
    b.sigma = sigma;
    return b;
}

SyntheticKernelGround SyntheticKernelGround::load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open ground-truth file: " + path);
    json j;
    in >> j;
    SyntheticKernelGround g;
    for (const auto& je : j.at("entries")) {
        GroundEntry e{je.at("base").get<double>(), je.at("per_iter").get<double>(), je.value("dispatch_gap", 0.0)};
        if (e.base <= 0 || e.per_iter < 0 || e.dispatch_gap < 0)
            throw std::invalid_argument("ground-truth costs must be positive");
        g.entries[{je.at("macro_id").get<int>(), je.at("micro_id").get<int>()}] = e;
    }
    return g;
}

void SyntheticKernelGround::save(const std::string& path) const {
    json j;
    j["entries"] = json::array();
    for (const auto& [k, e] : entries)
        j["entries"].push_back({{"macro_id", k.first}, {"micro_id", k.second}, {"base", e.base},
                                {"per_iter", e.per_iter}, {"dispatch_gap", e.dispatch_gap}});
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write ground-truth file: " + path);
    out << j.dump(2) << "\n";
}

namespace {
uint64_t host_splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t host_mix(uint64_t a, uint64_t b) { return host_splitmix(a ^ host_splitmix(b)); }

std::vector<double> run_sims(const std::vector<int64_t>& g, const std::vector<double>& mean, double sigma,
                             const std::vector<double>& eps, const std::vector<double>& gap,
                             const std::vector<uint64_t>& seed, int slots) {
    std::vector<double> sig(g.size(), sigma), out(g.size());
    int dev = 0;
    cudaGetDevice(&dev);
    ok(wt_simulate_batch(g.data(), mean.data(), sig.data(), eps.data(), gap.data(), seed.data(), int64_t(g.size()),
                         slots, out.data(), dev));
    return out;
}
}  // namespace

double simulate(const SimMachine& machine, i64 g, i64 l, const BlockLatencyModel& blm, int macro_id, int micro_id) {
    if (g < 1 || l < 1) throw std::invalid_argument("grid size and loop count must be >= 1");
    if (!blm.mean_fn) throw std::invalid_argument("latency model has no mean_fn");
    const double mean = blm.mean_fn(macro_id, micro_id, l);
    if (mean <= 0) throw std::invalid_argument("mean block duration must be positive");
    const double gap = blm.dispatch_gap ? blm.dispatch_gap(macro_id, micro_id) : 0.0;
    return run_sims({g}, {mean}, blm.sigma, {blm.floor_frac * mean}, {gap}, {machine.seed}, machine.hw.slots())[0];
}

std::vector<SweepPoint> sweep_profile(const SimMachine& machine, const std::vector<i64>& g_list, i64 l,
                                      const BlockLatencyModel& blm, int macro_id, int micro_id) {
    if (g_list.empty()) throw std::invalid_argument("g_list must be non-empty");
    if (!std::is_sorted(g_list.begin(), g_list.end())) throw std::invalid_argument("g_list must be ascending");
    if (!blm.mean_fn) throw std::invalid_argument("latency model has no mean_fn");
    const double mean = blm.mean_fn(macro_id, micro_id, l);
    if (mean <= 0) throw std::invalid_argument("mean block duration must be positive");
    const double gap = blm.dispatch_gap ? blm.dispatch_gap(macro_id, micro_id) : 0.0;
    const size_t n = g_list.size();
    std::vector<uint64_t> seeds(n);
    for (size_t i = 0; i < n; ++i) seeds[i] = host_mix(machine.seed, uint64_t(g_list[i]));
    auto m = run_sims(std::vector<int64_t>(g_list.begin(), g_list.end()), std::vector<double>(n, mean), blm.sigma,
                      std::vector<double>(n, blm.floor_frac * mean), std::vector<double>(n, gap), seeds,
                      machine.hw.slots());
    std::vector<SweepPoint> out;
    for (size_t i = 0; i < n; ++i) out.push_back({g_list[i], m[i]});
    return out;
}

OracleResult oracle_best(const SimMachine& machine, const KernelWorkload& x, const ConfigRegistry& registry,
                         const SyntheticKernelGround& ground, double sigma, int reps) {
    if (registry.feasible.empty()) throw std::invalid_argument("registry has no feasible pairs");
    if (reps < 1) throw std::invalid_argument("reps must be >= 1");
    std::vector<int64_t> g;
    std::vector<double> mean, eps, gap;
    std::vector<uint64_t> seed;
    std::vector<std::pair<int, int>> pairs(registry.feasible.begin(), registry.feasible.end());
    for (const auto& [ma, mi] : pairs) {
        const auto [gg, l] = map_workload(x, registry.macro(ma));
        const double mu = ground.mean(ma, mi, l);
        if (mu <= 0) throw std::invalid_argument("mean block duration must be positive");
        for (int r = 0; r < reps; ++r) {
            g.push_back(gg);
            mean.push_back(mu);
            eps.push_back(0.01 * mu);
            gap.push_back(ground.at(ma, mi).dispatch_gap);
            seed.push_back(host_mix(host_mix(host_mix(machine.seed, uint64_t(int64_t(ma))), uint64_t(int64_t(mi))),
                                    uint64_t(r)));
        }
    }
    const auto m = run_sims(g, mean, sigma, eps, gap, seed, machine.hw.slots());
    OracleResult best{-1, -1, std::numeric_limits<double>::infinity()};
    for (size_t p = 0; p < pairs.size(); ++p) {
        double total = 0.0;
        for (int r = 0; r < reps; ++r) total += m[p * reps + r];
        const double lat = total / reps;
        if (lat < best.latency_us) best = {pairs[p].first, pairs[p].second, lat};
    }
    return best;
}

SimulatorBackend::SimulatorBackend(HardwareSpec hw, SyntheticKernelGround ground, double sigma, std::uint64_t seed,
                                   int warmup, int measured)
    : hw_(std::move(hw)), ground_(std::move(ground)), sigma_(sigma), seed_(seed), warmup_(warmup),
      measured_(measured) {
    if (measured_ < 1) throw std::invalid_argument("measured iterations must be >= 1");
}

double SimulatorBackend::measure(const KernelWorkload& x, const MacroConfig& macro, const MicroConfig& micro) {
    const auto [g, l] = map_workload(x, macro);
    const double mean = ground_.mean(macro.id, micro.id, l);
    if (mean <= 0) throw std::invalid_argument("mean block duration must be positive");
    const int iters = warmup_ + measured_;
    const uint64_t inner = host_mix(host_mix(uint64_t(l), uint64_t(int64_t(macro.id))), uint64_t(int64_t(micro.id)));
    const uint64_t base = host_mix(host_mix(seed_, uint64_t(g)), inner);
    std::vector<uint64_t> seeds(iters);
    for (int it = 0; it < iters; ++it) seeds[it] = host_mix(base, uint64_t(it));
    const auto m = run_sims(std::vector<int64_t>(iters, g), std::vector<double>(iters, mean), sigma_,
                            std::vector<double>(iters, 0.01 * mean),
                            std::vector<double>(iters, ground_.at(macro.id, micro.id).dispatch_gap), seeds,
                            hw_.slots());
    double total = 0.0;
    for (int it = warmup_; it < iters; ++it) total += m[it];
    return total / measured_;
}

std::vector<ProfileRecord> SimulatorBackend::profile(const SamplingPlan& plan, const ConfigRegistry& registry) const {
    std::vector<int64_t> pg, al(plan.loop_anchors.begin(), plan.loop_anchors.end());
    for (const auto& p : plan.grid_points) pg.push_back(p.g);
    std::vector<MacroConfig> macros = registry.macros;
    std::sort(macros.begin(), macros.end(), [](const MacroConfig& a, const MacroConfig& b) { return a.id < b.id; });
    std::vector<int32_t> pm, pu;
    std::vector<double> base, per, gap;
    for (const auto& mc : macros)
        for (int mu : registry.feasible_micros(mc.id)) {
            const GroundEntry& e = ground_.at(mc.id, mu);
            pm.push_back(mc.id);
            pu.push_back(mu);
            base.push_back(e.base);
            per.push_back(e.per_iter);
            gap.push_back(e.dispatch_gap);
        }
    wt_sim_profile_desc d{};
    d.n_points = int64_t(pg.size());
    d.point_g = pg.data();
    d.n_anchors = int64_t(al.size());
    d.anchor_l = al.data();
    d.n_pairs = int64_t(pm.size());
    d.pair_macro = pm.data();
    d.pair_micro = pu.data();
    d.pair_base = base.data();
    d.pair_per_iter = per.data();
    d.pair_gap = gap.data();
    d.sigma = sigma_;
    d.floor_frac = 0.01;
    d.seed = seed_;
    d.warmup = warmup_;
    d.measured = measured_;
    d.slots = hw_.slots();
    const size_t total = pg.size() * al.size() * pm.size();
    std::vector<double> lat(total);
    std::vector<int32_t> st(total);
    int dev = 0;
    cudaGetDevice(&dev);
    double ms = 0;
    ok(wt_profile_sim(&d, lat.data(), st.data(), dev, &ms));
    std::vector<ProfileRecord> out;
    size_t r = 0, failed = 0;
    for (size_t p = 0; p < pg.size(); ++p)
        for (size_t a = 0; a < al.size(); ++a)
            for (size_t f = 0; f < pm.size(); ++f, ++r) {
                if (st[r]) {
                    ++failed;
                    std::cerr << "profile: skipped g=" << pg[p] << " l=" << al[a] << " macro=" << pm[f]
                              << " micro=" << pu[f] << ": mean block duration must be positive\n";
                    continue;
                }
                out.push_back({pg[p], al[a], wave_count(pg[p], plan.hw), pm[f], pu[f], lat[r]});
            }
    if (total > 0 && failed * 10 > total)
        throw std::runtime_error("profiling aborted: " + std::to_string(failed) + " of " + std::to_string(total) +
                                 " measurements failed (>10%)");
    return out;
}

// ------------------------------------------------------------------ model
FitResult fit_bucket(const std::vector<FitSample>& samples) {
    if (samples.empty()) throw std::invalid_argument("fit_bucket: no samples");
    const size_t n = samples.size();
    std::vector<double> g(n), l(n), t(n);
    for (size_t i = 0; i < n; ++i) {
        g[i] = samples[i].g;
        l[i] = samples[i].l;
        t[i] = samples[i].latency_us;
    }
    const int64_t off[2] = {0, int64_t(n)};
    double co[4], r2, mape;
    int32_t dg;
    int dev = 0;
    cudaGetDevice(&dev);
    ok(wt_fit_bucket_batch(g.data(), l.data(), t.data(), off, 1, co, &r2, &mape, &dg, dev));
    FitResult r;
    r.coeffs = {co[0], co[1], co[2], co[3]};
    r.r2 = r2;
    r.mape = mape;
    r.degenerate = dg != 0;
    return r;
}

namespace {

// One wt_fit_build call, converted back into DualTables (registry order).
std::vector<DualTable> device_build(const std::vector<ProfileRecord>& records, const std::vector<int>& ids,
                                    const std::string& hw_name, int W, int p) {
    const size_t n = records.size();
    std::vector<int64_t> g(n), l(n);
    std::vector<int32_t> w(n), ma(n), mi(n);
    std::vector<double> t(n);
    for (size_t i = 0; i < n; ++i) {
        g[i] = records[i].g;
        l[i] = records[i].l;
        w[i] = records[i].w;
        ma[i] = records[i].macro_id;
        mi[i] = records[i].micro_id;
        t[i] = records[i].latency_us;
    }
    wt_records_desc rd{int64_t(n), g.data(), l.data(), w.data(), ma.data(), mi.data(), t.data()};
    wt_build* b = nullptr;
    wt_build_result R{};
    int dev = 0;
    cudaGetDevice(&dev);
    std::vector<int32_t> ids32(ids.begin(), ids.end());
    ok(wt_fit_build(&rd, ids32.data(), int32_t(ids32.size()), W, p, dev, &b, &R));
    std::unique_ptr<wt_build, wt_status (*)(wt_build*)> guard(b, wt_build_free);
    std::vector<DualTable> out;
    for (int32_t q = 0; q < R.n_tables; ++q) {
        DualTable d;
        d.macro_id = R.macro_id[q];
        d.hardware = hw_name;
        d.W = R.W;
        d.p = R.p;
        d.theta_ext = {R.theta_ext[4 * q], R.theta_ext[4 * q + 1], R.theta_ext[4 * q + 2], R.theta_ext[4 * q + 3]};
        for (int32_t k = R.coeff_off[q]; k < R.coeff_off[q + 1]; ++k) {
            d.coeff_table[R.coeff_w[k]] = {R.coeff_theta[4 * k], R.coeff_theta[4 * k + 1], R.coeff_theta[4 * k + 2],
                                          R.coeff_theta[4 * k + 3]};
            WaveDiagnostics& dg = d.diagnostics[R.coeff_w[k]];
            dg.r2 = R.diag_r2[k];
            dg.mape = R.diag_mape[k];
            dg.samples = R.diag_samples[k];
        }
        for (int32_t k = R.awave_off[q]; k < R.awave_off[q + 1]; ++k) {
            const int wave = R.awave_w[k];
            WaveDiagnostics& dg = d.diagnostics[wave];
            for (int32_t a = R.awave_aoff[k]; a < R.awave_aoff[k + 1]; ++a) {
                d.anchor_table[wave][R.anchor_l[a]] = R.anchor_micro[a];
                if (R.anchor_partial[a]) dg.flags.push_back("partial_micro_coverage_l" + std::to_string(R.anchor_l[a]));
            }
        }
        for (int32_t k = R.coeff_off[q]; k < R.coeff_off[q + 1]; ++k) {
            WaveDiagnostics& dg = d.diagnostics[R.coeff_w[k]];
            if (R.diag_flags[k] & 1) dg.flags.push_back("degenerate_fit");
            if (R.diag_flags[k] & 2) dg.flags.push_back("sparse_bucket");
        }
        for (int32_t a = R.ext_aoff[q]; a < R.ext_aoff[q + 1]; ++a) d.ext_anchors[R.ext_l[a]] = R.ext_micro[a];
        if (R.ext_flags[q] & 1) d.ext_flags.push_back("ext_degenerate_fit");
        if (R.ext_flags[q] & 2) d.ext_flags.push_back("ext_insufficient_waves");
        out.push_back(std::move(d));
    }
    return out;
}

}  // namespace

SharedMicroSelection select_shared_micro(const std::vector<ProfileRecord>& group) {
    if (group.empty()) throw std::invalid_argument("select_shared_micro: empty group");
    // One (macro, w, l) group through the device build: the anchor carries the
    // selected micro and its partial-coverage bit; the samples are re-read
    // from the group in (g ascending, last write wins) order for that micro.
    std::vector<ProfileRecord> recs = group;
    for (auto& r : recs) {
        r.macro_id = 0;
        r.w = 1;
        r.l = 1;
    }
    const size_t n = recs.size();
    std::vector<int64_t> g(n), l(n, 1);
    std::vector<int32_t> w(n, 1), ma(n, 0), mi(n);
    std::vector<double> t(n);
    for (size_t i = 0; i < n; ++i) {
        g[i] = recs[i].g;
        mi[i] = recs[i].micro_id;
        t[i] = recs[i].latency_us;
    }
    wt_records_desc rd{int64_t(n), g.data(), l.data(), w.data(), ma.data(), mi.data(), t.data()};
    wt_build* b = nullptr;
    wt_build_result R{};
    int dev = 0;
    cudaGetDevice(&dev);
    const int32_t id0 = 0;
    ok(wt_fit_build(&rd, &id0, 1, 1, 10, dev, &b, &R));
    std::unique_ptr<wt_build, wt_status (*)(wt_build*)> guard(b, wt_build_free);
    SharedMicroSelection s;
    s.micro_id = R.anchor_micro[0];
    s.partial_coverage = R.anchor_partial[0] != 0;
    std::map<i64, double> per_g;
    for (const auto& r : group)
        if (r.micro_id == s.micro_id) per_g[r.g] = r.latency_us;
    s.samples.assign(per_g.begin(), per_g.end());
    return s;
}

ExtrapolationFit fit_extrapolation(const std::vector<ProfileRecord>& records, int W, int p) {
    if (records.empty()) throw std::invalid_argument("fit_extrapolation: no records");
    const int id = records.front().macro_id;
    std::vector<ProfileRecord> mine;
    for (const auto& r : records)
        if (r.macro_id == id) mine.push_back(r);
    auto tables = device_build(mine, {id}, "", W, p);
    ExtrapolationFit e;
    e.theta_ext = tables.at(0).theta_ext;
    e.ext_anchors = tables.at(0).ext_anchors;
    e.flags = tables.at(0).ext_flags;
    return e;
}

std::vector<DualTable> build_dual_table(const std::vector<ProfileRecord>& records, const ConfigRegistry& registry,
                                        const HardwareSpec& hw, const TableBuildParams& params) {
    if (records.empty()) throw std::invalid_argument("build_dual_table: empty record set");
    std::vector<int> ids;
    for (const auto& m : registry.macros) ids.push_back(m.id);
    auto tables = device_build(records, ids, hw.name, params.W, params.p);
    std::set<int> built;
    for (const auto& t : tables) built.insert(t.macro_id);
    for (int id : ids)
        if (!built.count(id)) std::cerr << "fit: macro " << id << " has no records, omitted\n";
    if (tables.empty()) throw std::runtime_error("build_dual_table: no macro produced a table");
    return tables;
}

// ------------------------------------------------------------- artefacts
namespace {
std::string hexf(double v) {
    char b[48];
    std::snprintf(b, sizeof b, "%a", v);
    return b;
}
double unhexf(const json& j, const char* field) {
    if (!j.is_string())
        throw std::runtime_error(std::string("table artifact field '") + field + "' must be a hex-float string");
    const std::string& s = j.get_ref<const std::string&>();
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end != '\0')
        throw std::runtime_error(std::string("malformed float in field '") + field + "': " + s);
    return v;
}
json coeff_json(const BilinearCoeffs& c) {
    return json::array({hexf(c.alpha), hexf(c.beta), hexf(c.gamma), hexf(c.delta)});
}
BilinearCoeffs coeff_from(const json& j, const char* field) {
    if (!j.is_array() || j.size() != 4)
        throw std::runtime_error(std::string("field '") + field + "' must be a 4-element coefficient array");
    return {unhexf(j[0], field), unhexf(j[1], field), unhexf(j[2], field), unhexf(j[3], field)};
}
}  // namespace

void save_tables(const TableArtifact& artifact, const std::string& path) {
    json j;
    j["schema_version"] = 1;
    j["kernel_family"] = family_name(artifact.family);
    j["tables"] = json::array();
    for (const auto& t : artifact.tables) {
        json jt;
        jt["macro_id"] = t.macro_id;
        jt["hardware"] = t.hardware;
        jt["W"] = t.W;
        jt["p"] = t.p;
        jt["coeffs"] = json::object();
        for (const auto& [w, c] : t.coeff_table) jt["coeffs"][std::to_string(w)] = coeff_json(c);
        jt["theta_ext"] = coeff_json(t.theta_ext);
        jt["anchors"] = json::object();
        for (const auto& [w, per_l] : t.anchor_table) {
            json ja = json::object();
            for (const auto& [l, m] : per_l) ja[std::to_string(l)] = m;
            jt["anchors"][std::to_string(w)] = ja;
        }
        jt["ext_anchors"] = json::object();
        for (const auto& [l, m] : t.ext_anchors) jt["ext_anchors"][std::to_string(l)] = m;
        jt["diagnostics"] = json::object();
        for (const auto& [w, d] : t.diagnostics)
            jt["diagnostics"][std::to_string(w)] = {
                {"r2", hexf(d.r2)}, {"mape", hexf(d.mape)}, {"samples", d.samples}, {"flags", d.flags}};
        jt["ext_flags"] = t.ext_flags;
        j["tables"].push_back(jt);
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write table artifact: " + path);
    out << j.dump(2) << "\n";
}

TableArtifact load_tables(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open table artifact: " + path);
    json j;
    in >> j;
    if (!j.contains("schema_version")) throw std::runtime_error("table artifact missing 'schema_version'");
    const int v = j.at("schema_version").get<int>();
    if (v != 1)
        throw std::runtime_error("table artifact schema mismatch: expected 1, found " + std::to_string(v));
    TableArtifact a;
    a.family = family_from_name(j.at("kernel_family").get<std::string>());
    for (const auto& jt : j.at("tables")) {
        DualTable t;
        t.macro_id = jt.at("macro_id").get<int>();
        t.hardware = jt.at("hardware").get<std::string>();
        t.W = jt.at("W").get<int>();
        t.p = jt.at("p").get<int>();
        for (const auto& [w, c] : jt.at("coeffs").items()) t.coeff_table[std::stoi(w)] = coeff_from(c, "coeffs");
        t.theta_ext = coeff_from(jt.at("theta_ext"), "theta_ext");
        for (const auto& [w, ja] : jt.at("anchors").items())
            for (const auto& [l, m] : ja.items()) t.anchor_table[std::stoi(w)][std::stoll(l)] = m.get<int>();
        for (const auto& [l, m] : jt.at("ext_anchors").items()) t.ext_anchors[std::stoll(l)] = m.get<int>();
        for (const auto& [w, jd] : jt.at("diagnostics").items()) {
            WaveDiagnostics d;
            d.r2 = unhexf(jd.at("r2"), "diagnostics.r2");
            d.mape = unhexf(jd.at("mape"), "diagnostics.mape");
            d.samples = jd.at("samples").get<int>();
            d.flags = jd.at("flags").get<std::vector<std::string>>();
            t.diagnostics[std::stoi(w)] = d;
        }
        t.ext_flags = jt.at("ext_flags").get<std::vector<std::string>>();
        a.tables.push_back(std::move(t));
    }
    return a;
}

// ------------------------------------------------------------------ engine
namespace {

struct Flat {  // DualTables as the C-ABI's CSR arrays
    std::vector<int32_t> macro_id, W, coeff_off{0}, coeff_w, awave_off{0}, awave_w, awave_aoff{0}, anchor_micro,
        ext_aoff{0}, ext_micro;
    std::vector<double> theta_ext, coeff_theta;
    std::vector<int64_t> anchor_l, ext_l;
    wt_tables_desc desc() const {
        return wt_tables_desc{int32_t(macro_id.size()), macro_id.data(), W.data(), theta_ext.data(),
                              coeff_off.data(), coeff_w.data(), coeff_theta.data(), awave_off.data(),
                              awave_w.data(), awave_aoff.data(), anchor_l.data(), anchor_micro.data(),
                              ext_aoff.data(), ext_l.data(), ext_micro.data()};
    }
};

Flat flatten(const std::vector<DualTable>& tables) {
    Flat f;
    for (const auto& t : tables) {
        f.macro_id.push_back(t.macro_id);
        f.W.push_back(t.W);
        for (double v : {t.theta_ext.alpha, t.theta_ext.beta, t.theta_ext.gamma, t.theta_ext.delta})
            f.theta_ext.push_back(v);
        for (const auto& [w, c] : t.coeff_table) {
            f.coeff_w.push_back(w);
            for (double v : {c.alpha, c.beta, c.gamma, c.delta}) f.coeff_theta.push_back(v);
        }
        f.coeff_off.push_back(int32_t(f.coeff_w.size()));
        for (const auto& [w, per_l] : t.anchor_table) {
            f.awave_w.push_back(w);
            for (const auto& [l, m] : per_l) {
                f.anchor_l.push_back(l);
                f.anchor_micro.push_back(m);
            }
            f.awave_aoff.push_back(int32_t(f.anchor_l.size()));
        }
        f.awave_off.push_back(int32_t(f.awave_w.size()));
        for (const auto& [l, m] : t.ext_anchors) {
            f.ext_l.push_back(l);
            f.ext_micro.push_back(m);
        }
        f.ext_aoff.push_back(int32_t(f.ext_l.size()));
    }
    // non-null pointers for empty pools
    for (auto* v : {&f.coeff_w, &f.awave_w, &f.anchor_micro, &f.ext_micro}) v->push_back(0);
    f.coeff_theta.insert(f.coeff_theta.end(), 4, 0.0);
    f.anchor_l.push_back(0);
    f.ext_l.push_back(0);
    return f;
}

}  // namespace

Engine::Engine(const std::vector<DualTable>& tables, const ConfigRegistry& registry, const HardwareSpec& hw,
               int device)
    : device_(device), family_(registry.family), hw_(hw) {
    if (tables.empty()) throw std::invalid_argument("no dual tables provided");
    Flat f = flatten(tables);
    std::vector<int32_t> ids;
    std::vector<int64_t> tm, tn, tk;
    for (const auto& m : registry.macros) {
        ids.push_back(m.id);
        if (const auto* g = std::get_if<GemmTiles>(&m.tiles)) {
            tm.push_back(g->t_m);
            tn.push_back(g->t_n);
            tk.push_back(g->t_k);
        } else {
            const auto& a = std::get<AttnTiles>(m.tiles);
            tm.push_back(a.t_q);
            tn.push_back(1);
            tk.push_back(a.t_kv);
        }
    }
    ids.push_back(0);
    tm.push_back(1);
    tn.push_back(1);
    tk.push_back(1);
    const int fam = registry.family == KernelFamily::DenseGemm ? WT_FAMILY_DENSE_GEMM
                    : registry.family == KernelFamily::GroupedGemm ? WT_FAMILY_GROUPED_GEMM
                                                                     : WT_FAMILY_FLASH_ATTENTION;
    wt_registry_desc rd{fam, int32_t(registry.macros.size()), ids.data(), tm.data(), tn.data(), tk.data()};
    wt_tables_desc td = f.desc();
    wt_hw h{hw.n_sm, hw.blocks_per_sm};
    wt_engine* e = nullptr;
    ok(wt_engine_create(&td, &rd, &h, device, &e));
    handle_ = e;
    wt_engine_info info{};
    wt_engine_info_get(e, &info);
    n_configs_ = info.n_configs;
    tables_sorted_ = tables;
    std::stable_sort(tables_sorted_.begin(), tables_sorted_.end(),
                     [](const DualTable& a, const DualTable& b) { return a.macro_id < b.macro_id; });
    for (const auto& t : tables_sorted_) macro_sorted_.push_back(t.macro_id);
}

Engine::~Engine() {
    if (handle_) wt_engine_destroy(static_cast<wt_engine*>(handle_));
}

namespace {
struct QueryOut {  // device block for one query
    int32_t macro, micro, wave, comps;
    uint32_t flags;
    int32_t pad;
    double lat, tail;
    int64_t g, l;
};
}  // namespace

Tuned Engine::tune_one(const KernelWorkload& x) const {
    auto* e = static_cast<wt_engine*>(handle_);
    cudaSetDevice(device_);
    const int C = n_configs_;
    // scratch: query (3 int32 + rows), outputs, explain arrays
    std::vector<int32_t> rows32;
    int64_t M = 1, N = 1, K = 1;
    const bool grouped = std::holds_alternative<GroupedGemm>(x);
    if (const auto* d = std::get_if<DenseGemm>(&x)) {
        if (family_ == KernelFamily::FlashAttention) throw std::invalid_argument("dense_gemm workload needs gemm tiles");
        M = d->m, N = d->n, K = d->k;
    } else if (const auto* a = std::get_if<FlashAttention>(&x)) {
        if (family_ != KernelFamily::FlashAttention)
            throw std::invalid_argument("attention workload needs attention tiles");
        M = a->s_q, N = a->n_heads, K = a->s_kv;
    } else {
        const auto& gg = std::get<GroupedGemm>(x);
        if (family_ == KernelFamily::FlashAttention)
            throw std::invalid_argument("grouped_gemm workload needs gemm tiles");
        N = gg.n, K = gg.k;
        for (i64 r : gg.group_rows) {
            if (r > INT32_MAX) throw std::invalid_argument("group row count above 2^31-1 is unsupported");
            rows32.push_back(int32_t(r));
        }
    }
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        throw std::invalid_argument("dims above 2^31-1 are outside the device path's range");
    const size_t need = 4096 + rows32.size() * 4 + size_t(C) * 40;
    char* base = static_cast<char*>(t_scratch.get(need, device_));
    int32_t* q = reinterpret_cast<int32_t*>(base);             // M, N, K
    int64_t* roff = reinterpret_cast<int64_t*>(base + 64);     // 2
    QueryOut* o = reinterpret_cast<QueryOut*>(base + 128);
    int32_t* rows = reinterpret_cast<int32_t*>(base + 4096);
    char* ex = base + 4096 + rows32.size() * 4;
    ex = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ex) + 15) & ~uintptr_t(15));
    int32_t hq[3] = {int32_t(std::max<i64>(M, INT32_MIN)), int32_t(std::max<i64>(N, INT32_MIN)),
                     int32_t(std::max<i64>(K, INT32_MIN))};
    const int64_t hro[2] = {0, int64_t(rows32.size())};
    QueryOut h{};
    if (!grouped) {  // one warp, result polled from pinned host memory
        wt_decision_one one{};
        ok(wt_tune_one(e, hq[0], hq[1], hq[2], &one));
        h.macro = one.macro_id;
        h.micro = one.micro_id;
        h.wave = one.wave;
        h.comps = one.comparisons;
        h.flags = one.flags;
        h.lat = one.latency_us;
        h.tail = one.tail_frac;
        h.g = one.g;
        h.l = one.l;
    } else {
        cu(cudaMemcpy(q, hq, sizeof hq, cudaMemcpyHostToDevice), "tune upload");
        cu(cudaMemcpy(roff, hro, sizeof hro, cudaMemcpyHostToDevice), "tune upload");
        if (!rows32.empty()) cu(cudaMemcpy(rows, rows32.data(), rows32.size() * 4, cudaMemcpyHostToDevice), "rows");
        wt_decisions d{};
        d.macro_id = &o->macro;
        d.micro_id = &o->micro;
        d.latency_us = &o->lat;
        d.g = &o->g;
        d.l = &o->l;
        d.wave = &o->wave;
        d.flags = &o->flags;
        d.comparisons = &o->comps;
        d.tail_frac = &o->tail;
        ok(wt_tune_grouped_batch(e, roff, rows, q + 1, q + 2, 1, &d, nullptr));
        cu(cudaMemcpy(&h, o, sizeof h, cudaMemcpyDeviceToHost), "tune download");
    }
    const int st = WT_FLAG_STATUS(h.flags);
    // per-table explanation (flag text, error attribution) for dense/attention
    std::vector<int64_t> eg(C), el(C);
    std::vector<int32_t> ew(C), eu(C), es(C);
    std::vector<double> elat(C);
    const bool need_explain = !grouped && (st != 0 || (h.flags & WT_FLAG_MISSING_WAVE));
    if (need_explain) {
        int64_t* dg = reinterpret_cast<int64_t*>(ex);
        int64_t* dl = dg + C;
        double* dlat = reinterpret_cast<double*>(dl + C);
        int32_t* dw = reinterpret_cast<int32_t*>(dlat + C);
        int32_t* du = dw + C;
        int32_t* ds = du + C;
        ok(wt_explain(e, M, N, K, dg, dl, dw, du, dlat, ds, nullptr));
        cu(cudaMemcpy(eg.data(), dg, C * 8, cudaMemcpyDeviceToHost), "explain");
        cu(cudaMemcpy(el.data(), dl, C * 8, cudaMemcpyDeviceToHost), "explain");
        cu(cudaMemcpy(elat.data(), dlat, C * 8, cudaMemcpyDeviceToHost), "explain");
        cu(cudaMemcpy(ew.data(), dw, C * 4, cudaMemcpyDeviceToHost), "explain");
        cu(cudaMemcpy(eu.data(), du, C * 4, cudaMemcpyDeviceToHost), "explain");
        cu(cudaMemcpy(es.data(), ds, C * 4, cudaMemcpyDeviceToHost), "explain");
    }
    if (st != 0) {
        if (st == WT_INVALID_ARGUMENT) {
            if (grouped) {
                const auto& gg = std::get<GroupedGemm>(x);
                if (gg.n < 1 || gg.k < 1) throw std::invalid_argument("grouped_gemm dims must be >= 1");
                for (i64 r : gg.group_rows)
                    if (r < 0) throw std::invalid_argument("negative group row count");
                throw std::invalid_argument("grouped_gemm maps to an empty grid");
            }
            throw std::invalid_argument(family_ == KernelFamily::FlashAttention ? "attention dims must be >= 1"
                                                                               : "dense_gemm dims must be >= 1");
        }
        if (st == WT_RUNTIME_ERROR && need_explain) {
            for (int c = 0; c < C; ++c)
                if (es[c] == WT_RUNTIME_ERROR)
                    throw std::runtime_error("dual table for macro " + std::to_string(macro_sorted_[c]) +
                                             " has no coefficient entries");
            // Stage II: the winner has no anchor map at all
            int win = -1;
            double best = INFINITY;
            for (int c = 0; c < C; ++c)
                if (elat[c] < best) {
                    best = elat[c];
                    win = c;
                }
            if (win >= 0)
                throw std::runtime_error("dual table for macro " + std::to_string(macro_sorted_[win]) +
                                         " has no anchor entries");
            throw std::runtime_error("no finite latency prediction among the dual tables");
        }
        rethrow(wt_status(st), "decision failed with status " + std::to_string(st));
    }
    Tuned t;
    t.macro_id = h.macro;
    t.micro_id = h.micro;
    t.predicted_latency_us = h.lat;
    t.g = h.g;
    t.l = h.l;
    t.regime = Regime{(h.flags & WT_FLAG_EXTRAPOLATED) != 0, h.wave};
    t.stats.model_evals = C;
    t.stats.anchor_comparisons = h.comps;
    if (h.flags & WT_FLAG_MISSING_WAVE) {
        for (int c = 0; c < C; ++c)
            if (eu[c] >= 0)
                t.flags.push_back("missing_wave_" + std::to_string(ew[c]) + "_used_" + std::to_string(eu[c]));
    }
    if (h.flags & WT_FLAG_ANCHOR_FALLBACK) {
        const int cfg = wt_engine_config_index(e, h.macro);
        int32_t fb = -1;
        wt_engine_anchor_map(e, cfg, h.wave, (h.flags & WT_FLAG_EXTRAPOLATED) ? 1 : 0, nullptr, nullptr, 0, &fb);
        t.flags.push_back("anchor_fallback_wave_" + std::to_string(fb));
    }
    return t;
}

void Engine::set_resident(int idle_us) { ok(wt_engine_set_resident(static_cast<wt_engine*>(handle_), idle_us)); }

void Engine::tune_host(const std::vector<int32_t>& M, const std::vector<int32_t>& N, const std::vector<int32_t>& K,
                       std::vector<int32_t>& macro, std::vector<int32_t>& micro, std::vector<double>& latency) const {
    const size_t n = M.size();
    if (N.size() != n || K.size() != n) throw std::invalid_argument("M, N, K must have equal length");
    macro.resize(n);
    micro.resize(n);
    latency.resize(n);
    ok(wt_decide_host_sync(static_cast<wt_engine*>(handle_), nullptr, M.data(), N.data(), K.data(), int64_t(n),
                           macro.data(), micro.data(), latency.data(), 0));
}

// ------------------------------------------------------------------ tuner
namespace {

// Engines are cached by content so repeated tune() calls on the same
// (tables, registry, hw) reuse the device image.
uint64_t fnv(uint64_t h, const void* p, size_t n) {  // FNV-style, 8 bytes per step
    const unsigned char* b = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = (h ^ w) * 0x100000001b3ULL;
        h ^= h >> 29;
    }
    for (; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
    return h;
}

uint64_t fingerprint(const std::vector<DualTable>& tables, const ConfigRegistry& reg, const HardwareSpec& hw) {
    uint64_t h = 0xcbf29ce484222325ULL;
    int dev = 0;
    cudaGetDevice(&dev);
    h = fnv(h, &dev, sizeof dev);
    h = fnv(h, &hw.n_sm, sizeof hw.n_sm);
    h = fnv(h, &hw.blocks_per_sm, sizeof hw.blocks_per_sm);
    const int fam = int(reg.family);
    h = fnv(h, &fam, sizeof fam);
    for (const auto& m : reg.macros) {
        h = fnv(h, &m.id, sizeof m.id);
        if (const auto* g = std::get_if<GemmTiles>(&m.tiles)) h = fnv(h, g, sizeof *g);
        else h = fnv(h, &std::get<AttnTiles>(m.tiles), sizeof(AttnTiles));
    }
    for (const auto& t : tables) {
        h = fnv(h, &t.macro_id, sizeof t.macro_id);
        h = fnv(h, &t.W, sizeof t.W);
        h = fnv(h, &t.theta_ext, sizeof t.theta_ext);
        for (const auto& [w, c] : t.coeff_table) {
            h = fnv(h, &w, sizeof w);
            h = fnv(h, &c, sizeof c);
        }
        const int sep = -7;
        for (const auto& [w, per_l] : t.anchor_table) {
            h = fnv(h, &w, sizeof w);
            for (const auto& [l, m] : per_l) {
                h = fnv(h, &l, sizeof l);
                h = fnv(h, &m, sizeof m);
            }
            h = fnv(h, &sep, sizeof sep);
        }
        for (const auto& [l, m] : t.ext_anchors) {
            h = fnv(h, &l, sizeof l);
            h = fnv(h, &m, sizeof m);
        }
        h = fnv(h, &sep, sizeof sep);
    }
    return h;
}

std::shared_ptr<Engine> cached_engine(const std::vector<DualTable>& tables, const ConfigRegistry& reg,
                                      const HardwareSpec& hw) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, std::shared_ptr<Engine>> cache;
    const uint64_t key = fingerprint(tables, reg, hw);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    auto e = std::make_shared<Engine>(tables, reg, hw, dev);
    // WT_RESIDENT_US=<idle us>: answer tune() from a resident polling CTA
    if (const char* r = std::getenv("WT_RESIDENT_US"); r && std::atoi(r) > 0) e->set_resident(std::atoi(r));
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 64) cache.clear();
    cache[key] = e;
    return e;
}

}  // namespace

Tuned tune(const KernelWorkload& x, const std::vector<DualTable>& tables, const ConfigRegistry& registry,
           const HardwareSpec& hw) {
    if (tables.empty()) throw std::invalid_argument("no dual tables provided");
    return cached_engine(tables, registry, hw)->tune_one(x);
}

std::pair<double, Regime> predict_latency(const DualTable& table, i64 g, i64 l, const HardwareSpec& hw,
                                          std::vector<std::string>* flags) {
    if (g < 1 || l < 1) throw std::invalid_argument("grid size and loop count must be >= 1");
    if (hw.n_sm < 1 || hw.blocks_per_sm < 1)
        throw std::invalid_argument("hardware spec must have positive capacities");
    ConfigRegistry reg;
    reg.macros.push_back(MacroConfig{table.macro_id, GemmTiles{1, 1, 1}});
    auto eng = cached_engine({table}, reg, hw);
    auto* e = static_cast<wt_engine*>(eng->handle());
    char* base = static_cast<char*>(t_scratch.get(4096, eng->device()));
    int32_t* cfg = reinterpret_cast<int32_t*>(base);
    int64_t* dg = reinterpret_cast<int64_t*>(base + 64);
    int64_t* dl = dg + 1;
    double* lat = reinterpret_cast<double*>(base + 128);
    int32_t* out4 = reinterpret_cast<int32_t*>(base + 256);  // wave, extrap, used, status
    const int32_t c0 = 0;
    cu(cudaMemcpy(cfg, &c0, 4, cudaMemcpyHostToDevice), "predict upload");
    const int64_t gl[2] = {g, l};
    cu(cudaMemcpy(dg, gl, 16, cudaMemcpyHostToDevice), "predict upload");
    ok(wt_predict_batch(e, cfg, dg, dl, 1, lat, out4, out4 + 1, out4 + 2, out4 + 3, nullptr));
    double v;
    int32_t o4[4];
    cu(cudaMemcpy(&v, lat, 8, cudaMemcpyDeviceToHost), "predict download");
    cu(cudaMemcpy(o4, out4, 16, cudaMemcpyDeviceToHost), "predict download");
    if (o4[3] == WT_RUNTIME_ERROR)
        throw std::runtime_error("dual table for macro " + std::to_string(table.macro_id) +
                                 " has no coefficient entries");
    if (o4[3] != WT_OK) rethrow(wt_status(o4[3]), "predict_latency failed");
    if (flags && o4[2] >= 0)
        flags->push_back("missing_wave_" + std::to_string(o4[0]) + "_used_" + std::to_string(o4[2]));
    return {v, Regime{o4[1] != 0, o4[0]}};
}

i64 nearest_anchor(const std::vector<i64>& sorted_anchors, i64 l, int* comparisons) {
    if (sorted_anchors.empty()) throw std::invalid_argument("nearest_anchor: empty anchor list");
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t n = sorted_anchors.size();
    char* base = static_cast<char*>(t_scratch.get(64 + 8 * n + 64, dev));
    int64_t* dl = reinterpret_cast<int64_t*>(base);
    int64_t* dout = dl + 1;
    int32_t* dc = reinterpret_cast<int32_t*>(dl + 2);
    int64_t* da = reinterpret_cast<int64_t*>(base + 64);
    cu(cudaMemcpy(da, sorted_anchors.data(), 8 * n, cudaMemcpyHostToDevice), "anchors");
    cu(cudaMemcpy(dl, &l, 8, cudaMemcpyHostToDevice), "anchor l");
    ok(wt_nearest_anchor_batch(da, int32_t(n), dl, 1, dout, dc, nullptr));
    i64 r;
    int32_t c;
    cu(cudaMemcpy(&r, dout, 8, cudaMemcpyDeviceToHost), "anchor out");
    cu(cudaMemcpy(&c, dc, 4, cudaMemcpyDeviceToHost), "anchor out");
    if (comparisons) *comparisons = c;
    return r;
}

// -------------------------------------------------------------- baselines
namespace {

BaselinePredictor device_baselines(const std::vector<ProfileRecord>& records, BaselinePredictor::Kind kind) {
    BaselinePredictor bp;
    bp.kind = kind;
    if (records.empty()) return bp;
    // every macro of the records: selected_samples() has no registry filter
    std::set<int> macros;
    for (const auto& r : records) macros.insert(r.macro_id);
    const size_t n = records.size();
    std::vector<int64_t> g(n), l(n);
    std::vector<int32_t> w(n), ma(n), mi(n);
    std::vector<double> t(n);
    for (size_t i = 0; i < n; ++i) {
        g[i] = records[i].g;
        l[i] = records[i].l;
        w[i] = records[i].w;
        ma[i] = records[i].macro_id;
        mi[i] = records[i].micro_id;
        t[i] = records[i].latency_us;
    }
    wt_records_desc rd{int64_t(n), g.data(), l.data(), w.data(), ma.data(), mi.data(), t.data()};
    std::vector<int32_t> ids(macros.begin(), macros.end());
    wt_build* b = nullptr;
    wt_build_result R{};
    int dev = 0;
    cudaGetDevice(&dev);
    ok(wt_fit_build(&rd, ids.data(), int32_t(ids.size()), 0, 10, dev, &b, &R));
    std::unique_ptr<wt_build, wt_status (*)(wt_build*)> guard(b, wt_build_free);
    for (int32_t q = 0; q < R.n_tables; ++q) {
        const int m = R.macro_id[q];
        if (kind == BaselinePredictor::Kind::Step)
            for (int32_t k = R.step_off[q]; k < R.step_off[q + 1]; ++k) bp.step.t_wave[{m, R.step_l[k]}] = R.step_t[k];
        else
            bp.linear.theta[m] = {R.lin_theta[4 * q], R.lin_theta[4 * q + 1], R.lin_theta[4 * q + 2],
                                  R.lin_theta[4 * q + 3]};
    }
    return bp;
}

// Flattened entries in the C-ABI's order (step: (macro, l); linear: macro).
struct BaselineArrays {
    int32_t kind;
    std::vector<int32_t> macro;
    std::vector<int64_t> l;
    std::vector<double> v;
};
BaselineArrays flatten(const BaselinePredictor& bp) {
    BaselineArrays a;
    a.kind = bp.kind == BaselinePredictor::Kind::Step ? WT_BASELINE_STEP : WT_BASELINE_LINEAR;
    if (a.kind == WT_BASELINE_STEP)
        for (const auto& [key, t] : bp.step.t_wave) {
            a.macro.push_back(key.first);
            a.l.push_back(key.second);
            a.v.push_back(t);
        }
    else
        for (const auto& [m, th] : bp.linear.theta) {
            a.macro.push_back(m);
            a.v.insert(a.v.end(), {th.alpha, th.beta, th.gamma, th.delta});
        }
    return a;
}

uint64_t bp_fingerprint(const BaselineArrays& a) {
    uint64_t h = fnv(0xcbf29ce484222325ULL, &a.kind, sizeof a.kind);
    h = fnv(h, a.macro.data(), a.macro.size() * 4);
    h = fnv(h, a.l.data(), a.l.size() * 8);
    return fnv(h, a.v.data(), a.v.size() * 8);
}

struct DeviceBaseline {
    std::shared_ptr<Engine> engine;  // keeps the bound engine alive
    wt_baseline* b = nullptr;
    ~DeviceBaseline() { wt_baseline_destroy(b); }
};

std::shared_ptr<DeviceBaseline> cached_baseline(const BaselinePredictor& bp, std::shared_ptr<Engine> eng) {
    static std::mutex mu;
    static std::map<std::pair<uint64_t, const void*>, std::shared_ptr<DeviceBaseline>> cache;
    const BaselineArrays a = flatten(bp);
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(bp_fingerprint(a) ^ uint64_t(dev), eng ? eng->handle() : nullptr);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    auto d = std::make_shared<DeviceBaseline>();
    d->engine = eng;
    ok(wt_baseline_create(eng ? static_cast<const wt_engine*>(eng->handle()) : nullptr, dev, a.kind, a.macro.data(),
                          a.l.data(), a.v.data(), int64_t(a.macro.size()), &d->b));
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 64) cache.clear();
    cache[key] = d;
    return d;
}

const char* baseline_name(const BaselinePredictor& bp) {
    return bp.kind == BaselinePredictor::Kind::GlobalLinear ? "linear" : "step";
}

bool has_entry(const BaselinePredictor& bp, int macro_id) {
    if (bp.kind == BaselinePredictor::Kind::GlobalLinear) return bp.linear.theta.count(macro_id) != 0;
    auto it = bp.step.t_wave.lower_bound({macro_id, std::numeric_limits<i64>::min()});
    return it != bp.step.t_wave.end() && it->first.first == macro_id;
}

}  // namespace

BaselinePredictor fit_step_baseline(const std::vector<ProfileRecord>& records) {
    return device_baselines(records, BaselinePredictor::Kind::Step);
}

BaselinePredictor fit_linear_baseline(const std::vector<ProfileRecord>& records) {
    return device_baselines(records, BaselinePredictor::Kind::GlobalLinear);
}

double baseline_predict(const BaselinePredictor& bp, int macro_id, i64 g, i64 l, const HardwareSpec& hw) {
    auto d = cached_baseline(bp, nullptr);
    int dev = 0;
    cudaGetDevice(&dev);
    char* base = static_cast<char*>(t_scratch.get(256, dev));
    int32_t* dm = reinterpret_cast<int32_t*>(base);
    int64_t* dg = reinterpret_cast<int64_t*>(base + 64);
    int64_t* dl = dg + 1;
    double* dlat = reinterpret_cast<double*>(base + 128);
    int32_t* dst = reinterpret_cast<int32_t*>(base + 192);
    const int64_t gl[2] = {g, l};
    cu(cudaMemcpy(dm, &macro_id, 4, cudaMemcpyHostToDevice), "baseline upload");
    cu(cudaMemcpy(dg, gl, 16, cudaMemcpyHostToDevice), "baseline upload");
    const wt_hw h{hw.n_sm, hw.blocks_per_sm};
    ok(wt_baseline_predict_batch(d->b, dm, dg, dl, 1, &h, dlat, dst, nullptr));
    double v;
    int32_t st;
    cu(cudaMemcpy(&v, dlat, 8, cudaMemcpyDeviceToHost), "baseline download");
    cu(cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost), "baseline download");
    if (st == WT_OUT_OF_RANGE)
        throw std::out_of_range(std::string("no ") + baseline_name(bp) + " baseline for macro " +
                                std::to_string(macro_id));
    if (st == WT_INVALID_ARGUMENT) (void)wave_count(g, hw);  // throws the reference's message
    if (st != WT_OK) rethrow(wt_status(st), "baseline_predict failed");
    return v;
}

Tuned baseline_tune(const KernelWorkload& x, const BaselinePredictor& bp, const std::vector<DualTable>& tables,
                    const ConfigRegistry& registry, const HardwareSpec& hw) {
    if (tables.empty()) throw std::invalid_argument("no dual tables provided");
    if (std::holds_alternative<GroupedGemm>(x))
        throw std::invalid_argument("baseline_tune: grouped_gemm queries are not supported by the device path");
    auto eng = cached_engine(tables, registry, hw);
    // the reference's exception order: map_workload's argument checks on the
    // first table, then baseline_predict's missing entry in ascending macro order
    i64 M, N, K;
    if (const auto* d = std::get_if<DenseGemm>(&x)) M = d->m, N = d->n, K = d->k;
    else {
        const auto& a = std::get<FlashAttention>(x);
        M = a.s_q, N = a.n_heads, K = a.s_kv;
    }
    std::vector<int> ids;
    for (const auto& t : tables) ids.push_back(t.macro_id);
    std::sort(ids.begin(), ids.end());
    (void)map_workload(x, registry.macro(ids.front()));
    for (int id : ids)
        if (!has_entry(bp, id))
            throw std::out_of_range(std::string("no ") + baseline_name(bp) + " baseline for macro " +
                                    std::to_string(id));
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        throw std::invalid_argument("dims above 2^31-1 are outside the device path's range");
    auto d = cached_baseline(bp, eng);
    auto* e = static_cast<const wt_engine*>(eng->handle());
    char* base = static_cast<char*>(t_scratch.get(4096, eng->device()));
    int32_t* q = reinterpret_cast<int32_t*>(base);
    QueryOut* o = reinterpret_cast<QueryOut*>(base + 128);
    const int32_t hq[3] = {int32_t(M), int32_t(N), int32_t(K)};
    cu(cudaMemcpy(q, hq, sizeof hq, cudaMemcpyHostToDevice), "baseline upload");
    wt_decisions dd{};
    dd.macro_id = &o->macro;
    dd.micro_id = &o->micro;
    dd.latency_us = &o->lat;
    dd.g = &o->g;
    dd.l = &o->l;
    dd.wave = &o->wave;
    dd.flags = &o->flags;
    dd.comparisons = &o->comps;
    dd.tail_frac = &o->tail;
    ok(wt_baseline_tune_batch(e, d->b, q, q + 1, q + 2, 1, &dd, nullptr));
    QueryOut h{};
    cu(cudaMemcpy(&h, o, sizeof h, cudaMemcpyDeviceToHost), "baseline download");
    const int st = WT_FLAG_STATUS(h.flags);
    if (st != 0) rethrow(wt_status(st), "baseline_tune: decision failed (no finite prediction or no anchor entries)");
    Tuned t;
    t.macro_id = h.macro;
    t.micro_id = h.micro;
    t.predicted_latency_us = h.lat;
    t.g = h.g;
    t.l = h.l;
    t.regime = Regime{(h.flags & WT_FLAG_EXTRAPOLATED) != 0, h.wave};
    t.stats.model_evals = int(tables.size());
    t.stats.anchor_comparisons = h.comps;
    if (h.flags & WT_FLAG_ANCHOR_FALLBACK) {
        const int cfg = wt_engine_config_index(e, h.macro);
        int32_t fb = -1;
        wt_engine_anchor_map(e, cfg, h.wave, (h.flags & WT_FLAG_EXTRAPOLATED) ? 1 : 0, nullptr, nullptr, 0, &fb);
        t.flags.push_back("anchor_fallback_wave_" + std::to_string(fb));
    }
    return t;
}

}  // namespace wavetune
