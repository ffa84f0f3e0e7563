// Reference-side binding of the B200 engine: the two entry points of the reference's replica hot
// path, implemented over the C-ABI (include/migsim_b200.h).  A reference build links this TU in
// place of the CPU definitions (oracle/Makefile's `shim` target weakens exactly these two symbols
// in the unmodified engine.o / harness.o); every other reference function -- scenario loading,
// audit, trace writers, experiment_json / experiment_csv / render_report -- is the reference's own.
//
//   migsim::engine::run_scenario  /root/reference/proj/include/migsim/engine.hpp:117
//                                 (impl engine.cpp:898-902): one replica = a 1x1 GPU batch
//   migsim::harness::run_plan     /root/reference/proj/include/migsim/harness.hpp:91
//                                 (impl harness.cpp:114-216): the std::async fan-out (:156-176)
//                                 becomes ONE migsim_gpu_run_batch over variants x seeds
//
// The ScenarioSpec crosses as an in-memory descriptor (migsim_gpu_load_spec), so specs the
// caller built or mutated (apply_variant, the e3 ControllerConfig edits) need no YAML round trip.
// Results come back as the engine's RunResult JSON (17 significant digits: exact round trip) and
// are rebuilt into engine::RunResult; keep_completions uses migsim_batch_completion_records.
// Errors: ABI code 1 -> model::ConfigError (where() = "<spec>" for descriptor checks), any other
// non-zero code -> std::runtime_error.  One device handle per host thread (MIGSIM_DEVICE, default 0).
#include <json.hpp>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "migsim/controller.hpp"
#include "migsim/engine.hpp"
#include "migsim/harness.hpp"
#include "migsim/model.hpp"
#include "migsim/scenario.hpp"
#include "migsim/trace.hpp"
#include "migsim_b200.h"

using namespace migsim;

namespace {

constexpr size_t kErr = 1024;

[[noreturn]] void fail(int rc, const char* err) {
    const std::string msg = std::string("migsim-b200: ") + err;
    if (rc == MIGSIM_ERR_CONFIG) {
        // "<where>: <message>" -> ConfigError(message, where), like model.hpp:29-37
        const std::string e = err;
        const size_t colon = e.find(": ");
        if (colon != std::string::npos && e.compare(0, 1, "<") == 0) throw model::ConfigError(e.substr(colon + 2), e.substr(0, colon));
        throw model::ConfigError(e);
    }
    throw std::runtime_error(msg);
}

struct Handle {
    migsim_gpu* g = nullptr;
    Handle() {
        char err[kErr] = {0};
        const char* dev = std::getenv("MIGSIM_DEVICE");
        const int rc = migsim_gpu_open(dev ? std::atoi(dev) : 0, &g, err, sizeof(err));
        if (rc != MIGSIM_OK) fail(rc, err);
    }
    ~Handle() {
        if (g) migsim_gpu_close(g);
    }
};

migsim_gpu* gpu() {
    thread_local Handle h;  // "one handle per host thread" (migsim_b200.h)
    return h.g;
}

// ScenarioSpec -> migsim_scenario_desc.  The descriptor points into this object's storage.
class SpecDesc {
public:
    explicit SpecDesc(const scenario::ScenarioSpec& s) {
        // reserve so the pointers taken below stay valid
        hosts_.reserve(s.topology.hosts.size());
        gpus_.reserve(s.topology.hosts.size());
        roots_.reserve(s.topology.hosts.size());
        irq_hot_.reserve(s.topology.hosts.size());
        for (const auto& h : s.topology.hosts) {
            gpus_.emplace_back();
            for (const auto& g : h.gpus)
                gpus_.back().push_back({g.id, g.pcie_root_id, g.numa_id, g.core_group, g.total_slices, g.mig_enabled ? 1 : 0});
            roots_.emplace_back();
            for (const auto& r : h.pcie_roots) roots_.back().push_back({r.id, r.capacity_Bps});
            irq_hot_.emplace_back(h.irq_hot_core_groups.begin(), h.irq_hot_core_groups.end());
            migsim_host_desc hd{};
            hd.gpus = gpus_.back().data();
            hd.n_gpus = gpus_.back().size();
            hd.numa_domains = h.numa_domains;
            hd.roots = roots_.back().data();
            hd.n_roots = roots_.back().size();
            hd.irq_hot_core_groups = irq_hot_.back().data();
            hd.n_irq_hot = irq_hot_.back().size();
            hd.io_capacity_Bps = h.io_capacity_Bps;
            hosts_.push_back(hd);
        }
        const size_t n_sched = s.tenants.size() + s.irq_bursts.size();
        ph_start_.reserve(n_sched);
        ph_end_.reserve(n_sched);
        mix_b_.reserve(s.tenants.size());
        mix_w_.reserve(s.tenants.size());
        for (const auto& t : s.tenants) {
            const auto& p = t.spec;
            mix_b_.emplace_back();
            mix_w_.emplace_back();
            for (const auto& m : p.transfer_mix) {
                mix_b_.back().push_back(m.bytes);
                mix_w_.back().push_back(m.weight);
            }
            migsim_tenant_desc td{};
            td.id = p.id.c_str();
            td.tclass = static_cast<int32_t>(p.tclass);
            td.arrival_rate_hz = p.arrival_rate_hz;
            td.arrival_cv = p.arrival_cv;
            td.mix_bytes = mix_b_.back().data();
            td.mix_weight = mix_w_.back().data();
            td.n_mix = mix_b_.back().size();
            td.base_compute_ms = p.base_compute_ms;
            td.service_cv = p.service_cv;
            td.slo_tail_ms = p.slo_tail_ms;
            td.weight = p.weight;
            td.pcie_cap_Bps = p.pcie_cap_Bps;
            td.host_io_Bps = p.host_io_Bps;
            td.sm_demand = p.sm_demand;
            td.noise_mean_ms = p.noise_mean_ms;
            td.host = t.placement.host;
            td.gpu = t.placement.gpu;
            td.first_slice = t.placement.slices.first;
            td.slice_count = t.placement.slices.count;
            td.profile = t.profile_name.c_str();
            td.schedule = sched(t.schedule);
            tenants_.push_back(td);
        }
        for (const auto& b : s.irq_bursts) irqs_.push_back({b.host, b.core_group, b.extra_noise_ms, sched(b.schedule)});
        const auto& c = s.controller;
        migsim_controller_desc& o = d_.controller;
        o.enabled = c.enabled;
        o.enable_mig = c.enable_mig;
        o.enable_placement = c.enable_placement;
        o.enable_guardrails = c.enable_guardrails;
        o.tail_threshold_ms = c.tail_threshold_ms;
        o.persistence_windows = c.persistence_windows;
        o.dwell_obs = c.dwell_obs;
        o.cooldown_obs = c.cooldown_obs;
        o.sample_interval_s = c.sample_interval_s;
        o.warmup_s = c.warmup_s;
        o.move_futility_ratio = c.move_futility_ratio;
        o.throttle_duration_s = c.throttle_duration_s;
        o.quota_duration_s = c.quota_duration_s;
        o.ema_alpha = c.ema_alpha;
        o.hysteresis_clear_ratio = c.hysteresis_clear_ratio;
        o.relax_stability_ratio = c.relax_stability_ratio;
        o.relax_score_threshold = c.relax_score_threshold;
        o.validation_obs = c.validation_obs;
        o.rollback_regress_ratio = c.rollback_regress_ratio;
        o.diag_pcie_util_threshold = c.diag_pcie_util_threshold;
        o.diag_host_io_threshold = c.diag_host_io_threshold;
        o.diag_sm_util_threshold = c.diag_sm_util_threshold;
        o.move_margin = c.move_margin;
        o.admission_queue_timeout_epochs = c.admission_queue_timeout_epochs;
        o.guardrail_io_throttle_Bps = c.guardrail_io_throttle_Bps;
        o.guardrail_mps_quota_pct = c.guardrail_mps_quota_pct;
        o.irq_lookback_s = c.irq_lookback_s;
        o.throughput_floor = c.throughput_floor;
        name_ = s.name;
        d_.name = name_.c_str();
        d_.duration_s = s.duration_s;
        d_.measure_start_s = s.measure_start_s;
        d_.fabric_redistribute = s.fabric_redistribute;
        d_.hosts = hosts_.data();
        d_.n_hosts = hosts_.size();
        d_.tenants = tenants_.data();
        d_.n_tenants = tenants_.size();
        d_.irq_bursts = irqs_.data();
        d_.n_irq_bursts = irqs_.size();
    }
    const migsim_scenario_desc* get() const { return &d_; }

private:
    migsim_schedule_desc sched(const workload::InterferenceSchedule& s) {
        migsim_schedule_desc d{};
        d.kind = static_cast<int32_t>(s.kind);
        d.period_s = s.period_s;
        d.duty = s.duty;
        d.offset_s = s.offset_s;
        ph_start_.emplace_back();
        ph_end_.emplace_back();
        for (const auto& p : s.phases) {
            ph_start_.back().push_back(p.start_s);
            ph_end_.back().push_back(p.end_s);
        }
        d.phase_start_s = ph_start_.back().data();
        d.phase_end_s = ph_end_.back().data();
        d.n_phases = ph_start_.back().size();
        return d;
    }
    std::string name_;
    std::vector<std::vector<migsim_gpu_desc>> gpus_;
    std::vector<std::vector<migsim_root_desc>> roots_;
    std::vector<std::vector<int32_t>> irq_hot_;
    std::vector<migsim_host_desc> hosts_;
    std::vector<std::vector<double>> mix_b_, mix_w_, ph_start_, ph_end_;
    std::vector<migsim_tenant_desc> tenants_;
    std::vector<migsim_irq_desc> irqs_;
    migsim_scenario_desc d_{};
};

// A loaded scenario on this thread's handle, released when the scope ends.
struct Loaded {
    int32_t id = -1;
    explicit Loaded(const scenario::ScenarioSpec& s) {
        SpecDesc d(s);
        char err[kErr] = {0};
        const int rc = migsim_gpu_load_spec(gpu(), d.get(), &id, err, sizeof(err));
        if (rc != MIGSIM_OK) fail(rc, err);
    }
    ~Loaded() { migsim_gpu_release_scenario(gpu(), id); }
    std::vector<std::string> tenant_ids() const {  // canonical (lexicographic) order of the engine
        std::vector<std::string> ids;
        const int n = migsim_scenario_n_tenants(gpu(), id);
        char buf[256];
        for (int i = 0; i < n; ++i) {
            migsim_scenario_tenant_id(gpu(), id, i, buf, sizeof(buf));
            ids.emplace_back(buf);
        }
        return ids;
    }
};

struct Batch {
    migsim_batch_result* r = nullptr;
    ~Batch() {
        if (r) migsim_batch_result_free(r);
    }
};

template <class E>
E enum_from(const std::string& s, int n, const char* what) {
    for (int k = 0; k < n; ++k)
        if (s == control::to_string(static_cast<E>(k))) return static_cast<E>(k);
    throw std::runtime_error(std::string("migsim-b200: unknown ") + what + " '" + s + "'");
}

// the engine's RunResult JSON (csrc/host/result_json.cpp) -> engine::RunResult (engine.hpp:101-113)
engine::RunResult from_json(const nlohmann::json& j) {
    engine::RunResult r;
    r.scenario_name = j.at("scenario").get<std::string>();
    r.seed = j.at("seed").get<uint64_t>();
    r.duration_s = j.at("duration_s").get<double>();
    r.measure_start_s = j.at("measure_start_s").get<double>();
    for (const auto& [id, t] : j.at("tenants").items()) {
        engine::TenantSummary s;
        s.id = id;
        s.completed_total = t.at("completed_total").get<uint64_t>();
        s.completed_window = t.at("completed_window").get<uint64_t>();
        s.mean_ms = t.at("mean_ms").get<double>();
        s.p50_ms = t.at("p50_ms").get<double>();
        s.p95_ms = t.at("p95_ms").get<double>();
        s.p99_ms = t.at("p99_ms").get<double>();
        s.miss_rate = t.at("miss_rate").get<double>();
        s.throughput_hz = t.at("throughput_hz").get<double>();
        s.slo_tail_ms = t.at("slo_tail_ms").get<double>();
        r.tenants[id] = s;
    }
    for (const auto& [id, e] : j.at("end_states").items()) {
        engine::EndState s;
        s.placement.host = e.at("host").get<int>();
        s.placement.gpu = e.at("gpu").get<int>();
        s.placement.slices.first = e.at("first_slice").get<int>();
        s.placement.slices.count = e.at("slice_count").get<int>();
        s.profile = e.at("profile").get<std::string>();
        s.claim_Bps = e.at("claim_Bps").get<double>();
        s.status = model::TenantStatus::admitted;  // every tenant is admitted on the engine path (engine.cpp:254)
        s.cpu_pinned = e.at("cpu_pinned").get<bool>();
        r.end_states[id] = s;
    }
    constexpr int kKinds = static_cast<int>(control::ActionKind::rollback) + 1;
    constexpr int kDiags = static_cast<int>(control::Diagnosis::compute_contention) + 1;
    for (const auto& a : j.at("actions")) {
        control::ActionRecord x;
        x.seq = a.at("seq").get<int>();
        x.t_s = a.at("t_s").get<double>();
        x.tenant = a.at("tenant").get<std::string>();
        x.target = a.at("target").get<std::string>();
        x.kind = enum_from<control::ActionKind>(a.at("kind").get<std::string>(), kKinds, "action kind");
        x.diagnosis = enum_from<control::Diagnosis>(a.at("diagnosis").get<std::string>(), kDiags, "diagnosis");
        x.p99_pre_ms = a.at("p99_pre_ms").get<double>();
        x.ema_p99_ms = a.at("ema_p99_ms").get<double>();
        x.breach_windows = a.at("breach_windows").get<int>();
        x.obs_since_prev = a.at("obs_since_prev").get<size_t>();
        x.throttle_Bps = a.at("throttle_Bps").get<double>();
        x.quota_pct = a.at("quota_pct").get<double>();
        x.detail = a.at("detail").get<std::string>();
        x.pause_s = a.at("pause_s").get<double>();
        x.rolled_back_seq = a.at("rolled_back_seq").get<int>();
        r.actions.push_back(std::move(x));
    }
    for (const auto& p : j.at("pauses")) {
        engine::PauseEvent e;
        e.t_s = p.at("t_s").get<double>();
        e.tenant = p.at("tenant").get<std::string>();
        e.kind = enum_from<control::ActionKind>(p.at("kind").get<std::string>(), kKinds, "pause kind");
        e.duration_s = p.at("duration_s").get<double>();
        r.pauses.push_back(std::move(e));
    }
    const auto& st = j.at("stability");
    r.stability.analytic_oversubscribed = st.at("analytic_oversubscribed").get<bool>();
    r.stability.unbounded_growth = st.at("unbounded_growth").get<bool>();
    for (const auto& n : st.at("notes")) r.stability.notes.push_back(n.get<std::string>());
    return r;
}

migsim_variant keep_all(const char* name) {
    migsim_variant v{};
    v.name = name;
    v.enabled = v.enable_mig = v.enable_placement = v.enable_guardrails = -1;
    v.sample_interval_s = std::nan("");
    v.persistence_windows = v.dwell_obs = v.cooldown_obs = v.validation_obs = MIGSIM_KEEP_INT;
    return v;
}

// one batch on the GPU; runs row-major (variant-major, seed-minor), like harness.cpp:125-152
std::vector<engine::RunResult> run_batch(const Loaded& sc, const std::vector<migsim_variant>& vs,
                                         const std::vector<uint64_t>& seeds, bool keep_completions) {
    migsim_run_opts o{};
    o.keep_completions = keep_completions ? 1 : 0;
    Batch b;
    char err[kErr] = {0};
    const int rc = migsim_gpu_run_batch(gpu(), sc.id, vs.data(), vs.size(), seeds.data(), seeds.size(), &o, &b.r, err,
                                        sizeof(err));
    if (rc != MIGSIM_OK) fail(rc, err);
    const size_t n = migsim_batch_n_runs(b.r);
    std::vector<engine::RunResult> runs(n);
    const std::vector<std::string> ids = keep_completions ? sc.tenant_ids() : std::vector<std::string>{};
    for (size_t i = 0; i < n; ++i) {
        runs[i] = from_json(nlohmann::json::parse(migsim_batch_run_json(b.r, i)));
        if (keep_completions) {
            const int64_t m = migsim_batch_completion_records(b.r, i, nullptr, 0);
            std::vector<migsim_completion> recs(static_cast<size_t>(m));
            migsim_batch_completion_records(b.r, i, recs.data(), m);
            runs[i].completions.reserve(recs.size());
            for (const auto& c : recs) {
                engine::CompletionRecord x;
                x.tenant = ids.at(static_cast<size_t>(c.tenant));
                x.seq = c.seq;
                x.arrived_s = c.arrived_s;
                x.done_s = c.done_s;
                x.total_ms = c.total_ms;
                x.compute_ms = c.compute_ms;
                x.transfer_ms = c.transfer_ms;
                x.noise_ms = c.noise_ms;
                x.transfer_bytes = c.transfer_bytes;
                runs[i].completions.push_back(x);
            }
        }
    }
    return runs;
}

std::string pick_focus_tenant(const scenario::ScenarioSpec& spec) {  // harness.cpp:80-87
    const scenario::TenantEntry* best = nullptr;
    for (const auto& t : spec.tenants)
        if (!best || t.spec.slo_tail_ms < best->spec.slo_tail_ms) best = &t;
    if (!best) throw model::ConfigError("scenario has no tenants");
    return best->spec.id;
}

}  // namespace

namespace migsim::engine {

RunResult run_scenario(const scenario::ScenarioSpec& spec, const RunOptions& opt) {
    const auto wall_start = std::chrono::steady_clock::now();
    spec.validate();
    Loaded sc(spec);
    RunResult r;
    if (!opt.out_dir.empty()) {
        // the engine writes summary.json + actions.jsonl (+ requests/counters/fabric.csv with
        // write_traces) byte-identical to the reference's (engine.cpp:279-288, 889-892)
        char* js = nullptr;
        char err[kErr] = {0};
        std::filesystem::create_directories(opt.out_dir);
        const int rc = migsim_gpu_run_scenario(gpu(), sc.id, nullptr, opt.seed, opt.out_dir.c_str(),
                                               opt.write_traces ? 1 : 0, &js, err, sizeof(err));
        if (rc != MIGSIM_OK) fail(rc, err);
        const std::string text = js;
        migsim_free(js);
        r = from_json(nlohmann::json::parse(text));
        if (opt.keep_completions) r.completions = std::move(run_batch(sc, {keep_all("")}, {opt.seed}, true)[0].completions);
    } else {
        r = std::move(run_batch(sc, {keep_all("")}, {opt.seed}, opt.keep_completions)[0]);
    }
    r.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall_start).count();
    return r;
}

}  // namespace migsim::engine

namespace migsim::harness {

ExperimentResult run_plan(const PlanOptions& opt) {
    const auto wall_start = std::chrono::steady_clock::now();
    if (opt.seeds < 1) throw model::ConfigError("experiment needs at least one seed");
    scenario::ScenarioSpec base = scenario::load_scenario(opt.scenario_path);

    ExperimentResult result;
    result.plan = opt.plan;
    result.scenario_name = base.name;
    result.focus_tenant = opt.focus_tenant.empty() ? pick_focus_tenant(base) : opt.focus_tenant;
    base.tenant(result.focus_tenant);  // throws if missing

    // plan -> variants (harness.cpp:139-152); e3 points as ControllerConfig knob overrides
    std::vector<std::string> names;
    std::vector<migsim_variant> vs;
    if (opt.plan == "e1" || opt.plan == "llm" || opt.plan == "e2") {
        for (const auto& v : opt.plan == "e2" ? ablation_variants() : main_variants()) names.push_back(v.name);
        const auto grid = opt.plan == "e2" ? ablation_variants() : main_variants();
        for (size_t k = 0; k < grid.size(); ++k) {
            migsim_variant mv = keep_all(names[k].c_str());
            mv.enabled = grid[k].enabled;
            mv.enable_mig = grid[k].enable_mig;
            mv.enable_placement = grid[k].enable_placement;
            mv.enable_guardrails = grid[k].enable_guardrails;
            vs.push_back(mv);
        }
    } else if (opt.plan == "e3") {
        // sweep_points (harness.cpp:89-110): interval 1/2/5 s, persistence 2/3/5, dwell 128/256/512
        struct Point {
            std::string name;
            std::function<void(model::ControllerConfig&, migsim_variant&)> set;
        };
        std::vector<Point> pts;
        for (double dt : {1.0, 2.0, 5.0}) {
            char n[48];
            std::snprintf(n, sizeof(n), "interval=%.0fs", dt);
            pts.push_back({n, [dt](model::ControllerConfig& c, migsim_variant& v) { c.sample_interval_s = v.sample_interval_s = dt; }});
        }
        for (int y : {2, 3, 5}) {
            char n[48];
            std::snprintf(n, sizeof(n), "persistence=%d", y);
            pts.push_back({n, [y](model::ControllerConfig& c, migsim_variant& v) { c.persistence_windows = v.persistence_windows = y; }});
        }
        for (int d : {128, 256, 512}) {
            char n[48];
            std::snprintf(n, sizeof(n), "dwell=%d", d);
            pts.push_back({n, [d](model::ControllerConfig& c, migsim_variant& v) {
                               c.dwell_obs = v.dwell_obs = d;
                               c.cooldown_obs = v.cooldown_obs = d / 2;
                           }});
        }
        for (const auto& p : pts) names.push_back(p.name);
        for (size_t k = 0; k < pts.size(); ++k) {
            model::ControllerConfig c = base.controller;
            migsim_variant mv = keep_all(names[k].c_str());
            pts[k].set(c, mv);
            c.validate();  // harness.cpp:147
            vs.push_back(mv);
        }
    } else {
        throw model::ConfigError("unknown experiment plan '" + opt.plan + "'");
    }
    std::vector<uint64_t> seeds;
    for (int s = 0; s < opt.seeds; ++s) seeds.push_back(opt.seed_base + static_cast<uint64_t>(s));

    // the fan-out (harness.cpp:156-176): one GPU batch instead of std::async batches of `jobs`
    Loaded sc(base);
    std::vector<engine::RunResult> runs = run_batch(sc, vs, seeds, false);

    // per-job artifacts (harness.cpp:131-133: <out>/<variant>/seed<N>, summary + actions only)
    if (!opt.out_dir.empty()) {
        for (size_t i = 0; i < runs.size(); ++i) {
            const std::string dir = opt.out_dir + "/" + names[i / seeds.size()] + "/seed" + std::to_string(runs[i].seed);
            std::filesystem::create_directories(dir);
            trace::write_actions_jsonl(dir + "/actions.jsonl", runs[i].actions);
            trace::write_summary(dir + "/summary.json", runs[i]);
        }
    }

    // aggregate per variant in plan order (harness.cpp:178-204)
    for (size_t v = 0; v < names.size(); ++v) {
        VariantOutcome out;
        out.variant = names[v];
        for (size_t s = 0; s < seeds.size(); ++s) {
            const auto& run = runs[v * seeds.size() + s];
            const auto it = run.tenants.find(result.focus_tenant);
            if (it == run.tenants.end()) throw std::runtime_error("focus tenant missing from run summary");
            out.seeds.push_back(seeds[s]);
            out.p99_ms.push_back(it->second.p99_ms);
            out.miss_rate.push_back(it->second.miss_rate);
            double thr = 0.0;
            for (const auto& [id, t] : run.tenants) thr += t.throughput_hz;
            out.throughput_hz.push_back(thr);
        }
        out.p99_ci = confidence_interval(out.p99_ms);
        out.miss_ci = confidence_interval(out.miss_rate);
        out.throughput_ci = confidence_interval(out.throughput_hz);
        result.variants.push_back(std::move(out));
    }
    result.runs = std::move(runs);
    result.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall_start).count();

    if (!opt.out_dir.empty()) {
        std::filesystem::create_directories(opt.out_dir);
        std::ofstream jf(opt.out_dir + "/experiment.json");
        jf << experiment_json(result).dump(2) << "\n";
        std::ofstream cf(opt.out_dir + "/summary.csv");
        cf << experiment_csv(result);
    }
    return result;
}

}  // namespace migsim::harness
