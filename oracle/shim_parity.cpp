// Oracle test infrastructure: diff of the B200 shim against the reference, in ONE process, through
// the reference's own C++ API.  engine::run_scenario / harness::run_plan resolve to the shim
// (paper_2508_20274_b200/shim/migsim_ref_shim.cpp -> C-ABI -> GPU); engine::run_scenario_cpu /
// harness::run_plan_cpu are the unmodified reference definitions (engine.cpp:898-902,
// harness.cpp:114-216) renamed by objcopy in oracle/Makefile.  Every field of RunResult
// (engine.hpp:44-113) and ExperimentResult (harness.hpp:56-76) is compared bit-for-bit.
//
//   shim_parity run  <scenario> <seed_base> <n_seeds> [keep]   all 5 ablation variants
//   shim_parity plan <plan> <scenario> <seeds>                 e1 | e2 | e3 | llm
//   shim_parity spec <scenario>                                in-memory spec edits + errors
// Prints one line per mismatch and "OK <n>" at the end; exit 0 iff no mismatch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "migsim/engine.hpp"
#include "migsim/harness.hpp"
#include "migsim/model.hpp"
#include "migsim/scenario.hpp"

namespace migsim::engine {
RunResult run_scenario_cpu(const scenario::ScenarioSpec& spec, const RunOptions& opt);
}
namespace migsim::harness {
ExperimentResult run_plan_cpu(const PlanOptions& opt);
}

using namespace migsim;

namespace {

int g_bad = 0;
long g_checked = 0;

bool same(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

template <class T>
void eq(const T& a, const T& b, const std::string& what) {
    ++g_checked;
    if (!(a == b)) {
        if (g_bad < 40) std::printf("MISMATCH %s\n", what.c_str());
        ++g_bad;
    }
}
void eqd(double a, double b, const std::string& what) {
    ++g_checked;
    if (!same(a, b)) {
        if (g_bad < 40) std::printf("MISMATCH %s: %.17g vs %.17g\n", what.c_str(), a, b);
        ++g_bad;
    }
}

void diff_run(const engine::RunResult& g, const engine::RunResult& c, const std::string& at) {
    eq(g.scenario_name, c.scenario_name, at + " scenario_name");
    eq(g.seed, c.seed, at + " seed");
    eqd(g.duration_s, c.duration_s, at + " duration_s");
    eqd(g.measure_start_s, c.measure_start_s, at + " measure_start_s");
    eq(g.tenants.size(), c.tenants.size(), at + " n_tenants");
    for (const auto& [id, s] : c.tenants) {
        auto it = g.tenants.find(id);
        if (it == g.tenants.end()) {
            eq(0, 1, at + " missing tenant " + id);
            continue;
        }
        const auto& m = it->second;
        const std::string p = at + " tenant " + id + " ";
        eq(m.id, s.id, p + "id");
        eq(m.completed_total, s.completed_total, p + "completed_total");
        eq(m.completed_window, s.completed_window, p + "completed_window");
        eqd(m.mean_ms, s.mean_ms, p + "mean_ms");
        eqd(m.p50_ms, s.p50_ms, p + "p50_ms");
        eqd(m.p95_ms, s.p95_ms, p + "p95_ms");
        eqd(m.p99_ms, s.p99_ms, p + "p99_ms");
        eqd(m.miss_rate, s.miss_rate, p + "miss_rate");
        eqd(m.throughput_hz, s.throughput_hz, p + "throughput_hz");
        eqd(m.slo_tail_ms, s.slo_tail_ms, p + "slo_tail_ms");
    }
    eq(g.end_states.size(), c.end_states.size(), at + " n_end_states");
    for (const auto& [id, e] : c.end_states) {
        auto it = g.end_states.find(id);
        if (it == g.end_states.end()) {
            eq(0, 1, at + " missing end state " + id);
            continue;
        }
        const auto& m = it->second;
        const std::string p = at + " end " + id + " ";
        eq(m.placement.host, e.placement.host, p + "host");
        eq(m.placement.gpu, e.placement.gpu, p + "gpu");
        eq(m.placement.slices.first, e.placement.slices.first, p + "first");
        eq(m.placement.slices.count, e.placement.slices.count, p + "count");
        eq(m.profile, e.profile, p + "profile");
        eqd(m.claim_Bps, e.claim_Bps, p + "claim_Bps");
        eq(static_cast<int>(m.status), static_cast<int>(e.status), p + "status");
        eq(m.cpu_pinned, e.cpu_pinned, p + "cpu_pinned");
    }
    eq(g.actions.size(), c.actions.size(), at + " n_actions");
    for (size_t k = 0; k < std::min(g.actions.size(), c.actions.size()); ++k) {
        const auto& a = g.actions[k];
        const auto& b = c.actions[k];
        const std::string p = at + " action " + std::to_string(k) + " ";
        eq(a.seq, b.seq, p + "seq");
        eqd(a.t_s, b.t_s, p + "t_s");
        eq(a.tenant, b.tenant, p + "tenant");
        eq(a.target, b.target, p + "target");
        eq(static_cast<int>(a.kind), static_cast<int>(b.kind), p + "kind");
        eq(static_cast<int>(a.diagnosis), static_cast<int>(b.diagnosis), p + "diagnosis");
        eqd(a.p99_pre_ms, b.p99_pre_ms, p + "p99_pre_ms");
        eqd(a.ema_p99_ms, b.ema_p99_ms, p + "ema_p99_ms");
        eq(a.breach_windows, b.breach_windows, p + "breach_windows");
        eq(a.obs_since_prev, b.obs_since_prev, p + "obs_since_prev");
        eqd(a.throttle_Bps, b.throttle_Bps, p + "throttle_Bps");
        eqd(a.quota_pct, b.quota_pct, p + "quota_pct");
        eq(a.detail, b.detail, p + "detail");
        eqd(a.pause_s, b.pause_s, p + "pause_s");
        eq(a.rolled_back_seq, b.rolled_back_seq, p + "rolled_back_seq");
    }
    eq(g.pauses.size(), c.pauses.size(), at + " n_pauses");
    for (size_t k = 0; k < std::min(g.pauses.size(), c.pauses.size()); ++k) {
        const std::string p = at + " pause " + std::to_string(k) + " ";
        eqd(g.pauses[k].t_s, c.pauses[k].t_s, p + "t_s");
        eq(g.pauses[k].tenant, c.pauses[k].tenant, p + "tenant");
        eq(static_cast<int>(g.pauses[k].kind), static_cast<int>(c.pauses[k].kind), p + "kind");
        eqd(g.pauses[k].duration_s, c.pauses[k].duration_s, p + "duration_s");
    }
    eq(g.stability.analytic_oversubscribed, c.stability.analytic_oversubscribed, at + " oversubscribed");
    eq(g.stability.unbounded_growth, c.stability.unbounded_growth, at + " unbounded_growth");
    eq(g.stability.notes, c.stability.notes, at + " stability notes");
    eq(g.completions.size(), c.completions.size(), at + " n_completions");
    for (size_t k = 0; k < std::min(g.completions.size(), c.completions.size()); ++k) {
        const auto& a = g.completions[k];
        const auto& b = c.completions[k];
        const std::string p = at + " completion " + std::to_string(k) + " ";
        eq(a.tenant, b.tenant, p + "tenant");
        eq(a.seq, b.seq, p + "seq");
        eqd(a.arrived_s, b.arrived_s, p + "arrived_s");
        eqd(a.done_s, b.done_s, p + "done_s");
        eqd(a.total_ms, b.total_ms, p + "total_ms");
        eqd(a.compute_ms, b.compute_ms, p + "compute_ms");
        eqd(a.transfer_ms, b.transfer_ms, p + "transfer_ms");
        eqd(a.noise_ms, b.noise_ms, p + "noise_ms");
        eqd(a.transfer_bytes, b.transfer_bytes, p + "transfer_bytes");
    }
}

void diff_interval(const harness::Interval& a, const harness::Interval& b, const std::string& at) {
    eqd(a.mean, b.mean, at + " mean");
    eqd(a.half_width, b.half_width, at + " half_width");
}

int cmd_run(const std::string& path, uint64_t seed_base, int n, bool keep) {
    const auto base = scenario::load_scenario(path);
    for (const auto& v : harness::ablation_variants()) {
        const auto spec = harness::apply_variant(base, v);
        for (int s = 0; s < n; ++s) {
            engine::RunOptions ro;
            ro.seed = seed_base + static_cast<uint64_t>(s);
            ro.write_traces = false;
            ro.keep_completions = keep;
            diff_run(engine::run_scenario(spec, ro), engine::run_scenario_cpu(spec, ro),
                     v.name + " seed " + std::to_string(ro.seed));
        }
    }
    return 0;
}

int cmd_plan(const std::string& plan, const std::string& path, int seeds) {
    harness::PlanOptions po;
    po.plan = plan;
    po.scenario_path = path;
    po.seeds = seeds;
    const auto g = harness::run_plan(po);
    const auto c = harness::run_plan_cpu(po);
    eq(g.plan, c.plan, "plan");
    eq(g.scenario_name, c.scenario_name, "scenario_name");
    eq(g.focus_tenant, c.focus_tenant, "focus_tenant");
    eq(g.variants.size(), c.variants.size(), "n_variants");
    for (size_t k = 0; k < std::min(g.variants.size(), c.variants.size()); ++k) {
        const auto& a = g.variants[k];
        const auto& b = c.variants[k];
        const std::string p = "variant " + b.variant + " ";
        eq(a.variant, b.variant, p + "name");
        eq(a.seeds, b.seeds, p + "seeds");
        eq(a.p99_ms.size(), b.p99_ms.size(), p + "n");
        for (size_t s = 0; s < std::min(a.p99_ms.size(), b.p99_ms.size()); ++s) {
            eqd(a.p99_ms[s], b.p99_ms[s], p + "p99_ms");
            eqd(a.miss_rate[s], b.miss_rate[s], p + "miss_rate");
            eqd(a.throughput_hz[s], b.throughput_hz[s], p + "throughput_hz");
        }
        diff_interval(a.p99_ci, b.p99_ci, p + "p99_ci");
        diff_interval(a.miss_ci, b.miss_ci, p + "miss_ci");
        diff_interval(a.throughput_ci, b.throughput_ci, p + "throughput_ci");
    }
    eq(g.runs.size(), c.runs.size(), "n_runs");
    for (size_t k = 0; k < std::min(g.runs.size(), c.runs.size()); ++k) diff_run(g.runs[k], c.runs[k], "run " + std::to_string(k));
    return 0;
}

// specs built / mutated in memory cross the ABI (no YAML): edited controller knobs, an edited
// tenant, and a spec the reference rejects must be rejected the same way (ConfigError)
int cmd_spec(const std::string& path) {
    auto spec = scenario::load_scenario(path);
    engine::RunOptions ro;
    ro.seed = 3;
    ro.write_traces = false;
    spec.controller.dwell_obs = 96;
    spec.controller.cooldown_obs = 40;
    spec.controller.persistence_windows = 2;
    spec.controller.validation_obs = 48;
    spec.controller.move_margin = 0.1;
    spec.controller.ema_alpha = 0.35;
    diff_run(engine::run_scenario(spec, ro), engine::run_scenario_cpu(spec, ro), "edited controller");
    spec.tenants[0].spec.arrival_rate_hz *= 1.25;
    spec.tenants[0].spec.noise_mean_ms += 0.5;
    spec.duration_s = 900;
    spec.measure_start_s = 300;
    diff_run(engine::run_scenario(spec, ro), engine::run_scenario_cpu(spec, ro), "edited tenant");
    auto bad = spec;
    bad.tenants[0].placement.slices.first = 6;  // overlaps / overflows the GPU's 7 slices
    bad.tenants[0].placement.slices.count = 4;
    std::string ge, ce;
    try {
        (void)engine::run_scenario(bad, ro);
    } catch (const model::ConfigError& e) {
        ge = "config";
    } catch (const std::exception& e) {
        ge = std::string("other: ") + e.what();
    }
    try {
        (void)engine::run_scenario_cpu(bad, ro);
    } catch (const model::ConfigError& e) {
        ce = "config";
    } catch (const std::exception& e) {
        ce = std::string("other: ") + e.what();
    }
    eq(ge, ce, "invalid spec error class (" + ge + " vs " + ce + ")");
    eq(ce, std::string("config"), "reference rejects the invalid spec");
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: shim_parity run <scenario> <seed_base> <n> [keep] | plan <plan> <scenario> <seeds> | spec <scenario>\n");
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "run" && argc >= 5)
            cmd_run(argv[2], std::stoull(argv[3]), std::stoi(argv[4]), argc > 5 && std::string(argv[5]) == "keep");
        else if (cmd == "plan" && argc >= 5)
            cmd_plan(argv[2], argv[3], std::stoi(argv[4]));
        else if (cmd == "spec")
            cmd_spec(argv[2]);
        else {
            std::fprintf(stderr, "bad arguments\n");
            return 2;
        }
    } catch (const std::exception& e) {
        std::printf("ERROR %s\n", e.what());
        return 1;
    }
    std::printf("%s %ld fields compared, %d mismatches\n", g_bad ? "FAIL" : "OK", g_checked, g_bad);
    return g_bad ? 1 : 0;
}
