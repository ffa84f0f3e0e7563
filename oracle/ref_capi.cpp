// Oracle test infrastructure -- NOT product code.
//
// A C API over the *unmodified* reference engine (compiled from /root/reference/proj/src into
// oracle/_ref/libmigsim_ref.so by oracle/Makefile).  tests/ call it through ctypes to get the
// reference's own outputs for differential parity; bench.py's `--impl reference` arm calls
// `ref_run_batch`, which reproduces the reference's replica fan-out (std::async batches of
// `jobs`, /root/reference/proj/src/harness.cpp:156-176) so the CPU baseline is the reference
// itself, timed on the box's host cores.
#include <json.hpp>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <future>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "migsim/audit.hpp"
#include "migsim/controller.hpp"
#include "migsim/engine.hpp"
#include "migsim/fabric.hpp"
#include "migsim/harness.hpp"
#include "migsim/scenario.hpp"
#include "migsim/telemetry.hpp"
#include "migsim/trace.hpp"
#include "migsim/workload.hpp"

using nlohmann::json;
using nlohmann::ordered_json;
using namespace migsim;

namespace {

thread_local std::string g_err;

char* dup_str(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

// Controller overrides for a variant: {"enabled":b, "enable_mig":b, ..., numeric keys}.
void apply_overrides(scenario::ScenarioSpec& spec, const char* overrides_json) {
    if (!overrides_json || !*overrides_json) return;
    json o = json::parse(overrides_json);
    auto& c = spec.controller;
    for (auto it = o.begin(); it != o.end(); ++it) {
        const std::string& k = it.key();
        const json& v = it.value();
        if (k == "enabled") c.enabled = v.get<bool>();
        else if (k == "enable_mig") c.enable_mig = v.get<bool>();
        else if (k == "enable_placement") c.enable_placement = v.get<bool>();
        else if (k == "enable_guardrails") c.enable_guardrails = v.get<bool>();
        else if (k == "sample_interval_s") c.sample_interval_s = v.get<double>();
        else if (k == "persistence_windows") c.persistence_windows = v.get<int>();
        else if (k == "dwell_obs") c.dwell_obs = v.get<int>();
        else if (k == "cooldown_obs") c.cooldown_obs = v.get<int>();
        else if (k == "validation_obs") c.validation_obs = v.get<int>();
        else if (k == "tail_threshold_ms") c.tail_threshold_ms = v.get<double>();
        else throw std::runtime_error("unsupported override key " + k);
    }
    spec.controller.validate();
}

ordered_json result_json(const engine::RunResult& r) {
    ordered_json j;
    j["summary"] = trace::summary_json(r);  // reference's own formatter (trace.cpp:118-189)
    ordered_json acts = ordered_json::array();
    for (const auto& a : r.actions) {
        ordered_json e = trace::action_json(a);  // trace.cpp:98-116
        // full-precision record for parity (the jsonl drops zero pause/rolled_back fields)
        e["_pause_s"] = a.pause_s;
        e["_rolled_back_seq"] = a.rolled_back_seq;
        e["_throttle_Bps"] = a.throttle_Bps;
        e["_quota_pct"] = a.quota_pct;
        acts.push_back(std::move(e));
    }
    j["actions"] = std::move(acts);
    ordered_json ps = ordered_json::array();
    for (const auto& p : r.pauses) {
        ordered_json e;
        e["t_s"] = p.t_s;
        e["tenant"] = p.tenant;
        e["kind"] = control::to_string(p.kind);
        e["duration_s"] = p.duration_s;
        ps.push_back(std::move(e));
    }
    j["pauses"] = std::move(ps);
    j["wall_s"] = r.wall_s;
    return j;
}

struct Handle {
    engine::RunResult result;
    std::vector<std::string> tenant_ids;  // lexicographic
    std::string json_text;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

// Parse a scenario (JSON from oracle/yaml_to_json.py) and return the normalised spec as JSON.
char* ref_scenario_dump(const char* scenario_json, const char* source) {
    try {
        auto spec = scenario::parse_scenario(scenario_json, source ? source : "<scenario>");
        ordered_json j;
        j["name"] = spec.name;
        j["duration_s"] = spec.duration_s;
        j["measure_start_s"] = spec.measure_start_s;
        j["fabric_redistribute"] = spec.fabric_redistribute;
        ordered_json hosts = ordered_json::array();
        for (const auto& h : spec.topology.hosts) {
            ordered_json hj;
            hj["numa_domains"] = h.numa_domains;
            hj["io_capacity_Bps"] = h.io_capacity_Bps;
            hj["irq_hot_core_groups"] = std::vector<int>(h.irq_hot_core_groups.begin(), h.irq_hot_core_groups.end());
            ordered_json roots = ordered_json::array();
            for (const auto& r : h.pcie_roots) roots.push_back({{"id", r.id}, {"capacity_Bps", r.capacity_Bps}});
            hj["pcie_roots"] = roots;
            ordered_json gpus = ordered_json::array();
            for (const auto& g : h.gpus)
                gpus.push_back({{"id", g.id}, {"pcie_root_id", g.pcie_root_id}, {"numa_id", g.numa_id},
                                {"core_group", g.core_group}, {"total_slices", g.total_slices},
                                {"mig_enabled", g.mig_enabled}});
            hj["gpus"] = gpus;
            hosts.push_back(hj);
        }
        j["hosts"] = hosts;
        auto sched = [](const workload::InterferenceSchedule& s) {
            ordered_json o;
            o["kind"] = s.kind == workload::InterferenceSchedule::Kind::always        ? "always"
                        : s.kind == workload::InterferenceSchedule::Kind::square_wave ? "square_wave"
                                                                                       : "phases";
            o["period_s"] = s.period_s;
            o["duty"] = s.duty;
            o["offset_s"] = s.offset_s;
            ordered_json ph = ordered_json::array();
            for (const auto& p : s.phases) ph.push_back({p.start_s, p.end_s});
            o["phases"] = ph;
            return o;
        };
        ordered_json ts = ordered_json::array();
        for (const auto& t : spec.tenants) {
            ordered_json tj;
            const auto& s = t.spec;
            tj["id"] = s.id;
            tj["class"] = model::to_string(s.tclass);
            tj["arrival_rate_hz"] = s.arrival_rate_hz;
            tj["arrival_cv"] = s.arrival_cv;
            ordered_json mix = ordered_json::array();
            for (const auto& m : s.transfer_mix) mix.push_back({m.bytes, m.weight});
            tj["transfer_mix"] = mix;
            tj["base_compute_ms"] = s.base_compute_ms;
            tj["service_cv"] = s.service_cv;
            tj["slo_tail_ms"] = s.slo_tail_ms;
            tj["weight"] = s.weight;
            tj["pcie_cap_Bps"] = s.pcie_cap_Bps;
            tj["host_io_Bps"] = s.host_io_Bps;
            tj["sm_demand"] = s.sm_demand;
            tj["noise_mean_ms"] = s.noise_mean_ms;
            tj["host"] = t.placement.host;
            tj["gpu"] = t.placement.gpu;
            tj["first_slice"] = t.placement.slices.first;
            tj["slice_count"] = t.placement.slices.count;
            tj["profile"] = t.profile_name;
            tj["schedule"] = sched(t.schedule);
            ts.push_back(tj);
        }
        j["tenants"] = ts;
        ordered_json irqs = ordered_json::array();
        for (const auto& b : spec.irq_bursts)
            irqs.push_back({{"host", b.host}, {"core_group", b.core_group}, {"extra_noise_ms", b.extra_noise_ms},
                            {"schedule", sched(b.schedule)}});
        j["irq_bursts"] = irqs;
        const auto& c = spec.controller;
        j["controller"] = {{"enabled", c.enabled},
                           {"enable_mig", c.enable_mig},
                           {"enable_placement", c.enable_placement},
                           {"enable_guardrails", c.enable_guardrails},
                           {"tail_threshold_ms", c.tail_threshold_ms},
                           {"persistence_windows", c.persistence_windows},
                           {"dwell_obs", c.dwell_obs},
                           {"cooldown_obs", c.cooldown_obs},
                           {"sample_interval_s", c.sample_interval_s},
                           {"warmup_s", c.warmup_s},
                           {"move_futility_ratio", c.move_futility_ratio},
                           {"throttle_duration_s", c.throttle_duration_s},
                           {"quota_duration_s", c.quota_duration_s},
                           {"ema_alpha", c.ema_alpha},
                           {"hysteresis_clear_ratio", c.hysteresis_clear_ratio},
                           {"relax_stability_ratio", c.relax_stability_ratio},
                           {"relax_score_threshold", c.relax_score_threshold},
                           {"validation_obs", c.validation_obs},
                           {"rollback_regress_ratio", c.rollback_regress_ratio},
                           {"diag_pcie_util_threshold", c.diag_pcie_util_threshold},
                           {"diag_host_io_threshold", c.diag_host_io_threshold},
                           {"diag_sm_util_threshold", c.diag_sm_util_threshold},
                           {"move_margin", c.move_margin},
                           {"admission_queue_timeout_epochs", c.admission_queue_timeout_epochs},
                           {"guardrail_io_throttle_Bps", c.guardrail_io_throttle_Bps},
                           {"guardrail_mps_quota_pct", c.guardrail_mps_quota_pct},
                           {"irq_lookback_s", c.irq_lookback_s},
                           {"throughput_floor", c.throughput_floor}};
        return dup_str(j.dump());
    } catch (const model::ConfigError& e) {
        g_err = std::string("{\"error\":\"config\",\"message\":") + json(e.what()).dump() +
                ",\"where\":" + json(e.where()).dump() + "}";
        return nullptr;
    } catch (const std::exception& e) {
        g_err = std::string("{\"error\":\"runtime\",\"message\":") + json(e.what()).dump() + "}";
        return nullptr;
    }
}

// One replica through engine::run_scenario (engine.hpp:117).
void* ref_run(const char* scenario_json, const char* overrides_json, uint64_t seed, int keep_completions) {
    try {
        auto spec = scenario::parse_scenario(scenario_json, "<scenario>");
        apply_overrides(spec, overrides_json);
        engine::RunOptions ro;
        ro.seed = seed;
        ro.write_traces = false;
        ro.keep_completions = keep_completions != 0;
        auto* h = new Handle();
        h->result = engine::run_scenario(spec, ro);
        for (const auto& [id, s] : h->result.tenants) h->tenant_ids.push_back(id);
        h->json_text = result_json(h->result).dump();
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// engine::run_scenario with files: RunOptions{seed, out_dir, write_traces} -- the reference's own
// trace/summary/actions writers (engine.cpp:279-288, 889-892; trace.cpp).  Returns 0 on success.
int ref_run_artifacts(const char* scenario_json, const char* overrides_json, uint64_t seed, const char* out_dir,
                      int write_traces) {
    try {
        auto spec = scenario::parse_scenario(scenario_json, "<scenario>");
        apply_overrides(spec, overrides_json);
        engine::RunOptions ro;
        ro.seed = seed;
        ro.out_dir = out_dir;
        ro.write_traces = write_traces != 0;
        ro.keep_completions = false;
        (void)engine::run_scenario(spec, ro);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// harness::run_plan (harness.cpp:114-216) with out_dir: experiment.json, summary.csv and the per-run
// <variant>/seed<N>/{actions.jsonl,summary.json}.  `scenario_json_path` is a scenario-v1 document
// already converted to JSON (the restated loader's input).  Returns the experiment JSON (dump(2)).
char* ref_run_plan(const char* plan, const char* scenario_json_path, int seeds, uint64_t seed_base, const char* focus,
                   const char* out_dir, int jobs) {
    try {
        harness::PlanOptions o;
        o.plan = plan;
        o.scenario_path = scenario_json_path;
        o.seeds = seeds;
        o.seed_base = seed_base;
        o.focus_tenant = focus ? focus : "";
        o.out_dir = out_dir ? out_dir : "";
        o.jobs = jobs;
        auto r = harness::run_plan(o);
        return dup_str(harness::experiment_json(r).dump(2));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// harness::render_report (harness.cpp:272-313) of an experiment.json text
char* ref_render_report(const char* experiment_json_text) {
    try {
        return dup_str(harness::render_report(nlohmann::json::parse(experiment_json_text)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Controller::admit (controller.cpp:637-692) on explicit cases: tenants in canonical (lexicographic
// id) order, states [n][T] (admitted, host, gpu id, first, count), snapshot fields [n][T] and
// irq_recent [n][H] bitmasks, request (tenant index, lattice index).  A fresh Controller per case.
// out: [n][6] ints (outcome 0/1/2, host, gpu, first, count, reason code) and score[n].
// ref_admit_repeat: the same request `repeat` times on ONE controller per case (its queue_epochs_
// carries across the calls, controller.cpp:671-691); out/score hold [n][repeat] decisions.
int ref_admit_repeat(const char* scenario_json, int n, const int32_t* tenant, const int32_t* profile,
                     const int32_t* admitted, const int32_t* host, const int32_t* gpu_id, const int32_t* first,
                     const int32_t* count, const double* pcie, const double* hio, const uint32_t* irq, int repeat,
                     int32_t* out, double* score) {
    try {
        const auto spec = scenario::parse_scenario(scenario_json, "<scenario>");
        std::vector<const scenario::TenantEntry*> canon;
        for (const auto& t : spec.tenants) canon.push_back(&t);
        std::sort(canon.begin(), canon.end(),
                  [](const scenario::TenantEntry* a, const scenario::TenantEntry* b) { return a->spec.id < b->spec.id; });
        const int T = static_cast<int>(canon.size());
        const int H = static_cast<int>(spec.topology.hosts.size());
        const auto& lattice = model::mig_lattice();
        for (int c = 0; c < n; ++c) {
            control::TenantStates states;
            control::ClusterSnapshot snap;
            for (int j = 0; j < T; ++j) {
                const int x = c * T + j;
                model::TenantState st;
                st.spec = &canon[j]->spec;
                st.placement = {host[x], gpu_id[x], {first[x], count[x]}};
                st.profile = lattice[0];
                for (const auto& p : lattice)
                    if (p.slices == count[x]) st.profile = p;
                st.status = admitted[x] ? model::TenantStatus::admitted : model::TenantStatus::queued;
                states[canon[j]->spec.id] = st;
                snap.tenant_pcie_Bps[canon[j]->spec.id] = pcie[x];
                snap.tenant_host_io_Bps[canon[j]->spec.id] = hio[x];
            }
            for (int h = 0; h < H; ++h)
                for (int g = 0; g < 32; ++g)
                    if ((irq[c * H + h] >> g) & 1u) snap.irq_recent.insert({h, g});
            control::Controller ctl(spec.controller, spec.topology);
            for (int rep = 0; rep < repeat; ++rep) {
            const int oc = c * repeat + rep;
            const auto d = ctl.admit(canon[tenant[c]]->spec, lattice[profile[c]].name, snap, states);
            int32_t* o = out + 6 * oc;
            o[0] = d.outcome == control::AdmissionOutcome::admitted ? 0
                   : d.outcome == control::AdmissionOutcome::queued ? 1 : 2;
            o[1] = o[0] == 0 ? d.placement.host : -1;
            o[2] = o[0] == 0 ? d.placement.gpu : -1;
            o[3] = o[0] == 0 ? d.placement.slices.first : -1;
            o[4] = o[0] == 0 ? d.placement.slices.count : -1;
            o[5] = o[0] == 0 ? 0
                   : d.reason.find("service rate") != std::string::npos ? 1
                   : d.reason.find("timeout") != std::string::npos ? 3 : 2;
            score[oc] = 0.0;
            if (o[0] == 0)
                score[oc] = control::placement_score(spec.topology, states, snap, canon[tenant[c]]->spec.id,
                                                     d.placement.host, d.placement.gpu).total();
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_admit(const char* scenario_json, int n, const int32_t* tenant, const int32_t* profile,
              const int32_t* admitted, const int32_t* host, const int32_t* gpu_id, const int32_t* first,
              const int32_t* count, const double* pcie, const double* hio, const uint32_t* irq, int32_t* out,
              double* score) {
    return ref_admit_repeat(scenario_json, n, tenant, profile, admitted, host, gpu_id, first, count, pcie, hio, irq, 1,
                            out, score);
}

const char* ref_result_json(void* hp) { return static_cast<Handle*>(hp)->json_text.c_str(); }

size_t ref_result_n_completions(void* hp) { return static_cast<Handle*>(hp)->result.completions.size(); }

void ref_result_completions(void* hp, int32_t* tenant, uint64_t* seq, double* arrived, double* done, double* total,
                            double* compute, double* transfer, double* noise, double* bytes) {
    auto* h = static_cast<Handle*>(hp);
    size_t i = 0;
    for (const auto& c : h->result.completions) {
        int32_t ti = -1;
        for (size_t k = 0; k < h->tenant_ids.size(); ++k)
            if (h->tenant_ids[k] == c.tenant) ti = static_cast<int32_t>(k);
        tenant[i] = ti;
        seq[i] = c.seq;
        arrived[i] = c.arrived_s;
        done[i] = c.done_s;
        total[i] = c.total_ms;
        compute[i] = c.compute_ms;
        transfer[i] = c.transfer_ms;
        noise[i] = c.noise_ms;
        bytes[i] = c.transfer_bytes;
        ++i;
    }
}

// Audit the run (audit.cpp:52-122): returns the number of issues, fills a JSON list.
int ref_result_audit(void* hp, const char* scenario_json, const char* overrides_json, char** issues_json) {
    auto* h = static_cast<Handle*>(hp);
    auto spec = scenario::parse_scenario(scenario_json, "<scenario>");
    apply_overrides(spec, overrides_json);
    auto rep = audit::audit_run(spec, h->result);
    ordered_json arr = ordered_json::array();
    for (const auto& i : rep.issues) arr.push_back({{"rule", i.rule}, {"message", i.message}});
    if (issues_json) *issues_json = dup_str(arr.dump());
    return static_cast<int>(rep.issues.size());
}

void ref_result_free(void* hp) { delete static_cast<Handle*>(hp); }

// The reference's audit::audit_run (audit.cpp:52-122) over a RunResult produced by the GPU engine:
// `gpu_result_json` is the engine's RunResult JSON (migsim_batch_run_json); the fields the audit
// reads (action kind/tenant/target/seq/obs_since_prev/guardrail values, end-state placement and
// claim) are rebuilt into an engine::RunResult.  Returns the issue count, -1 on error.
int ref_audit_gpu_result(const char* scenario_json, const char* overrides_json, const char* gpu_result_json,
                         char** issues_json) {
    try {
        auto spec = scenario::parse_scenario(scenario_json, "<scenario>");
        apply_overrides(spec, overrides_json);
        const json g = json::parse(gpu_result_json);
        engine::RunResult r;
        r.duration_s = g.at("duration_s").get<double>();
        r.measure_start_s = g.at("measure_start_s").get<double>();
        auto kind_of = [](const std::string& s) {
            for (int k = 0; k <= static_cast<int>(control::ActionKind::rollback); ++k)
                if (s == control::to_string(static_cast<control::ActionKind>(k))) return static_cast<control::ActionKind>(k);
            throw std::runtime_error("unknown action kind " + s);
        };
        for (const auto& a : g.at("actions")) {
            control::ActionRecord rec;
            rec.seq = a.at("seq").get<int>();
            rec.t_s = a.at("t_s").get<double>();
            rec.tenant = a.at("tenant").get<std::string>();
            rec.target = a.at("target").get<std::string>();
            rec.kind = kind_of(a.at("kind").get<std::string>());
            rec.obs_since_prev = a.at("obs_since_prev").get<size_t>();
            rec.throttle_Bps = a.at("throttle_Bps").get<double>();
            rec.quota_pct = a.at("quota_pct").get<double>();
            rec.pause_s = a.at("pause_s").get<double>();
            rec.rolled_back_seq = a.at("rolled_back_seq").get<int>();
            r.actions.push_back(rec);
        }
        for (const auto& [id, e] : g.at("end_states").items()) {
            engine::EndState es;
            es.placement.host = e.at("host").get<int>();
            es.placement.gpu = e.at("gpu").get<int>();
            es.placement.slices.first = e.at("first_slice").get<int>();
            es.profile = e.at("profile").get<std::string>();
            es.claim_Bps = e.at("claim_Bps").get<double>();
            es.cpu_pinned = e.at("cpu_pinned").get<bool>();
            r.end_states[id] = es;
        }
        auto rep = audit::audit_run(spec, r);
        ordered_json arr = ordered_json::array();
        for (const auto& i : rep.issues) arr.push_back({{"rule", i.rule}, {"message", i.message}});
        if (issues_json) *issues_json = dup_str(arr.dump());
        return static_cast<int>(rep.issues.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Reference replica fan-out for the CPU baseline: jobs = variants x seeds, run in std::async
// batches of `jobs` exactly like harness.cpp:156-176.  Per job writes (focus p99, focus miss,
// sum throughput, total completions).  Returns wall seconds, or -1 on error.
double ref_run_batch(const char* scenario_json, const char* const* variant_overrides, int n_variants,
                     uint64_t seed_base, int n_seeds, int jobs, const char* focus_tenant, double* out_p99,
                     double* out_miss, double* out_thr, uint64_t* out_completions) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        auto base = scenario::parse_scenario(scenario_json, "<scenario>");
        struct Job {
            scenario::ScenarioSpec spec;
            uint64_t seed;
        };
        std::vector<Job> js;
        for (int v = 0; v < n_variants; ++v) {
            auto spec = base;
            apply_overrides(spec, variant_overrides ? variant_overrides[v] : nullptr);
            for (int s = 0; s < n_seeds; ++s) js.push_back({spec, seed_base + static_cast<uint64_t>(s)});
        }
        const unsigned limit = jobs > 0 ? static_cast<unsigned>(jobs) : std::max(1u, std::thread::hardware_concurrency());
        size_t next = 0;
        while (next < js.size()) {
            const size_t batch = std::min<size_t>(limit, js.size() - next);
            std::vector<std::future<engine::RunResult>> futs;
            for (size_t i = 0; i < batch; ++i) {
                const Job& j = js[next + i];
                futs.push_back(std::async(std::launch::async, [&j]() {
                    engine::RunOptions ro;
                    ro.seed = j.seed;
                    ro.write_traces = false;
                    return engine::run_scenario(j.spec, ro);
                }));
            }
            for (size_t i = 0; i < batch; ++i) {
                auto r = futs[i].get();
                const size_t k = next + i;
                double thr = 0.0;
                uint64_t comp = 0;
                for (const auto& [id, t] : r.tenants) {
                    thr += t.throughput_hz;
                    comp += t.completed_total;
                }
                const auto it = r.tenants.find(focus_tenant ? focus_tenant : "");
                if (out_p99) out_p99[k] = it != r.tenants.end() ? it->second.p99_ms : 0.0;
                if (out_miss) out_miss[k] = it != r.tenants.end() ? it->second.miss_rate : 0.0;
                if (out_thr) out_thr[k] = thr;
                if (out_completions) out_completions[k] = comp;
            }
            next += batch;
        }
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// ---- primitive access for known-answer / restatement tests ---------------------------------

// Raw mt19937_64 outputs of make_substream (workload.cpp:42-47).
void ref_substream(uint64_t seed, const char* name, int purpose, uint64_t* out, size_t n) {
    auto g = workload::make_substream(seed, name, static_cast<workload::StreamPurpose>(purpose));
    for (size_t i = 0; i < n; ++i) out[i] = g();
}

// generate_arrivals (workload.cpp:271-282) for one tenant of a scenario; returns the count
// (or -1), writes up to `cap` records as 4 doubles {t, bytes, mult, noise}.
long ref_generate_arrivals(const char* scenario_json, const char* tenant_id, uint64_t seed, double horizon,
                           double* out, long cap) {
    try {
        auto spec = scenario::parse_scenario(scenario_json, "<scenario>");
        const auto& t = spec.tenant(tenant_id);
        auto arr = workload::generate_arrivals(t.spec, seed, horizon, t.schedule);
        const long n = static_cast<long>(arr.size());
        for (long i = 0; i < n && i < cap; ++i) {
            out[4 * i + 0] = arr[i].t_s;
            out[4 * i + 1] = arr[i].transfer_bytes;
            out[4 * i + 2] = arr[i].service_mult;
            out[4 * i + 3] = arr[i].noise_ms;
        }
        return n;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// fabric::allocate_bandwidth (fabric.cpp:31-87). caps[i] < 0 means uncapped (nullopt).
int ref_allocate_bandwidth(int n, const double* weights, const double* caps, double capacity, int water_filling,
                           double* grants, double* residual) {
    try {
        std::vector<fabric::FlowRequest> fl(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            fl[i].tenant = "f" + std::to_string(1000 + i);
            fl[i].weight = weights[i];
            if (caps[i] >= 0.0) fl[i].cap_Bps = caps[i];
        }
        auto g = fabric::allocate_bandwidth(fl, capacity, water_filling != 0);
        for (int i = 0; i < n; ++i) grants[i] = g.grants[i].bandwidth_Bps;
        *residual = g.residual_Bps;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// TailWindow push/quantile sequence (telemetry.cpp:30-56): out[i] = quantile(q) after push i.
void ref_tailwindow_run(size_t capacity, const double* xs, size_t n, double q, double* out) {
    telemetry::TailWindow w(capacity);
    for (size_t i = 0; i < n; ++i) out[i] = *telemetry::push_and_quantile(w, xs[i], q);
}

// SmoothedSignal::update sequence (telemetry.cpp:81-95): ema + state per step.
void ref_ema_run(double alpha, double trigger, double clear, const double* xs, size_t n, double* ema, int* state) {
    telemetry::SmoothedSignal s(alpha, trigger, clear);
    for (size_t i = 0; i < n; ++i) {
        ema[i] = s.update(xs[i]);
        state[i] = s.state() == telemetry::SmoothedSignal::State::triggered ? 1 : 0;
    }
}

// sample_truncated_normal (engine.cpp:33-39) draws on a fresh substream.
void ref_truncated_normal(uint64_t seed, const char* name, int purpose, double mean, double sd, double lo, double hi,
                          double* out, size_t n) {
    auto g = workload::make_substream(seed, name, static_cast<workload::StreamPurpose>(purpose));
    for (size_t i = 0; i < n; ++i) out[i] = engine::sample_truncated_normal(g, mean, sd, lo, hi);
}

// harness::confidence_interval (harness.cpp:32-43).
void ref_confidence_interval(const double* v, size_t n, double* mean, double* half) {
    std::vector<double> vals(v, v + n);
    auto ci = harness::confidence_interval(vals);
    *mean = ci.mean;
    *half = ci.half_width;
}

}  // extern "C"
