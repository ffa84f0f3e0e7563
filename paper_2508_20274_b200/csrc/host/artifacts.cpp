#include "artifacts.hpp"

#include <json.hpp>  // nlohmann 3.11.3: the reference's own serializer (number formatting, key order)

#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <numeric>
#include <stdexcept>

namespace mgb {

namespace {

using ojson = nlohmann::ordered_json;

void put_file(const std::string& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path);
    out << text;
}

ojson interval_obj(double mean, double half) {
    ojson j;
    j["mean"] = mean;
    j["half_width"] = half;
    return j;
}

// control::ActionRecord -> one actions.jsonl object, fixed key order (trace.cpp:98-116)
ojson action_obj(const ActionRecord& r) {
    ojson j;
    j["seq"] = r.seq;
    j["t_s"] = r.t_s;
    j["tenant"] = r.tenant;
    j["target"] = r.target;
    j["kind"] = r.kind;
    j["diagnosis"] = r.diagnosis;
    j["p99_pre_ms"] = r.p99_pre_ms;
    j["ema_p99_ms"] = r.ema_p99_ms;
    j["breach_windows"] = r.breach_windows;
    j["obs_since_prev"] = r.obs_since_prev;
    if (r.kind == "guardrail_io_throttle") j["throttle_Bps"] = r.throttle_Bps;
    if (r.kind == "guardrail_mps_quota") j["quota_pct"] = r.quota_pct;
    if (r.pause_s > 0.0) j["pause_s"] = r.pause_s;
    if (r.rolled_back_seq >= 0) j["rolled_back_seq"] = r.rolled_back_seq;
    if (!r.detail.empty()) j["detail"] = r.detail;
    return j;
}

}  // namespace

std::string fmt_double(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.9g", v);
    return buf;
}

// trace.cpp:118-189
std::string summary_json_text(const RunResult& r) {
    ojson j;
    j["scenario"] = r.scenario_name;
    j["seed"] = r.seed;
    j["duration_s"] = r.duration_s;
    j["measure_start_s"] = r.measure_start_s;
    ojson tenants = ojson::object();
    for (const auto& [id, s] : r.tenants) {
        ojson t;
        t["completed_total"] = s.completed_total;
        t["completed_window"] = s.completed_window;
        t["mean_ms"] = s.mean_ms;
        t["p50_ms"] = s.p50_ms;
        t["p95_ms"] = s.p95_ms;
        t["p99_ms"] = s.p99_ms;
        t["miss_rate"] = s.miss_rate;
        t["throughput_hz"] = s.throughput_hz;
        t["slo_tail_ms"] = s.slo_tail_ms;
        tenants[id] = std::move(t);
    }
    j["tenants"] = std::move(tenants);
    ojson ends = ojson::object();
    for (const auto& [id, e] : r.end_states) {
        ojson t;
        t["host"] = e.placement.host;
        t["gpu"] = e.placement.gpu;
        t["first_slice"] = e.placement.slices.first;
        t["profile"] = e.profile;
        t["claim_Bps"] = e.claim_Bps;
        t["status"] = "admitted";  // every tenant is admitted on the engine path (engine.cpp:254)
        t["cpu_pinned"] = e.cpu_pinned;
        ends[id] = std::move(t);
    }
    j["end_states"] = std::move(ends);
    std::map<std::string, std::pair<int, double>> pause_kinds;
    double pause_max = 0.0;
    for (const auto& p : r.pauses) {
        auto& agg = pause_kinds[p.kind];
        agg.first += 1;
        agg.second += p.duration_s;
        pause_max = std::max(pause_max, p.duration_s);
    }
    ojson pauses = ojson::object();
    pauses["count"] = r.pauses.size();
    pauses["max_s"] = pause_max;
    ojson by_kind = ojson::object();
    for (const auto& [kind, agg] : pause_kinds) {
        ojson k;
        k["count"] = agg.first;
        k["mean_s"] = agg.second / agg.first;
        by_kind[kind] = std::move(k);
    }
    pauses["by_kind"] = std::move(by_kind);
    j["pauses"] = std::move(pauses);
    std::map<std::string, int> action_counts;
    for (const auto& a : r.actions) action_counts[a.kind] += 1;
    ojson actions = ojson::object();
    actions["total"] = r.actions.size();
    for (const auto& [kind, n] : action_counts) actions[kind] = n;
    j["actions"] = std::move(actions);
    ojson stab;
    stab["analytic_oversubscribed"] = r.stability.analytic_oversubscribed;
    stab["unbounded_growth"] = r.stability.unbounded_growth;
    stab["notes"] = r.stability.notes;
    j["stability"] = std::move(stab);
    return j.dump(2) + "\n";
}

std::string actions_jsonl_text(const std::vector<ActionRecord>& a) {
    std::string o;
    for (const auto& r : a) o += action_obj(r).dump() + "\n";
    return o;
}

// requests.csv: completions in event order (engine.cpp:503, trace.cpp:30-50)
std::string requests_csv_text(const Packed& p, const TraceRows& t) {
    const int T = static_cast<int>(p.tenant_ids.size());
    struct Ref {
        int64_t order;
        int32_t tenant;
        int64_t k;
    };
    std::vector<Ref> refs;
    for (int i = 0; i < T; ++i)
        for (uint64_t c = 0; c < t.n_done[i]; ++c)
            refs.push_back({t.order[t.off[i] + static_cast<int64_t>(c)], i, static_cast<int64_t>(c)});
    std::sort(refs.begin(), refs.end(), [](const Ref& a, const Ref& b) { return a.order < b.order; });
    std::string o = "t_s,tenant,seq,arrived_s,total_ms,compute_ms,transfer_ms,noise_ms,transfer_bytes\n";
    o.reserve(o.size() + refs.size() * 96);
    for (const Ref& r : refs) {
        const int64_t x = t.off[r.tenant] + r.k;
        o += fmt_double(t.done[x]);
        o += ',';
        o += p.tenant_ids[r.tenant];
        o += ',';
        o += std::to_string(r.k);  // req.seq = per-tenant emitted-arrival index (engine.cpp:425)
        o += ',';
        o += fmt_double(t.arrived[x]);
        o += ',';
        o += fmt_double(t.total[x]);
        o += ',';
        o += fmt_double(t.compute[x]);
        o += ',';
        o += fmt_double(t.transfer[x]);
        o += ',';
        o += fmt_double(t.noise[x]);
        o += ',';
        o += fmt_double(t.bytes[x]);
        o += '\n';
    }
    return o;
}

// counters.csv: per tick, tenants in id order (engine.cpp:767-774, trace.cpp:52-76)
std::string counters_csv_text(const Packed& p, const TraceRows& t) {
    const int T = static_cast<int>(p.tenant_ids.size());
    std::string o = "t_s,tenant,completed,queue_len,window_p99_ms,grant_Bps,profile,host,gpu\n";
    for (int j = 0; j < t.n_ticks; ++j) {
        const std::string ts = fmt_double(static_cast<double>(j + 1));
        for (int i = 0; i < T; ++i) {
            const mg::CounterRow& c = t.counters[static_cast<size_t>(j) * T + i];
            o += ts;
            o += ',';
            o += p.tenant_ids[i];
            o += ',';
            o += std::to_string(c.completed);
            o += ',';
            o += std::to_string(c.queue_len);
            o += ',';
            o += fmt_double(c.window_p99_ms);
            o += ',';
            o += fmt_double(c.grant_Bps);
            o += ',';
            o += mig_lattice()[static_cast<size_t>(c.profile)].name;
            o += ',';
            o += std::to_string(c.host);
            o += ',';
            o += std::to_string(c.gpu_id);
            o += '\n';
        }
    }
    return o;
}

// fabric.csv: per tick, roots in (host, id) order (engine.cpp:746-765, trace.cpp:78-96)
std::string fabric_csv_text(const ScenarioSpec&, const Packed& p, const TraceRows& t) {
    const int R = p.scen.n_roots;
    std::string o = "t_s,host,root,offered_Bps,capacity_Bps,active_flows,backlog_bytes\n";
    for (int j = 0; j < t.n_ticks; ++j) {
        const std::string ts = fmt_double(static_cast<double>(j + 1));
        for (int r = 0; r < R; ++r) {
            const mg::FabricRow& f = t.fabric[static_cast<size_t>(j) * R + r];
            const mg::PRoot& root = p.scen.roots[r];
            o += ts;
            o += ',';
            o += std::to_string(root.host);
            o += ',';
            o += std::to_string(root.id);
            o += ',';
            o += fmt_double(f.offered_Bps);
            o += ',';
            o += fmt_double(root.capacity);
            o += ',';
            o += std::to_string(f.active_flows);
            o += ',';
            o += fmt_double(f.backlog_bytes);
            o += '\n';
        }
    }
    return o;
}

void put_text_file(const std::string& path, const std::string& text) { put_file(path, text); }

std::string experiment_json_text(const std::string& plan, const std::string& scenario, const std::string& focus,
                                 double wall_s, const std::vector<PlanVariantOut>& vs) {
    ojson j;
    j["plan"] = plan;
    j["scenario"] = scenario;
    j["focus_tenant"] = focus;
    j["wall_s"] = wall_s;
    const PlanVariantOut* base = nullptr;
    for (const auto& v : vs)
        if (v.name == "static") {
            base = &v;
            break;
        }
    ojson variants = ojson::array();
    for (const auto& v : vs) {
        ojson e;
        e["name"] = v.name;
        e["seeds"] = v.seeds;
        e["p99_ms"] = v.p99_ms;
        e["miss_rate"] = v.miss_rate;
        e["throughput_hz"] = v.throughput_hz;
        e["p99_ci"] = interval_obj(v.mean[0], v.half[0]);
        e["miss_ci"] = interval_obj(v.mean[1], v.half[1]);
        e["throughput_ci"] = interval_obj(v.mean[2], v.half[2]);
        if (base && v.name != "static" && base->mean[0] > 0.0) {
            e["p99_delta_pct"] = 100.0 * (v.mean[0] - base->mean[0]) / base->mean[0];
            if (base->mean[1] > 0.0) e["miss_delta_pct"] = 100.0 * (v.mean[1] - base->mean[1]) / base->mean[1];
            if (base->mean[2] > 0.0)
                e["throughput_delta_pct"] = 100.0 * (v.mean[2] - base->mean[2]) / base->mean[2];
        }
        variants.push_back(std::move(e));
    }
    j["variants"] = std::move(variants);
    return j.dump(2);
}

std::string experiment_csv_text(const std::vector<PlanVariantOut>& vs) {
    std::string out = "variant,seed,p99_ms,miss_rate,throughput_hz\n";
    char buf[160];
    for (const auto& v : vs)
        for (size_t i = 0; i < v.seeds.size(); ++i) {
            std::snprintf(buf, sizeof(buf), "%s,%llu,%.9g,%.9g,%.9g\n", v.name.c_str(),
                          static_cast<unsigned long long>(v.seeds[i]), v.p99_ms[i], v.miss_rate[i], v.throughput_hz[i]);
            out += buf;
        }
    return out;
}

std::string render_report_text(const std::string& text) {
    const nlohmann::json e = nlohmann::json::parse(text);
    std::string out = "plan: " + e.value("plan", std::string("?")) + "  scenario: " +
                      e.value("scenario", std::string("?")) + "  tenant: " + e.value("focus_tenant", std::string("?")) +
                      "\n\n";
    char line[240];
    std::snprintf(line, sizeof(line), "%-16s %7s %22s %14s %16s %12s\n", "variant", "seeds", "p99_ms (CI)", "vs static",
                  "miss_rate", "thr_hz");
    out += line;
    out += std::string(92, '-') + "\n";
    if (!e.contains("variants")) return out;
    for (const auto& v : e["variants"]) {
        const auto& p99 = v["p99_ci"];
        char ci[48];
        std::snprintf(ci, sizeof(ci), "%.2f +/- %.2f", p99["mean"].get<double>(), p99["half_width"].get<double>());
        char delta[24];
        if (v.contains("p99_delta_pct"))
            std::snprintf(delta, sizeof(delta), "%+.1f%%", v["p99_delta_pct"].get<double>());
        else
            std::snprintf(delta, sizeof(delta), "-");
        std::snprintf(line, sizeof(line), "%-16s %7zu %22s %14s %16.4f %12.2f\n", v["name"].get<std::string>().c_str(),
                      v["seeds"].size(), ci, delta, v["miss_ci"]["mean"].get<double>(),
                      v["throughput_ci"]["mean"].get<double>());
        out += line;
    }
    return out;
}

void write_run_artifacts(const std::string& out_dir, const ScenarioSpec& spec, const Packed& p, const RunResult& r,
                         const TraceRows* traces) {
    if (out_dir.empty()) return;
    std::filesystem::create_directories(out_dir);
    if (traces) {
        put_file(out_dir + "/requests.csv", requests_csv_text(p, *traces));
        put_file(out_dir + "/counters.csv", counters_csv_text(p, *traces));
        put_file(out_dir + "/fabric.csv", fabric_csv_text(spec, p, *traces));
    }
    put_file(out_dir + "/actions.jsonl", actions_jsonl_text(r.actions));
    put_file(out_dir + "/summary.json", summary_json_text(r));
}

}  // namespace mgb
