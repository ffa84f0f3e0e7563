// Host packing of scenarios into the device POD and assembly of per-replica results.
#include "packer.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "../common/rng.h"

namespace mgb {

ControllerConfig apply_variant(const ControllerConfig& base, const Variant& v) {
    ControllerConfig c = base;
    auto flag = [](int f, bool& dst) {
        if (f == -1) return;
        if (f != 0 && f != 1) throw ConfigError("variant flag must be -1 (keep), 0 or 1");
        dst = f != 0;
    };
    flag(v.enabled, c.enabled);
    flag(v.enable_mig, c.enable_mig);
    flag(v.enable_placement, c.enable_placement);
    flag(v.enable_guardrails, c.enable_guardrails);
    if (!std::isnan(v.sample_interval_s)) c.sample_interval_s = v.sample_interval_s;
    if (v.persistence_windows != kKeepInt) c.persistence_windows = v.persistence_windows;
    if (v.dwell_obs != kKeepInt) c.dwell_obs = v.dwell_obs;
    if (v.cooldown_obs != kKeepInt) c.cooldown_obs = v.cooldown_obs;
    if (v.validation_obs != kKeepInt) c.validation_obs = v.validation_obs;
    if (!std::isnan(v.tail_threshold_ms)) c.tail_threshold_ms = v.tail_threshold_ms;
    c.validate();
    return c;
}

namespace {

void pack_schedule(const InterferenceSchedule& s, mg::Schedule& o) {
    o.kind = s.kind == InterferenceSchedule::Kind::always ? mg::kAlways
             : s.kind == InterferenceSchedule::Kind::square_wave ? mg::kSquareWave
                                                                 : mg::kPhases;
    o.period_s = s.period_s;
    o.duty = s.duty;
    o.offset_s = s.offset_s;
    if (s.phases.size() > static_cast<size_t>(mg::kMaxPhases)) throw ConfigError("too many schedule phases for the device");
    o.n_phases = static_cast<int32_t>(s.phases.size());
    for (size_t i = 0; i < s.phases.size(); ++i) {
        o.ph_start[i] = s.phases[i].start_s;
        o.ph_end[i] = s.phases[i].end_s;
    }
}

mg::PController pack_controller(const ControllerConfig& c) {
    mg::PController p{};
    p.enabled = c.enabled;
    p.enable_mig = c.enable_mig;
    p.enable_placement = c.enable_placement;
    p.enable_guardrails = c.enable_guardrails;
    p.persistence_windows = c.persistence_windows;
    p.dwell_obs = c.dwell_obs;
    p.cooldown_obs = c.cooldown_obs;
    p.validation_obs = c.validation_obs;
    p.tail_threshold_ms = c.tail_threshold_ms;
    p.sample_interval_s = c.sample_interval_s;
    p.warmup_s = c.warmup_s;
    p.move_futility_ratio = c.move_futility_ratio;
    p.throttle_duration_s = c.throttle_duration_s;
    p.quota_duration_s = c.quota_duration_s;
    p.ema_alpha = c.ema_alpha;
    p.hysteresis_clear_ratio = c.hysteresis_clear_ratio;
    p.relax_stability_ratio = c.relax_stability_ratio;
    p.relax_score_threshold = c.relax_score_threshold;
    p.rollback_regress_ratio = c.rollback_regress_ratio;
    p.diag_pcie_util_threshold = c.diag_pcie_util_threshold;
    p.diag_host_io_threshold = c.diag_host_io_threshold;
    p.diag_sm_util_threshold = c.diag_sm_util_threshold;
    p.move_margin = c.move_margin;
    p.guardrail_io_throttle_Bps = c.guardrail_io_throttle_Bps;
    p.guardrail_mps_quota_pct = c.guardrail_mps_quota_pct;
    p.irq_lookback_s = c.irq_lookback_s;
    p.throughput_floor = c.throughput_floor;
    return p;
}

}  // namespace

Packed pack(const ScenarioSpec& spec, const std::vector<Variant>& variants, double cap_sigmas) {
    spec.validate();
    Packed P;
    mg::PScenario& S = P.scen;
    S = mg::PScenario{};
    const auto& topo = spec.topology;
    if (topo.hosts.size() > static_cast<size_t>(mg::kMaxHosts)) throw ConfigError("too many hosts for the device");
    if (spec.tenants.size() > static_cast<size_t>(mg::kMaxTenants)) throw ConfigError("too many tenants for the device (max 64)");
    if (spec.irq_bursts.size() > static_cast<size_t>(mg::kMaxIrq)) throw ConfigError("too many irq bursts for the device");
    S.n_hosts = static_cast<int32_t>(topo.hosts.size());
    S.duration_s = spec.duration_s;
    S.measure_start_s = spec.measure_start_s;
    S.fabric_redistribute = spec.fabric_redistribute;
    S.n_ticks = spec.duration_s >= 1.0 ? static_cast<int32_t>(std::floor(spec.duration_s)) : 0;

    // roots in (host, id) order
    std::map<std::pair<int, int>, int> root_index;
    for (size_t h = 0; h < topo.hosts.size(); ++h) {
        S.host_io_capacity[h] = topo.hosts[h].io_capacity_Bps;
        for (const auto& r : topo.hosts[h].pcie_roots) root_index[{static_cast<int>(h), r.id}] = 0;
    }
    if (root_index.size() > static_cast<size_t>(mg::kMaxRoots)) throw ConfigError("too many PCIe roots for the device");
    int ri = 0;
    for (auto& kv : root_index) {
        kv.second = ri;
        S.roots[ri].host = kv.first.first;
        S.roots[ri].id = kv.first.second;
        S.roots[ri].capacity = topo.pcie_root(kv.first.first, kv.first.second).capacity_Bps;
        ++ri;
    }
    S.n_roots = ri;
    // gpus in topology order
    std::map<std::pair<int, int>, int> gpu_index;
    int gi = 0;
    for (size_t h = 0; h < topo.hosts.size(); ++h) {
        for (const auto& g : topo.hosts[h].gpus) {
            if (gi >= mg::kMaxGpus) throw ConfigError("too many GPUs for the device");
            if (g.total_slices > 64) throw ConfigError("total_slices > 64 is not supported on the device");
            mg::PGpu& o = S.gpus[gi];
            o.host = static_cast<int32_t>(h);
            o.id = g.id;
            o.root = root_index.at({static_cast<int>(h), g.pcie_root_id});
            o.numa = g.numa_id;
            o.core_group = g.core_group;
            o.total_slices = g.total_slices;
            o.mig_enabled = g.mig_enabled;
            gpu_index[{static_cast<int>(h), g.id}] = gi;
            ++gi;
        }
    }
    S.n_gpus = gi;
    for (size_t b = 0; b < spec.irq_bursts.size(); ++b) {
        const auto& q = spec.irq_bursts[b];
        mg::PIrq& o = S.irq[b];
        o.host = q.host;
        o.core_group = q.core_group;
        o.extra_noise_ms = q.extra_noise_ms;
        o.lambda = q.extra_noise_ms > 0.0 ? 1.0 / q.extra_noise_ms : 0.0;
        pack_schedule(q.schedule, o.sched);
        if (q.extra_noise_ms > 0.0) P.any_irq_noise = true;
    }
    S.n_irq = static_cast<int32_t>(spec.irq_bursts.size());

    // tenants, lexicographic
    std::vector<int> order(spec.tenants.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(),
              [&](int a, int b) { return spec.tenants[a].spec.id < spec.tenants[b].spec.id; });
    std::vector<int> canon_of_file(spec.tenants.size());
    S.n_tenants = static_cast<int32_t>(order.size());
    P.cap.resize(order.size());
    P.off.resize(order.size());
    for (size_t c = 0; c < order.size(); ++c) {
        const TenantEntry& e = spec.tenants[order[c]];
        canon_of_file[order[c]] = static_cast<int>(c);
        P.tenant_ids.push_back(e.spec.id);
        const TenantSpec& t = e.spec;
        mg::PTenant& o = S.tenants[c];
        o.name_hash = mg::fnv1a(t.id.data(), t.id.size());
        o.tclass = t.tclass == TenantClass::latency_sensitive ? mg::kLatencySensitive
                   : t.tclass == TenantClass::bandwidth_heavy ? mg::kBandwidthHeavy
                                                              : mg::kComputeHeavy;
        o.host = e.placement.host;
        o.gpu = gpu_index.at({e.placement.host, e.placement.gpu});
        o.first = e.placement.slices.first;
        o.count = e.placement.slices.count;
        o.profile = mig_profile_index(e.profile_name);
        o.arrival_rate_hz = t.arrival_rate_hz;
        o.weight = t.weight;
        o.pcie_cap = t.pcie_cap_Bps;
        o.host_io = t.host_io_Bps;
        o.sm_demand = t.sm_demand;
        o.base_compute_ms = t.base_compute_ms;
        o.slo_tail_ms = t.slo_tail_ms;
        o.claim = bandwidth_claim(t);
        // ArrivalGen (workload.cpp:103-127)
        const double cv = t.arrival_cv;
        o.deterministic = cv <= 0.0;
        o.det_step = 1.0 / t.arrival_rate_hz;
        if (!o.deterministic) {
            const double shape = 1.0 / (cv * cv);
            const double scale = 1.0 / (t.arrival_rate_hz * shape);
            o.g_alpha = shape;
            o.g_beta = scale;
            o.g_malpha = shape < 1.0 ? shape + 1.0 : shape;  // random.tcc:2341
            o.g_a1 = o.g_malpha - 1.0 / 3.0;
            o.g_a2 = 1.0 / std::sqrt(9.0 * o.g_a1);
            o.g_inv_alpha = 1.0 / shape;
        }
        if (t.transfer_mix.size() > static_cast<size_t>(mg::kMaxMix)) throw ConfigError("transfer_mix too long for the device");
        o.n_mix = static_cast<int32_t>(t.transfer_mix.size());
        double acc = 0.0;
        for (size_t m = 0; m < t.transfer_mix.size(); ++m) {
            acc += t.transfer_mix[m].weight;
            o.mix_cdf[m] = acc;
            o.mix_bytes[m] = t.transfer_mix[m].bytes;
        }
        o.has_service = t.service_cv > 0.0;
        if (o.has_service) {
            const double s2 = std::log(1.0 + t.service_cv * t.service_cv);
            o.svc_sigma = std::sqrt(s2);
            o.svc_mu = -0.5 * s2;
        }
        o.has_noise = t.noise_mean_ms > 0.0;
        o.noise_lambda = o.has_noise ? 1.0 / t.noise_mean_ms : 0.0;
        pack_schedule(e.schedule, o.sched);
        if (o.sched.kind != mg::kAlways) P.any_thinned = true;
        // record capacity: mean count + cap_sigmas standard deviations of a renewal count
        const double mean = t.arrival_rate_hz * spec.duration_s;
        const double cvx = std::max(cv, 0.5);
        // (rounded to 16 records so every tenant's arrays start on a 128-byte line)
        P.cap[c] = (static_cast<int64_t>(std::ceil(mean + cap_sigmas * cvx * std::sqrt(mean) + 64.0)) + 15) / 16 * 16;
    }
    for (size_t f = 0; f < spec.tenants.size(); ++f) P.file_order.push_back(canon_of_file[f]);
    int64_t s = 0;
    for (size_t c = 0; c < P.cap.size(); ++c) {
        P.off[c] = s;
        s += P.cap[c];
    }
    P.cap_sum = s;
    std::vector<Variant> vs = variants.empty() ? std::vector<Variant>{Variant{}} : variants;
    for (const auto& v : vs) {
        const ControllerConfig cc = apply_variant(spec.controller, v);
        P.ctrl.push_back(pack_controller(cc));
        P.max_dwell = std::max(P.max_dwell, cc.dwell_obs);
        P.max_validation = std::max(P.max_validation, cc.validation_obs);
    }
    return P;
}

const char* action_kind_name(int k) {
    switch (k) {
        case mg::kActNone: return "none";
        case mg::kActIoThrottle: return "guardrail_io_throttle";
        case mg::kActMpsQuota: return "guardrail_mps_quota";
        case mg::kActExpire: return "guardrail_expire";
        case mg::kActMove: return "move";
        case mg::kActMigUp: return "mig_up";
        case mg::kActMigDown: return "mig_down";
        case mg::kActRollback: return "rollback";
    }
    return "?";
}

const char* diagnosis_name(int d) {
    switch (d) {
        case mg::kDiagNone: return "none";
        case mg::kDiagIo: return "io_pressure";
        case mg::kDiagCompute: return "compute_contention";
    }
    return "?";
}

std::string action_detail(const mg::ActionRec& r, const Packed& p) {
    char buf[160];
    const std::string target = r.target >= 0 ? p.tenant_ids[static_cast<size_t>(r.target)] : std::string();
    switch (r.kind) {
        case mg::kActIoThrottle:
            std::snprintf(buf, sizeof(buf), "%.0f MB/s", r.throttle_Bps / 1e6);
            return "throttle " + target + " to " + buf;
        case mg::kActMpsQuota:
            std::snprintf(buf, sizeof(buf), "quota %s to %.0f%%", target.c_str(), r.quota_pct);
            return buf;
        case mg::kActMove:
            std::snprintf(buf, sizeof(buf), "move to host%d gpu%d slices [%d,%d)", r.new_host, r.new_gpu_id, r.new_first,
                          r.new_end);
            return buf;
        case mg::kActMigUp:
        case mg::kActMigDown:
            std::snprintf(buf, sizeof(buf), "%s -> %s slices [%d,%d)", r.kind == mg::kActMigUp ? "grow" : "shrink",
                          mig_lattice()[static_cast<size_t>(r.new_profile)].name.c_str(), r.new_first, r.new_end);
            return buf;
        case mg::kActRollback: return "restore previous configuration";
        case mg::kActNone: return "no feasible action";
        case mg::kActExpire: return std::string("guardrail expired (") + action_kind_name(r.expire_kind) + ")";
    }
    return "";
}

RunResult assemble(const ScenarioSpec& spec, const Packed& p, const std::string& variant, uint64_t seed,
                   const mg::TenantOut* tout, const double* quant, const mg::ActionRec* acts, int n_actions,
                   const mg::PauseRec* pauses, int n_pauses, const double* backlog, uint64_t n_events) {
    RunResult r;
    r.scenario_name = spec.name;
    r.variant = variant;
    r.seed = seed;
    r.duration_s = spec.duration_s;
    r.measure_start_s = spec.measure_start_s;
    r.n_events = n_events;
    const double window_s = spec.duration_s - spec.measure_start_s;
    const int T = p.scen.n_tenants;
    for (int i = 0; i < T; ++i) {
        const auto& id = p.tenant_ids[static_cast<size_t>(i)];
        const mg::TenantOut& o = tout[i];
        TenantSummary s;
        s.id = id;
        s.completed_total = o.completed_total;
        s.completed_window = o.completed_window;
        s.slo_tail_ms = p.scen.tenants[i].slo_tail_ms;
        if (o.completed_window > 0) {
            const double n = static_cast<double>(o.completed_window);
            s.p50_ms = quant[4 * i + 0];
            s.p95_ms = quant[4 * i + 1];
            s.p99_ms = quant[4 * i + 2];
            s.p999_ms = quant[4 * i + 3];
            s.mean_ms = o.sum_total_ms / n;
            s.miss_rate = static_cast<double>(o.window_misses) / n;
            s.throughput_hz = n / window_s;
        }
        r.tenants[id] = s;
        EndState e;
        e.placement.host = o.host;
        e.placement.gpu = o.gpu_id;
        e.placement.slices.first = o.first;
        e.placement.slices.count = mig_lattice()[static_cast<size_t>(o.profile)].slices;
        e.profile = mig_lattice()[static_cast<size_t>(o.profile)].name;
        e.claim_Bps = p.scen.tenants[i].claim;
        e.cpu_pinned = o.cpu_pinned != 0;
        r.end_states[id] = e;
    }
    for (int k = 0; k < n_actions; ++k) {
        const mg::ActionRec& a = acts[k];
        ActionRecord x;
        x.seq = a.seq;
        x.t_s = a.t_s;
        x.tenant = a.tenant >= 0 ? p.tenant_ids[static_cast<size_t>(a.tenant)] : "";
        x.target = a.target >= 0 ? p.tenant_ids[static_cast<size_t>(a.target)] : "";
        x.kind = action_kind_name(a.kind);
        x.diagnosis = diagnosis_name(a.diagnosis);
        x.detail = action_detail(a, p);
        x.p99_pre_ms = a.p99_pre_ms;
        x.ema_p99_ms = a.ema_p99_ms;
        x.breach_windows = a.breach_windows;
        x.obs_since_prev = a.obs_since_prev;
        x.throttle_Bps = a.throttle_Bps;
        x.quota_pct = a.quota_pct;
        x.pause_s = a.pause_s;
        x.rolled_back_seq = a.rolled_back_seq;
        r.actions.push_back(x);
    }
    for (int k = 0; k < n_pauses; ++k) {
        PauseEvent e;
        e.t_s = pauses[k].t_s;
        e.tenant = p.tenant_ids[static_cast<size_t>(pauses[k].tenant)];
        e.kind = action_kind_name(pauses[k].kind);
        e.duration_s = pauses[k].duration_s;
        r.pauses.push_back(e);
    }
    // Stability (engine.cpp:829-861): claims per root over end states, backlog-growth test.
    for (int ri = 0; ri < p.scen.n_roots; ++ri) {
        const mg::PRoot& root = p.scen.roots[ri];
        double claims = 0.0;
        for (int i = 0; i < T; ++i) {
            const mg::TenantOut& o = tout[i];
            const GpuSpec& g = spec.topology.gpu(o.host, o.gpu_id);
            if (o.host != root.host || g.pcie_root_id != root.id) continue;
            claims += p.scen.tenants[i].claim;
        }
        char buf[160];
        if (claims >= root.capacity) {
            r.stability.analytic_oversubscribed = true;
            std::snprintf(buf, sizeof(buf), "host %d root %d: claims %.3g B/s >= capacity %.3g B/s", root.host, root.id,
                          claims, root.capacity);
            r.stability.notes.push_back(buf);
        }
        const int n = p.scen.n_ticks;
        if (n >= 10) {
            const int third = n / 3;
            const double first = backlog[2 * ri] / static_cast<double>(third);
            const double last = backlog[2 * ri + 1] / static_cast<double>(third);
            if (last > 3.0 * std::max(first, 1.0) && last > root.capacity) {
                r.stability.unbounded_growth = true;
                std::snprintf(buf, sizeof(buf), "host %d root %d: backlog grew %.3g -> %.3g bytes", root.host, root.id,
                              first, last);
                r.stability.notes.push_back(buf);
            }
        }
    }
    return r;
}

}  // namespace mgb
