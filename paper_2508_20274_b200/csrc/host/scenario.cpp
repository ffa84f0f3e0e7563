// scenario-v1 loader and model validation for the B200 engine (host side).
// Semantics follow /root/reference/proj/src/scenario.cpp:26-384 and model.cpp:57-206;
// presets follow workload.cpp:172-236.
#include "scenario.hpp"

#include <cmath>
#include <fstream>
#include <sstream>

#include "yaml_lite.hpp"

namespace mgb {

const std::vector<MigProfile>& mig_lattice() {
    static const std::vector<MigProfile> lattice = {
        {"1g.10gb", 1, 10.0}, {"2g.20gb", 2, 20.0}, {"3g.40gb", 3, 40.0}, {"4g.40gb", 4, 40.0}, {"7g.80gb", 7, 80.0},
    };
    return lattice;
}

int mig_profile_index(const std::string& name) {
    const auto& l = mig_lattice();
    for (size_t i = 0; i < l.size(); ++i)
        if (l[i].name == name) return static_cast<int>(i);
    throw ConfigError("unknown MIG profile '" + name + "'");
}

void TopologySpec::validate() const {
    if (hosts.empty()) throw ConfigError("topology has no hosts");
    for (size_t h = 0; h < hosts.size(); ++h) {
        const auto& host = hosts[h];
        if (host.pcie_roots.empty()) throw ConfigError("host " + std::to_string(h) + " has no PCIe roots");
        if (host.io_capacity_Bps <= 0.0) throw ConfigError("host " + std::to_string(h) + " has non-positive I/O capacity");
        std::set<int> roots;
        for (const auto& r : host.pcie_roots) {
            if (r.capacity_Bps <= 0.0) throw ConfigError("PCIe root " + std::to_string(r.id) + " has non-positive capacity");
            if (!roots.insert(r.id).second) throw ConfigError("duplicate PCIe root id " + std::to_string(r.id));
        }
        std::set<int> gpus;
        for (const auto& g : host.gpus) {
            if (!gpus.insert(g.id).second) throw ConfigError("duplicate GPU id " + std::to_string(g.id));
            if (!roots.count(g.pcie_root_id))
                throw ConfigError("GPU " + std::to_string(g.id) + " references unknown PCIe root " +
                                  std::to_string(g.pcie_root_id));
            if (g.numa_id < 0 || g.numa_id >= host.numa_domains)
                throw ConfigError("GPU " + std::to_string(g.id) + " references unknown NUMA domain " +
                                  std::to_string(g.numa_id));
            if (g.total_slices <= 0) throw ConfigError("GPU " + std::to_string(g.id) + " has non-positive slice count");
        }
    }
}

const GpuSpec& TopologySpec::gpu(int host, int gpu_id) const {
    if (host < 0 || host >= static_cast<int>(hosts.size())) throw std::out_of_range("host index");
    for (const auto& g : hosts[static_cast<size_t>(host)].gpus)
        if (g.id == gpu_id) return g;
    throw ConfigError("unknown GPU " + std::to_string(gpu_id) + " on host " + std::to_string(host));
}

const PcieRootSpec& TopologySpec::pcie_root(int host, int root_id) const {
    if (host < 0 || host >= static_cast<int>(hosts.size())) throw std::out_of_range("host index");
    for (const auto& r : hosts[static_cast<size_t>(host)].pcie_roots)
        if (r.id == root_id) return r;
    throw ConfigError("unknown PCIe root " + std::to_string(root_id) + " on host " + std::to_string(host));
}

const char* to_string(TenantClass c) {
    switch (c) {
        case TenantClass::latency_sensitive: return "latency_sensitive";
        case TenantClass::bandwidth_heavy: return "bandwidth_heavy";
        case TenantClass::compute_heavy: return "compute_heavy";
    }
    return "?";
}

TenantClass tenant_class_from_string(const std::string& s) {
    if (s == "latency_sensitive") return TenantClass::latency_sensitive;
    if (s == "bandwidth_heavy") return TenantClass::bandwidth_heavy;
    if (s == "compute_heavy") return TenantClass::compute_heavy;
    throw ConfigError("unknown tenant class '" + s + "'");
}

double TenantSpec::mean_transfer_bytes() const {
    double w = 0.0, acc = 0.0;
    for (const auto& e : transfer_mix) {
        w += e.weight;
        acc += e.weight * e.bytes;
    }
    return w > 0.0 ? acc / w : 0.0;
}

void TenantSpec::validate() const {
    if (id.empty()) throw ConfigError("tenant id is empty");
    if (arrival_rate_hz <= 0.0) throw ConfigError("tenant " + id + ": arrival rate must be > 0");
    if (arrival_cv < 0.0) throw ConfigError("tenant " + id + ": arrival_cv must be >= 0");
    if (base_compute_ms <= 0.0) throw ConfigError("tenant " + id + ": base_compute_ms must be > 0");
    if (service_cv < 0.0) throw ConfigError("tenant " + id + ": service_cv must be >= 0");
    if (weight <= 0.0) throw ConfigError("tenant " + id + ": weight must be > 0");
    if (pcie_cap_Bps < 0.0) throw ConfigError("tenant " + id + ": pcie_cap must be >= 0");
    if (sm_demand < 0.0 || sm_demand > 1.0) throw ConfigError("tenant " + id + ": sm_demand must be in [0,1]");
    if (noise_mean_ms < 0.0) throw ConfigError("tenant " + id + ": noise_mean_ms must be >= 0");
    double w = 0.0;
    for (const auto& e : transfer_mix) {
        if (e.bytes < 0.0) throw ConfigError("tenant " + id + ": transfer bytes must be >= 0");
        if (e.weight < 0.0) throw ConfigError("tenant " + id + ": transfer mix weight must be >= 0");
        w += e.weight;
    }
    if (!transfer_mix.empty() && w <= 0.0) throw ConfigError("tenant " + id + ": transfer mix has zero total weight");
}

void ControllerConfig::validate() const {
    if (sample_interval_s < 1.0 || sample_interval_s > 5.0) throw ConfigError("sample_interval_s must lie in [1,5]");
    if (tail_threshold_ms <= 0.0) throw ConfigError("tail_threshold_ms must be > 0");
    if (persistence_windows < 1) throw ConfigError("persistence_windows must be >= 1");
    if (dwell_obs < 1) throw ConfigError("dwell_obs must be >= 1");
    if (cooldown_obs < 0) throw ConfigError("cooldown_obs must be >= 0");
    if (ema_alpha <= 0.0 || ema_alpha > 1.0) throw ConfigError("ema_alpha must be in (0,1]");
    if (hysteresis_clear_ratio <= 0.0 || hysteresis_clear_ratio >= 1.0)
        throw ConfigError("hysteresis_clear_ratio must be in (0,1)");
    if (relax_stability_ratio <= 0.0 || relax_stability_ratio >= 1.0)
        throw ConfigError("relax_stability_ratio must be in (0,1)");
    if (validation_obs < 1) throw ConfigError("validation_obs must be >= 1");
    if (rollback_regress_ratio < 0.0) throw ConfigError("rollback_regress_ratio must be >= 0");
    if (warmup_s < 0.0) throw ConfigError("warmup_s must be >= 0");
    if (move_futility_ratio <= 0.0) throw ConfigError("move_futility_ratio must be > 0");
    if (guardrail_io_throttle_Bps < 100e6 || guardrail_io_throttle_Bps > 500e6)
        throw ConfigError("guardrail_io_throttle outside the 100-500 MB/s bounds");
    if (guardrail_mps_quota_pct < 50.0 || guardrail_mps_quota_pct > 100.0)
        throw ConfigError("guardrail_mps_quota outside the 50-100% bounds");
    if (throttle_duration_s <= 0.0 || quota_duration_s <= 0.0) throw ConfigError("guardrail durations must be > 0");
}

void InterferenceSchedule::validate() const {
    if (kind == Kind::square_wave) {
        if (period_s <= 0.0) throw ConfigError("square_wave schedule needs period > 0");
        if (duty < 0.0 || duty > 1.0) throw ConfigError("square_wave duty must lie in [0,1]");
    }
    if (kind == Kind::phases) {
        for (const auto& p : phases)
            if (p.end_s <= p.start_s) throw ConfigError("schedule phase must have end > start");
    }
}

TenantSpec workload_preset(const std::string& name) {
    TenantSpec t;
    if (name == "t1-inference") {
        t.id = "t1";
        t.tclass = TenantClass::latency_sensitive;
        t.arrival_rate_hz = 40.0;
        t.arrival_cv = 1.3;
        t.transfer_mix = {{2e6, 0.70}, {8e6, 0.25}, {24e6, 0.05}};
        t.base_compute_ms = 2.2;
        t.service_cv = 0.28;
        t.slo_tail_ms = 15.0;
        t.weight = 1.0;
        t.pcie_cap_Bps = 0.0;
        t.host_io_Bps = 20e6;
        t.sm_demand = 0.9;
        t.noise_mean_ms = 0.15;
    } else if (name == "t2-etl") {
        t.id = "t2";
        t.tclass = TenantClass::bandwidth_heavy;
        t.arrival_rate_hz = 8.0;
        t.arrival_cv = 1.0;
        t.transfer_mix = {{1.2e9, 0.85}, {2.4e9, 0.15}};
        t.base_compute_ms = 8.0;
        t.service_cv = 0.4;
        t.slo_tail_ms = 30000.0;
        t.weight = 4.0;
        t.pcie_cap_Bps = 9.5e9;
        t.host_io_Bps = 450e6;
        t.sm_demand = 0.15;
        t.noise_mean_ms = 0.0;
    } else if (name == "t3-train") {
        t.id = "t3";
        t.tclass = TenantClass::compute_heavy;
        t.arrival_rate_hz = 3.0;
        t.arrival_cv = 1.0;
        t.transfer_mix = {{4e6, 1.0}};
        t.base_compute_ms = 30.0;
        t.service_cv = 0.3;
        t.slo_tail_ms = 30000.0;
        t.weight = 1.0;
        t.pcie_cap_Bps = 1e9;
        t.host_io_Bps = 50e6;
        t.sm_demand = 0.6;
        t.noise_mean_ms = 0.0;
    } else if (name == "llm-ttft") {
        t.id = "llm";
        t.tclass = TenantClass::latency_sensitive;
        t.arrival_rate_hz = 3.0;
        t.arrival_cv = 1.2;
        t.transfer_mix = {{1e6, 0.55}, {4e6, 0.30}, {12e6, 0.15}};
        t.base_compute_ms = 52.0;
        t.service_cv = 0.35;
        t.slo_tail_ms = 200.0;
        t.weight = 1.0;
        t.pcie_cap_Bps = 0.0;
        t.host_io_Bps = 30e6;
        t.sm_demand = 0.9;
        t.noise_mean_ms = 0.5;
    } else {
        throw ConfigError("unknown workload preset '" + name + "'");
    }
    t.validate();
    return t;
}

double bandwidth_claim(const TenantSpec& spec) {
    if (spec.pcie_cap_Bps > 0.0) return spec.pcie_cap_Bps;
    return spec.arrival_rate_hz * spec.mean_transfer_bytes();
}

void ScenarioSpec::validate() const {
    if (duration_s <= 0.0) throw ConfigError("scenario duration must be > 0");
    if (measure_start_s < 0.0 || measure_start_s >= duration_s)
        throw ConfigError("measure_start_s must lie in [0, duration)");
    topology.validate();
    controller.validate();
    if (tenants.empty()) throw ConfigError("scenario has no tenants");
    std::set<std::string> ids;
    for (const auto& t : tenants) {
        t.spec.validate();
        if (!ids.insert(t.spec.id).second) throw ConfigError("duplicate tenant id '" + t.spec.id + "'");
        const auto& gpu = topology.gpu(t.placement.host, t.placement.gpu);
        const int p = mig_profile_index(t.profile_name);
        if (t.placement.slices.count != mig_lattice()[static_cast<size_t>(p)].slices)
            throw ConfigError("tenant " + t.spec.id + ": slice count disagrees with profile " + t.profile_name);
        if (gpu.mig_enabled && (t.placement.slices.first < 0 || t.placement.slices.end() > gpu.total_slices))
            throw ConfigError("tenant " + t.spec.id + ": slices outside GPU " + std::to_string(gpu.id));
    }
    for (size_t h = 0; h < topology.hosts.size(); ++h) {
        for (const auto& gpu : topology.hosts[h].gpus) {
            if (!gpu.mig_enabled) continue;
            for (size_t i = 0; i < tenants.size(); ++i) {
                const auto& a = tenants[i];
                if (a.placement.host != static_cast<int>(h) || a.placement.gpu != gpu.id) continue;
                for (size_t j = i + 1; j < tenants.size(); ++j) {
                    const auto& b = tenants[j];
                    if (b.placement.host != static_cast<int>(h) || b.placement.gpu != gpu.id) continue;
                    if (a.placement.slices.overlaps(b.placement.slices))
                        throw ConfigError("tenants " + a.spec.id + " and " + b.spec.id + " overlap on GPU " +
                                          std::to_string(gpu.id));
                }
            }
        }
    }
    for (const auto& irq : irq_bursts) {
        if (irq.host < 0 || irq.host >= static_cast<int>(topology.hosts.size()))
            throw ConfigError("irq_burst references unknown host " + std::to_string(irq.host));
        if (irq.extra_noise_ms < 0.0) throw ConfigError("irq_burst extra_noise_ms must be >= 0");
        irq.schedule.validate();
    }
}

const TenantEntry& ScenarioSpec::tenant(const std::string& id) const {
    for (const auto& t : tenants)
        if (t.spec.id == id) return t;
    throw ConfigError("unknown tenant '" + id + "'");
}

// ---------------------------------------------------------------------------------------------
namespace {

using yaml::Node;

struct Doc {
    std::string source;
    std::string at(int line) const { return source + ":" + std::to_string(line); }
    [[noreturn]] void fail(int line, const std::string& msg) const { throw ConfigError(msg, at(line)); }
};

void check_keys(const Doc& d, const Node* n, const std::string& ctx, const std::set<std::string>& allowed) {
    if (!n || n->kind != Node::kMap) d.fail(n ? n->line : 1, ctx + " must be a mapping");
    for (size_t i = 0; i < n->map.size(); ++i)
        if (!allowed.count(n->map[i].first)) d.fail(n->key_lines[i], "unknown key '" + n->map[i].first + "' in " + ctx);
}

std::string get_str(const Doc& d, const Node* n) {
    if (!n || n->kind != Node::kScalar) d.fail(n ? n->line : 1, "expected a scalar");
    return n->text;
}

// yaml-cpp convert<double>: full stream extraction, plus .inf/.nan spellings
double get_double(const Doc& d, const Node* n, const std::string& key) {
    if (!n || n->kind != Node::kScalar) d.fail(n ? n->line : 1, "value of '" + key + "' is not a number");
    const std::string& s = n->text;
    if (s == ".inf" || s == ".Inf" || s == ".INF" || s == "+.inf" || s == "+.Inf" || s == "+.INF") return HUGE_VAL;
    if (s == "-.inf" || s == "-.Inf" || s == "-.INF") return -HUGE_VAL;
    if (s == ".nan" || s == ".NaN" || s == ".NAN") return std::nan("");
    std::istringstream is(s);
    double v;
    is >> v;
    if (is.fail() || !(is >> std::ws).eof()) d.fail(n->line, "value of '" + key + "' is not a number");
    return v;
}

int get_int(const Doc& d, const Node* n, const std::string& key) {
    if (!n || n->kind != Node::kScalar) d.fail(n ? n->line : 1, "value of '" + key + "' is not an integer");
    std::istringstream is(n->text);
    is.unsetf(std::ios::dec);
    int v;
    is >> v;
    if (is.fail() || !(is >> std::ws).eof()) d.fail(n->line, "value of '" + key + "' is not an integer");
    return v;
}

bool get_bool(const Doc& d, const Node* n, const std::string& key) {
    if (n && n->kind == Node::kScalar) {
        static const std::set<std::string> yes = {"y", "Y", "yes", "Yes", "YES", "true", "True", "TRUE", "on", "On", "ON"};
        static const std::set<std::string> no = {"n", "N", "no", "No", "NO", "false", "False", "FALSE", "off", "Off", "OFF"};
        if (yes.count(n->text)) return true;
        if (no.count(n->text)) return false;
    }
    d.fail(n ? n->line : 1, "value of '" + key + "' is not a boolean");
}

InterferenceSchedule parse_schedule(const Doc& d, const Node* n) {
    check_keys(d, n, "schedule", {"kind", "period_s", "duty", "offset_s", "phases"});
    InterferenceSchedule s;
    const Node* k = n->get("kind");
    if (!k) d.fail(n->line, "schedule needs a 'kind'");
    const std::string kind = get_str(d, k);
    if (kind == "always") {
        s.kind = InterferenceSchedule::Kind::always;
    } else if (kind == "square_wave") {
        s.kind = InterferenceSchedule::Kind::square_wave;
        if (!n->get("period_s")) d.fail(n->line, "square_wave schedule needs 'period_s'");
        s.period_s = get_double(d, n->get("period_s"), "period_s");
        if (n->get("duty")) s.duty = get_double(d, n->get("duty"), "duty");
        if (n->get("offset_s")) s.offset_s = get_double(d, n->get("offset_s"), "offset_s");
    } else if (kind == "phases") {
        s.kind = InterferenceSchedule::Kind::phases;
        const Node* ph = n->get("phases");
        if (!ph || ph->kind != Node::kSeq) d.fail(n->line, "phases schedule needs a 'phases' list");
        for (const auto& p : ph->seq) {
            check_keys(d, p.get(), "phase", {"start_s", "end_s"});
            if (!p->get("start_s") || !p->get("end_s")) d.fail(p->line, "phase needs 'start_s' and 'end_s'");
            InterferenceSchedule::Phase x;
            x.start_s = get_double(d, p->get("start_s"), "start_s");
            x.end_s = get_double(d, p->get("end_s"), "end_s");
            s.phases.push_back(x);
        }
    } else {
        d.fail(k->line, "unknown schedule kind '" + kind + "'");
    }
    try {
        s.validate();
    } catch (const ConfigError& e) {
        d.fail(n->line, e.what());
    }
    return s;
}

TopologySpec parse_topology(const Doc& d, const Node* n) {
    TopologySpec topo;
    check_keys(d, n, "topology", {"hosts"});
    const Node* hs = n->get("hosts");
    if (!hs || hs->kind != Node::kSeq) d.fail(n->line, "topology needs a 'hosts' list");
    for (const auto& hp : hs->seq) {
        const Node* hn = hp.get();
        check_keys(d, hn, "host", {"numa_domains", "io_capacity_Bps", "irq_hot_core_groups", "pcie_roots", "gpus"});
        HostSpec host;
        if (hn->get("numa_domains")) host.numa_domains = get_int(d, hn->get("numa_domains"), "numa_domains");
        if (hn->get("io_capacity_Bps")) host.io_capacity_Bps = get_double(d, hn->get("io_capacity_Bps"), "io_capacity_Bps");
        if (const Node* g = hn->get("irq_hot_core_groups")) {
            for (const auto& x : g->seq) host.irq_hot_core_groups.insert(get_int(d, x.get(), "irq_hot_core_groups"));
        }
        const Node* rs = hn->get("pcie_roots");
        if (!rs || rs->kind != Node::kSeq) d.fail(hn->line, "host needs a 'pcie_roots' list");
        for (const auto& rp : rs->seq) {
            check_keys(d, rp.get(), "pcie_root", {"id", "capacity_Bps"});
            if (!rp->get("id") || !rp->get("capacity_Bps")) d.fail(rp->line, "pcie_root needs 'id' and 'capacity_Bps'");
            PcieRootSpec r;
            r.id = get_int(d, rp->get("id"), "id");
            r.capacity_Bps = get_double(d, rp->get("capacity_Bps"), "capacity_Bps");
            host.pcie_roots.push_back(r);
        }
        const Node* gs = hn->get("gpus");
        if (!gs || gs->kind != Node::kSeq) d.fail(hn->line, "host needs a 'gpus' list");
        for (const auto& gp : gs->seq) {
            check_keys(d, gp.get(), "gpu", {"id", "pcie_root_id", "numa_id", "core_group", "total_slices", "mig_enabled"});
            if (!gp->get("id") || !gp->get("pcie_root_id")) d.fail(gp->line, "gpu needs 'id' and 'pcie_root_id'");
            GpuSpec g;
            g.id = get_int(d, gp->get("id"), "id");
            g.pcie_root_id = get_int(d, gp->get("pcie_root_id"), "pcie_root_id");
            if (gp->get("numa_id")) g.numa_id = get_int(d, gp->get("numa_id"), "numa_id");
            if (gp->get("core_group")) g.core_group = get_int(d, gp->get("core_group"), "core_group");
            if (gp->get("total_slices")) g.total_slices = get_int(d, gp->get("total_slices"), "total_slices");
            if (gp->get("mig_enabled")) g.mig_enabled = get_bool(d, gp->get("mig_enabled"), "mig_enabled");
            host.gpus.push_back(g);
        }
        topo.hosts.push_back(host);
    }
    return topo;
}

void apply_tenant_overrides(const Doc& d, const Node* n, TenantSpec& t) {
    check_keys(d, n, "tenant",
               {"preset", "id", "class", "arrival_rate_hz", "arrival_cv", "transfer_mix", "base_compute_ms", "service_cv",
                "slo_tail_ms", "weight", "pcie_cap_Bps", "host_io_Bps", "sm_demand", "noise_mean_ms", "placement",
                "schedule"});
    if (n->get("id")) t.id = get_str(d, n->get("id"));
    if (const Node* c = n->get("class")) {
        try {
            t.tclass = tenant_class_from_string(get_str(d, c));
        } catch (const ConfigError& e) {
            d.fail(c->line, e.what());
        }
    }
    auto dbl = [&](const char* k, double& out) {
        if (const Node* v = n->get(k)) out = get_double(d, v, k);
    };
    dbl("arrival_rate_hz", t.arrival_rate_hz);
    dbl("arrival_cv", t.arrival_cv);
    if (const Node* m = n->get("transfer_mix")) {
        if (m->kind != Node::kSeq) d.fail(m->line, "transfer_mix must be a list");
        t.transfer_mix.clear();
        for (const auto& e : m->seq) {
            check_keys(d, e.get(), "transfer_mix entry", {"bytes", "weight"});
            if (!e->get("bytes")) d.fail(e->line, "transfer_mix entry needs 'bytes'");
            TransferMixEntry x;
            x.bytes = get_double(d, e->get("bytes"), "bytes");
            x.weight = e->get("weight") ? get_double(d, e->get("weight"), "weight") : 1.0;
            t.transfer_mix.push_back(x);
        }
    }
    dbl("base_compute_ms", t.base_compute_ms);
    dbl("service_cv", t.service_cv);
    dbl("slo_tail_ms", t.slo_tail_ms);
    dbl("weight", t.weight);
    dbl("pcie_cap_Bps", t.pcie_cap_Bps);
    dbl("host_io_Bps", t.host_io_Bps);
    dbl("sm_demand", t.sm_demand);
    dbl("noise_mean_ms", t.noise_mean_ms);
}

TenantEntry parse_tenant(const Doc& d, const Node* n) {
    TenantEntry e;
    if (const Node* p = n->get("preset")) {
        try {
            e.spec = workload_preset(get_str(d, p));
        } catch (const ConfigError& err) {
            d.fail(p->line, err.what());
        }
    }
    apply_tenant_overrides(d, n, e.spec);
    const Node* pn = n->get("placement");
    if (!pn) d.fail(n->line, "tenant needs a 'placement'");
    check_keys(d, pn, "placement", {"host", "gpu", "profile", "first_slice"});
    if (!pn->get("gpu") || !pn->get("profile")) d.fail(pn->line, "placement needs 'gpu' and 'profile'");
    e.placement.host = pn->get("host") ? get_int(d, pn->get("host"), "host") : 0;
    e.placement.gpu = get_int(d, pn->get("gpu"), "gpu");
    e.profile_name = get_str(d, pn->get("profile"));
    try {
        e.placement.slices.count = mig_lattice()[static_cast<size_t>(mig_profile_index(e.profile_name))].slices;
    } catch (const ConfigError& err) {
        d.fail(pn->get("profile")->line, err.what());
    }
    e.placement.slices.first = pn->get("first_slice") ? get_int(d, pn->get("first_slice"), "first_slice") : 0;
    if (const Node* s = n->get("schedule")) e.schedule = parse_schedule(d, s);
    try {
        e.spec.validate();
    } catch (const ConfigError& err) {
        d.fail(n->line, err.what());
    }
    return e;
}

void apply_controller_overrides(const Doc& d, const Node* n, ControllerConfig& c) {
    check_keys(d, n, "controller",
               {"enabled", "enable_mig", "enable_placement", "enable_guardrails", "tail_threshold_ms",
                "persistence_windows", "dwell_obs", "cooldown_obs", "sample_interval_s", "warmup_s",
                "move_futility_ratio", "throttle_duration_s", "quota_duration_s", "ema_alpha", "hysteresis_clear_ratio",
                "relax_stability_ratio", "relax_score_threshold", "validation_obs", "rollback_regress_ratio",
                "diag_pcie_util_threshold", "diag_host_io_threshold", "diag_sm_util_threshold", "move_margin",
                "admission_queue_timeout_epochs", "guardrail_io_throttle_Bps", "guardrail_mps_quota_pct",
                "irq_lookback_s", "throughput_floor"});
    auto b = [&](const char* k, bool& o) {
        if (const Node* v = n->get(k)) o = get_bool(d, v, k);
    };
    auto f = [&](const char* k, double& o) {
        if (const Node* v = n->get(k)) o = get_double(d, v, k);
    };
    auto i = [&](const char* k, int& o) {
        if (const Node* v = n->get(k)) o = get_int(d, v, k);
    };
    b("enabled", c.enabled);
    b("enable_mig", c.enable_mig);
    b("enable_placement", c.enable_placement);
    b("enable_guardrails", c.enable_guardrails);
    f("tail_threshold_ms", c.tail_threshold_ms);
    i("persistence_windows", c.persistence_windows);
    i("dwell_obs", c.dwell_obs);
    i("cooldown_obs", c.cooldown_obs);
    f("sample_interval_s", c.sample_interval_s);
    f("warmup_s", c.warmup_s);
    f("move_futility_ratio", c.move_futility_ratio);
    f("throttle_duration_s", c.throttle_duration_s);
    f("quota_duration_s", c.quota_duration_s);
    f("ema_alpha", c.ema_alpha);
    f("hysteresis_clear_ratio", c.hysteresis_clear_ratio);
    f("relax_stability_ratio", c.relax_stability_ratio);
    f("relax_score_threshold", c.relax_score_threshold);
    i("validation_obs", c.validation_obs);
    f("rollback_regress_ratio", c.rollback_regress_ratio);
    f("diag_pcie_util_threshold", c.diag_pcie_util_threshold);
    f("diag_host_io_threshold", c.diag_host_io_threshold);
    f("diag_sm_util_threshold", c.diag_sm_util_threshold);
    f("move_margin", c.move_margin);
    i("admission_queue_timeout_epochs", c.admission_queue_timeout_epochs);
    f("guardrail_io_throttle_Bps", c.guardrail_io_throttle_Bps);
    f("guardrail_mps_quota_pct", c.guardrail_mps_quota_pct);
    f("irq_lookback_s", c.irq_lookback_s);
    f("throughput_floor", c.throughput_floor);
}

}  // namespace

ScenarioSpec parse_scenario(const std::string& yaml_text, const std::string& source_name) {
    Doc d{source_name};
    std::shared_ptr<Node> root;
    try {
        root = yaml::parse(yaml_text);
    } catch (const yaml::ParseError& e) {
        throw ConfigError(std::string("YAML parse error: ") + e.what(), source_name + ":" + std::to_string(e.line));
    }
    if (root->kind != Node::kMap) throw ConfigError("scenario document must be a mapping", source_name + ":1");
    check_keys(d, root.get(), "scenario",
               {"version", "name", "duration_s", "measure_start_s", "fabric", "topology", "tenants", "irq_bursts",
                "controller"});
    const Node* v = root->get("version");
    if (!v) throw ConfigError("scenario is missing 'version'", source_name + ":1");
    const std::string version = get_str(d, v);
    if (version != "scenario-v1")
        d.fail(v->line, "unsupported scenario version '" + version + "' (expected scenario-v1)");
    ScenarioSpec spec;
    spec.name = root->get("name") ? get_str(d, root->get("name")) : "unnamed";
    if (!root->get("duration_s")) throw ConfigError("scenario is missing 'duration_s'", source_name + ":1");
    spec.duration_s = get_double(d, root->get("duration_s"), "duration_s");
    if (root->get("measure_start_s")) spec.measure_start_s = get_double(d, root->get("measure_start_s"), "measure_start_s");
    if (const Node* f = root->get("fabric")) {
        check_keys(d, f, "fabric", {"redistribute"});
        if (f->get("redistribute")) spec.fabric_redistribute = get_bool(d, f->get("redistribute"), "redistribute");
    }
    if (!root->get("topology")) throw ConfigError("scenario is missing 'topology'", source_name + ":1");
    spec.topology = parse_topology(d, root->get("topology"));
    const Node* ts = root->get("tenants");
    if (!ts || ts->kind != Node::kSeq) throw ConfigError("scenario needs a 'tenants' list", source_name + ":1");
    for (const auto& t : ts->seq) spec.tenants.push_back(parse_tenant(d, t.get()));
    if (const Node* irqs = root->get("irq_bursts")) {
        for (const auto& ip : irqs->seq) {
            const Node* in = ip.get();
            check_keys(d, in, "irq_burst", {"host", "core_group", "extra_noise_ms", "schedule"});
            IrqBurstSpec b;
            if (in->get("host")) b.host = get_int(d, in->get("host"), "host");
            if (in->get("core_group")) b.core_group = get_int(d, in->get("core_group"), "core_group");
            if (in->get("extra_noise_ms")) b.extra_noise_ms = get_double(d, in->get("extra_noise_ms"), "extra_noise_ms");
            if (in->get("schedule")) b.schedule = parse_schedule(d, in->get("schedule"));
            spec.irq_bursts.push_back(b);
        }
    }
    if (const Node* c = root->get("controller")) apply_controller_overrides(d, c, spec.controller);
    spec.validate();
    return spec;
}

ScenarioSpec load_scenario(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open scenario file '" + path + "'");
    std::stringstream buf;
    buf << in.rdbuf();
    return parse_scenario(buf.str(), path);
}

}  // namespace mgb
