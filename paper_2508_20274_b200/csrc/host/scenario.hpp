// Host-side scenario model + scenario-v1 loader of the B200 engine.
//
// Mirrors the reference's input types and their semantics so the engine is a drop-in for the
// same files:
//   model types      /root/reference/proj/include/migsim/model.hpp:45-232
//   schedule         /root/reference/proj/include/migsim/workload.hpp:56-74
//   presets          /root/reference/proj/src/workload.cpp:172-236
//   scenario + load  /root/reference/proj/include/migsim/scenario.hpp:30-68, src/scenario.cpp:26-384
#pragma once

#include <cstdint>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace mgb {

// model::ConfigError (model.hpp:29-37): where() carries "file:line" for document errors.
class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& msg, std::string where = {})
        : std::runtime_error(where.empty() ? msg : where + ": " + msg), where_(std::move(where)) {}
    const std::string& where() const { return where_; }

private:
    std::string where_;
};

struct MigProfile {
    std::string name;
    int slices = 0;
    double mem_gb = 0.0;
};
const std::vector<MigProfile>& mig_lattice();
int mig_profile_index(const std::string& name);  // throws ConfigError (model.cpp:35-41)

struct PcieRootSpec {
    int id = 0;
    double capacity_Bps = 0.0;
};
struct GpuSpec {
    int id = 0;
    int pcie_root_id = 0;
    int numa_id = 0;
    int core_group = 0;
    int total_slices = 7;
    bool mig_enabled = true;
};
struct HostSpec {
    std::vector<GpuSpec> gpus;
    int numa_domains = 1;
    std::vector<PcieRootSpec> pcie_roots;
    std::set<int> irq_hot_core_groups;
    double io_capacity_Bps = 1e9;
};
struct TopologySpec {
    std::vector<HostSpec> hosts;
    void validate() const;
    const GpuSpec& gpu(int host, int gpu_id) const;
    const PcieRootSpec& pcie_root(int host, int root_id) const;
};

enum class TenantClass { latency_sensitive, bandwidth_heavy, compute_heavy };
const char* to_string(TenantClass c);
TenantClass tenant_class_from_string(const std::string& s);

struct TransferMixEntry {
    double bytes = 0.0;
    double weight = 0.0;
};
struct TenantSpec {
    std::string id;
    TenantClass tclass = TenantClass::latency_sensitive;
    double arrival_rate_hz = 0.0;
    double arrival_cv = 1.0;
    std::vector<TransferMixEntry> transfer_mix;
    double base_compute_ms = 0.0;
    double service_cv = 0.0;
    double slo_tail_ms = 0.0;
    double weight = 1.0;
    double pcie_cap_Bps = 0.0;
    double host_io_Bps = 0.0;
    double sm_demand = 1.0;
    double noise_mean_ms = 0.0;
    double mean_transfer_bytes() const;
    void validate() const;
};
struct SliceRange {
    int first = 0;
    int count = 0;
    int end() const { return first + count; }
    bool overlaps(const SliceRange& o) const { return first < o.end() && o.first < end(); }
};
struct Placement {
    int host = 0;
    int gpu = 0;
    SliceRange slices;
};

struct ControllerConfig {
    bool enabled = true;
    bool enable_mig = true;
    bool enable_placement = true;
    bool enable_guardrails = true;
    double tail_threshold_ms = 15.0;
    int persistence_windows = 3;
    int dwell_obs = 256;
    int cooldown_obs = 128;
    double sample_interval_s = 2.0;
    double warmup_s = 60.0;
    double move_futility_ratio = 2.0;
    double throttle_duration_s = 30.0;
    double quota_duration_s = 30.0;
    double ema_alpha = 0.2;
    double hysteresis_clear_ratio = 0.9;
    double relax_stability_ratio = 0.8;
    double relax_score_threshold = 0.3;
    int validation_obs = 64;
    double rollback_regress_ratio = 0.05;
    double diag_pcie_util_threshold = 0.8;
    double diag_host_io_threshold = 0.8;
    double diag_sm_util_threshold = 0.7;
    double move_margin = 0.25;
    int admission_queue_timeout_epochs = 10;
    double guardrail_io_throttle_Bps = 250e6;
    double guardrail_mps_quota_pct = 50.0;
    double irq_lookback_s = 30.0;
    double throughput_floor = 0.95;
    void validate() const;
};

struct InterferenceSchedule {
    enum class Kind { always, square_wave, phases };
    struct Phase {
        double start_s = 0.0;
        double end_s = 0.0;
    };
    Kind kind = Kind::always;
    double period_s = 0.0;
    double duty = 1.0;
    double offset_s = 0.0;
    std::vector<Phase> phases;
    void validate() const;
};

struct TenantEntry {
    TenantSpec spec;
    Placement placement;
    std::string profile_name;
    InterferenceSchedule schedule;
};
struct IrqBurstSpec {
    int host = 0;
    int core_group = 0;
    double extra_noise_ms = 0.0;
    InterferenceSchedule schedule;
};
struct ScenarioSpec {
    std::string name;
    double duration_s = 0.0;
    double measure_start_s = 0.0;
    bool fabric_redistribute = false;
    TopologySpec topology;
    std::vector<TenantEntry> tenants;
    std::vector<IrqBurstSpec> irq_bursts;
    ControllerConfig controller;
    void validate() const;
    const TenantEntry& tenant(const std::string& id) const;
};

TenantSpec workload_preset(const std::string& name);
ScenarioSpec parse_scenario(const std::string& yaml_text, const std::string& source_name);
ScenarioSpec load_scenario(const std::string& path);

// Controller::bandwidth_claim (controller.cpp:166-169)
double bandwidth_claim(const TenantSpec& spec);

}  // namespace mgb
