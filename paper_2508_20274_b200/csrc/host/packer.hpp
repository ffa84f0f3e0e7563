// ScenarioSpec -> device POD (PScenario / PController), plus the result model returned to callers.
//
// Canonical orders (what the reference's std::map iteration implies):
//   tenants lexicographic by id (engine.cpp:194 `std::map<std::string, TenantRt>`),
//   roots by (host, id) (engine.cpp:196), GPUs in topology order (controller.cpp:268-269).
// ArrivalGen constants (gamma shape/scale, lognormal mu/sigma, mixture cdf ...) are computed here
// on the host with glibc, exactly as ArrivalGen's constructor does (workload.cpp:103-127), so the
// device only evaluates per-draw arithmetic.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include <climits>
#include <cstdint>
#include <limits>

#include "../common/des_types.h"
#include "../common/packed.h"
#include "scenario.hpp"

namespace mgb {

// harness::Variant (harness.hpp:40-46) + the e3 sweep overrides (harness.cpp:89-110)
// Only the sentinels keep the scenario's value (flags -1, integers kKeepInt, doubles NaN); every
// other value is applied and then checked by ControllerConfig::validate (model.cpp:184-206).
constexpr int kKeepInt = INT32_MIN;
struct Variant {
    std::string name = "as-is";
    int enabled = -1, enable_mig = -1, enable_placement = -1, enable_guardrails = -1;  // -1: keep scenario value
    double sample_interval_s = std::numeric_limits<double>::quiet_NaN();
    int persistence_windows = kKeepInt, dwell_obs = kKeepInt, cooldown_obs = kKeepInt, validation_obs = kKeepInt;
    double tail_threshold_ms = std::numeric_limits<double>::quiet_NaN();
};

ControllerConfig apply_variant(const ControllerConfig& base, const Variant& v);

struct Packed {
    mg::PScenario scen;
    std::vector<mg::PController> ctrl;      // per variant
    std::vector<std::string> tenant_ids;    // canonical (lexicographic) order
    std::vector<int32_t> file_order;        // canonical indices in scenario-file order
    std::vector<int64_t> cap;               // arrival-record capacity per canonical tenant
    std::vector<int64_t> off;               // prefix offsets of `cap`
    int64_t cap_sum = 0;
    int max_dwell = 0, max_validation = 0;
    bool any_irq_noise = false;
    bool any_thinned = false;  // some tenant's arrivals are schedule-thinned (needs the unthinned clock)
};

// Throws ConfigError when the scenario exceeds the device representation limits.
Packed pack(const ScenarioSpec& spec, const std::vector<Variant>& variants, double cap_sigmas = 12.0);

// ---- results (mirror engine::RunResult, engine.hpp:47-113) ---------------------------------
struct TenantSummary {
    std::string id;
    uint64_t completed_total = 0, completed_window = 0;
    double mean_ms = 0.0, p50_ms = 0.0, p95_ms = 0.0, p99_ms = 0.0, p999_ms = 0.0;
    double miss_rate = 0.0, throughput_hz = 0.0, slo_tail_ms = 0.0;
};
struct EndState {
    Placement placement;
    std::string profile;
    double claim_Bps = 0.0;
    bool cpu_pinned = false;
};
struct ActionRecord {
    int seq = 0;
    double t_s = 0.0;
    std::string tenant, target, kind, diagnosis, detail;
    double p99_pre_ms = 0.0, ema_p99_ms = 0.0;
    int breach_windows = 0;
    uint64_t obs_since_prev = 0;
    double throttle_Bps = 0.0, quota_pct = 0.0, pause_s = 0.0;
    int rolled_back_seq = -1;
};
struct PauseEvent {
    double t_s = 0.0;
    std::string tenant, kind;
    double duration_s = 0.0;
};
struct Stability {
    bool analytic_oversubscribed = false, unbounded_growth = false;
    std::vector<std::string> notes;
};
struct RunResult {
    std::string scenario_name, variant;
    uint64_t seed = 1;
    double duration_s = 0.0, measure_start_s = 0.0;
    std::map<std::string, TenantSummary> tenants;
    std::map<std::string, EndState> end_states;
    std::vector<ActionRecord> actions;
    std::vector<PauseEvent> pauses;
    Stability stability;
    uint64_t n_events = 0;
};

const char* action_kind_name(int k);
const char* diagnosis_name(int d);
// ActionRecord.detail exactly as controller.cpp:361-396 / :633 format it
std::string action_detail(const mg::ActionRec& r, const Packed& p);

// Assemble one replica's RunResult from the raw device outputs (host side of Sim::finish,
// engine.cpp:784-862).  `quant` = p50,p95,p99,p999 per canonical tenant.
RunResult assemble(const ScenarioSpec& spec, const Packed& p, const std::string& variant, uint64_t seed,
                   const mg::TenantOut* tout, const double* quant, const mg::ActionRec* acts, int n_actions,
                   const mg::PauseRec* pauses, int n_pauses, const double* backlog, uint64_t n_events);

}  // namespace mgb
