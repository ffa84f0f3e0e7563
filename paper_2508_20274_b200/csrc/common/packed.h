// Device-side (POD) form of one scenario + the per-variant controller configs.
//
// Produced on the host by host/packer.cpp from the reference-format scenario
// (`ScenarioSpec`, /root/reference/proj/include/migsim/scenario.hpp:46-61) with
// the canonical orders the reference's std::map iterations imply:
//   tenants  lexicographic by id       (std::map<std::string,...>, engine.cpp:194-196)
//   roots    by (host, root id)        (std::map<std::pair<int,int>,RootRt>, engine.cpp:196)
//   gpus     topology order per host   (controller.cpp:268-269)
#pragma once

#include <stdint.h>

namespace mg {

constexpr int kMaxTenants = 64;   // root.active is a 64-bit tenant mask
constexpr int kMaxMix = 8;
constexpr int kMaxPhases = 8;
constexpr int kMaxRoots = 64;
constexpr int kMaxGpus = 128;
constexpr int kMaxHosts = 16;
constexpr int kMaxIrq = 16;
constexpr int kNumProfiles = 5;   // A100 lattice 1g,2g,3g,4g,7g (model.cpp:23-32)

enum TenantClass : int32_t { kLatencySensitive = 0, kBandwidthHeavy = 1, kComputeHeavy = 2 };
enum SchedKind : int32_t { kAlways = 0, kSquareWave = 1, kPhases = 2 };

struct Schedule {
    int32_t kind;
    int32_t n_phases;
    double period_s, duty, offset_s;
    double ph_start[kMaxPhases];
    double ph_end[kMaxPhases];
};

struct PGpu {
    int32_t host, id, root;  // root = canonical root index
    int32_t numa, core_group, total_slices, mig_enabled;
    int32_t pad;
};

struct PRoot {
    int32_t host, id;
    double capacity;
};

struct PIrq {
    int32_t host, core_group;
    double extra_noise_ms;
    double lambda;  // 1.0 / extra_noise_ms (exponential_distribution ctor arg, engine.cpp:403)
    Schedule sched;
};

struct PTenant {
    uint64_t name_hash;  // fnv1a(id)
    int32_t tclass;
    int32_t host, gpu, first, count, profile;  // initial placement; gpu = canonical gpu index
    double arrival_rate_hz, weight, pcie_cap, host_io, sm_demand, base_compute_ms, slo_tail_ms;
    double claim;  // Controller::bandwidth_claim (controller.cpp:166-169)
    // --- ArrivalGen parameters (workload.cpp:103-127), computed on the host with glibc
    int32_t deterministic, n_mix;
    double det_step;  // 1.0 / arrival_rate_hz
    double g_alpha, g_beta, g_malpha, g_a1, g_a2, g_inv_alpha;
    double mix_cdf[kMaxMix];
    double mix_bytes[kMaxMix];
    int32_t has_service, has_noise;
    double svc_mu, svc_sigma, noise_lambda;
    Schedule sched;
};

// ControllerConfig (model.hpp:186-224) after variant overrides (harness.cpp:62-69)
struct PController {
    int32_t enabled, enable_mig, enable_placement, enable_guardrails;
    int32_t persistence_windows, dwell_obs, cooldown_obs, validation_obs;
    double tail_threshold_ms, sample_interval_s, warmup_s, move_futility_ratio;
    double throttle_duration_s, quota_duration_s, ema_alpha, hysteresis_clear_ratio;
    double relax_stability_ratio, relax_score_threshold, rollback_regress_ratio;
    double diag_pcie_util_threshold, diag_host_io_threshold, diag_sm_util_threshold;
    double move_margin, guardrail_io_throttle_Bps, guardrail_mps_quota_pct, irq_lookback_s;
    double throughput_floor;
};

struct PScenario {
    int32_t n_tenants, n_roots, n_gpus, n_hosts, n_irq, fabric_redistribute;
    int32_t n_ticks;  // ticks at t = 1..floor(duration) (engine.cpp:273-276,776-781)
    int32_t pad;
    double duration_s, measure_start_s;
    double host_io_capacity[kMaxHosts];
    PRoot roots[kMaxRoots];
    PGpu gpus[kMaxGpus];
    PIrq irq[kMaxIrq];
    PTenant tenants[kMaxTenants];
};

// MIG lattice slice counts (model.cpp:23-32)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int profile_slices(int p) {
    return p == 0 ? 1 : p == 1 ? 2 : p == 2 ? 3 : p == 3 ? 4 : 7;
}

}  // namespace mg
