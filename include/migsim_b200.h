/*
 * migsim-b200: C-ABI of the B200 batched engine for the reference's replica hot path.
 *
 * The reference evaluates its multi-tenancy controller by fanning (variant, seed) replicas of
 * `engine::run_scenario` out over std::async threads
 *   - replica entry  : RunResult run_scenario(const ScenarioSpec&, const RunOptions&)
 *                      /root/reference/proj/include/migsim/engine.hpp:117 (impl engine.cpp:898-902)
 *   - fan-out        : harness::run_plan, /root/reference/proj/src/harness.cpp:156-176
 *   - scenario input : scenario-v1 YAML, /root/reference/proj/src/scenario.cpp:322-374
 * This ABI replaces that fan-out with one batched GPU call.  Plain C types only; all buffers are
 * caller-owned except results, which are freed with migsim_batch_result_free.  No exceptions
 * cross the ABI.  Calls are synchronous; one handle per host thread.
 *
 * Return codes: 0 ok; 1 config error (message carries "file:line" like model::ConfigError,
 * model.hpp:29-37); 2 runtime/CUDA error; 3 parity guard (a device-sized buffer would have
 * truncated; nothing is silently dropped).
 */
#ifndef MIGSIM_B200_H
#define MIGSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MIGSIM_API __attribute__((visibility("default")))
#else
#define MIGSIM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MIGSIM_OK 0
#define MIGSIM_ERR_CONFIG 1
#define MIGSIM_ERR_RUNTIME 2
#define MIGSIM_ERR_PARITY_GUARD 3

typedef struct migsim_gpu migsim_gpu;
typedef struct migsim_batch_result migsim_batch_result;

/* harness::Variant (harness.hpp:40-46) plus the e3 sweep knobs (harness.cpp:89-110).
 * Flags: -1 keeps the scenario's value, 0/1 set it.  Numeric knobs: MIGSIM_KEEP_INT / NaN keep
 * the scenario's value; every other value is applied and checked by ControllerConfig::validate
 * (model.cpp:184-206), so e.g. dwell_obs = 0 is a config error, as in the reference. */
#define MIGSIM_KEEP_INT INT32_MIN
typedef struct migsim_variant {
    const char* name;
    int32_t enabled, enable_mig, enable_placement, enable_guardrails;
    double sample_interval_s;    /* NaN: keep */
    int32_t persistence_windows; /* MIGSIM_KEEP_INT: keep */
    int32_t dwell_obs;           /* MIGSIM_KEEP_INT: keep */
    int32_t cooldown_obs;        /* MIGSIM_KEEP_INT: keep */
    int32_t validation_obs;      /* MIGSIM_KEEP_INT: keep */
} migsim_variant;

/* engine::RunOptions (engine.hpp:94-99) batch form. */
typedef struct migsim_run_opts {
    int32_t keep_completions;   /* store per-completion records (parity/debug; memory heavy) */
    int32_t max_wave_replicas;  /* 0: sized from free device memory */
    int32_t action_cap;         /* per-replica action-log capacity, 0: default 1024 */
    int32_t pause_cap;          /* per-replica pause-log capacity, 0: default 1024 */
    int32_t write_traces;       /* RunOptions::write_traces: per-completion + per-tick trace rows
                                   (requests/counters/fabric streams, engine.cpp:279-288) */
} migsim_run_opts;

/* device-side timing of the last batch (CUDA events on the batch stream), milliseconds */
typedef struct migsim_timing {
    double gen_ms, des_ms, select_ms, total_device_ms, wall_ms;
    int64_t replicas, tenant_ticks, completions, arrivals, events, waves;
    int64_t select_samples;  /* measurement-window latencies fed to the select kernel */
    int64_t des_form;        /* DES kernel: 0 warp per replica, 1 SIMT (thread per replica),
                                2 warp per replica register-capped (saturated batches) */
    int64_t des_blocks_per_sm; /* occupancy of the DES launch (resident blocks per SM) */
    int64_t des_smem_bytes;    /* dynamic shared memory per DES block */
    int64_t kernel_launches;   /* engine kernels launched by the call */
    int64_t h2d_bytes, d2h_bytes; /* host<->device bytes copied by the call */
    int64_t pipeline_slots;       /* 2: waves double-buffered on two streams (total_device_ms = span) */
} migsim_timing;

/* per (run, tenant) flat summary row, tenants in lexicographic id order
 * (engine::TenantSummary, engine.hpp:67-78, plus p999) */
typedef struct migsim_tenant_row {
    uint64_t completed_total, completed_window, window_misses;
    double mean_ms, p50_ms, p95_ms, p99_ms, p999_ms, miss_rate, throughput_hz;
} migsim_tenant_row;

MIGSIM_API int migsim_gpu_open(int device, migsim_gpu** out, char* err, size_t errlen);
MIGSIM_API void migsim_gpu_close(migsim_gpu* g);

/* scenario::parse_scenario / load_scenario (scenario.hpp:65-68) */
MIGSIM_API int migsim_gpu_load_scenario(migsim_gpu* g, const char* yaml_text, const char* source_name, int32_t* scenario_id,
                             char* err, size_t errlen);
MIGSIM_API int migsim_gpu_load_scenario_file(migsim_gpu* g, const char* path, int32_t* scenario_id, char* err, size_t errlen);
/* ---- in-memory scenario specs ----------------------------------------------------------
 * Plain-C mirror of scenario::ScenarioSpec (scenario.hpp:30-61) with its model/workload parts
 * (TopologySpec/HostSpec/GpuSpec/PcieRootSpec model.hpp:74-105, TenantSpec model.hpp:122-139,
 * ControllerConfig model.hpp:186-224, InterferenceSchedule workload.hpp:56-74), presets already
 * applied, every field explicit.  Tenants, hosts, GPUs and roots in the spec's own order.  This is
 * how a spec the caller built or mutated in memory (e.g. harness::apply_variant, the e3 sweep's
 * ControllerConfig edits, harness.cpp:89-110) crosses the ABI without a YAML round trip; the
 * engine copies it, runs ScenarioSpec::validate (scenario.cpp:270-313 checks) and canonicalises
 * the orders itself. */
typedef struct migsim_schedule_desc {
    int32_t kind; /* 0 always, 1 square_wave, 2 phases */
    double period_s, duty, offset_s;
    const double* phase_start_s; /* [n_phases] */
    const double* phase_end_s;   /* [n_phases] */
    size_t n_phases;
} migsim_schedule_desc;
typedef struct migsim_gpu_desc {
    int32_t id, pcie_root_id, numa_id, core_group, total_slices, mig_enabled;
} migsim_gpu_desc;
typedef struct migsim_root_desc {
    int32_t id;
    double capacity_Bps;
} migsim_root_desc;
typedef struct migsim_host_desc {
    const migsim_gpu_desc* gpus;
    size_t n_gpus;
    int32_t numa_domains;
    const migsim_root_desc* roots;
    size_t n_roots;
    const int32_t* irq_hot_core_groups;
    size_t n_irq_hot;
    double io_capacity_Bps;
} migsim_host_desc;
typedef struct migsim_tenant_desc {
    const char* id;
    int32_t tclass; /* 0 latency_sensitive, 1 bandwidth_heavy, 2 compute_heavy */
    double arrival_rate_hz, arrival_cv;
    const double* mix_bytes;  /* transfer_mix, [n_mix] */
    const double* mix_weight; /* [n_mix] */
    size_t n_mix;
    double base_compute_ms, service_cv, slo_tail_ms, weight, pcie_cap_Bps, host_io_Bps, sm_demand, noise_mean_ms;
    int32_t host, gpu, first_slice, slice_count; /* TenantEntry::placement */
    const char* profile;                         /* TenantEntry::profile_name, e.g. "2g" */
    migsim_schedule_desc schedule;
} migsim_tenant_desc;
typedef struct migsim_irq_desc {
    int32_t host, core_group;
    double extra_noise_ms;
    migsim_schedule_desc schedule;
} migsim_irq_desc;
typedef struct migsim_controller_desc {
    int32_t enabled, enable_mig, enable_placement, enable_guardrails;
    double tail_threshold_ms;
    int32_t persistence_windows, dwell_obs, cooldown_obs;
    double sample_interval_s, warmup_s, move_futility_ratio, throttle_duration_s, quota_duration_s, ema_alpha,
        hysteresis_clear_ratio, relax_stability_ratio, relax_score_threshold;
    int32_t validation_obs;
    double rollback_regress_ratio, diag_pcie_util_threshold, diag_host_io_threshold, diag_sm_util_threshold,
        move_margin;
    int32_t admission_queue_timeout_epochs;
    double guardrail_io_throttle_Bps, guardrail_mps_quota_pct, irq_lookback_s, throughput_floor;
} migsim_controller_desc;
typedef struct migsim_scenario_desc {
    const char* name;
    double duration_s, measure_start_s;
    int32_t fabric_redistribute;
    const migsim_host_desc* hosts;
    size_t n_hosts;
    const migsim_tenant_desc* tenants;
    size_t n_tenants;
    const migsim_irq_desc* irq_bursts;
    size_t n_irq_bursts;
    migsim_controller_desc controller;
} migsim_scenario_desc;
/* load an in-memory spec; same ids and errors as migsim_gpu_load_scenario (code 1 = ConfigError
 * from ScenarioSpec::validate, message prefixed "<spec>") */
MIGSIM_API int migsim_gpu_load_spec(migsim_gpu* g, const migsim_scenario_desc* spec, int32_t* scenario_id, char* err,
                                    size_t errlen);
/* drop a loaded scenario's host copy (its id is not reused; later use is a config error) */
MIGSIM_API int migsim_gpu_release_scenario(migsim_gpu* g, int32_t scenario_id);

/* canonical tenant order of a loaded scenario: writes the i-th id (lexicographic) */
MIGSIM_API int migsim_scenario_n_tenants(migsim_gpu* g, int32_t scenario_id);
MIGSIM_API int migsim_scenario_tenant_id(migsim_gpu* g, int32_t scenario_id, int32_t i, char* buf, size_t buflen);

/* variants x seeds replicas, row-major (variant-major, seed-minor) like harness.cpp:125-152 */
MIGSIM_API int migsim_gpu_run_batch(migsim_gpu* g, int32_t scenario_id, const migsim_variant* variants, size_t n_variants,
                         const uint64_t* seeds, size_t n_seeds, const migsim_run_opts* opts,
                         migsim_batch_result** out, char* err, size_t errlen);

/* engine::run_scenario(spec, RunOptions{seed, out_dir, write_traces}) (engine.hpp:94-99,117): one
 * replica on the GPU; the host writes the reference's artifacts into out_dir byte-for-byte
 * (summary.json, actions.jsonl and, with write_traces, requests.csv / counters.csv / fabric.csv;
 * engine.cpp:279-288,889-892, trace.cpp).  *result_json (optional, free with migsim_free) receives
 * the RunResult as JSON. */
MIGSIM_API int migsim_gpu_run_scenario(migsim_gpu* g, int32_t scenario_id, const migsim_variant* variant, uint64_t seed,
                            const char* out_dir, int32_t write_traces, char** result_json, char* err, size_t errlen);

MIGSIM_API size_t migsim_batch_n_runs(const migsim_batch_result* r);
MIGSIM_API int migsim_batch_n_tenants(const migsim_batch_result* r);
MIGSIM_API int migsim_batch_timing(const migsim_batch_result* r, migsim_timing* t);
/* rows [n_runs * n_tenants] */
MIGSIM_API int migsim_batch_tenant_rows(const migsim_batch_result* r, migsim_tenant_row* rows, size_t cap);
/* full engine::RunResult of one run as JSON (summary + actions + pauses + stability);
 * the pointer stays valid until the result is freed */
MIGSIM_API const char* migsim_batch_run_json(migsim_batch_result* r, size_t run);
/* per-completion records of one run (only with keep_completions): 7 doubles per completion
 * {tenant, seq, done_s, total_ms, compute_ms, transfer_ms, noise_ms}, tenant-major order */
MIGSIM_API int64_t migsim_batch_completions(const migsim_batch_result* r, size_t run, double* out, int64_t cap);
/* engine::CompletionRecord (engine.hpp:44-54) of one run, only with keep_completions: in the
 * reference's RunResult::completions order (completion order, engine.cpp:504); tenant = canonical
 * (lexicographic) index, seq = the tenant's request sequence number (engine.cpp:425,482).  Returns
 * the record count (out may be NULL to query it), -1 without keep_completions. */
typedef struct migsim_completion {
    int32_t tenant, pad;
    uint64_t seq;
    double arrived_s, done_s, total_ms, compute_ms, transfer_ms, noise_ms, transfer_bytes;
} migsim_completion;
MIGSIM_API int64_t migsim_batch_completion_records(const migsim_batch_result* r, size_t run, migsim_completion* out,
                                                   int64_t cap);
MIGSIM_API void migsim_batch_result_free(migsim_batch_result* r);

/* Per-(variant, tenant) aggregates of a batch, summed over its seeds on the device -- the payload
 * the multi-GPU reduction all-reduces (the per-variant aggregation of harness.cpp:
 * 178-204 extended to whole distributions).  Histograms: every measurement-window latency
 * (engine.cpp:498-502) counted in MIGSIM_HIST_BINS fixed log-spaced bins (64 per binary octave,
 * bin 0 starting at 2^-10 ms; values below / above the range clamp into the first / last bin;
 * edges from migsim_hist_bin_edges).  out[(v * T + t) * MIGSIM_HIST_BINS + b], tenants in
 * lexicographic id order, variants in the batch's order.  Counts: out[(v * T + t) * 3 + k] =
 * completed_total, completed_window, window_misses (engine.cpp:497-501). */
#define MIGSIM_HIST_BINS 2048
MIGSIM_API size_t migsim_batch_n_variants(const migsim_batch_result* r);
MIGSIM_API int migsim_batch_latency_hist(const migsim_batch_result* r, uint64_t* out, size_t cap);
MIGSIM_API int migsim_batch_tenant_counts(const migsim_batch_result* r, uint64_t* out, size_t cap);
/* lower edge (ms) of each histogram bin; n >= MIGSIM_HIST_BINS */
MIGSIM_API int migsim_hist_bin_edges(double* lo, size_t n);

/* Standalone nearest-rank select (telemetry.cpp:38-56 / engine.cpp:800-816 semantics) over
 * n_segments host segments vals[seg_off[s] .. seg_off[s+1]); out[s * n_q + j] = quantile qs[j]. */
MIGSIM_API int migsim_gpu_select(migsim_gpu* g, const double* vals, const int64_t* seg_off, size_t n_segments, const double* qs,
                      size_t n_q, double* out, double* device_ms, char* err, size_t errlen);

/* Batched admission control: Controller::admit (controller.cpp:637-692; declared controller.hpp:
 * 152-153) for n independent cases on the GPU -- exhaustive placement-candidate scoring over every
 * (host, gpu).  Tenants are the loaded scenario's, canonical (lexicographic id) order, T of them;
 * case c requests tenant tenant[c] at MIG profile profile[c] (lattice index 0..4 = 1g..7g) given
 * TenantStates admitted/host/gpu_id/first/count [n][T] and the ClusterSnapshot fields the scoring
 * reads: tenant_pcie_Bps, tenant_host_io_Bps [n][T] and irq_recent [n][n_hosts] (bit g = core
 * group g of that host had a recent IRQ burst).  queue_epochs [n] (in/out, may be NULL = fresh
 * controllers) is the case's controller state Controller::queue_epochs_[tenant] (controller.hpp:
 * 214; 0 = no entry): a request without a feasible slot increments it and is rejected (entry
 * erased) once it exceeds admission_queue_timeout_epochs, an admitted request erases it
 * (controller.cpp:671-691) -- carry the array across calls to retry queued requests.
 * outcome: 0 admitted, 1 queued, 2 rejected; reason: 0 none, 1 service rate, 2 no feasible slot,
 * 3 queue timeout. */
typedef struct migsim_admit_decision {
    int32_t outcome, host, gpu, first, count, profile, reason, pad;
    double score; /* placement_score(...).total() of the chosen slot */
} migsim_admit_decision;
MIGSIM_API int migsim_gpu_admit(migsim_gpu* g, int32_t scenario_id, size_t n_cases, const int32_t* tenant,
                     const int32_t* profile, const int32_t* admitted, const int32_t* host, const int32_t* gpu_id,
                     const int32_t* first, const int32_t* count, const double* tenant_pcie_Bps,
                     const double* tenant_host_io_Bps, const uint32_t* irq_recent, int32_t* queue_epochs,
                     migsim_admit_decision* out,
                     double* device_ms, char* err, size_t errlen);

/* Batched experiment plans (harness::run_plan, harness.cpp:114-216; PlanOptions harness.hpp:84-92):
 * plan in {e1,e2,e3,llm}; returns experiment.json (same keys/aggregation: population-sigma CIs in
 * seed order).  With out_dir: experiment.json + summary.csv and <variant>/seed<N>/{actions.jsonl,
 * summary.json} per job, like the reference (harness.cpp:131-133,208-214). */
MIGSIM_API int migsim_run_plan(migsim_gpu* g, const char* plan, const char* scenario_path, int32_t seeds, uint64_t seed_base,
                    const char* focus_tenant, const char* out_dir, char** experiment_json, char* err, size_t errlen);
/* harness::render_report (harness.cpp:285-313) of an experiment.json text; host only */
MIGSIM_API int migsim_render_report(const char* experiment_json, char** report, char* err, size_t errlen);
MIGSIM_API void migsim_free(void* p);

/* ---- diagnostics used by the parity tests ---------------------------------------------- */
/* Host-only: parse a scenario (path) with the engine's scenario-v1 loader and return the
 * normalised spec as JSON (no GPU needed). */
MIGSIM_API int migsim_scenario_dump(const char* path, char** json, char* err, size_t errlen);
/* Device glibc-exact math: fn 0 = log(x), 1 = exp(x), 2 = pow(x, y), 3 = fmod(x, y) (the
 * schedule phase, arrivals.h sched_active); n values. */
MIGSIM_API int migsim_gpu_libm(migsim_gpu* g, int fn, const double* x, const double* y, double* out, size_t n,
                               char* err, size_t errlen);
/* Device-generated arrival records of one tenant (canonical index) for one seed:
 * 4 doubles per kept arrival {t_s, transfer_bytes, service_mult, noise_ms}; *n_out = count. */
MIGSIM_API int migsim_gpu_arrivals(migsim_gpu* g, int32_t scenario_id, uint64_t seed, int32_t tenant, double* out,
                                   int64_t cap, int64_t* n_out, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* MIGSIM_B200_H */
