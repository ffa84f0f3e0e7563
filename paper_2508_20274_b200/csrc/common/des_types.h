// Output records of the batched engine (device -> host), POD.
// Field meanings follow the reference's result types:
//   ActionRecord  /root/reference/proj/include/migsim/controller.hpp:61-80
//   PauseEvent    /root/reference/proj/include/migsim/engine.hpp:59-64
//   TenantSummary /root/reference/proj/include/migsim/engine.hpp:67-78 (order statistics by the
//                 select kernel), EndState engine.hpp:80-86, StabilityReport engine.hpp:88-92
#pragma once

#include <stdint.h>

namespace mg {

// control::ActionKind (controller.hpp:32-41)
enum ActionKind : int32_t {
    kActNone = 0,
    kActIoThrottle = 1,
    kActMpsQuota = 2,
    kActExpire = 3,
    kActMove = 4,
    kActMigUp = 5,
    kActMigDown = 6,
    kActRollback = 7,
};
// control::Diagnosis (controller.hpp:29)
enum Diagnosis : int32_t { kDiagNone = 0, kDiagIo = 1, kDiagCompute = 2 };

struct ActionRec {
    int32_t seq, kind, tenant, target;
    int32_t diagnosis, breach_windows, rolled_back_seq, expire_kind;
    int32_t new_host, new_gpu_id, new_first, new_end;
    int32_t new_profile, pad;
    uint64_t obs_since_prev;
    double t_s, p99_pre_ms, ema_p99_ms, throttle_Bps, quota_pct, pause_s;
};

struct PauseRec {
    double t_s, duration_s;
    int32_t tenant, kind;
};

struct TenantOut {
    uint64_t completed_total;
    uint64_t completed_window;
    uint64_t window_misses;
    double sum_total_ms;
    int32_t host, gpu_id, first, profile;
    int32_t cpu_pinned, pad;
    double win_min, win_max;  // range of the measurement-window latencies (seeds the radix select)
};

// Per-tick trace rows (engine.cpp:744-775 with RunOptions::write_traces; formatted on the host by
// the trace.cpp equivalents).  counters.csv: one row per (tick, tenant in id order);
// fabric.csv: one row per (tick, root in (host, id) order).
struct CounterRow {
    uint64_t completed, queue_len;
    double window_p99_ms, grant_Bps;
    int32_t profile, host, gpu_id, pad;
};
struct FabricRow {
    double offered_Bps, backlog_bytes;
    int32_t active_flows, pad;
};

// error codes (C-ABI return codes, include/migsim_b200.h)
enum : int32_t {
    kErrNone = 0,
    kErrActionOverflow = 1,
    kErrPauseOverflow = 2,
    kErrArrivalOverflow = 3,
    kErrSeqOverflow = 4,  // > 2^29 event pushes in one replica
    kErrOpOverflow = 5,   // continuation-op word overflow (des_core.h run_ops; structurally impossible)
};

struct ReplicaOut {
    int32_t n_actions, n_pauses, error, pad;
    uint64_t n_events;  // live events dispatched
};

}  // namespace mg
