// One replica of the reference's discrete-event simulator + Algorithm-1 controller.
//
// Semantics are the reference's, restated for a flat, allocation-free state so that one warp
// can run one replica out of shared memory:
//   event loop          engine.cpp:864-894 (total order (t, kind, seq), seq bumps per push)
//   tenant pipeline     engine.cpp:298-508 (settle/reallocate root, transfer -> compute)
//   actuation           engine.cpp:553-742 (guardrails, pause/resume, expiry)
//   ticks               engine.cpp:744-782 (backlog series -> stability sums)
//   controller          controller.cpp:72-635 (on_observation, ladder, scoring, validation)
//   fabric              fabric.cpp:31-87 (PS share + water-filling)
//   telemetry           telemetry.cpp:30-125 (nearest-rank window, EMA, SLO account)
//
// Representation choices (all exactness-preserving):
// * Events live in fixed slots, one per (tenant, kind) plus the tick: in the reference every
//   cancellable event is superseded by a generation bump, so at most one event per (tenant,kind)
//   is live; stale heap entries have no observable effect (they only set `now_` before being
//   dropped, and the next live event overwrites it).  Each push still takes the next `seq`.
// * Transfer/compute FIFOs are index ranges over the tenant's pre-generated arrival records:
//   requests enter transfer_q in arrival order and leave both queues in FIFO order.
// * The controller's TailWindow quantile (a full copy+sort per observation in the reference,
//   ~84% of its CPU time) is answered from a cached top-K of the sliding window, rebuilt by a
//   scan only when evictions exhaust it; nearest rank is an index, so values are identical.
// * The ClusterSnapshot (engine.cpp:518-551) is evaluated lazily: on_observation only reads it
//   on the rare breach/relax/validation paths, and the engine state cannot change between the
//   snapshot and those reads, so the same sums in the same (tenant-id) order are reproduced.
#pragma once

#include "arrivals.h"
#include "des_types.h"
#include "lat_hist.h"
#include "packed.h"

#if defined(__CUDA_ARCH__)
#define MG_DEV_INLINE __device__ __forceinline__
#endif
// A/B switch (build flag -DMG_OUTLINE_HOT): the shared pipeline helpers as single out-of-line copies
// instead of one inlined copy per call site (instruction-cache footprint of the event loop)
#if defined(MG_OUTLINE_HOT) && defined(__CUDACC__)
#define MG_HOT __host__ __device__ __noinline__
#else
#define MG_HOT MG_HD
#endif

namespace mg {

constexpr int kTopK = 8;
constexpr int kEvKinds = 5;  // resume, expire, transfer, compute, arrival (+ one tick slot)
enum EvKind : int32_t { kEvResume = 0, kEvExpire = 1, kEvTransfer = 2, kEvCompute = 3, kEvArrival = 4, kEvTick = 5 };

constexpr double kEpsBytes = 1e-6;   // engine.cpp:48
constexpr double kMpsKappa = 0.5;    // engine.hpp:42

struct TailWin;

// ---------------------------------------------------------------------------------------------
// per-replica inputs/outputs in global memory
struct ReplicaIO {
    // arrival records of this replica: tenant t owns [off[t], off[t] + count[t])
    const double* arr_t;
    const double* arr_bytes;
    const double* arr_mult;
    const double* arr_noise;
    const double* irq_e;  // -log(1-u) draws of the irq stream, same offsets
    const int64_t* off;
    const int32_t* count;
    uint64_t seed;
    // scratch
    double* req_transfer_ms;  // same offsets
    uint64_t* mt_pause;       // n_tenants * 312
    // outputs
    double* win_lat;          // measurement-window latencies, same offsets
    uint32_t* win_hist;       // optional [T][kHistBins] histogram of the same latencies (lat_hist.h)
    ActionRec* actions;
    int32_t action_cap;
    PauseRec* pauses;
    int32_t pause_cap;
    TenantOut* tout;
    ReplicaOut* rout;
    double* backlog;          // n_roots * 2 : sum over first third, sum over last third of ticks
    // optional per-completion records (keep_completions), same offsets
    double* c_done;
    double* c_total;
    double* c_compute;
    double* c_transfer;
    double* c_noise;
    int64_t* c_order;  // position of the completion in the replica's completion sequence
    // optional per-tick traces (write_traces): rows [n_ticks][T] / [n_ticks][R], and the per-tenant
    // 256-sample trace window (engine.cpp:115, pushed on every completion, :497)
    CounterRow* tr_cnt;
    FabricRow* tr_fab;
    TailWin* tr_win;
};

// ---------------------------------------------------------------------------------------------
// sliding nearest-rank window with a cached top-K (telemetry.cpp:30-56) + SLO misses
// (telemetry.cpp:106-125; same capacity and push sequence as the window, controller.cpp:544-545)
struct TailWin {
    double* ring;
    int32_t cap, n, head, m;  // m = number of valid cached top values
    int32_t misses;
    int32_t pad;
    double tau;
    double top[kTopK];
};

MG_HD void tw_reset(TailWin& w, double tau) {
    w.n = 0;
    w.head = 0;
    w.m = 0;
    w.misses = 0;
    w.tau = tau;
}

MG_HD void tw_top_insert(TailWin& w, double x) {
    int j = w.m < kTopK ? w.m : kTopK - 1;
    if (w.m < kTopK) w.m += 1;
    while (j > 0 && w.top[j - 1] < x) {
        w.top[j] = w.top[j - 1];
        --j;
    }
    w.top[j] = x;
}

MG_HD void tw_push(TailWin& w, double x) {
    if (w.n == w.cap) {
        const double old = w.ring[w.head];
        w.ring[w.head] = x;
        w.head = w.head + 1 == w.cap ? 0 : w.head + 1;
        if (old > w.tau) w.misses -= 1;
        // evict `old` from the cached top (one copy of its value)
        if (w.m > 0 && old >= w.top[w.m - 1]) {
            int j = w.m - 1;
            while (j > 0 && w.top[j] != old) --j;
            for (int k = j; k + 1 < w.m; ++k) w.top[k] = w.top[k + 1];
            w.m -= 1;
        }
        w.n -= 1;  // transiently n-1 (for the insertion rule below)
    } else {
        int idx = w.head + w.n;
        if (idx >= w.cap) idx -= w.cap;
        w.ring[idx] = x;
    }
    if (x > w.tau) w.misses += 1;
    // insert x: complete cache (m == n) takes everything; otherwise only values >= smallest cached
    if (w.m == w.n) {
        if (w.m < kTopK) tw_top_insert(w, x);
        else if (x > w.top[kTopK - 1]) tw_top_insert(w, x);
    } else if (w.m > 0 && x >= w.top[w.m - 1]) {
        tw_top_insert(w, x);
    }
    w.n += 1;
}

// rebuild the cached top-K by a scan of the ring
MG_HD void tw_rebuild(TailWin& w) {
    w.m = 0;
    for (int i = 0; i < w.n; ++i) {
        int idx = w.head + i;
        if (idx >= w.cap) idx -= w.cap;
        const double x = w.ring[idx];
        if (w.m < kTopK || x > w.top[kTopK - 1]) tw_top_insert(w, x);
    }
}

// j-th largest (0-based) of n values ring[(head + i) % cap], i < n -- the order statistic that
// std::sort + nearest rank picks (telemetry.cpp:38-56, controller.cpp:446).  Bitwise bisection on
// the order-preserving 64-bit keys: after 64 counting passes K is the largest key with at least
// j+1 values >= K, i.e. exactly the j-th largest.  O(64 n), no scratch memory (used where the
// cached top-K does not reach the rank: validation verdicts and windows longer than ~8/(1-q)).
MG_HD uint64_t order_key(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
MG_HD double from_order_key(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & ~0x8000000000000000ull) : ~k;
    double x;
    std::memcpy(&x, &b, 8);
    return x;
}
MG_HD double ring_jth_largest(const double* ring, int cap, int head, int n, int j) {
    if (j < kTopK) {
        // small rank (the p99 of windows up to ~800 samples, e.g. every validation verdict): one
        // pass keeping the j+1 largest values, a sorted multiset -- the same order statistic
        double top[kTopK];
        int m = 0;
        int idx = head;
        for (int i = 0; i < n; ++i) {
            const double x = ring[idx];
            idx = idx + 1 == cap ? 0 : idx + 1;
            if (m <= j || x > top[m - 1]) {
                int k = m <= j ? m++ : m - 1;
                while (k > 0 && top[k - 1] < x) {
                    top[k] = top[k - 1];
                    --k;
                }
                top[k] = x;
            }
        }
        return top[j];
    }
    uint64_t K = 0;
    for (int bit = 63; bit >= 0; --bit) {
        const uint64_t c = K | (1ull << bit);
        int cnt = 0;
        int idx = head;
        for (int i = 0; i < n; ++i) {
            cnt += order_key(ring[idx]) >= c;
            idx = idx + 1 == cap ? 0 : idx + 1;
        }
        if (cnt >= j + 1) K = c;
    }
    return from_order_key(K);
}
MG_HD double select_jth_largest(const double* vals, int n, int j) { return ring_jth_largest(vals, n, 0, n, j); }

// nearest rank index from the top: rank = clamp(ceil(q*n), 1, n) (telemetry.cpp:52-55)
MG_HD int nr_from_top(double q, int n) {
    long rank = static_cast<long>(ceil(fmul(q, static_cast<double>(n))));
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    return n - static_cast<int>(rank);
}

MG_HD double tw_quantile(TailWin& w, double q) {
    const int j = nr_from_top(q, w.n);
    if (j < w.m) return w.top[j];
    if (j < kTopK) {
        tw_rebuild(w);
        return w.top[j];
    }
    // rank beyond the cache (q far below the tail, or windows longer than ~8/(1-q)): linear selection
    return ring_jth_largest(w.ring, w.cap, w.head, w.n, j);
}

// ---------------------------------------------------------------------------------------------
// pending action (control::Action, controller.hpp:46-58)
struct Action {
    int32_t kind, tenant, target, diagnosis;
    int32_t new_host, new_gpu, new_first, new_count, new_profile;
    int32_t pin_cpu, restore_throttle, valid;
    double throttle_Bps, quota_pct, expires_at_s;
};

// per-tenant controller state (Controller::TenantCtl, controller.hpp:167-195)
struct TenantCtl {
    TailWin win;
    double* vwin;  // validation window storage (capacity validation_obs)
    int32_t vn;
    int32_t breach_windows, next_rung, acted_ever, backfired, none_logged, relax_blocked, validating, drain_seen;
    int32_t action_seq, prior_host, prior_gpu, prior_first, prior_count, prior_profile, ema_has, ema_trig;
    uint32_t obs_in_window, obs_since_action, relax_run, obs_total;  // 32-bit: < 2^32 per run
    double window_end_s, ignore_before_s, validation_start_s, pre_p99_ms, ema, trigger, clear;
    int32_t app_kind, app_target, app_diag, pad;
};

// per-tenant engine state (TenantState + TenantRt, model.hpp:164-176, engine.cpp:89-129)
struct TenantDyn {
    int32_t host, gpu, first, count, profile, cpu_pinned, paused, transferring, computing, has_throttle;
    int32_t n_arrived, tq_head, cq_head, cur_compute, irq_cursor, pend_kind, has_pend, mt_p, mt_init, pad;
    double mps_quota, io_throttle, paused_until;
    double remaining, started_s, transfer_ms, last_settle, grant;
    double compute_done_ms, svc_ms, extra_ms, compute_end, cur_transfer_ms;
    double pend_pause;
    uint32_t completed, n_window, misses, pad_c;  // 32-bit counters (widened in finish)
    double sum_total;
    double win_min, win_max;
    int64_t base;   // offset of this tenant's records inside the replica's arrays
    int32_t n_count, root;  // root: canonical PCIe root of the current placement
    double frac;    // sm_fraction of the current (gpu, profile) (engine.cpp:330-334)
    double cap_eff; // effective_pcie_cap_Bps of the current throttle state (model.cpp:155-159)
    double obs_lat, obs_arrived;  // the completion handed to the deferred controller step (kOpObserve)
};

MG_HD int __popcll_hd(uint64_t m) {
#if defined(__CUDA_ARCH__)
    return __popcll(static_cast<unsigned long long>(m));
#else
    return __builtin_popcountll(m);
#endif
}

// per_thread: the replica is run by this thread alone (SIMT kernel, host harness); otherwise the
// handlers run warp-uniformly (every lane executes them) and one lane counts.
MG_HD void hist_add(uint32_t* p, bool per_thread = false) {
#if defined(__CUDA_ARCH__)
    if (per_thread || (threadIdx.x & 31) == 0) atomicAdd(p, 1u);  // result unused: a fire-and-forget RED
#else
    (void)per_thread;
    *p += 1;
#endif
}

// Execution model of a Lanes type: kPerThread = one thread runs one replica (no warp redundancy).
// kDefer: the hot handlers queue the pipeline helpers as continuation ops (one copy each in the
// event loop: the instruction-fetch-bound saturated regime) instead of inlining them per call site
// (the latency-bound regime, where the op loop's extra instructions sit on the critical path).
template <class Lanes>
struct LanesTraits {
    static constexpr bool kPerThread = false;
    static constexpr bool kDefer = true;
};

MG_HD void prefetch_l1(const void* p) {
#if defined(__CUDA_ARCH__)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
    (void)p;
#endif
}

// Grant cache of a root: the bandwidth split of reallocate_root (PS shares + water-filling,
// fabric.cpp:31-87) is a pure function of the active flow set, given the root capacity, the flow
// weights and the tenants' effective PCIe caps; the caps change only in Sim::refresh, which empties
// every cache.  Replaying a cached split writes the identical doubles.  Direct-mapped on the mask.
#ifndef MG_GC_ENTRIES
#define MG_GC_ENTRIES 4
#endif
constexpr int kGcEntries = MG_GC_ENTRIES, kGcFlows = 4;
struct RootDyn {
    uint64_t active;  // tenant bitmask, iteration in id order == sorted root.active
    uint64_t gc_mask[kGcEntries];           // cached active sets (0 = empty entry)
    double gc_grant[kGcEntries][kGcFlows];  // their grants, members in id order
};
MG_HD int gc_entry(uint64_t m) { return static_cast<int>((m ^ (m >> 2) ^ (m >> 5) ^ (m >> 11)) & (kGcEntries - 1)); }

struct Slot {
    double t;
    uint64_t key;  // (kind << 48) | seq ; ~0 when empty
};

// Everything one replica mutates; lives in shared memory on the device.
// (The clock, the push counter and the live-slot masks are Sim members instead: registers on
// the device.)
struct SimState {
    int32_t n_actions, n_pauses, error, next_action_seq;
    int32_t tick_index, pad;
    int64_t done_seq;  // completions so far (order of the requests.csv stream)
    TenantDyn* td;   // n_tenants
    TenantCtl* ctl;  // n_tenants
    RootDyn* rd;     // n_roots
};

// Byte layout of one replica's working set: [SimState][TenantDyn*T][TenantCtl*T][RootDyn*R]
// [Slot*(5T+1)] then, when `rings` is set, the controller windows [T*W] and validation windows [T*V].
struct SimLayout {
    int64_t td, ctl, rd, slots, win, vwin, total;
    // read-only scenario tables copied to shared memory (device only)
    int64_t sc_tn, sc_gp, sc_rt, sc_iq, sc_hio, sc_ctrl, st;
};
MG_HD int64_t align16(int64_t x) { return (x + 15) & ~static_cast<int64_t>(15); }
// global_tables: the read-only scenario tables stay in global memory (read through L1 by every
// replica of the SM; sc_* = -1) and only the PController is staged -- for the T > 10 kernel, where a
// per-replica copy of 64 PTenant rows (30 KB) caps the DES at 3 replicas per SM.
MG_HD SimLayout sim_layout(int T, int R, int W, int V, bool rings, int G = 0, int I = 0, int H = 0,
                           bool global_tables = false) {
    SimLayout L;
    int64_t o = 0;
    if (global_tables) {
        L.sc_tn = L.sc_gp = L.sc_rt = L.sc_iq = L.sc_hio = -1;
    } else {
        L.sc_tn = o;
        o = align16(o + static_cast<int64_t>(sizeof(PTenant)) * T);
        L.sc_gp = o;
        o = align16(o + static_cast<int64_t>(sizeof(PGpu)) * G);
        L.sc_rt = o;
        o = align16(o + static_cast<int64_t>(sizeof(PRoot)) * R);
        L.sc_iq = o;
        o = align16(o + static_cast<int64_t>(sizeof(PIrq)) * I);
        L.sc_hio = o;
        o = align16(o + 8ll * H);
    }
    L.sc_ctrl = o;
    o = align16(o + static_cast<int64_t>(sizeof(PController)));
    if (G == 0) o = 0;  // host harness: no copies
    L.st = o;
    o = align16(o + sizeof(SimState));
    L.td = o;
    o = align16(o + static_cast<int64_t>(sizeof(TenantDyn)) * T);
    L.ctl = o;
    o = align16(o + static_cast<int64_t>(sizeof(TenantCtl)) * T);
    L.rd = o;
    o = align16(o + static_cast<int64_t>(sizeof(RootDyn)) * R);
    L.slots = o;
    o = align16(o + static_cast<int64_t>(sizeof(Slot)) * (kEvKinds * T + 1));
    L.win = o;
    if (rings) o = align16(o + 8ll * T * W);
    L.vwin = o;
    if (rings) o = align16(o + 8ll * T * V);
    L.total = o;
    return L;
}

// ---------------------------------------------------------------------------------------------
// The replica simulator.  `Lanes` abstracts the warp: on the device all 32 lanes execute this
// code redundantly on identical shared-memory state, with the event-slot argmin done lane-parallel.
// Tenant-set words: 32-bit when the lane-register event slots are used (T <= 10), else 64-bit.
template <class Lanes>
struct MaskOf {
    using type = uint64_t;
};

template <class Lanes>
struct Sim {
    using Mask = typename MaskOf<Lanes>::type;
    const PScenario& S;
    const PController& C;
    ReplicaIO io;
    SimState& st;
    Lanes lanes;  // owns the 5T+1 event slots (host: an array; device: lane registers or smem)
    int T;
    // per-event scalars kept out of shared memory (registers once inlined into the kernel)
    double now;
    uint32_t next_seq, n_events;  // seq < 2^29 is checked in finish
    // hot scenario scalars held in registers (PScenario itself stays in global memory)
    double measure_start;
    int n_irq, redistribute;
    Mask live_resume, live_expire;  // tenants with a live resume / guardrail-expire event
    // Continuation ops (warp-uniform registers).  The hot handlers do not inline the shared
    // pipeline helpers at each call site; they queue them, and the event loop runs every queued op
    // from ONE copy of each helper (run_ops), so the event loop's instruction working set holds one
    // reallocate_root / start_compute / start_transfer instead of 3 / 2 / 2 inlined copies (the
    // saturated-regime DES is instruction-fetch bound).  An op is
    // (code << 7 | arg) in a 10-bit field; `ops` runs front (low bits) first; ops queued while an
    // op runs go to `cont` and run before the rest of `ops`, so the order of every state change and
    // push is exactly the nested-call order of the reference.  At most 3 ops are ever pending (a
    // transfer completion queues 3; only the last of them, a start_transfer, queues more, <= 2).
    uint32_t ops, cont;
    int n_cont;
    // Working-set arrays held as registers (not re-loaded from SimState) so that, after inlining
    // into the kernel, the compiler sees shared-memory provenance and emits LDS/STS.
    TenantDyn* td;
    TenantCtl* ctl;
    RootDyn* rd;
    // Scenario tables; the kernel points these at shared-memory copies (see ScenCopy).
    const PTenant* tn;
    const PGpu* gp;
    const PRoot* rt;
    const PIrq* iq;
    const double* hio;

    MG_HD Sim(const PScenario& s, const PController& c, const ReplicaIO& i, SimState& state, Lanes l,
              TenantDyn* tdp, TenantCtl* ctlp, RootDyn* rdp)
        : S(s), C(c), io(i), st(state), lanes(l), T(s.n_tenants), now(0.0), next_seq(0), n_events(0),
          live_resume(0), live_expire(0), ops(0), cont(0), n_cont(0), measure_start(s.measure_start_s), n_irq(s.n_irq),
          redistribute(s.fabric_redistribute), td(tdp), ctl(ctlp), rd(rdp), tn(s.tenants), gp(s.gpus), rt(s.roots),
          iq(s.irq), hio(s.host_io_capacity) {}

    // ---- small helpers -------------------------------------------------------------------
    MG_HD const PTenant& spec(int i) const { return tn[i]; }
    MG_HD const PGpu& gpu_of(int i) const { return gp[td[i].gpu]; }
    MG_HD int root_of(int i) const { return td[i].root; }
    // placement or throttle changed: refresh the cached derived values
    MG_HD void refresh(int i) {
        TenantDyn& d = td[i];
        d.root = gp[d.gpu].root;
        d.frac = calc_frac(i);
        const double base = spec(i).pcie_cap;
        d.cap_eff = !d.has_throttle ? base : base > 0.0 ? (d.io_throttle < base ? d.io_throttle : base) : d.io_throttle;
        for (int r = 0; r < S.n_roots; ++r)
            for (int e = 0; e < kGcEntries; ++e) rd[r].gc_mask[e] = 0;
    }
    // Slot layout: the three per-request kinds first, then the tick, then the rare kinds, so the
    // device argmin scans only 3T+1 slots while no resume/expire event is live (any_rare() false).
    MG_HD int slot_base(int kind) const {
        return kind == kEvCompute ? 0 : kind == kEvTransfer ? T : kind == kEvArrival ? 2 * T
               : kind == kEvTick ? 3 * T : kind == kEvResume ? 3 * T + 1 : 4 * T + 1;
    }
    MG_HD int slot_index(int kind, int i) const { return slot_base(kind) + (kind == kEvTick ? 0 : i); }
    MG_HD static bool rare_kind(int kind) { return kind == kEvResume || kind == kEvExpire; }
    MG_HD bool any_rare() const { return (live_resume | live_expire) != 0; }
    MG_HD void mark_rare(int kind, int i, bool live) {
        Mask& m = kind == kEvResume ? live_resume : live_expire;
        m = live ? (m | (Mask(1) << i)) : (m & ~(Mask(1) << i));
    }

    MG_HD void push(int kind, int i, double t) {
        if (rare_kind(kind)) mark_rare(kind, i, true);
        lanes.set(slot_index(kind, i), t, (static_cast<uint64_t>(kind) << 48) | static_cast<uint64_t>(next_seq));
        next_seq += 1;
    }
    MG_HD void cancel(int kind, int i) {
        if (rare_kind(kind)) mark_rare(kind, i, false);
        lanes.clear(slot_index(kind, i));
    }

    MG_HD double calc_frac(int i) const {
        const PGpu& g = gpu_of(i);
        if (!g.mig_enabled) return 1.0;
        return fdiv_exact(static_cast<double>(profile_slices(td[i].profile)), static_cast<double>(g.total_slices));
    }
    MG_HD double sm_fraction(int i) const { return td[i].frac; }
    MG_HD double eff_pcie_cap(int i) const { return td[i].cap_eff; }  // model.cpp:155-159, cached
    MG_HD uint64_t queue_len(int i) const {  // engine.cpp:245-247
        const TenantDyn& d = td[i];
        const int cq_end = d.transferring ? d.tq_head - 1 : d.tq_head;
        return static_cast<uint64_t>(d.n_arrived - d.tq_head) + static_cast<uint64_t>(cq_end - d.cq_head) +
               static_cast<uint64_t>(d.transferring ? 1 : 0) + static_cast<uint64_t>(d.computing ? 1 : 0);
    }
    MG_HD double eff_host_io(int i) const {  // engine.cpp:336-344
        const TenantDyn& d = td[i];
        if (d.paused) return 0.0;
        if (queue_len(i) == 0) return 0.0;
        double v = spec(i).host_io;
        if (d.has_throttle && d.io_throttle < v) v = d.io_throttle;
        return v;
    }
    MG_HD double tenant_pcie(int i) const { return td[i].transferring ? td[i].grant : 0.0; }
    MG_HD double tenant_sm_util(int i) const {  // engine.cpp:657-659
        const TenantDyn& d = td[i];
        if (!(d.computing && !d.paused)) return 0.0;
        return fdiv_exact(fmul(fmul(spec(i).sm_demand, sm_fraction(i)), d.mps_quota), 100.0);
    }
    MG_HD double root_offered(int r) const {
        double s = 0.0;
        for (Mask m = static_cast<Mask>(rd[r].active); m; m &= m - 1) s = fadd(s, td[ctz64(m)].grant);
        return s;
    }
    MG_HD double host_io(int h) const {
        double s = 0.0;
        for (int j = 0; j < T; ++j)
            if (td[j].host == h) s = fadd(s, eff_host_io(j));
        return s;
    }
    MG_HD double gpu_sm_util(int h, int g) const {
        double s = 0.0;
        for (int j = 0; j < T; ++j)
            if (td[j].host == h && td[j].gpu == g) s = fadd(s, tenant_sm_util(j));
        return s;
    }
    MG_HD bool irq_recent(int h, int core_group) const {  // engine.cpp:664-668
        for (int b = 0; b < n_irq; ++b) {
            const PIrq& q = iq[b];
            if (q.host == h && q.core_group == core_group &&
                sched_active_within(q.sched, fsub(now, C.irq_lookback_s), now))
                return true;
        }
        return false;
    }
    MG_HD static int ctz64(uint64_t m) {
#if defined(__CUDA_ARCH__)
        return __ffsll(static_cast<long long>(m)) - 1;
#else
        return __builtin_ctzll(m);
#endif
    }
    MG_HD static int ctz64(uint32_t m) {
#if defined(__CUDA_ARCH__)
        return __ffs(static_cast<int>(m)) - 1;
#else
        return __builtin_ctz(m);
#endif
    }

    // ---- fabric (fabric.cpp:31-87 via engine.cpp:312-347) ----------------------------------
    MG_HOT void settle_root(int r) {
        for (Mask m = static_cast<Mask>(rd[r].active); m; m &= m - 1) {
            TenantDyn& d = td[ctz64(m)];
            const double dt = fsub(now, d.last_settle);
            if (dt > 0.0 && d.grant > 0.0) {
                const double x = fsub(d.remaining, fmul(d.grant, dt));
                d.remaining = 0.0 < x ? x : 0.0;
                if (d.remaining < kEpsBytes) d.remaining = 0.0;
            }
            d.last_settle = now;
        }
    }

    MG_HOT void reallocate_root(int r) {
        const Mask act = static_cast<Mask>(rd[r].active);
        const double cap = rt[r].capacity;
        const int ge = gc_entry(act);
        const bool cacheable = __popcll_hd(act) <= kGcFlows;
        if (act && cacheable && rd[r].gc_mask[ge] == act) {
            int k = 0;
            for (Mask m = act; m; m &= m - 1) td[ctz64(m)].grant = rd[r].gc_grant[ge][k++];
        } else if (act) {
            double wsum = 0.0;
            for (Mask m = act; m; m &= m - 1) wsum = fadd(wsum, spec(ctz64(m)).weight);
            double granted = 0.0;
            for (Mask m = act; m; m &= m - 1) {
                const int i = ctz64(m);
                const double share = fdiv_exact(fmul(cap, spec(i).weight), wsum);
                const double c = eff_pcie_cap(i);
                const double b = c > 0.0 ? (c < share ? c : share) : share;
                td[i].grant = b;
                granted = fadd(granted, b);
            }
            if (redistribute) {
                double residual = fsub(cap, granted);
                for (int iter = 0; iter < 64 && residual > fmul(1e-9, cap); ++iter) {
                    double open_w = 0.0;
                    for (Mask m = act; m; m &= m - 1) {
                        const int i = ctz64(m);
                        const double c = eff_pcie_cap(i);
                        if (!(c > 0.0) || td[i].grant < fsub(c, 1e-12)) open_w = fadd(open_w, spec(i).weight);
                    }
                    if (open_w <= 0.0) break;
                    double moved = 0.0;
                    for (Mask m = act; m; m &= m - 1) {
                        const int i = ctz64(m);
                        const double c = eff_pcie_cap(i);
                        double& g = td[i].grant;
                        if (c > 0.0 && g >= fsub(c, 1e-12)) continue;
                        double add = fdiv_exact(fmul(residual, spec(i).weight), open_w);
                        if (c > 0.0) {
                            const double room = fsub(c, g);
                            add = room < add ? room : add;
                        }
                        g = fadd(g, add);
                        moved = fadd(moved, add);
                    }
                    residual = fsub(residual, moved);
                    if (moved <= fmul(1e-12, cap)) break;
                }
            }
            if (cacheable) {
                int k = 0;
                for (Mask m = act; m; m &= m - 1) rd[r].gc_grant[ge][k++] = td[ctz64(m)].grant;
                rd[r].gc_mask[ge] = act;
            }
        }
        for (Mask m = act; m; m &= m - 1) {
            const int i = ctz64(m);
            TenantDyn& d = td[i];
            d.last_settle = now;
            if (d.grant > 0.0 && d.remaining > kEpsBytes) {
                push(kEvTransfer, i, fadd(now, fdiv_exact(d.remaining, d.grant)));
            } else if (d.remaining <= kEpsBytes) {
                push(kEvTransfer, i, now);
            } else {
                cancel(kEvTransfer, i);  // starved: generation bumped, nothing scheduled
            }
        }
    }

    // ---- pipeline stages (engine.cpp:349-420) --------------------------------------------
    MG_HD bool irq_exposed(int i) const {
        const TenantDyn& d = td[i];
        if (d.cpu_pinned) return false;
        const PGpu& g = gpu_of(i);
        for (int b = 0; b < n_irq; ++b) {
            const PIrq& q = iq[b];
            if (q.host == d.host && q.core_group == g.core_group && sched_active(q.sched, now)) return true;
        }
        return false;
    }

    MG_HOT void start_compute(int i) {
        TenantDyn& d = td[i];
        const int cq_end = d.transferring ? d.tq_head - 1 : d.tq_head;
        if (d.computing || d.paused || d.cq_head >= cq_end) return;
        const int64_t base = d.base;
        const int k = d.cq_head++;
        const double frac = sm_fraction(i);
        double service = fdiv_exact(fmul(spec(i).base_compute_ms, io.arr_mult[base + k]), frac);
        const PGpu& g = gpu_of(i);
        if (!g.mig_enabled) {
            service = fmul(service, fdiv_exact(100.0, d.mps_quota));
            double pressure = 0.0;
            for (int j = 0; j < T; ++j) {
                if (j == i) continue;
                const TenantDyn& o = td[j];
                if (o.paused) continue;
                if (o.host != d.host || o.gpu != d.gpu) continue;
                if (!o.computing) continue;
                pressure = fadd(pressure, fdiv_exact(fmul(spec(j).sm_demand, o.mps_quota), 100.0));
            }
            service = fmul(service, fadd(1.0, fmul(kMpsKappa, pressure)));
        }
        double extra = io.arr_noise[base + k];
        if (irq_exposed(i)) {
            for (int b = 0; b < n_irq; ++b) {
                const PIrq& q = iq[b];
                if (q.host == d.host && q.core_group == g.core_group) {
                    if (q.extra_noise_ms > 0.0) {
                        const double e = io.irq_e[base + d.irq_cursor];
                        d.irq_cursor += 1;
                        extra = fadd(extra, fdiv_exact(e, q.lambda));
                    }
                    break;
                }
            }
        }
        d.cur_compute = k;
        d.computing = 1;
        d.svc_ms = service;
        d.extra_ms = extra;
        d.compute_done_ms = 0.0;
        d.cur_transfer_ms = io.req_transfer_ms[base + k];
        d.compute_end = fadd(now, fdiv_exact(fadd(service, extra), 1000.0));
        push(kEvCompute, i, d.compute_end);
    }

    // kDefer: the tail calls are queued as continuation ops (hot callers); otherwise run in place
    template <bool kDefer>
    MG_HD void start_transfer_t(int i) {
        TenantDyn& d = td[i];
        if (d.transferring || d.paused) return;
        const int64_t base = d.base;
        while (d.tq_head < d.n_arrived) {
            const int k = d.tq_head++;
            const double bytes = io.arr_bytes[base + k];
            if (bytes <= 0.0) {
                io.req_transfer_ms[base + k] = 0.0;
                if (kDefer) {  // start_compute, then this loop again (re-entry sees the same flags)
                    then(kOpStartCompute, i);
                    then(kOpStartTransfer, i);
                    return;
                }
                start_compute(i);
                continue;
            }
            d.started_s = now;
            d.remaining = bytes;
            d.transfer_ms = 0.0;
            d.transferring = 1;
            const int r = root_of(i);
            settle_root(r);
            rd[r].active |= 1ull << i;
            if (kDefer) then(kOpRealloc, r);
            else reallocate_root(r);
            return;
        }
    }
    MG_HOT void start_transfer(int i) { start_transfer_t<false>(i); }

    // ---- continuation ops ----------------------------------------------------------------
    enum : uint32_t { kOpRealloc = 1, kOpStartCompute = 2, kOpStartTransfer = 3, kOpObserve = 4 };
    MG_HD void then(uint32_t code, int arg) {  // arg: a tenant (< 64) or root (< 16) index
        cont |= ((code << 7) | static_cast<uint32_t>(arg)) << (10 * n_cont);
        n_cont += 1;
    }
    // the deferred controller step of a completion (engine.cpp:497-503: on_observation, then the
    // returned action is applied)
    MG_HD void observe(int i) {
        const TenantDyn& d = td[i];
        Action a = on_observation(i, d.obs_lat, now, d.obs_arrived);
        if (a.valid) apply_action(a);
    }
    MG_HD void run_op(uint32_t code, int arg) {  // if-chain in frequency order: no indirect branch
        if (code == kOpRealloc) reallocate_root(arg);
        else if (code == kOpStartCompute) start_compute(arg);
        else if (code == kOpStartTransfer) start_transfer_t<LanesTraits<Lanes>::kDefer>(arg);
        else observe(arg);
    }
    // a helper call of a hot handler: queued (kDefer) or run in place (`code` is a literal at every
    // call site, so the in-place form folds to the one helper)
    MG_HD void call(uint32_t code, int arg) {
        if (LanesTraits<Lanes>::kDefer) then(code, arg);
        else run_op(code, arg);
    }
    // run the ops the handler queued, depth first
    MG_HD void run_ops() {
        ops = cont;
        cont = 0;
        n_cont = 0;
        while (ops) {
            const uint32_t code = (ops >> 7) & 7u;
            const int arg = static_cast<int>(ops & 0x7fu);
            ops >>= 10;
            run_op(code, arg);
            if (n_cont) {
                if (n_cont > 3 || (ops >> (30 - 10 * n_cont)) != 0) st.error = kErrOpOverflow;
                ops = cont | (ops << (10 * n_cont));
                cont = 0;
                n_cont = 0;
            }
        }
    }

    // ---- event handlers (engine.cpp:422-782) ---------------------------------------------
    MG_HD void on_arrival(int i) {
        TenantDyn& d = td[i];
        const int k = d.n_arrived;
        // (no software prefetch of the arrival records: an L1 prefetch per 16 records measured 2%
        //  slower than letting the in-order loads miss)
        d.n_arrived = k + 1;
        // start_transfer is deferred past the next-arrival push: only same-kind pushes compare by
        // seq, and their relative order is unchanged
        if (d.n_arrived < d.n_count) push(kEvArrival, i, io.arr_t[d.base + d.n_arrived]);
        call(kOpStartTransfer, i);
    }

    MG_HD void on_transfer_complete(int i) {
        TenantDyn& d = td[i];
        const int r = root_of(i);
        settle_root(r);
        const double rem = d.remaining;
        const bool done =
            rem <= kEpsBytes || (d.grant > 0.0 && fadd(now, fdiv_exact(rem, d.grant)) <= now);
        if (!done) {
            call(kOpRealloc, r);
            return;
        }
        d.remaining = 0.0;
        d.transferring = 0;
        const int k = d.tq_head - 1;
        io.req_transfer_ms[d.base + k] = fadd(d.transfer_ms, fmul(fsub(now, d.started_s), 1000.0));
        rd[r].active &= ~(1ull << i);
        d.grant = 0.0;
        call(kOpRealloc, r);
        call(kOpStartCompute, i);
        call(kOpStartTransfer, i);
    }

    MG_HD void on_compute_complete(int i) {
        TenantDyn& d = td[i];
        d.computing = 0;
        const int64_t base = d.base;
        const int k = d.cur_compute;
        const double arrived = io.arr_t[base + k];
        double total = fmul(fsub(now, arrived), 1000.0);
        const double compute = fadd(d.compute_done_ms, d.svc_ms);
        const double transfer = d.cur_transfer_ms;
        double noise = fsub(fsub(total, compute), transfer);
        if (noise < 0.0 && noise > -1e-9) noise = 0.0;
        total = fadd(fadd(compute, transfer), noise);
        const uint64_t idx = d.completed;
        d.completed += 1;
        if (now >= measure_start) {
            io.win_lat[base + static_cast<int64_t>(d.n_window)] = total;
            d.n_window += 1;
            d.sum_total = fadd(d.sum_total, total);
            if (total < d.win_min) d.win_min = total;
            if (total > d.win_max) d.win_max = total;
            if (total > spec(i).slo_tail_ms) d.misses += 1;
            if (io.win_hist)
                hist_add(io.win_hist + static_cast<int64_t>(i) * kHistBins + lat_bin(total), LanesTraits<Lanes>::kPerThread);
        }
        if (io.c_total) {
            const int64_t o = base + static_cast<int64_t>(idx);
            io.c_done[o] = now;
            io.c_total[o] = total;
            io.c_compute[o] = compute;
            io.c_transfer[o] = transfer;
            io.c_noise[o] = noise;
            if (io.c_order) io.c_order[o] = st.done_seq;
        }
        st.done_seq += 1;
        if (io.tr_win) tw_push(io.tr_win[i], total);
        call(kOpStartCompute, i);
        if (C.enabled) {
            d.obs_lat = total;
            d.obs_arrived = arrived;
            call(kOpObserve, i);
        }
    }

    // counters.csv / fabric.csv rows of tick j (engine.cpp:746-775)
    MG_HD void trace_tick(int j) {
        for (int r = 0; r < S.n_roots; ++r) {
            double backlog = 0.0;
            for (int i = 0; i < T; ++i) {
                const TenantDyn& d = td[i];
                if (d.host != rt[r].host || root_of(i) != r) continue;
                if (d.transferring) backlog = fadd(backlog, d.remaining);
                for (int k = d.tq_head; k < d.n_arrived; ++k) backlog = fadd(backlog, io.arr_bytes[d.base + k]);
            }
            FabricRow& f = io.tr_fab[static_cast<int64_t>(j) * S.n_roots + r];
            f.offered_Bps = root_offered(r);
            f.backlog_bytes = backlog;
            f.active_flows = __popcll_hd(rd[r].active);
            f.pad = 0;
        }
        for (int i = 0; i < T; ++i) {
            const TenantDyn& d = td[i];
            CounterRow& c = io.tr_cnt[static_cast<int64_t>(j) * T + i];
            c.completed = d.completed;
            c.queue_len = queue_len(i);
            c.window_p99_ms = io.tr_win[i].n > 0 ? tw_quantile(io.tr_win[i], 0.99) : 0.0;
            c.grant_Bps = d.transferring ? d.grant : 0.0;
            c.profile = d.profile;
            c.host = d.host;
            c.gpu_id = gp[d.gpu].id;
            c.pad = 0;
        }
    }

    MG_HD void on_tick() {
        const int third = S.n_ticks / 3;
        const int j = st.tick_index++;
        if (io.tr_cnt) trace_tick(j);
        if (S.n_ticks >= 10 && third > 0) {
            for (int r = 0; r < S.n_roots; ++r) {
                const bool in_first = j < third, in_last = j >= S.n_ticks - third;
                if (!in_first && !in_last) continue;
                double backlog = 0.0;
                for (int i = 0; i < T; ++i) {
                    const TenantDyn& d = td[i];
                    if (d.host != rt[r].host || root_of(i) != r) continue;
                    if (d.transferring) backlog = fadd(backlog, d.remaining);
                    const int64_t base = d.base;
                    for (int k = d.tq_head; k < d.n_arrived; ++k) backlog = fadd(backlog, io.arr_bytes[base + k]);
                }
                if (in_first) io.backlog[2 * r] = fadd(io.backlog[2 * r], backlog);
                if (in_last) io.backlog[2 * r + 1] = fadd(io.backlog[2 * r + 1], backlog);
            }
        }
        const double nt = fadd(now, 1.0);
        if (nt <= S.duration_s) push(kEvTick, 0, nt);
    }

    // ---- pause / actuation (engine.cpp:553-742) --------------------------------------------
    MG_HD double pause_draw(int i, double mean, double sd, double lo, double hi) {
        TenantDyn& d = td[i];
        Mt64Ref g{io.mt_pause + static_cast<int64_t>(i) * kMtN, d.mt_p};
        if (!d.mt_init) {
            g.seed(substream_seed(io.seed, spec(i).name_hash, kPause));
            d.mt_init = 1;
        }
        const double v = truncated_normal_draw(g, mean, sd, lo, hi);
        d.mt_p = g.p;
        return v;
    }

    MG_HD void pause_tenant(int i, double duration, int cause_kind) {
        TenantDyn& d = td[i];
        if (d.transferring) {
            const int r = root_of(i);
            settle_root(r);
            rd[r].active &= ~(1ull << i);
            d.grant = 0.0;
            cancel(kEvTransfer, i);
            if (d.started_s >= 0.0) {
                d.transfer_ms = fadd(d.transfer_ms, fmul(fsub(now, d.started_s), 1000.0));
                d.started_s = -1.0;
            }
            reallocate_root(r);
        }
        if (d.computing) {
            const double rm = fmul(fsub(d.compute_end, now), 1000.0);
            const double remaining_ms = 0.0 < rm ? rm : 0.0;
            const double stage = fadd(d.svc_ms, d.extra_ms);
            const double frac = stage > 0.0 ? fdiv_exact(remaining_ms, stage) : 0.0;
            const double rem_service = fmul(d.svc_ms, frac);
            d.compute_done_ms = fadd(d.compute_done_ms, fsub(d.svc_ms, rem_service));
            d.svc_ms = fmul(rem_service, sm_fraction(i));
            d.extra_ms = fmul(d.extra_ms, frac);
            cancel(kEvCompute, i);
        }
        d.paused = 1;
        d.paused_until = fadd(now, duration);
        if (st.n_pauses < io.pause_cap) {
            PauseRec& p = io.pauses[st.n_pauses];
            p.t_s = now;
            p.duration_s = duration;
            p.tenant = i;
            p.kind = cause_kind;
        } else {
            st.error = kErrPauseOverflow;
        }
        st.n_pauses += 1;
        d.has_pend = 1;
        d.pend_kind = cause_kind;
        d.pend_pause = duration;
        push(kEvResume, i, d.paused_until);
    }

    MG_HD void on_resume(int i) {
        TenantDyn& d = td[i];
        d.paused = 0;
        if (d.computing) {
            const double service = fdiv_exact(d.svc_ms, sm_fraction(i));
            d.svc_ms = service;
            d.compute_end = fadd(now, fdiv_exact(fadd(service, d.extra_ms), 1000.0));
            push(kEvCompute, i, d.compute_end);
        }
        if (d.transferring) {
            d.started_s = now;
            const int r = root_of(i);
            settle_root(r);
            rd[r].active |= 1ull << i;
            reallocate_root(r);
        }
        start_transfer(i);
        start_compute(i);
        if (d.has_pend) {
            d.has_pend = 0;
            on_action_applied(i, d.pend_kind, now, d.pend_pause);
        }
    }

    MG_HD void on_guardrail_expire(int i) {
        TenantDyn& d = td[i];
        int kind;
        if (d.has_throttle) {
            d.has_throttle = 0;
            refresh(i);
            kind = kActIoThrottle;
        } else if (d.mps_quota < 100.0) {
            d.mps_quota = 100.0;
            kind = kActMpsQuota;
        } else {
            return;
        }
        if (d.transferring) {
            const int r = root_of(i);
            settle_root(r);
            reallocate_root(r);
        }
        // Controller::on_guardrail_expired (controller.cpp:625-635)
        ActionRec* rec = new_record();
        if (rec) {
            rec->kind = kActExpire;
            rec->tenant = i;
            rec->target = i;
            rec->diagnosis = kDiagNone;
            rec->expire_kind = kind;
            rec->t_s = now;
        }
    }

    MG_HD void apply_action(const Action& a) {
        TenantDyn& tgt = td[a.target];
        switch (a.kind) {
            case kActIoThrottle: {
                tgt.has_throttle = 1;
                tgt.io_throttle = a.throttle_Bps;
                refresh(a.target);
                push(kEvExpire, a.target, a.expires_at_s);
                if (tgt.transferring) {
                    const int r = root_of(a.target);
                    settle_root(r);
                    reallocate_root(r);
                }
                on_action_applied(a.tenant, a.kind, now, 0.0);
                break;
            }
            case kActMpsQuota: {
                tgt.mps_quota = a.quota_pct;
                push(kEvExpire, a.target, a.expires_at_s);
                on_action_applied(a.tenant, a.kind, now, 0.0);
                break;
            }
            case kActMove: {
                const double pause = pause_draw(a.tenant, 9.0, 3.0, 2.5, 15.0);
                pause_tenant(a.tenant, pause, a.kind);
                TenantDyn& d = td[a.tenant];
                d.host = a.new_host;
                d.gpu = a.new_gpu;
                d.first = a.new_first;
                d.count = a.new_count;
                if (a.pin_cpu) d.cpu_pinned = 1;
                refresh(a.tenant);
                break;
            }
            case kActMigUp:
            case kActMigDown: {
                const double pause = pause_draw(a.tenant, 18.0, 6.0, 5.0, 30.0);
                pause_tenant(a.tenant, pause, a.kind);
                TenantDyn& d = td[a.tenant];
                d.host = a.new_host;
                d.gpu = a.new_gpu;
                d.first = a.new_first;
                d.count = a.new_count;
                d.profile = a.new_profile;
                refresh(a.tenant);
                break;
            }
            case kActRollback: {
                if (a.restore_throttle) {
                    tgt.has_throttle = 0;
                    refresh(a.target);
                    tgt.mps_quota = 100.0;
                    cancel(kEvExpire, a.target);
                    if (tgt.transferring) {
                        const int r = root_of(a.target);
                        settle_root(r);
                        reallocate_root(r);
                    }
                    on_action_applied(a.tenant, a.kind, now, 0.0);
                    break;
                }
                TenantDyn& d = td[a.tenant];
                const bool profile_change = d.profile != a.new_profile;
                const double pause = profile_change ? pause_draw(a.tenant, 18.0, 6.0, 5.0, 30.0)
                                                    : pause_draw(a.tenant, 9.0, 3.0, 2.5, 15.0);
                pause_tenant(a.tenant, pause, a.kind);
                d.host = a.new_host;
                d.gpu = a.new_gpu;
                d.first = a.new_first;
                d.count = a.new_count;
                d.profile = a.new_profile;
                refresh(a.tenant);
                break;
            }
            default:
                break;
        }
    }

    // ---- controller (controller.cpp) -----------------------------------------------------
    MG_HD ActionRec* new_record() {
        const int seq = st.next_action_seq++;
        if (st.n_actions >= io.action_cap) {
            st.error = kErrActionOverflow;
            st.n_actions += 1;
            return nullptr;
        }
        ActionRec* r = &io.actions[st.n_actions];
        st.n_actions += 1;
        r->seq = seq;
        r->kind = kActNone;
        r->tenant = r->target = -1;
        r->diagnosis = kDiagNone;
        r->breach_windows = 0;
        r->rolled_back_seq = -1;
        r->expire_kind = 0;
        r->new_host = r->new_gpu_id = r->new_first = r->new_end = r->new_profile = -1;
        r->pad = 0;
        r->obs_since_prev = 0;
        r->t_s = r->p99_pre_ms = r->ema_p99_ms = r->throttle_Bps = r->quota_pct = r->pause_s = 0.0;
        return r;
    }

    // Controller::record (controller.cpp:347-399); returns the record seq
    MG_HD int record(const Action& a, double t, TenantCtl& c) {
        ActionRec* r = new_record();
        const int seq = st.next_action_seq - 1;
        if (!r) return seq;
        r->t_s = t;
        r->tenant = a.tenant;
        r->target = a.target;
        r->kind = a.kind;
        r->diagnosis = a.diagnosis;
        r->p99_pre_ms = c.win.n > 0 ? tw_quantile(c.win, 0.99) : 0.0;
        r->ema_p99_ms = c.ema_has ? c.ema : 0.0;
        r->breach_windows = c.breach_windows;
        r->obs_since_prev = c.acted_ever ? c.obs_since_action : c.obs_total;
        if (a.kind == kActIoThrottle) r->throttle_Bps = a.throttle_Bps;
        if (a.kind == kActMpsQuota) r->quota_pct = a.quota_pct;
        if (a.kind == kActMove || a.kind == kActMigUp || a.kind == kActMigDown || a.kind == kActRollback) {
            if (!(a.kind == kActRollback && a.restore_throttle)) {
                r->new_host = a.new_host;
                r->new_gpu_id = a.new_gpu >= 0 ? gp[a.new_gpu].id : -1;
                r->new_first = a.new_first;
                r->new_end = a.new_first + a.new_count;
                r->new_profile = a.new_profile;
            }
        }
        return seq;
    }

    MG_HD void reset_signal(TenantCtl& c, double t) {  // controller.cpp:154-164
        tw_reset(c.win, c.trigger);
        c.ema_has = 0;
        c.ema_trig = 0;
        c.breach_windows = 0;
        c.obs_in_window = 0;
        c.relax_run = 0;
        c.window_end_s = fadd(t, C.sample_interval_s);
    }

    MG_HD void ema_update(TenantCtl& c, double x) {  // telemetry.cpp:81-95
        if (!c.ema_has) {
            c.ema = x;
            c.ema_has = 1;
        } else {
            c.ema = fadd(fmul(C.ema_alpha, x), fmul(fsub(1.0, C.ema_alpha), c.ema));
        }
        if (!c.ema_trig && c.ema > c.trigger) c.ema_trig = 1;
        else if (c.ema_trig && c.ema < c.clear) c.ema_trig = 0;
    }

    // find_slice_run (controller.cpp:72-99); returns first or -1
    MG_HD int find_slice_run(int gidx, int host, int count, int prefer, int ignore) const {
        const PGpu& g = gp[gidx];
        if (count <= 0 || count > g.total_slices) return -1;
        uint64_t used = 0;
        for (int j = 0; j < T; ++j) {
            if (j == ignore) continue;
            const TenantDyn& o = td[j];
            if (o.host != host || o.gpu != gidx) continue;
            for (int s = o.first; s < o.first + o.count; ++s)
                if (s >= 0 && s < g.total_slices) used |= 1ull << s;
        }
        auto fits = [&](int first) {
            if (first < 0 || first + count > g.total_slices) return false;
            for (int s = first; s < first + count; ++s)
                if (used >> s & 1ull) return false;
            return true;
        };
        if (prefer >= 0 && fits(prefer)) return prefer;
        for (int f = 0; f + count <= g.total_slices; ++f)
            if (fits(f)) return f;
        return -1;
    }

    // placement_score(...).total() (controller.cpp:101-123)
    MG_HD double placement_score(int i, int host, int gidx) const {
        const PGpu& g = gp[gidx];
        const double root_cap = rt[g.root].capacity;
        const double io_cap = hio[host];
        double pcie = 0.0, numa = 0.0, irq = 0.0;
        for (int j = 0; j < T; ++j) {
            if (j == i) continue;
            const TenantDyn& o = td[j];
            if (o.host != host) continue;
            const PGpu& og = gp[o.gpu];
            if (spec(j).tclass == kBandwidthHeavy && og.root == g.root) pcie = fadd(pcie, fdiv_exact(tenant_pcie(j), root_cap));
            if (og.numa == g.numa) numa = fadd(numa, fdiv_exact(eff_host_io(j), io_cap));
        }
        if (irq_recent(host, g.core_group)) irq = 1.0;
        return fadd(fadd(pcie, numa), irq);
    }

    MG_HD int diagnose(int i) const {  // controller.cpp:171-189
        const TenantDyn& d = td[i];
        const int r = root_of(i);
        const double root_util = fdiv_exact(root_offered(r), rt[r].capacity);
        const double io_util = fdiv_exact(host_io(d.host), hio[d.host]);
        if (root_util > C.diag_pcie_util_threshold || io_util > C.diag_host_io_threshold) return kDiagIo;
        const double gu = gpu_sm_util(d.host, d.gpu);
        const double own = tenant_sm_util(i);
        if (fsub(gu, own) > C.diag_sm_util_threshold) return kDiagCompute;
        return kDiagNone;
    }

    MG_HD Action no_action() const {
        Action a;
        a.valid = 0;
        a.kind = kActNone;
        a.tenant = a.target = -1;
        a.diagnosis = kDiagNone;
        a.new_host = a.new_gpu = a.new_first = a.new_count = a.new_profile = -1;
        a.pin_cpu = a.restore_throttle = 0;
        a.throttle_Bps = 0.0;
        a.quota_pct = 100.0;
        a.expires_at_s = 0.0;
        return a;
    }

    MG_HD Action try_guardrail(int i, int diag) {  // controller.cpp:191-257
        const TenantDyn& d = td[i];
        Action a = no_action();
        if (diag == kDiagIo) {
            const int myroot = root_of(i);
            const bool io_disjunct =
                fdiv_exact(host_io(d.host), hio[d.host]) > C.diag_host_io_threshold;
            int off = -1;
            double best = 0.0;
            for (int j = 0; j < T; ++j) {
                if (j == i) continue;
                if (spec(j).tclass == kLatencySensitive) continue;
                if (td[j].host != d.host) continue;
                double load;
                if (io_disjunct) {
                    load = eff_host_io(j);
                } else {
                    if (root_of(j) != myroot) continue;
                    load = tenant_pcie(j);
                }
                if (load > best) {
                    best = load;
                    off = j;
                }
            }
            if (off < 0 || best <= 0.0) return a;
            if (td[off].has_throttle) return a;
            a.valid = 1;
            a.kind = kActIoThrottle;
            a.tenant = i;
            a.target = off;
            a.diagnosis = diag;
            a.throttle_Bps = C.guardrail_io_throttle_Bps;
            a.expires_at_s = fadd(now, C.throttle_duration_s);
            return a;
        }
        if (diag == kDiagCompute) {
            if (gpu_of(i).mig_enabled) return a;
            int off = -1;
            double best = 0.0;
            for (int j = 0; j < T; ++j) {
                if (j == i) continue;
                if (spec(j).tclass == kLatencySensitive) continue;
                if (td[j].host != d.host || td[j].gpu != d.gpu) continue;
                const double u = tenant_sm_util(j);
                if (u > best) {
                    best = u;
                    off = j;
                }
            }
            if (off < 0) return a;
            if (td[off].mps_quota < 100.0) return a;
            a.valid = 1;
            a.kind = kActMpsQuota;
            a.tenant = i;
            a.target = off;
            a.diagnosis = diag;
            a.quota_pct = C.guardrail_mps_quota_pct;
            a.expires_at_s = fadd(now, C.quota_duration_s);
            return a;
        }
        return a;
    }

    MG_HD Action try_move(int i) {  // controller.cpp:259-303
        const TenantDyn& d = td[i];
        Action a = no_action();
        const double current = placement_score(i, d.host, d.gpu);
        const double claim = spec(i).claim;
        int best_g = -1, best_first = -1;
        double best_score = 0.0;
        for (int g = 0; g < S.n_gpus; ++g) {
            const PGpu& cg = gp[g];
            const int host = cg.host;
            if (host == d.host && g == d.gpu) continue;
            const int run = find_slice_run(g, host, d.count, -1, i);
            if (run < 0) continue;
            double claims = claim;
            for (int j = 0; j < T; ++j) {
                if (j == i) continue;
                if (td[j].host != host) continue;
                if (root_of(j) != cg.root) continue;
                claims = fadd(claims, spec(j).claim);
            }
            if (claims >= rt[cg.root].capacity) continue;
            const double score = placement_score(i, host, g);
            bool take = best_g < 0 || score < best_score;
            if (!take && score == best_score) {
                const PGpu& bg = gp[best_g];
                take = host < bg.host || (host == bg.host && (cg.id < bg.id || (cg.id == bg.id && run < best_first)));
            }
            if (take) {
                best_g = g;
                best_first = run;
                best_score = score;
            }
        }
        if (best_g < 0) return a;
        if (fsub(current, best_score) < C.move_margin) return a;
        a.valid = 1;
        a.kind = kActMove;
        a.tenant = i;
        a.target = i;
        a.new_host = gp[best_g].host;
        a.new_gpu = best_g;
        a.new_first = best_first;
        a.new_count = d.count;
        a.new_profile = d.profile;
        a.pin_cpu = 1;
        return a;
    }

    MG_HD Action try_mig_up(int i) {  // controller.cpp:305-319
        const TenantDyn& d = td[i];
        Action a = no_action();
        if (d.profile + 1 >= kNumProfiles) return a;
        const int np = d.profile + 1;
        const int run = find_slice_run(d.gpu, d.host, profile_slices(np), d.first, i);
        if (run < 0) return a;
        a.valid = 1;
        a.kind = kActMigUp;
        a.tenant = i;
        a.target = i;
        a.new_host = d.host;
        a.new_gpu = d.gpu;
        a.new_first = run;
        a.new_count = profile_slices(np);
        a.new_profile = np;
        return a;
    }

    MG_HD Action try_relax(int i, TenantCtl& c) {  // controller.cpp:321-345
        const TenantDyn& d = td[i];
        Action a = no_action();
        if (d.profile == 0) return a;
        if (c.relax_blocked >= 0 && d.profile == c.relax_blocked) return a;
        if (c.win.n < C.dwell_obs) return a;
        if (c.win.n == 0) return a;
        const double m = fdiv_exact(static_cast<double>(c.win.misses), static_cast<double>(c.win.n));
        if (m > fsub(1.0, C.throughput_floor)) return a;
        const double score = placement_score(i, d.host, d.gpu);
        if (score >= C.relax_score_threshold) return a;
        const int dp = d.profile - 1;
        a.valid = 1;
        a.kind = kActMigDown;
        a.tenant = i;
        a.target = i;
        a.new_host = d.host;
        a.new_gpu = d.gpu;
        a.new_first = d.first;
        a.new_count = profile_slices(dp);
        a.new_profile = dp;
        return a;
    }

    MG_HD Action evaluate_breach(int i, TenantCtl& c) {  // controller.cpp:401-442
        const int diag = diagnose(i);
        for (int rung = c.next_rung; rung <= 2; ++rung) {
            Action act = no_action();
            if (rung == 0 && C.enable_guardrails) {
                act = try_guardrail(i, diag);
            } else if (rung == 1 && C.enable_placement) {
                if (C.enable_mig && c.ema_has && c.ema > fmul(C.move_futility_ratio, c.trigger)) continue;
                act = try_move(i);
                if (act.valid) act.diagnosis = diag;
            } else if (rung == 2 && C.enable_mig) {
                act = try_mig_up(i);
                if (act.valid) act.diagnosis = diag;
            }
            if (act.valid) {
                c.next_rung = rung + 1 < 2 ? rung + 1 : 2;
                return act;
            }
        }
        if (!c.none_logged) {
            Action n = no_action();
            n.kind = kActNone;
            n.tenant = i;
            n.target = i;
            n.diagnosis = diag;
            record(n, now, c);
            c.none_logged = 1;
        }
        c.next_rung = 0;
        c.breach_windows = 0;
        return no_action();
    }

    MG_HD Action finish_validation(int i, TenantCtl& c, double t) {  // controller.cpp:444-487
        c.validating = 0;
        double post = 0.0;
        if (c.vn > 0) post = select_jth_largest(c.vwin, c.vn, nr_from_top(0.99, c.vn));
        bool ok;
        if (c.app_kind == kActMigDown) {
            ok = post < c.clear;
        } else {
            ok = post <= fmul(fadd(1.0, C.rollback_regress_ratio), c.pre_p99_ms) || post < c.trigger;
        }
        if (ok) {
            c.backfired = 0;
            reset_signal(c, t);
            return no_action();
        }
        c.backfired = 1;
        if (c.app_kind == kActMigDown) c.relax_blocked = c.prior_profile;
        Action rb = no_action();
        rb.valid = 1;
        rb.kind = kActRollback;
        rb.tenant = i;
        rb.diagnosis = c.app_diag;
        if (c.app_kind == kActIoThrottle || c.app_kind == kActMpsQuota) {
            rb.target = c.app_target;
            rb.restore_throttle = 1;
        } else {
            rb.target = i;
            rb.new_host = c.prior_host;
            rb.new_gpu = c.prior_gpu;
            rb.new_first = c.prior_first;
            rb.new_count = c.prior_count;
            rb.new_profile = c.prior_profile;
        }
        const int seq = record(rb, t, c);
        if (seq < io.action_cap && st.n_actions <= io.action_cap) io.actions[seq].rolled_back_seq = c.action_seq;
        c.obs_since_action = 0;
        reset_signal(c, t);
        return rb;
    }

    MG_HD void adopt(int i, TenantCtl& c, const Action& act, double p99, double t) {
        const TenantDyn& d = td[i];
        c.pre_p99_ms = p99;
        c.prior_host = d.host;
        c.prior_gpu = d.gpu;
        c.prior_first = d.first;
        c.prior_count = d.count;
        c.prior_profile = d.profile;
        c.app_kind = act.kind;
        c.app_target = act.target;
        c.app_diag = act.diagnosis;
        c.action_seq = record(act, t, c);
    }

    MG_HD Action on_observation(int i, double lat, double t, double arrived) {  // controller.cpp:489-603
        TenantCtl& c = ctl[i];
        c.obs_total += 1;
        if (c.acted_ever) c.obs_since_action += 1;
        if (c.validating) {
            if (!c.drain_seen) {
                if (queue_len(i) <= 1) {
                    c.drain_seen = 1;
                    c.validation_start_s = t;
                } else if (fsub(t, c.validation_start_s) > 180.0) {
                    if (c.vn < C.validation_obs) c.vwin[c.vn++] = lat;
                    return finish_validation(i, c, t);
                }
            } else if (arrived >= c.validation_start_s) {
                c.vwin[c.vn++] = lat;
                if (c.vn >= C.validation_obs) return finish_validation(i, c, t);
            }
            return no_action();
        }
        if (arrived < c.ignore_before_s) return no_action();
        while (t >= c.window_end_s) {
            if (c.obs_in_window > 0) {
                if (c.ema_has) {
                    if (c.ema > c.trigger) {
                        c.breach_windows += 1;
                    } else if (c.ema < c.clear) {
                        c.breach_windows = 0;
                        c.next_rung = 0;
                        c.none_logged = 0;
                    }
                }
                c.obs_in_window = 0;
            }
            c.window_end_s = fadd(c.window_end_s, C.sample_interval_s);
        }
        tw_push(c.win, lat);
        const double p99 = tw_quantile(c.win, 0.99);
        ema_update(c, p99);
        c.obs_in_window += 1;
        if (p99 < fmul(C.relax_stability_ratio, c.trigger)) c.relax_run += 1;
        else c.relax_run = 0;
        if (t < C.warmup_s) return no_action();
        uint64_t required = static_cast<uint64_t>(C.dwell_obs);
        if (c.backfired) required += static_cast<uint64_t>(C.cooldown_obs);
        const bool gates = !c.acted_ever || static_cast<uint64_t>(c.obs_since_action) >= required;
        const bool eligible = spec(i).tclass == kLatencySensitive;
        if (eligible && c.breach_windows >= C.persistence_windows && gates) {
            Action act = evaluate_breach(i, c);
            if (act.valid) {
                if (act.kind == kActMigUp) c.relax_blocked = act.new_profile;
                adopt(i, c, act, p99, t);
                c.breach_windows = 0;
                c.obs_since_action = 0;
                c.acted_ever = 1;
                c.none_logged = 0;
                return act;
            }
            return no_action();
        }
        if (C.enable_mig && gates && static_cast<uint64_t>(c.relax_run) >= static_cast<uint64_t>(C.dwell_obs) && !c.ema_trig) {
            Action act = try_relax(i, c);
            if (act.valid) {
                adopt(i, c, act, p99, t);
                c.relax_run = 0;
                c.obs_since_action = 0;
                c.acted_ever = 1;
                return act;
            }
        }
        return no_action();
    }

    // Controller::on_action_applied (controller.cpp:605-623)
    MG_HD void on_action_applied(int i, int kind, double t, double pause) {
        TenantCtl& c = ctl[i];
        if (c.action_seq >= 0 && c.action_seq < st.n_actions && c.action_seq < io.action_cap)
            io.actions[c.action_seq].pause_s = pause;
        if (kind == kActRollback) {
            c.validating = 0;
            c.ignore_before_s = t;
            reset_signal(c, t);
            return;
        }
        c.validating = 1;
        c.drain_seen = 0;
        c.validation_start_s = t;
        c.ignore_before_s = t;
        c.vn = 0;
    }

    // ---- setup and main loop (engine.cpp:239-277, 864-894) -------------------------------
    MG_HD void init(const int32_t* file_order, double* win_storage, double* vwin_storage) {
        now = 0.0;
        next_seq = n_events = live_resume = live_expire = 0;
        st.n_actions = st.n_pauses = st.error = st.next_action_seq = 0;
        st.tick_index = st.pad = 0;
        st.done_seq = 0;
        for (int r = 0; r < S.n_roots; ++r) {
            rd[r].active = 0;
            for (int e = 0; e < kGcEntries; ++e) rd[r].gc_mask[e] = 0;
            io.backlog[2 * r] = 0.0;
            io.backlog[2 * r + 1] = 0.0;
        }
        for (int s = 0; s <= kEvKinds * T; ++s) lanes.clear(s);
        for (int i = 0; i < T; ++i) {
            const PTenant& p = spec(i);
            TenantDyn& d = td[i];
            d.host = p.host;
            d.gpu = p.gpu;
            d.first = p.first;
            d.count = p.count;
            d.profile = p.profile;
            d.base = io.off[i];
            d.n_count = io.count[i];
            d.cpu_pinned = d.paused = d.transferring = d.computing = d.has_throttle = 0;
            d.n_arrived = d.tq_head = d.cq_head = d.cur_compute = d.irq_cursor = 0;
            d.pend_kind = d.has_pend = d.mt_p = d.mt_init = d.pad = 0;
            d.mps_quota = 100.0;
            d.io_throttle = 0.0;
            refresh(i);
            d.paused_until = 0.0;
            d.remaining = d.transfer_ms = d.last_settle = d.grant = 0.0;
            d.started_s = -1.0;
            d.compute_done_ms = d.svc_ms = d.extra_ms = d.compute_end = d.cur_transfer_ms = 0.0;
            d.pend_pause = 0.0;
            d.obs_lat = d.obs_arrived = 0.0;
            d.completed = d.n_window = d.misses = d.pad_c = 0;
            d.sum_total = 0.0;
            d.win_min = k_inf();
            d.win_max = -k_inf();
            TenantCtl& c = ctl[i];
            const double tau = p.slo_tail_ms > 0.0 ? p.slo_tail_ms : C.tail_threshold_ms;
            c.trigger = tau;
            c.clear = fmul(C.hysteresis_clear_ratio, tau);
            c.win.ring = win_storage + static_cast<int64_t>(i) * C.dwell_obs;
            c.win.cap = C.dwell_obs;
            tw_reset(c.win, tau);
            c.vwin = vwin_storage + static_cast<int64_t>(i) * C.validation_obs;
            c.vn = 0;
            c.breach_windows = c.next_rung = c.acted_ever = c.backfired = c.none_logged = 0;
            c.validating = c.drain_seen = 0;
            c.relax_blocked = -1;
            c.action_seq = -1;
            c.prior_host = c.prior_gpu = c.prior_first = c.prior_count = c.prior_profile = -1;
            c.ema_has = c.ema_trig = 0;
            c.obs_in_window = c.obs_since_action = c.relax_run = c.obs_total = 0;
            c.window_end_s = C.sample_interval_s;
            c.ignore_before_s = c.validation_start_s = c.pre_p99_ms = c.ema = 0.0;
            c.app_kind = c.app_target = c.app_diag = 0;
            if (io.tr_win) tw_reset(io.tr_win[i], k_inf());
        }
        for (int n = 0; n < T; ++n) {
            const int i = file_order[n];
            if (io.count[i] > 0) push(kEvArrival, i, io.arr_t[io.off[i]]);
        }
        push(kEvTick, 0, 1.0);
    }

    // tenant of slot s holding an event of `kind`
    MG_HD int slot_tenant(int kind, int s) const { return kind == kEvTick ? 0 : s - slot_base(kind); }

    // run the popped event (its slot already cleared by the caller) (engine.cpp:873-881)
    MG_HD void dispatch(int kind, int i, double t) {
        if (rare_kind(kind)) mark_rare(kind, i, false);
        now = t;
        n_events += 1;
        switch (kind) {
            case kEvResume: on_resume(i); break;
            case kEvExpire: on_guardrail_expire(i); break;
            case kEvTransfer: on_transfer_complete(i); break;
            case kEvCompute: on_compute_complete(i); break;
            case kEvArrival: on_arrival(i); break;
            default: on_tick(); break;
        }
        if (LanesTraits<Lanes>::kDefer) run_ops();
    }

    // host event loop (engine.cpp:864-894); the device loop lives in des_kernel
    MG_HD void run() {
        const int nslots = kEvKinds * T + 1;
        for (;;) {
            const int s = lanes.argmin(nslots);
            const Slot e = lanes.slots[s];
            if (e.key == ~0ull || e.t > S.duration_s) break;  // engine.cpp:869-872
            lanes.clear(s);
            const int kind = static_cast<int>(e.key >> 48);
            dispatch(kind, slot_tenant(kind, s), e.t);
        }
        now = S.duration_s;
    }

    MG_HD void finish() {
        for (int i = 0; i < T; ++i) {
            const TenantDyn& d = td[i];
            TenantOut& o = io.tout[i];
            o.completed_total = d.completed;
            o.completed_window = d.n_window;
            o.window_misses = d.misses;
            o.sum_total_ms = d.sum_total;
            o.host = d.host;
            o.gpu_id = gp[d.gpu].id;
            o.first = d.first;
            o.profile = d.profile;
            o.cpu_pinned = d.cpu_pinned;
            o.win_min = d.win_min;
            o.win_max = d.win_max;
            o.pad = 0;
        }
        io.rout->n_actions = st.n_actions;
        io.rout->n_pauses = st.n_pauses;
        // the device event order packs seq into 29 bits (engine_kernels.cu); never silently wrap
        io.rout->error = next_seq >= (1u << 29) ? kErrSeqOverflow : st.error;
        io.rout->pad = 0;
        io.rout->n_events = n_events;
    }
};

// Event slots in memory with a linear argmin: the host harness (one lane) and the device
// fallback for tenant counts too large for lane-register slots (des_kernel scans them).
struct HostLanes {
    Slot* slots;  // 5T + 1
    MG_HD void set(int s, double t, uint64_t key) {
        slots[s].t = t;
        slots[s].key = key;
    }
    MG_HD void clear(int s) {
        slots[s].t = k_inf();
        slots[s].key = ~0ull;
    }
    MG_HD int argmin(int n) const {
        int best = 0;
        for (int k = 1; k < n; ++k)
            if (slots[k].t < slots[best].t || (slots[k].t == slots[best].t && slots[k].key < slots[best].key))
                best = k;
        return best;
    }
};

}  // namespace mg
