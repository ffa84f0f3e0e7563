// sm_100a kernels of the batched controller engine (see engine_kernels.cuh for the map to the
// reference).  Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -lineinfo
#include "engine_kernels.cuh"
#include "gen_warp.cuh"

namespace mg {

// ---------------------------------------------------------------------------------------------
// arrival-record generation
// one warp per (replica, tenant); blocks are tenant-major so neighbouring warps have equal rates
__global__ void __launch_bounds__(32) gen_times_kernel(const PScenario* __restrict__ S, WaveBuffers B, int n_rep) {
    extern __shared__ __align__(16) unsigned char smem[];
    GammaSmem& g = *reinterpret_cast<GammaSmem*>(smem);
    const int T = S->n_tenants;
    const int b = blockIdx.x;
    if (b >= n_rep * T) return;
    const int t = b / n_rep;
    const int r = b % n_rep;
    const int lane = threadIdx.x;
    const PTenant& p = S->tenants[t];
    const int64_t base = static_cast<int64_t>(r) * B.cap_sum + B.off[t];
    int32_t* n_all = B.n_all + r * T + t;
    int32_t* n_kept = B.n_kept + r * T + t;
    const bool ok = warp_gen_times(g, p, substream_seed(B.seeds[r], p.name_hash, kArrivals), S->duration_s,
                                   B.t_all ? B.t_all + base : nullptr, B.arr_t + base, B.cap[t], n_all, n_kept, lane);
    if (!ok && lane == 0) atomicExch(B.gen_overflow, 1);
}

// one warp per (replica, tenant, mark stream); purpose-major grid
__global__ void __launch_bounds__(32) gen_marks_kernel(const PScenario* __restrict__ S, WaveBuffers B, int n_rep) {
    __shared__ WarpMtSmem mt;
    const int T = S->n_tenants;
    const int per = n_rep * T;
    const int b = blockIdx.x;
    if (b >= 4 * per) return;
    const int purpose = b / per;
    const int rest = b % per;
    const int t = rest / n_rep;
    const int r = rest % n_rep;
    const int lane = threadIdx.x;
    const PTenant& p = S->tenants[t];
    const int64_t base = static_cast<int64_t>(r) * B.cap_sum + B.off[t];
    if (purpose == kMarkIrq) {
        if (!B.any_irq_noise) return;
        warp_gen_marks(mt, kMarkIrq, p, substream_seed(B.seeds[r], p.name_hash, kIrq), nullptr,
                       B.n_kept[r * T + t], false, B.irq_e ? B.irq_e + base : nullptr, lane);
        return;
    }
    const uint64_t sp = purpose == kMarkSize ? kTransferSize : purpose == kMarkService ? kService : kNoise;
    double* out = purpose == kMarkSize ? B.arr_bytes : purpose == kMarkService ? B.arr_mult : B.arr_noise;
    warp_gen_marks(mt, purpose, p, substream_seed(B.seeds[r], p.name_hash, sp), B.t_all ? B.t_all + base : nullptr,
                   B.n_all[r * T + t],
                   p.sched.kind != kAlways, out + base, lane);
}

size_t gen_times_smem_bytes() { return sizeof(GammaSmem); }

// ---------------------------------------------------------------------------------------------
// replica DES: one warp per replica, working set in dynamic shared memory
//
// Event order.  Event times are >= 0, so the IEEE bit pattern orders them as unsigned integers;
// the total order (t, kind, seq) (engine.cpp:69-75) becomes (t_hi, t_lo, kind<<29 | seq) and the
// warp minimum is one to three redux.sync.min.u32 steps.  seq < 2^29 per replica is checked by
// Sim::finish.
__device__ __forceinline__ uint32_t order_q(uint64_t key) {
    return static_cast<uint32_t>((key >> 48) << 29) | static_cast<uint32_t>(key & 0x1fffffffu);
}

// Event slots as lane registers (T <= kRegSlotMaxTenants): lane k owns hot slot k (< 3T+1:
// compute, transfer, arrival, tick) and rare slot k (< 2T: resume, expire).  A push is a
// predicated register write in the owning lane; the argmin reads no memory.
struct RegLanes {
    int lane, nhot;
    uint32_t hh, hl, hq;  // hot slot (t_hi, t_lo, q); hh == ~0 when empty
    uint32_t rh, rl, rq;  // rare slot
    __device__ __forceinline__ void put(int s, uint32_t h, uint32_t l, uint32_t q) {
        if (s < nhot) {
            if (lane == s) {
                hh = h;
                hl = l;
                hq = q;
            }
        } else if (lane == s - nhot) {
            rh = h;
            rl = l;
            rq = q;
        }
    }
    __device__ __forceinline__ void set(int s, double t, uint64_t key) {
        const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(t));
        put(s, static_cast<uint32_t>(tb >> 32), static_cast<uint32_t>(tb), order_q(key));
    }
    __device__ __forceinline__ void clear(int s) { put(s, 0xffffffffu, 0xffffffffu, 0xffffffffu); }
};

template <>
struct MaskOf<RegLanes> {
    using type = uint32_t;  // T <= kRegSlotMaxTenants
};
// the same lanes with the pipeline helpers inlined at their call sites (latency-bound batches)
struct RegLanesDirect : RegLanes {};
template <>
struct MaskOf<RegLanesDirect> {
    using type = uint32_t;
};
template <>
struct LanesTraits<RegLanesDirect> {
    static constexpr bool kPerThread = false;
    static constexpr bool kDefer = false;
};

template <class Lanes>
__device__ __forceinline__ Lanes make_lanes(unsigned char* smem, const SimLayout& L, int T);
template <>
__device__ __forceinline__ HostLanes make_lanes<HostLanes>(unsigned char* smem, const SimLayout& L, int) {
    return HostLanes{reinterpret_cast<Slot*>(smem + L.slots)};
}
template <>
__device__ __forceinline__ RegLanes make_lanes<RegLanes>(unsigned char*, const SimLayout&, int T) {
    RegLanes r;
    r.lane = static_cast<int>(threadIdx.x);
    r.nhot = 3 * T + 1;
    r.hh = r.hl = r.hq = r.rh = r.rl = r.rq = 0xffffffffu;
    return r;
}
template <>
__device__ __forceinline__ RegLanesDirect make_lanes<RegLanesDirect>(unsigned char* smem, const SimLayout& L, int T) {
    RegLanesDirect r;
    static_cast<RegLanes&>(r) = make_lanes<RegLanes>(smem, L, T);
    return r;
}

// Warp argmin of the next event.  Returns false when no live event is left.  On success every
// lane holds the winner's slot index and (t, q).
template <class Lanes>
__device__ __forceinline__ bool next_event(Sim<Lanes>& sim, int T, int& s_out, double& t_out, uint32_t& q_out);

template <class SimT>
__device__ __forceinline__ bool reg_next_event(SimT& sim, int& s_out, double& t_out, uint32_t& q_out);
template <>
__device__ __forceinline__ bool next_event<RegLanes>(Sim<RegLanes>& sim, int, int& s_out, double& t_out,
                                                     uint32_t& q_out) {
    return reg_next_event(sim, s_out, t_out, q_out);
}
template <>
__device__ __forceinline__ bool next_event<RegLanesDirect>(Sim<RegLanesDirect>& sim, int, int& s_out, double& t_out,
                                                           uint32_t& q_out) {
    return reg_next_event(sim, s_out, t_out, q_out);
}
template <class SimT>
__device__ __forceinline__ bool reg_next_event(SimT& sim, int& s_out, double& t_out, uint32_t& q_out) {
    RegLanes& R = sim.lanes;
    uint32_t h = R.hh, l = R.hl, q = R.hq;
    int s = R.lane;
    if (sim.any_rare() && (R.rh < h || (R.rh == h && (R.rl < l || (R.rl == l && R.rq < q))))) {
        h = R.rh;
        l = R.rl;
        q = R.rq;
        s = R.nhot + R.lane;
    }
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, h);
    if (m1 == 0xffffffffu) return false;  // no live event (every t >= 0 has a smaller high word)
    unsigned win = __ballot_sync(0xffffffffu, h == m1);
    if (win & (win - 1)) {  // equal high words: low words decide, then (kind, seq)
        const uint32_t m2 = __reduce_min_sync(0xffffffffu, h == m1 ? l : 0xffffffffu);
        win = __ballot_sync(0xffffffffu, h == m1 && l == m2);
        if (win & (win - 1)) {
            const uint32_t m3 = __reduce_min_sync(0xffffffffu, (h == m1 && l == m2) ? q : 0xffffffffu);
            win = __ballot_sync(0xffffffffu, h == m1 && l == m2 && q == m3);
        }
    }
    const int wl = __ffs(win) - 1;
    const uint32_t lo = __shfl_sync(0xffffffffu, l, wl);
    q_out = __shfl_sync(0xffffffffu, q, wl);
    s_out = __shfl_sync(0xffffffffu, s, wl);
    t_out = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(m1) << 32) | lo));
    return true;
}

template <>
__device__ __forceinline__ bool next_event<HostLanes>(Sim<HostLanes>& sim, int T, int& s_out, double& t_out,
                                                      uint32_t& q_out) {
    const Slot* slots = sim.lanes.slots;
    const int lane = threadIdx.x;
    uint32_t hi = 0xffffffffu, lo = 0xffffffffu, kq = 0xffffffffu;
    int bi = -1;
    const int nslots = sim.any_rare() ? kEvKinds * T + 1 : 3 * T + 1;
    // all of this lane's slot loads first (independent LDS.128s in flight), then the compares
    constexpr int KS = (kEvKinds * kMaxTenants + 1 + 31) / 32;
    uint64_t keys[KS], tbs[KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) {
        const int k = lane + 32 * j;
        keys[j] = ~0ull;
        tbs[j] = 0;
        if (k < nslots) {
            keys[j] = slots[k].key;
            tbs[j] = static_cast<uint64_t>(__double_as_longlong(slots[k].t));
        }
    }
#pragma unroll
    for (int j = 0; j < KS; ++j) {
        if (keys[j] == ~0ull) continue;
        const uint32_t h = static_cast<uint32_t>(tbs[j] >> 32), l = static_cast<uint32_t>(tbs[j]), q = order_q(keys[j]);
        if (h < hi || (h == hi && (l < lo || (l == lo && q < kq)))) {
            hi = h;
            lo = l;
            kq = q;
            bi = lane + 32 * j;
        }
    }
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, hi);
    if (m1 == 0xffffffffu) return false;
    const uint32_t m2 = __reduce_min_sync(0xffffffffu, hi == m1 ? lo : 0xffffffffu);
    unsigned win = __ballot_sync(0xffffffffu, bi >= 0 && hi == m1 && lo == m2);
    if (win & (win - 1)) {  // equal times: (kind, seq) decides
        const uint32_t m3 = __reduce_min_sync(0xffffffffu, (hi == m1 && lo == m2) ? kq : 0xffffffffu);
        win = __ballot_sync(0xffffffffu, bi >= 0 && hi == m1 && lo == m2 && kq == m3);
    }
    const int wl = __ffs(win) - 1;
    s_out = __shfl_sync(0xffffffffu, bi, wl);
    q_out = __shfl_sync(0xffffffffu, kq, wl);
    t_out = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(m1) << 32) | m2));
    return true;
}

// read-only scenario tables -> shared memory (cooperative 8-B copies; all PODs are 8-B multiples)
__device__ __forceinline__ void copy_tables(unsigned char* smem, const SimLayout& L, const PScenario* __restrict__ S,
                                            int tid, int nthreads) {
    auto copy8 = [&](int64_t dst_off, const void* src, int64_t bytes) {
        const uint64_t* s8 = reinterpret_cast<const uint64_t*>(src);
        uint64_t* d8 = reinterpret_cast<uint64_t*>(smem + dst_off);
        for (int64_t k = tid; k < bytes / 8; k += nthreads) d8[k] = s8[k];
    };
    copy8(L.sc_tn, S->tenants, static_cast<int64_t>(sizeof(PTenant)) * S->n_tenants);
    copy8(L.sc_gp, S->gpus, static_cast<int64_t>(sizeof(PGpu)) * S->n_gpus);
    copy8(L.sc_rt, S->roots, static_cast<int64_t>(sizeof(PRoot)) * S->n_roots);
    copy8(L.sc_iq, S->irq, static_cast<int64_t>(sizeof(PIrq)) * S->n_irq);
    copy8(L.sc_hio, S->host_io_capacity, align16(8ll * S->n_hosts));
}

// global-memory side of replica r (arrival records, scratch, outputs)
__device__ __forceinline__ ReplicaIO replica_io(const WaveBuffers& B, const PScenario* __restrict__ S, int r, int T) {
    const int64_t base = static_cast<int64_t>(r) * B.cap_sum;
    ReplicaIO io;
    io.arr_t = B.arr_t + base;
    io.arr_bytes = B.arr_bytes + base;
    io.arr_mult = B.arr_mult + base;
    io.arr_noise = B.arr_noise + base;
    io.irq_e = B.irq_e ? B.irq_e + base : nullptr;
    io.off = B.off;
    io.count = B.n_kept + static_cast<int64_t>(r) * T;
    io.seed = B.seeds[r];
    io.req_transfer_ms = B.req_ms + base;
    io.mt_pause = B.mt_pause + static_cast<int64_t>(r) * T * kMtN;
    io.win_lat = B.win_lat + base;
    io.win_hist = B.win_hist ? B.win_hist + static_cast<int64_t>(r) * T * kHistBins : nullptr;
    io.actions = B.actions + static_cast<int64_t>(r) * B.action_cap;
    io.action_cap = B.action_cap;
    io.pauses = B.pauses + static_cast<int64_t>(r) * B.pause_cap;
    io.pause_cap = B.pause_cap;
    io.tout = B.tout + static_cast<int64_t>(r) * T;
    io.rout = B.rout + r;
    io.backlog = B.backlog + static_cast<int64_t>(r) * 2 * S->n_roots;
    if (B.c_total) {
        io.c_done = B.c_done + base;
        io.c_total = B.c_total + base;
        io.c_compute = B.c_compute + base;
        io.c_transfer = B.c_transfer + base;
        io.c_noise = B.c_noise + base;
        io.c_order = B.c_order + base;
    } else {
        io.c_done = io.c_total = io.c_compute = io.c_transfer = io.c_noise = nullptr;
        io.c_order = nullptr;
    }
    if (B.tr_cnt) {
        io.tr_cnt = B.tr_cnt + static_cast<int64_t>(r) * S->n_ticks * T;
        io.tr_fab = B.tr_fab + static_cast<int64_t>(r) * S->n_ticks * S->n_roots;
        io.tr_win = B.tr_win + static_cast<int64_t>(r) * T;
    } else {
        io.tr_cnt = nullptr;
        io.tr_fab = nullptr;
        io.tr_win = nullptr;
    }
    return io;
}

// kGlobalTables: the scenario tables are read from global memory (layout sc_* = -1; T > 10 kernel)
template <class Lanes, bool kGlobalTables = false>
__device__ __forceinline__ void des_body(const PScenario* __restrict__ S, const PController* __restrict__ C,
                                         const WaveBuffers& B, int n_rep, const SimLayout& L) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int r = blockIdx.x;
    if (r >= n_rep) return;
    const int T = S->n_tenants;
    const int lane = threadIdx.x;
    if (!kGlobalTables) copy_tables(smem, L, S, lane, 32);
    {
        const uint64_t* s8 = reinterpret_cast<const uint64_t*>(C + B.variant[r]);
        uint64_t* d8 = reinterpret_cast<uint64_t*>(smem + L.sc_ctrl);
        for (int k = lane; k < static_cast<int>(sizeof(PController) / 8); k += 32) d8[k] = s8[k];
    }
    __syncwarp();
    const PController& Cv = *reinterpret_cast<const PController*>(smem + L.sc_ctrl);
    SimState& st = *reinterpret_cast<SimState*>(smem + L.st);
    TenantDyn* td = reinterpret_cast<TenantDyn*>(smem + L.td);
    TenantCtl* ctl = reinterpret_cast<TenantCtl*>(smem + L.ctl);
    RootDyn* rd = reinterpret_cast<RootDyn*>(smem + L.rd);
    double* win;
    double* vwin;
    if (B.rings_in_smem) {
        win = reinterpret_cast<double*>(smem + L.win);
        vwin = reinterpret_cast<double*>(smem + L.vwin);
    } else {
        win = B.rings + static_cast<int64_t>(r) * T * (B.dwell + B.validation);
        vwin = win + static_cast<int64_t>(T) * B.dwell;
    }
    const ReplicaIO io = replica_io(B, S, r, T);
    Sim<Lanes> sim(*S, Cv, io, st, make_lanes<Lanes>(smem, L, T), td, ctl, rd);
    if (!kGlobalTables) {
        sim.tn = reinterpret_cast<const PTenant*>(smem + L.sc_tn);
        sim.gp = reinterpret_cast<const PGpu*>(smem + L.sc_gp);
        sim.rt = reinterpret_cast<const PRoot*>(smem + L.sc_rt);
        sim.iq = reinterpret_cast<const PIrq*>(smem + L.sc_iq);
        sim.hio = reinterpret_cast<const double*>(smem + L.sc_hio);
    }  // else: the Sim constructor's S->tenants / gpus / roots / irq / host_io_capacity
    // The handlers run warp-uniformly: every lane executes the same instructions on the same
    // shared-memory words (broadcast loads, same-value stores), so no lane-0 divergence region
    // (BSSY/BSYNC) wraps the hot path.
    sim.init(B.file_order, win, vwin);
    __syncwarp();
    const double duration = S->duration_s;
#ifdef MG_PROFILE_EVENTS
    // build-time instrumentation (make PROFILE=1): SM cycles spent choosing vs running events
    unsigned long long c_pick[6] = {0, 0, 0, 0, 0, 0}, c_run[6] = {0, 0, 0, 0, 0, 0}, n_ev[6] = {0, 0, 0, 0, 0, 0};
#endif
    for (;;) {
#ifdef MG_PROFILE_EVENTS
        const long long c0 = clock64();
#endif
        int s;
        double t;
        uint32_t q;
        if (!next_event(sim, T, s, t, q)) break;
        if (t > duration) break;  // engine.cpp:872
        const int kind = static_cast<int>(q >> 29);
        sim.lanes.clear(s);
#ifdef MG_PROFILE_EVENTS
        const long long c1 = clock64();
#endif
        sim.dispatch(kind, sim.slot_tenant(kind, s), t);
        __syncwarp();
#ifdef MG_PROFILE_EVENTS
        const long long c2 = clock64();
        c_pick[kind] += c1 - c0;
        c_run[kind] += c2 - c1;
        n_ev[kind] += 1;
#endif
    }
    sim.now = duration;
    sim.finish();
#ifdef MG_PROFILE_EVENTS
    if (lane == 0 && B.prof)
        for (int k = 0; k < 6; ++k) {
            atomicAdd(B.prof + 3 * k + 0, c_pick[k]);
            atomicAdd(B.prof + 3 * k + 1, c_run[k]);
            atomicAdd(B.prof + 3 * k + 2, n_ev[k]);
        }
#endif
}

// T > 10 kernel register budget: with __launch_bounds__(32) alone ptxas settles on 80 registers
// and spills 404 B; 168 (148 used, no spills) measured -12% DES on C5 (occupancy is shared-memory
// bound at 5 replicas/SM either way; profiles/r2_ab_c5_regs.txt)
#ifndef MG_DESK_MAXNREG
#define MG_DESK_MAXNREG 168
#endif
#define MG_DESK_BOUNDS __maxnreg__(MG_DESK_MAXNREG)
__global__ void MG_DESK_BOUNDS des_kernel(const PScenario* __restrict__ S, const PController* __restrict__ C,
                                                 WaveBuffers B, int n_rep, SimLayout L) {
    des_body<HostLanes, true>(S, C, B, n_rep, L);
}

// the latency-regime kernel: helpers inlined at their call sites (RegLanesDirect) and a register
// budget large enough that ptxas does not spill (it settles on 128 + spills under launch_bounds)
#ifndef MG_DES_MAXNREG
#define MG_DES_MAXNREG 168
#endif
#define MG_DES_BOUNDS __maxnreg__(MG_DES_MAXNREG)
__global__ void MG_DES_BOUNDS des_kernel_reg(const PScenario* __restrict__ S,
                                                     const PController* __restrict__ C, WaveBuffers B, int n_rep,
                                                     SimLayout L) {
    des_body<RegLanesDirect>(S, C, B, n_rep, L);
}
// Saturated regime: with the event loop no longer instruction-fetch bound (continuation ops),
// dependent-latency stalls dominate and twice the resident warps hide them (C4 wave: 780 -> 676 ms
// at 64 vs 124 registers, no spills).  A latency-bound batch (fewer replicas than resident slots,
// e.g. C2's 256) keeps the uncapped kernel, whose per-replica event chain is shorter.
#ifndef MG_OCC_MAXNREG
#define MG_OCC_MAXNREG 64  // 48 / 56 measured slower: spills, and 1-warp blocks cap residency at 32/SM anyway
#endif
__global__ void __maxnreg__(MG_OCC_MAXNREG) des_kernel_reg_occ(const PScenario* __restrict__ S, const PController* __restrict__ C,
                                                   WaveBuffers B, int n_rep, SimLayout L) {
    des_body<RegLanes>(S, C, B, n_rep, L);
}

// ---------------------------------------------------------------------------------------------
// replica DES, SIMT form: one THREAD per replica.
//
// The warp kernels above run one replica per warp with every lane repeating the scalar handler
// work.  Here each lane owns a replica: its working set (SimState, TenantDyn/Ctl, RootDyn, event
// slots) lives in a private shared-memory slab at a stride that is an odd multiple of 8 bytes, so
// the 32 lanes' same-field loads hit 32 distinct bank pairs; the controller rings go to global
// memory.  Lanes diverge by event kind, so one pass of the warp executes each kind's handler once
// for all lanes that drew that kind -- per event, an order of magnitude fewer issued instructions
// than the warp-redundant form.  The scenario tables and every variant's PController are staged
// once per block.  Used for large waves (the saturated regime); small waves keep the warp kernel,
// whose lane-parallel argmin gives lower per-replica latency.
struct SimtLanes {
    Slot* slots;  // this thread's 5T+1 slots
    __device__ __forceinline__ void set(int s, double t, uint64_t key) {
        slots[s].t = t;
        slots[s].key = key;
    }
    __device__ __forceinline__ void clear(int s) {
        slots[s].t = k_inf();
        slots[s].key = ~0ull;
    }
};
template <>
struct MaskOf<SimtLanes> {
    using type = uint32_t;  // T <= kSimtMaxTenants
};
template <>
struct LanesTraits<SimtLanes> {
    static constexpr bool kPerThread = true;
    static constexpr bool kDefer = true;
};

__global__ void __launch_bounds__(kSimtBlock) des_simt_kernel(const PScenario* __restrict__ S,
                                                              const PController* __restrict__ C, WaveBuffers B,
                                                              int n_rep, SimtLayout Y) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    copy_tables(smem, Y.tab, S, tid, blockDim.x);
    {
        const uint64_t* s8 = reinterpret_cast<const uint64_t*>(C);
        uint64_t* d8 = reinterpret_cast<uint64_t*>(smem + Y.ctrl);
        const int n8 = B.n_variants * static_cast<int>(sizeof(PController) / 8);
        for (int k = tid; k < n8; k += blockDim.x) d8[k] = s8[k];
    }
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + tid;
    if (r >= n_rep) return;
    const int T = S->n_tenants;
    unsigned char* ln = smem + Y.lanes + static_cast<int64_t>(tid) * Y.stride;
    const SimLayout& L = Y.lane;
    const PController& Cv = reinterpret_cast<const PController*>(smem + Y.ctrl)[B.variant[r]];
    SimState& st = *reinterpret_cast<SimState*>(ln + L.st);
    TenantDyn* td = reinterpret_cast<TenantDyn*>(ln + L.td);
    TenantCtl* ctl = reinterpret_cast<TenantCtl*>(ln + L.ctl);
    RootDyn* rd = reinterpret_cast<RootDyn*>(ln + L.rd);
    double* win = B.rings + static_cast<int64_t>(r) * T * (B.dwell + B.validation);
    double* vwin = win + static_cast<int64_t>(T) * B.dwell;
    const ReplicaIO io = replica_io(B, S, r, T);
    Sim<SimtLanes> sim(*S, Cv, io, st, SimtLanes{reinterpret_cast<Slot*>(ln + L.slots)}, td, ctl, rd);
    sim.tn = reinterpret_cast<const PTenant*>(smem + Y.tab.sc_tn);
    sim.gp = reinterpret_cast<const PGpu*>(smem + Y.tab.sc_gp);
    sim.rt = reinterpret_cast<const PRoot*>(smem + Y.tab.sc_rt);
    sim.iq = reinterpret_cast<const PIrq*>(smem + Y.tab.sc_iq);
    sim.hio = reinterpret_cast<const double*>(smem + Y.tab.sc_hio);
    sim.init(B.file_order, win, vwin);
    const double duration = S->duration_s;
    const Slot* slots = sim.lanes.slots;
    const int nhot = 3 * T + 1;
    for (;;) {
        // this replica's next event: linear argmin over its live slots in (t, kind, seq) order;
        // t >= 0, so the IEEE bits order as unsigned and (t_bits, key) compares lexicographically
        const int n = sim.any_rare() ? kEvKinds * T + 1 : nhot;
        uint64_t bt = ~0ull, bk = ~0ull;
        int bs = -1;
        for (int k = 0; k < n; ++k) {
            const uint64_t kk = slots[k].key;
            const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(slots[k].t));
            if (kk != ~0ull && (tb < bt || (tb == bt && kk < bk))) {
                bt = tb;
                bk = kk;
                bs = k;
            }
        }
        if (bs < 0) break;
        const double t = __longlong_as_double(static_cast<long long>(bt));
        if (t > duration) break;  // engine.cpp:872
        const int kind = static_cast<int>(bk >> 48);
        sim.lanes.clear(bs);
        sim.dispatch(kind, sim.slot_tenant(kind, bs), t);
    }
    sim.now = duration;
    sim.finish();
}

SimtLayout simt_layout(int T, int R, int G, int I, int H, int n_variants) {
    SimtLayout Y;
    Y.tab = sim_layout(T, R, 0, 0, false, G, I, H);
    Y.ctrl = Y.tab.sc_ctrl;  // the per-variant controllers replace the single staged one
    Y.lanes = align16(Y.ctrl + static_cast<int64_t>(sizeof(PController)) * n_variants);
    Y.lane = sim_layout(T, R, 0, 0, false);  // G = 0: per-lane part only, st at offset 0
    int64_t stride = (Y.lane.total + 7) & ~static_cast<int64_t>(7);
    if (((stride / 8) & 1) == 0) stride += 8;  // odd multiple of 8 B: conflict-free same-field access
    Y.stride = stride;
    return Y;
}

// ---------------------------------------------------------------------------------------------
__global__ void compact_actions_kernel(const ActionRec* __restrict__ src, int cap, const ReplicaOut* __restrict__ rout,
                                       const int64_t* __restrict__ dst_off, ActionRec* __restrict__ dst, int n_rep) {
    const int r = blockIdx.x;
    if (r >= n_rep) return;
    const int n = rout[r].n_actions < cap ? rout[r].n_actions : cap;
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[dst_off[r] + k] = src[static_cast<int64_t>(r) * cap + k];
}

__global__ void compact_pauses_kernel(const PauseRec* __restrict__ src, int cap, const ReplicaOut* __restrict__ rout,
                                      const int64_t* __restrict__ dst_off, PauseRec* __restrict__ dst, int n_rep) {
    const int r = blockIdx.x;
    if (r >= n_rep) return;
    const int n = rout[r].n_pauses < cap ? rout[r].n_pauses : cap;
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[dst_off[r] + k] = src[static_cast<int64_t>(r) * cap + k];
}

}  // namespace mg

namespace mg {
__global__ void libm_kernel(int fn, const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ out,
                            int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = fn == 0 ? gl_log(x[i]) : fn == 1 ? gl_exp(x[i]) : fn == 2 ? gl_pow(x[i], y[i]) : fmod_fast(x[i], y[i]);
}
}  // namespace mg

namespace mg {
// ---------------------------------------------------------------------------------------------
// Per-(variant, tenant) latency histograms of a wave: sum the DES's per-(replica, tenant) window
// histograms (lat_hist.h bins) over replicas into int64 accumulators [n_var][T][kHistBins] that
// persist across waves -- the payload the multi-GPU reduction all-reduces.
// Thread = one (tenant, bin); blockIdx.y = a chunk of replicas; replicas are variant-major, so a
// thread flushes its running sum whenever the variant changes (few atomics, coalesced reads).
__global__ void hist_reduce_kernel(const uint32_t* __restrict__ win_hist, const int32_t* __restrict__ variant,
                                   int n_rep, int T, int chunk, unsigned long long* __restrict__ out) {
    const int tb = blockIdx.x * blockDim.x + threadIdx.x;  // t * kHistBins + bin
    if (tb >= T * kHistBins) return;
    const int r0 = blockIdx.y * chunk;
    const int r1 = min(n_rep, r0 + chunk);
    unsigned long long acc = 0;
    int v = r0 < r1 ? variant[r0] : 0;
    for (int r = r0; r < r1; ++r) {
        const int vr = variant[r];
        if (vr != v) {
            if (acc) atomicAdd(out + (static_cast<int64_t>(v) * T * kHistBins + tb), acc);
            acc = 0;
            v = vr;
        }
        acc += win_hist[static_cast<int64_t>(r) * T * kHistBins + tb];
    }
    if (acc) atomicAdd(out + (static_cast<int64_t>(v) * T * kHistBins + tb), acc);
}
}  // namespace mg
