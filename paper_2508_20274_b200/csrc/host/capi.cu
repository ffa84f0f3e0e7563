// C-ABI of the B200 engine (include/migsim_b200.h): scenario loading, wave-batched replica
// execution on one GPU, result assembly, the standalone select, and batched experiment plans.
// There is no CPU execution path: every replica runs in the CUDA kernels of engine_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/migsim_b200.h"
#include "../kernels/admit_kernel.cuh"
#include "../kernels/engine_kernels.cuh"
#include "artifacts.hpp"
#include "packer.hpp"
#include "result_json.hpp"

namespace mg {
size_t select_smem_bytes();
size_t select_cluster_smem_bytes();
int select_cluster_size();
int select_cluster_threads();
int select_threads();
size_t gen_times_smem_bytes();
}

namespace {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParityGuard : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// The SIMT DES (one thread per replica) is opt-in (MIGSIM_DES=simt): measured slower than the
// warp form at every batch size that fits HBM, so "auto" never picks it.
constexpr size_t kSimtMinJobs = SIZE_MAX;
// controller rings stay in shared memory while a replica's working set is at most this
constexpr int64_t kRingsSmemMax = 96 * 1024;

#define CK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess)                                                                         \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" + \
                            std::to_string(__LINE__) + ")");                                           \
    } while (0)

void set_err(char* err, size_t len, const std::string& msg) {
    if (!err || len == 0) return;
    std::snprintf(err, len, "%s", msg.c_str());
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return MIGSIM_OK;
    } catch (const mgb::ConfigError& e) {
        set_err(err, errlen, e.what());
        return MIGSIM_ERR_CONFIG;
    } catch (const ParityGuard& e) {
        set_err(err, errlen, e.what());
        return MIGSIM_ERR_PARITY_GUARD;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return MIGSIM_ERR_RUNTIME;
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    // keeps an existing allocation when it is large enough (wave buffers persist across batches
    // of a handle, so repeated batches do no cudaMalloc/cudaFree)
    void alloc(size_t count) {
        n = count;
        if (p && count <= cap) return;
        free();
        n = count;
        if (count) CK(cudaMalloc(&p, sizeof(T) * count));
        cap = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = cap = 0;
    }
    size_t bytes() const { return sizeof(T) * cap; }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { free(); }
};


struct WaveAlloc {
    DevBuf<double> arr_t, arr_bytes, arr_mult, arr_noise, irq_e, t_all, req_ms, win_lat;
    DevBuf<double> c_done, c_total, c_compute, c_transfer, c_noise;
    DevBuf<int32_t> n_all, n_kept, variant, gen_overflow, file_order, sel_order;
    DevBuf<uint64_t> mt_pause, seeds;
    DevBuf<mg::ActionRec> actions, actions_c;
    DevBuf<mg::PauseRec> pauses, pauses_c;
    DevBuf<mg::TenantOut> tout;
    DevBuf<mg::ReplicaOut> rout;
    DevBuf<double> backlog, quant, rings;
    DevBuf<int64_t> off, cap, act_off, pause_off, c_order;
    DevBuf<mg::CounterRow> tr_cnt;
    DevBuf<mg::FabricRow> tr_fab;
    DevBuf<mg::TailWin> tr_win;
    DevBuf<uint32_t> win_hist;
    DevBuf<unsigned long long> hist_sum;  // [n_var][T][kHistBins] over all waves of a batch
    DevBuf<double> tr_ring;
    DevBuf<mg::PScenario> scen;
    DevBuf<mg::PController> ctrl;
    size_t bytes() const {
        return arr_t.bytes() + arr_bytes.bytes() + arr_mult.bytes() + arr_noise.bytes() + irq_e.bytes() + t_all.bytes() +
               req_ms.bytes() + win_lat.bytes() + c_done.bytes() + c_total.bytes() + c_compute.bytes() +
               c_transfer.bytes() + c_noise.bytes() + mt_pause.bytes() + actions.bytes() + actions_c.bytes() +
               pauses.bytes() + pauses_c.bytes() + rings.bytes() + win_hist.bytes() + c_order.bytes() + tr_cnt.bytes() +
               tr_fab.bytes() + tr_ring.bytes();
    }
};

}  // namespace

struct migsim_gpu {
    int device = 0;
    WaveAlloc wave[2];  // device buffers of the last batch (two pipeline slots), reused by the next
    cudaStream_t stream = nullptr, stream2 = nullptr;
    cudaEvent_t ev[6] = {}, ev2[6] = {}, span[3] = {};
    std::vector<mgb::ScenarioSpec> scenarios;
    std::vector<char> released;  // migsim_gpu_release_scenario
};

struct migsim_batch_result {
    mgb::ScenarioSpec spec;
    mgb::Packed P;
    std::vector<mgb::Variant> variants;
    std::vector<uint64_t> seeds;
    size_t n_runs = 0;
    int T = 0, R = 0;
    std::vector<mg::TenantOut> tout;
    std::vector<double> quant;
    std::vector<mg::ReplicaOut> rout;
    std::vector<double> backlog;
    std::vector<mg::ActionRec> actions;
    std::vector<int64_t> act_off;
    std::vector<mg::PauseRec> pauses;
    std::vector<int64_t> pause_off;
    std::vector<double> comps;
    std::vector<int64_t> comp_off;
    std::vector<migsim_completion> crec;  // keep_completions: engine::CompletionRecord per run, kept_ order
    std::vector<int64_t> crec_off;
    std::vector<std::string> json;
    std::vector<mgb::TraceRows> traces;  // per run, with write_traces
    std::vector<uint64_t> hist;          // [n_var][T][kHistBins] window-latency histograms (lat_hist.h bins)
    std::vector<uint64_t> counts;        // [n_var][T][3] completed_total, completed_window, window_misses
    migsim_timing timing{};
};

namespace {



void check_scenario_id(const migsim_gpu* g, int32_t id) {
    if (!g || id < 0 || id >= static_cast<int32_t>(g->scenarios.size()))
        throw mgb::ConfigError("unknown scenario id");
    if (static_cast<size_t>(id) < g->released.size() && g->released[static_cast<size_t>(id)])
        throw mgb::ConfigError("scenario id " + std::to_string(id) + " was released");
}

void run_batch_impl(migsim_gpu* g, const mgb::ScenarioSpec& spec, const std::vector<mgb::Variant>& variants,
                    const std::vector<uint64_t>& seeds, const migsim_run_opts& opts, migsim_batch_result& res,
                    double cap_sigmas, int action_cap, int pause_cap) {
    const auto wall0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(g->device));
    res.spec = spec;
    res.variants = variants;
    res.seeds = seeds;
    res.P = mgb::pack(spec, variants, cap_sigmas);
    const mgb::Packed& P = res.P;
    const int T = P.scen.n_tenants, R = P.scen.n_roots;
    const size_t n_var = P.ctrl.size();
    const size_t n_jobs = n_var * seeds.size();
    res.n_runs = n_jobs;
    res.T = T;
    res.R = R;
    // every host<->device byte of the call, reported in migsim_timing (bench.py's e2e h2d/d2h)
    int64_t h2d_bytes = 0, d2h_bytes = 0;
    auto count = [&](size_t n, cudaMemcpyKind k) {
        if (k == cudaMemcpyHostToDevice) h2d_bytes += static_cast<int64_t>(n);
        else if (k == cudaMemcpyDeviceToHost) d2h_bytes += static_cast<int64_t>(n);
    };
    auto cpy_async = [&](void* d, const void* src, size_t n, cudaMemcpyKind k, cudaStream_t st) {
        count(n, k);
        return cudaMemcpyAsync(d, src, n, k, st);
    };
    auto cpy_sync = [&](void* d, const void* src, size_t n, cudaMemcpyKind k) {
        count(n, k);
        return cudaMemcpy(d, src, n, k);
    };
    const bool traces = opts.write_traces != 0;
    const bool keep = opts.keep_completions != 0 || traces;
    // working-set layout: controller rings in shared memory when a replica stays under 96 KB
    const int G = P.scen.n_gpus, I = P.scen.n_irq, H = P.scen.n_hosts;
    // T > 10 (des_kernel): scenario tables read from global memory, not staged per replica
    const bool global_tables = T > mg::kRegSlotMaxTenants;
    mg::SimLayout L = mg::sim_layout(T, R, P.max_dwell, P.max_validation, true, G, I, H, global_tables);
    // DES form: SIMT (one thread per replica) for large batches, warp-per-replica otherwise
    // (MIGSIM_DES=warp|simt overrides)
    const mg::SimtLayout Y = mg::simt_layout(T, R, G, I, H, static_cast<int>(n_var));
    const char* des_env = std::getenv("MIGSIM_DES");
    const std::string des_mode = des_env ? des_env : "auto";
    int simt_lanes = mg::kSimtBlock;
    while (simt_lanes > 1 && Y.bytes(simt_lanes) > 200 * 1024) simt_lanes /= 2;
    const bool simt_fits = T <= mg::kSimtMaxTenants && Y.bytes(1) <= 200 * 1024;
    const bool use_simt = simt_fits && (des_mode == "simt" || (des_mode == "auto" && n_jobs >= kSimtMinJobs));
    // MIGSIM_RINGS=global|smem overrides where the controller rings live (A/B of occupancy vs latency)
    const char* rings_env = std::getenv("MIGSIM_RINGS");
    const std::string rings_mode = rings_env ? rings_env : "auto";
    // auto: rings in shared memory only while every replica of the batch can be resident at once
    // with them there (latency-bound, few replicas: C2); otherwise in global memory, where the
    // smaller block footprint raises DES occupancy to the register limit (the saturated regime:
    // 6.77 -> 5.73 s for 16,384 default.yaml replicas)
    bool rings_in_smem = !use_simt && rings_mode != "global" && (rings_mode == "smem" || L.total <= kRingsSmemMax);
    if (rings_in_smem && rings_mode == "auto") {
        auto* des_k = T <= mg::kRegSlotMaxTenants ? mg::des_kernel_reg : mg::des_kernel;
        CK(cudaFuncSetAttribute(des_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.total)));
        int occ = 0, n_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, des_k, 32, static_cast<size_t>(L.total)));
        CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, g->device));
        if (n_jobs > static_cast<size_t>(occ) * static_cast<size_t>(n_sm)) rings_in_smem = false;
    }
    if (!rings_in_smem) L = mg::sim_layout(T, R, P.max_dwell, P.max_validation, false, G, I, H, global_tables);
    auto* des = T <= mg::kRegSlotMaxTenants ? mg::des_kernel_reg : mg::des_kernel;
    // register-capped form when the batch saturates the uncapped kernel's resident slots
    // (MIGSIM_DES_REGS=full|capped overrides)
    bool des_capped = false;
    if (!use_simt && T <= mg::kRegSlotMaxTenants) {
        const char* regs_env = std::getenv("MIGSIM_DES_REGS");
        const std::string regs_mode = regs_env ? regs_env : "auto";
        int occ_full = 0, nsm = 0;
        CK(cudaFuncSetAttribute(mg::des_kernel_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.total)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_full, mg::des_kernel_reg, 32, static_cast<size_t>(L.total)));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
        des_capped = regs_mode == "capped" ||
                     (regs_mode == "auto" && n_jobs > static_cast<size_t>(occ_full) * static_cast<size_t>(nsm));
        if (des_capped) des = mg::des_kernel_reg_occ;
    }
    if (use_simt)
        CK(cudaFuncSetAttribute(mg::des_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(Y.bytes(simt_lanes))));
    else
        CK(cudaFuncSetAttribute(des, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.total)));
    int des_blocks_per_sm = 0, n_sm = 0;
    if (use_simt)
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&des_blocks_per_sm, mg::des_simt_kernel, simt_lanes,
                                                         static_cast<size_t>(Y.bytes(simt_lanes))));
    else
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&des_blocks_per_sm, des, 32, static_cast<size_t>(L.total)));
    CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, g->device));
    // replicas the DES keeps resident at once (one "round" of a wave)
    const size_t resident = static_cast<size_t>(std::max(1, des_blocks_per_sm)) * static_cast<size_t>(n_sm) *
                            static_cast<size_t>(use_simt ? simt_lanes : 1);
    // wave size from free memory
    // record streams per arrival slot: t, bytes, mult, noise, req_ms, win_lat (+ irq draws when some
    // IRQ burst adds noise, + the unthinned clock when some tenant is schedule-thinned, + 5 with
    // keep_completions)
    const int n_streams = 6 + (P.any_irq_noise ? 1 : 0) + (P.any_thinned ? 1 : 0) + (keep ? 5 : 0);
    const size_t per_rep = static_cast<size_t>(P.cap_sum) * 8 * static_cast<size_t>(n_streams) + static_cast<size_t>(T) * 8 +
                           static_cast<size_t>(T) * mg::kMtN * 8 + static_cast<size_t>(action_cap) * sizeof(mg::ActionRec) * 2 +
                           static_cast<size_t>(pause_cap) * sizeof(mg::PauseRec) * 2 + T * sizeof(mg::TenantOut) +
                           sizeof(mg::ReplicaOut) + static_cast<size_t>(R) * 16 + static_cast<size_t>(T) * 32 + 64 +
                           static_cast<size_t>(T) * mg::kHistBins * 4 +
                           (rings_in_smem ? 0 : static_cast<size_t>(T) * (P.max_dwell + P.max_validation) * 8);
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    free_b += g->wave[0].bytes() + g->wave[1].bytes();  // the handle's cached wave buffers are reusable
    // MIGSIM_MEM_FRACTION: share of free HBM a batch's waves may use (default 0.70; processes that
    // share one device, e.g. test launches of several ranks on one GPU, pass their share)
    const char* frac_env = std::getenv("MIGSIM_MEM_FRACTION");
    const double mem_frac = frac_env ? std::min(0.9, std::max(0.01, std::atof(frac_env))) : 0.70;
    size_t W = std::max<size_t>(1, static_cast<size_t>(mem_frac * static_cast<double>(free_b)) / per_rep);
    if (opts.max_wave_replicas > 0) W = std::min<size_t>(W, static_cast<size_t>(opts.max_wave_replicas));
    // A multi-wave batch wastes the last, partly filled round of every wave (the event loop of a
    // wave ends with its slowest resident replicas).  Round the wave down to whole rounds of
    // resident replicas, so only the batch's final wave has a partial round (C4: 5 waves of 5.53
    // rounds = 30 executed rounds -> 28 for the same 27.7 rounds of work).
    if (W < n_jobs && W > resident && opts.max_wave_replicas <= 0) W -= W % resident;
    W = std::min(W, n_jobs);
    if (W == 0) W = 1;

    // ---- wave slots ------------------------------------------------------------------------
    // MIGSIM_PIPELINE=1: multi-wave batches run as a two-slot pipeline on two streams (the
    // generator of wave k+1 and its event loop start while wave k's event loop drains; wave k's
    // host-side assembly overlaps wave k+1).  Off by default: measured 12.0 vs 12.5 M tenant-ticks/s
    // on 16,384 default.yaml replicas (the half-size waves cost more than the overlap recovers;
    // DESIGN.md section 6).  keep_completions / traces always use one slot.
    const bool want_prof = std::getenv("MIGSIM_PROFILE_EVENTS") != nullptr;
    const char* pipe_env = std::getenv("MIGSIM_PIPELINE");
    const bool pipe_allowed = pipe_env && std::string(pipe_env) == "1" && !keep && !want_prof;
    const int n_slots = (pipe_allowed && n_jobs > W) ? 2 : 1;
    if (n_slots == 2) W = std::max<size_t>(1, W / 2);
    WaveAlloc& A = g->wave[0];  // also holds the batch-wide buffers (scenario, controllers, histograms)
    const size_t big = W * static_cast<size_t>(P.cap_sum);
    const int n_ticks = P.scen.n_ticks;
    constexpr int kTraceWin = 256;  // engine.cpp:115
    for (int si = 0; si < n_slots; ++si) {
        WaveAlloc& S = g->wave[si];
        S.arr_t.alloc(big);
        S.arr_bytes.alloc(big);
        S.arr_mult.alloc(big);
        S.arr_noise.alloc(big);
        // (optional streams not needed by this batch are released: the wave sizing above counts
        //  every cached buffer of the handle as reusable)
        if (P.any_irq_noise) S.irq_e.alloc(big);
        else S.irq_e.free();
        if (P.any_thinned) S.t_all.alloc(big);
        else S.t_all.free();
        S.req_ms.alloc(big);
        S.win_lat.alloc(big);
        S.win_hist.alloc(W * T * mg::kHistBins);
        S.n_all.alloc(W * T);
        S.n_kept.alloc(W * T);
        S.variant.alloc(W);
        S.seeds.alloc(W);
        S.gen_overflow.alloc(1);
        S.mt_pause.alloc(W * T * mg::kMtN);
        S.actions.alloc(W * action_cap);
        S.actions_c.alloc(W * action_cap);
        S.pauses.alloc(W * pause_cap);
        S.pauses_c.alloc(W * pause_cap);
        S.tout.alloc(W * T);
        S.rout.alloc(W);
        S.backlog.alloc(W * R * 2);
        S.quant.alloc(W * T * 4);
        if (!rings_in_smem) S.rings.alloc(W * T * (P.max_dwell + P.max_validation));
        S.act_off.alloc(W + 1);
        S.pause_off.alloc(W + 1);
    }
    if (keep) {
        A.c_done.alloc(big);
        A.c_total.alloc(big);
        A.c_compute.alloc(big);
        A.c_transfer.alloc(big);
        A.c_noise.alloc(big);
        A.c_order.alloc(big);
    }
    if (traces) {
        A.tr_cnt.alloc(W * static_cast<size_t>(n_ticks) * T);
        A.tr_fab.alloc(W * static_cast<size_t>(n_ticks) * R);
        A.tr_win.alloc(W * T);
        A.tr_ring.alloc(W * T * kTraceWin);
        std::vector<mg::TailWin> tw(W * T);
        for (size_t k = 0; k < W * T; ++k) {
            std::memset(&tw[k], 0, sizeof(mg::TailWin));
            tw[k].ring = A.tr_ring.p + k * kTraceWin;
            tw[k].cap = kTraceWin;
        }
        CK(cpy_sync(A.tr_win.p, tw.data(), sizeof(mg::TailWin) * W * T, cudaMemcpyHostToDevice));
        res.traces.resize(n_jobs);
    }
    A.file_order.alloc(T);
    A.sel_order.alloc(T);
    A.off.alloc(T);
    A.cap.alloc(T);
    A.scen.alloc(1);
    A.ctrl.alloc(n_var);
    A.hist_sum.alloc(n_var * T * mg::kHistBins);
    cudaStream_t s = g->stream;
    CK(cudaMemsetAsync(A.hist_sum.p, 0, sizeof(unsigned long long) * n_var * T * mg::kHistBins, s));
    CK(cpy_async(A.scen.p, &P.scen, sizeof(mg::PScenario), cudaMemcpyHostToDevice, s));
    CK(cpy_async(A.ctrl.p, P.ctrl.data(), sizeof(mg::PController) * n_var, cudaMemcpyHostToDevice, s));
    CK(cpy_async(A.off.p, P.off.data(), sizeof(int64_t) * T, cudaMemcpyHostToDevice, s));
    CK(cpy_async(A.cap.p, P.cap.data(), sizeof(int64_t) * T, cudaMemcpyHostToDevice, s));
    CK(cpy_async(A.file_order.p, P.file_order.data(), sizeof(int32_t) * T, cudaMemcpyHostToDevice, s));
    std::vector<int32_t> sel_order(T);
    for (int t = 0; t < T; ++t) sel_order[t] = t;
    std::stable_sort(sel_order.begin(), sel_order.end(), [&](int32_t a, int32_t b) { return P.cap[a] > P.cap[b]; });
    CK(cpy_async(A.sel_order.p, sel_order.data(), sizeof(int32_t) * T, cudaMemcpyHostToDevice, s));

    mg::WaveBuffers B0{};
    B0.file_order = A.file_order.p;
    B0.sel_order = A.sel_order.p;
    B0.off = A.off.p;
    B0.cap = A.cap.p;
    // optional streams: only when this batch asks for them (the cached buffers may hold others)
    B0.c_done = keep ? A.c_done.p : nullptr;
    B0.c_total = keep ? A.c_total.p : nullptr;
    B0.c_compute = keep ? A.c_compute.p : nullptr;
    B0.c_transfer = keep ? A.c_transfer.p : nullptr;
    B0.c_noise = keep ? A.c_noise.p : nullptr;
    B0.c_order = keep ? A.c_order.p : nullptr;
    B0.tr_cnt = traces ? A.tr_cnt.p : nullptr;
    B0.tr_fab = traces ? A.tr_fab.p : nullptr;
    B0.tr_win = traces ? A.tr_win.p : nullptr;
    B0.cap_sum = P.cap_sum;
    B0.action_cap = action_cap;
    B0.pause_cap = pause_cap;
    B0.any_irq_noise = P.any_irq_noise;
    B0.rings_in_smem = rings_in_smem;
    B0.dwell = P.max_dwell;
    B0.validation = P.max_validation;
    B0.n_variants = static_cast<int32_t>(n_var);
    DevBuf<unsigned long long> prof;
    if (want_prof) {
        prof.alloc(18);
        CK(cudaMemsetAsync(prof.p, 0, 18 * 8, s));
        B0.prof = prof.p;
    }
    struct Slot {
        WaveAlloc* A = nullptr;
        cudaStream_t st = nullptr;
        cudaEvent_t* ev = nullptr;
        mg::WaveBuffers B{};
        std::vector<uint64_t> wseeds;
        std::vector<int32_t> wvar, nkept;
        std::vector<int64_t> aoff, poff;
        int32_t overflow = 0;
        size_t j0 = 0;
        int w = 0;
        bool busy = false;
    };
    Slot slots[2];
    for (int si = 0; si < n_slots; ++si) {
        Slot& sl = slots[si];
        WaveAlloc& S = g->wave[si];
        sl.A = &S;
        sl.st = si == 0 ? g->stream : g->stream2;
        sl.ev = si == 0 ? g->ev : g->ev2;
        sl.B = B0;
        mg::WaveBuffers& B = sl.B;
        B.arr_t = S.arr_t.p;
        B.arr_bytes = S.arr_bytes.p;
        B.arr_mult = S.arr_mult.p;
        B.arr_noise = S.arr_noise.p;
        B.irq_e = P.any_irq_noise ? S.irq_e.p : nullptr;
        B.t_all = P.any_thinned ? S.t_all.p : nullptr;
        B.req_ms = S.req_ms.p;
        B.win_lat = S.win_lat.p;
        B.win_hist = S.win_hist.p;
        B.n_all = S.n_all.p;
        B.n_kept = S.n_kept.p;
        B.mt_pause = S.mt_pause.p;
        B.actions = S.actions.p;
        B.pauses = S.pauses.p;
        B.tout = S.tout.p;
        B.rout = S.rout.p;
        B.backlog = S.backlog.p;
        B.quant = S.quant.p;
        B.rings = rings_in_smem ? nullptr : S.rings.p;
        B.seeds = S.seeds.p;
        B.variant = S.variant.p;
        B.gen_overflow = S.gen_overflow.p;
        sl.wseeds.resize(W);
        sl.wvar.resize(W);
        sl.nkept.resize(W * T);
        sl.aoff.resize(W + 1);
        sl.poff.resize(W + 1);
    }

    const size_t sel_smem = mg::select_smem_bytes();
    CK(cudaFuncSetAttribute(mg::select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sel_smem)));
    const size_t cl_smem = mg::select_cluster_smem_bytes();
    CK(cudaFuncSetAttribute(mg::select_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cl_smem)));
    // MIGSIM_SELECT=cluster: the one-HBM-pass cluster select (same results; measured slower on the
    // C2 wave, 0.24 vs 0.15 ms -- DESIGN.md section 6)
    const char* sel_env = std::getenv("MIGSIM_SELECT");
    const bool sel_cluster = sel_env && std::string(sel_env) == "cluster";
    // MIGSIM_SELECT=two-pass: ignore the producer histogram (the two-pass digit select)
    const bool sel_two_pass = sel_env && std::string(sel_env) == "two-pass";

    res.tout.resize(n_jobs * T);
    res.quant.resize(n_jobs * T * 4);
    res.rout.resize(n_jobs);
    res.backlog.resize(n_jobs * R * 2);
    res.act_off.assign(n_jobs + 1, 0);
    res.pause_off.assign(n_jobs + 1, 0);
    if (keep) res.comp_off.assign(n_jobs + 1, 0);
    if (keep) res.crec_off.assign(n_jobs + 1, 0);

    double gen_ms = 0, des_ms = 0, sel_ms = 0;
    int64_t completions = 0, arrivals = 0, events = 0, waves = 0, samples = 0, launches = 0;
    // device span of the whole batch: first enqueue to the last kernel of either stream
    CK(cudaEventRecord(g->span[0], s));
    if (n_slots == 2) CK(cudaStreamWaitEvent(g->stream2, g->span[0], 0));

    // enqueue one wave: H2D of its seeds/variants, generator, event loop, select, histogram fold,
    // D2H of the per-replica status it needs before compaction
    auto launch_wave = [&](Slot& sl, size_t j0, int w) {
        WaveAlloc& S = *sl.A;
        const cudaStream_t st = sl.st;
        const mg::WaveBuffers& B = sl.B;
        sl.j0 = j0;
        sl.w = w;
        sl.busy = true;
        ++waves;
        launches += 7;  // gen_times, gen_marks, des, select, hist_reduce, compact_actions, compact_pauses
        for (int k = 0; k < w; ++k) {
            sl.wseeds[k] = seeds[(j0 + k) % seeds.size()];
            sl.wvar[k] = static_cast<int32_t>((j0 + k) / seeds.size());
        }
        CK(cpy_async(S.seeds.p, sl.wseeds.data(), sizeof(uint64_t) * w, cudaMemcpyHostToDevice, st));
        CK(cpy_async(S.variant.p, sl.wvar.data(), sizeof(int32_t) * w, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(S.gen_overflow.p, 0, sizeof(int32_t), st));
        CK(cudaEventRecord(sl.ev[0], st));
        CK(cudaMemsetAsync(S.win_hist.p, 0, sizeof(uint32_t) * w * T * mg::kHistBins, st));  // timed with gen
        const int64_t nt = static_cast<int64_t>(w) * T;
        mg::gen_times_kernel<<<static_cast<unsigned>(nt), 32, mg::gen_times_smem_bytes(), st>>>(A.scen.p, B, w);
        mg::gen_marks_kernel<<<static_cast<unsigned>(4 * nt), 32, 0, st>>>(A.scen.p, B, w);
        CK(cudaGetLastError());
        CK(cudaEventRecord(sl.ev[1], st));
        if (use_simt)
            mg::des_simt_kernel<<<static_cast<unsigned>((w + simt_lanes - 1) / simt_lanes), simt_lanes,
                                  static_cast<size_t>(Y.bytes(simt_lanes)), st>>>(A.scen.p, A.ctrl.p, B, w, Y);
        else
            des<<<static_cast<unsigned>(w), 32, static_cast<size_t>(L.total), st>>>(A.scen.p, A.ctrl.p, B, w, L);
        CK(cudaGetLastError());
        CK(cudaEventRecord(sl.ev[2], st));
        if (sel_cluster)
            mg::select_cluster_kernel<<<static_cast<unsigned>(nt * mg::select_cluster_size()), mg::select_cluster_threads(),
                                        cl_smem, st>>>(B, T, w);
        else {
            mg::WaveBuffers Bs = B;
            if (sel_two_pass) Bs.win_hist = nullptr;
            mg::select_kernel<<<static_cast<unsigned>(nt), mg::select_threads(), sel_smem, st>>>(Bs, T, w);
        }
        {
            constexpr int kChunk = 256;
            const dim3 grid(static_cast<unsigned>((T * mg::kHistBins + 255) / 256),
                            static_cast<unsigned>((w + kChunk - 1) / kChunk));
            mg::hist_reduce_kernel<<<grid, 256, 0, st>>>(S.win_hist.p, S.variant.p, w, T, kChunk, A.hist_sum.p);
        }
        CK(cudaGetLastError());
        CK(cudaEventRecord(sl.ev[3], st));
        CK(cpy_async(&sl.overflow, S.gen_overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        CK(cpy_async(res.rout.data() + j0, S.rout.p, sizeof(mg::ReplicaOut) * w, cudaMemcpyDeviceToHost, st));
        CK(cpy_async(sl.nkept.data(), S.n_kept.p, sizeof(int32_t) * w * T, cudaMemcpyDeviceToHost, st));
    };

    // keep_completions / traces: per-run completion records and trace rows (single-slot path)
    auto collect_keep = [&](size_t j0, int w) {

        std::vector<double> tmp(static_cast<size_t>(P.cap_sum) * 5);
        for (int k = 0; k < w; ++k) {
            const size_t job = j0 + k;
            const int64_t base = static_cast<int64_t>(k) * P.cap_sum;
            CK(cpy_sync(tmp.data() + 0 * P.cap_sum, A.c_done.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
            CK(cpy_sync(tmp.data() + 1 * P.cap_sum, A.c_total.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
            CK(cpy_sync(tmp.data() + 2 * P.cap_sum, A.c_compute.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
            CK(cpy_sync(tmp.data() + 3 * P.cap_sum, A.c_transfer.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
            CK(cpy_sync(tmp.data() + 4 * P.cap_sum, A.c_noise.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
            for (int i = 0; i < T; ++i) {
                const uint64_t n = res.tout[job * T + i].completed_total;
                for (uint64_t c = 0; c < n; ++c) {
                    const int64_t o = P.off[i] + static_cast<int64_t>(c);
                    const double rec[7] = {static_cast<double>(i), static_cast<double>(c), tmp[o],
                                           tmp[P.cap_sum + o], tmp[2 * P.cap_sum + o], tmp[3 * P.cap_sum + o],
                                           tmp[4 * P.cap_sum + o]};
                    res.comps.insert(res.comps.end(), rec, rec + 7);
                }
            }
            res.comp_off[job + 1] = static_cast<int64_t>(res.comps.size() / 7);
            {
                // engine::CompletionRecord list in the reference's kept_ order (engine.cpp:482-504):
                // requests complete FIFO per tenant, so completion c of tenant i is its c-th kept
                // arrival; c_order is the completion's position in the replica's sequence
                std::vector<double> arr(P.cap_sum), byt(P.cap_sum);
                std::vector<int64_t> ord(P.cap_sum);
                CK(cpy_sync(arr.data(), A.arr_t.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
                CK(cpy_sync(byt.data(), A.arr_bytes.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
                CK(cpy_sync(ord.data(), A.c_order.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
                const size_t c0 = res.crec.size();
                int64_t n_all = 0;
                for (int i = 0; i < T; ++i) n_all += static_cast<int64_t>(res.tout[job * T + i].completed_total);
                res.crec.resize(c0 + static_cast<size_t>(n_all));
                for (int i = 0; i < T; ++i) {
                    const uint64_t n = res.tout[job * T + i].completed_total;
                    for (uint64_t c = 0; c < n; ++c) {
                        const int64_t o = P.off[i] + static_cast<int64_t>(c);
                        if (ord[o] < 0 || ord[o] >= n_all) throw ParityGuard("completion order out of range");
                        migsim_completion& m = res.crec[c0 + static_cast<size_t>(ord[o])];
                        m.tenant = i;
                        m.seq = c;
                        m.arrived_s = arr[o];
                        m.done_s = tmp[o];
                        m.total_ms = tmp[P.cap_sum + o];
                        m.compute_ms = tmp[2 * P.cap_sum + o];
                        m.transfer_ms = tmp[3 * P.cap_sum + o];
                        m.noise_ms = tmp[4 * P.cap_sum + o];
                        m.transfer_bytes = byt[o];
                    }
                }
                res.crec_off[job + 1] = static_cast<int64_t>(res.crec.size());
            }
            if (traces) {
                mgb::TraceRows& tr = res.traces[job];
                tr.off = P.off;
                tr.n_done.resize(T);
                for (int i = 0; i < T; ++i) tr.n_done[i] = res.tout[job * T + i].completed_total;
                tr.done.assign(tmp.begin(), tmp.begin() + P.cap_sum);
                tr.total.assign(tmp.begin() + P.cap_sum, tmp.begin() + 2 * P.cap_sum);
                tr.compute.assign(tmp.begin() + 2 * P.cap_sum, tmp.begin() + 3 * P.cap_sum);
                tr.transfer.assign(tmp.begin() + 3 * P.cap_sum, tmp.begin() + 4 * P.cap_sum);
                tr.noise.assign(tmp.begin() + 4 * P.cap_sum, tmp.begin() + 5 * P.cap_sum);
                tr.arrived.resize(P.cap_sum);
                tr.bytes.resize(P.cap_sum);
                tr.order.resize(P.cap_sum);
                CK(cpy_sync(tr.arrived.data(), A.arr_t.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
                CK(cpy_sync(tr.bytes.data(), A.arr_bytes.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
                CK(cpy_sync(tr.order.data(), A.c_order.p + base, 8 * P.cap_sum, cudaMemcpyDeviceToHost));
                tr.n_ticks = n_ticks;
                tr.counters.resize(static_cast<size_t>(n_ticks) * T);
                tr.fabric.resize(static_cast<size_t>(n_ticks) * R);
                CK(cpy_sync(tr.counters.data(), A.tr_cnt.p + static_cast<size_t>(k) * n_ticks * T,
                              sizeof(mg::CounterRow) * n_ticks * T, cudaMemcpyDeviceToHost));
                CK(cpy_sync(tr.fabric.data(), A.tr_fab.p + static_cast<size_t>(k) * n_ticks * R,
                              sizeof(mg::FabricRow) * n_ticks * R, cudaMemcpyDeviceToHost));
            }
        }
            };

    // wait for a wave, compact its logs, copy its results back and fold them into the batch result
    auto finish_wave = [&](Slot& sl) {
        WaveAlloc& S = *sl.A;
        const cudaStream_t st = sl.st;
        const size_t j0 = sl.j0;
        const int w = sl.w;
        std::vector<int64_t>& aoff = sl.aoff;
        std::vector<int64_t>& poff = sl.poff;
        sl.busy = false;
        CK(cudaStreamSynchronize(st));
        if (sl.overflow) throw ParityGuard("arrival-record capacity exceeded");
        if (want_prof) {
            unsigned long long h[18];
            CK(cpy_sync(h, prof.p, sizeof(h), cudaMemcpyDeviceToHost));
            static const char* names[6] = {"resume", "expire", "transfer", "compute", "arrival", "tick"};
            for (int k = 0; k < 6; ++k)
                if (h[3 * k + 2])
                    std::fprintf(stderr, "[event-profile] %-8s n=%llu pick=%.0f run=%.0f cycles/event\n", names[k],
                                 h[3 * k + 2], static_cast<double>(h[3 * k]) / h[3 * k + 2],
                                 static_cast<double>(h[3 * k + 1]) / h[3 * k + 2]);
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, sl.ev[0], sl.ev[1]));
        gen_ms += ms;
        CK(cudaEventElapsedTime(&ms, sl.ev[1], sl.ev[2]));
        des_ms += ms;
        CK(cudaEventElapsedTime(&ms, sl.ev[2], sl.ev[3]));
        sel_ms += ms;
        aoff[0] = poff[0] = 0;
        for (int k = 0; k < w; ++k) {
            const mg::ReplicaOut& ro = res.rout[j0 + k];
            if (ro.error) throw ParityGuard("device log capacity exceeded (code " + std::to_string(ro.error) + ")");
            aoff[k + 1] = aoff[k] + ro.n_actions;
            poff[k + 1] = poff[k] + ro.n_pauses;
            events += static_cast<int64_t>(ro.n_events);
        }
        for (int k = 0; k < w * T; ++k) arrivals += sl.nkept[k];
        CK(cpy_async(S.act_off.p, aoff.data(), sizeof(int64_t) * (w + 1), cudaMemcpyHostToDevice, st));
        CK(cpy_async(S.pause_off.p, poff.data(), sizeof(int64_t) * (w + 1), cudaMemcpyHostToDevice, st));
        mg::compact_actions_kernel<<<static_cast<unsigned>(w), 64, 0, st>>>(S.actions.p, action_cap, S.rout.p,
                                                                            S.act_off.p, S.actions_c.p, w);
        mg::compact_pauses_kernel<<<static_cast<unsigned>(w), 64, 0, st>>>(S.pauses.p, pause_cap, S.rout.p,
                                                                           S.pause_off.p, S.pauses_c.p, w);
        CK(cudaGetLastError());
        const size_t a0 = res.actions.size(), p0 = res.pauses.size();
        res.actions.resize(a0 + static_cast<size_t>(aoff[w]));
        res.pauses.resize(p0 + static_cast<size_t>(poff[w]));
        for (int k = 0; k < w; ++k) {
            res.act_off[j0 + k + 1] = static_cast<int64_t>(a0) + aoff[k + 1];
            res.pause_off[j0 + k + 1] = static_cast<int64_t>(p0) + poff[k + 1];
        }
        if (aoff[w]) CK(cpy_async(res.actions.data() + a0, S.actions_c.p, sizeof(mg::ActionRec) * aoff[w], cudaMemcpyDeviceToHost, st));
        if (poff[w]) CK(cpy_async(res.pauses.data() + p0, S.pauses_c.p, sizeof(mg::PauseRec) * poff[w], cudaMemcpyDeviceToHost, st));
        CK(cpy_async(res.tout.data() + j0 * T, S.tout.p, sizeof(mg::TenantOut) * w * T, cudaMemcpyDeviceToHost, st));
        CK(cpy_async(res.quant.data() + j0 * T * 4, S.quant.p, sizeof(double) * w * T * 4, cudaMemcpyDeviceToHost, st));
        CK(cpy_async(res.backlog.data() + j0 * R * 2, S.backlog.p, sizeof(double) * w * R * 2, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int k = 0; k < w * T; ++k) {
            completions += static_cast<int64_t>(res.tout[j0 * T + k].completed_total);
            samples += static_cast<int64_t>(res.tout[j0 * T + k].completed_window);
        }
        if (keep) collect_keep(j0, w);
    };

    std::vector<size_t> starts;
    for (size_t j0 = 0; j0 < n_jobs; j0 += W) starts.push_back(j0);
    for (size_t k = 0; k < starts.size(); ++k) {
        Slot& sl = slots[k % n_slots];
        if (sl.busy) finish_wave(sl);
        launch_wave(sl, starts[k], static_cast<int>(std::min(W, n_jobs - starts[k])));
        if (n_slots == 2 && k >= 1 && slots[(k - 1) % 2].busy) finish_wave(slots[(k - 1) % 2]);
    }
    for (size_t k = starts.size() >= 2 ? starts.size() - 2 : 0; k < starts.size(); ++k)
        if (slots[k % n_slots].busy) finish_wave(slots[k % n_slots]);
    CK(cudaEventRecord(g->span[1], g->stream));
    if (n_slots == 2) CK(cudaEventRecord(g->span[2], g->stream2));
    CK(cudaStreamSynchronize(g->stream));
    if (n_slots == 2) CK(cudaStreamSynchronize(g->stream2));
    float span_ms = 0;
    CK(cudaEventElapsedTime(&span_ms, g->span[0], g->span[1]));
    if (n_slots == 2) {
        float ms2 = 0;
        CK(cudaEventElapsedTime(&ms2, g->span[0], g->span[2]));
        span_ms = std::max(span_ms, ms2);
    }
    res.hist.resize(n_var * T * mg::kHistBins);
    CK(cpy_async(res.hist.data(), A.hist_sum.p, sizeof(uint64_t) * res.hist.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    res.counts.assign(n_var * T * 3, 0);
    for (size_t job = 0; job < n_jobs; ++job) {
        const size_t v = job / seeds.size();
        for (int i = 0; i < T; ++i) {
            const mg::TenantOut& o = res.tout[job * T + i];
            uint64_t* c = res.counts.data() + (v * T + i) * 3;
            c[0] += o.completed_total;
            c[1] += o.completed_window;
            c[2] += o.window_misses;
        }
    }
    res.json.assign(n_jobs, std::string());
    res.timing.gen_ms = gen_ms;
    res.timing.des_ms = des_ms;
    res.timing.select_ms = sel_ms;
    // single slot: the kernels' own time; two slots: the device span (kernels overlap)
    res.timing.total_device_ms = n_slots == 2 ? static_cast<double>(span_ms) : gen_ms + des_ms + sel_ms;
    res.timing.pipeline_slots = n_slots;
    res.timing.replicas = static_cast<int64_t>(n_jobs);
    res.timing.tenant_ticks = static_cast<int64_t>(n_jobs) * T * P.scen.n_ticks;
    res.timing.completions = completions;
    res.timing.arrivals = arrivals;
    res.timing.events = events;
    res.timing.waves = waves;
    res.timing.select_samples = samples;
    res.timing.des_form = use_simt ? 1 : des_capped ? 2 : 0;
    res.timing.des_blocks_per_sm = des_blocks_per_sm;
    res.timing.des_smem_bytes = use_simt ? Y.bytes(simt_lanes) : L.total;
    res.timing.kernel_launches = launches;
    res.timing.h2d_bytes = h2d_bytes;
    res.timing.d2h_bytes = d2h_bytes;
    res.timing.wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
}

mgb::Variant to_variant(const migsim_variant& v) {
    mgb::Variant o;
    o.name = v.name ? v.name : "as-is";
    o.enabled = v.enabled;
    o.enable_mig = v.enable_mig;
    o.enable_placement = v.enable_placement;
    o.enable_guardrails = v.enable_guardrails;
    o.sample_interval_s = v.sample_interval_s;
    o.persistence_windows = v.persistence_windows;
    o.dwell_obs = v.dwell_obs;
    o.cooldown_obs = v.cooldown_obs;
    o.validation_obs = v.validation_obs;
    return o;
}

void run_batch_checked(migsim_gpu* g, const mgb::ScenarioSpec& spec, const std::vector<mgb::Variant>& vs,
                       const std::vector<uint64_t>& seeds, const migsim_run_opts& o, migsim_batch_result& res) {
    const int acap = o.action_cap > 0 ? o.action_cap : 1024;
    const int pcap = o.pause_cap > 0 ? o.pause_cap : 1024;
    try {
        run_batch_impl(g, spec, vs, seeds, o, res, 12.0, acap, pcap);
    } catch (const ParityGuard&) {
        // never truncate: rerun once with much larger device buffers
        res = migsim_batch_result{};
        run_batch_impl(g, spec, vs, seeds, o, res, 48.0, acap * 16, pcap * 16);
    }
}

// harness.cpp:32-43 (population sigma, summed in seed order)
void ci(const std::vector<double>& v, double& mean, double& half) {
    mean = half = 0.0;
    if (v.empty()) return;
    const double n = static_cast<double>(v.size());
    double sum = 0.0;
    for (double x : v) sum += x;
    mean = sum / n;
    double ss = 0.0;
    for (double x : v) ss += (x - mean) * (x - mean);
    half = 1.96 * std::sqrt(ss / n) / std::sqrt(n);
}

// RunResult of run 0 + its files (engine.cpp:889-892)
std::string write_artifacts(const migsim_batch_result& res, const std::string& dir, bool traces);

char* dup_c(const std::string& j) {
    char* o = static_cast<char*>(std::malloc(j.size() + 1));
    if (!o) throw std::bad_alloc();
    std::memcpy(o, j.c_str(), j.size() + 1);
    return o;
}

std::string num(double v) {
    char b[40];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

}  // namespace

extern "C" {

int migsim_gpu_open(int device, migsim_gpu** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw CudaError("no CUDA device " + std::to_string(device));
        CK(cudaSetDevice(device));
        auto* g = new migsim_gpu();
        g->device = device;
        CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&g->stream2, cudaStreamNonBlocking));
        for (auto& e : g->ev) CK(cudaEventCreate(&e));
        for (auto& e : g->ev2) CK(cudaEventCreate(&e));
        for (auto& e : g->span) CK(cudaEventCreate(&e));
        *out = g;
    });
}

void migsim_gpu_close(migsim_gpu* g) {
    if (!g) return;
    cudaSetDevice(g->device);
    for (auto* evs : {g->ev, g->ev2})
        for (int k = 0; k < 6; ++k)
            if (evs[k]) cudaEventDestroy(evs[k]);
    for (auto& e : g->span)
        if (e) cudaEventDestroy(e);
    if (g->stream) cudaStreamDestroy(g->stream);
    if (g->stream2) cudaStreamDestroy(g->stream2);
    delete g;
}

int migsim_gpu_load_scenario(migsim_gpu* g, const char* yaml_text, const char* source_name, int32_t* scenario_id,
                             char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        g->scenarios.push_back(mgb::parse_scenario(yaml_text, source_name ? source_name : "<scenario>"));
        *scenario_id = static_cast<int32_t>(g->scenarios.size() - 1);
    });
}

namespace {
mgb::InterferenceSchedule schedule_from(const migsim_schedule_desc& d) {
    mgb::InterferenceSchedule s;
    if (d.kind < 0 || d.kind > 2) throw mgb::ConfigError("unknown schedule kind " + std::to_string(d.kind), "<spec>");
    s.kind = static_cast<mgb::InterferenceSchedule::Kind>(d.kind);
    s.period_s = d.period_s;
    s.duty = d.duty;
    s.offset_s = d.offset_s;
    for (size_t k = 0; k < d.n_phases; ++k) s.phases.push_back({d.phase_start_s[k], d.phase_end_s[k]});
    return s;
}

// migsim_scenario_desc -> the engine's host ScenarioSpec, field for field (scenario.hpp:30-61)
mgb::ScenarioSpec spec_from(const migsim_scenario_desc& d) {
    mgb::ScenarioSpec s;
    s.name = d.name ? d.name : "";
    s.duration_s = d.duration_s;
    s.measure_start_s = d.measure_start_s;
    s.fabric_redistribute = d.fabric_redistribute != 0;
    for (size_t h = 0; h < d.n_hosts; ++h) {
        const migsim_host_desc& hd = d.hosts[h];
        mgb::HostSpec host;
        for (size_t k = 0; k < hd.n_gpus; ++k) {
            const migsim_gpu_desc& gd = hd.gpus[k];
            host.gpus.push_back({gd.id, gd.pcie_root_id, gd.numa_id, gd.core_group, gd.total_slices, gd.mig_enabled != 0});
        }
        host.numa_domains = hd.numa_domains;
        for (size_t k = 0; k < hd.n_roots; ++k) host.pcie_roots.push_back({hd.roots[k].id, hd.roots[k].capacity_Bps});
        for (size_t k = 0; k < hd.n_irq_hot; ++k) host.irq_hot_core_groups.insert(hd.irq_hot_core_groups[k]);
        host.io_capacity_Bps = hd.io_capacity_Bps;
        s.topology.hosts.push_back(std::move(host));
    }
    for (size_t i = 0; i < d.n_tenants; ++i) {
        const migsim_tenant_desc& td = d.tenants[i];
        mgb::TenantEntry e;
        if (!td.id) throw mgb::ConfigError("tenant " + std::to_string(i) + " has no id", "<spec>");
        e.spec.id = td.id;
        if (td.tclass < 0 || td.tclass > 2) throw mgb::ConfigError("unknown tenant class " + std::to_string(td.tclass), "<spec>");
        e.spec.tclass = static_cast<mgb::TenantClass>(td.tclass);
        e.spec.arrival_rate_hz = td.arrival_rate_hz;
        e.spec.arrival_cv = td.arrival_cv;
        for (size_t k = 0; k < td.n_mix; ++k) e.spec.transfer_mix.push_back({td.mix_bytes[k], td.mix_weight[k]});
        e.spec.base_compute_ms = td.base_compute_ms;
        e.spec.service_cv = td.service_cv;
        e.spec.slo_tail_ms = td.slo_tail_ms;
        e.spec.weight = td.weight;
        e.spec.pcie_cap_Bps = td.pcie_cap_Bps;
        e.spec.host_io_Bps = td.host_io_Bps;
        e.spec.sm_demand = td.sm_demand;
        e.spec.noise_mean_ms = td.noise_mean_ms;
        e.placement = {td.host, td.gpu, {td.first_slice, td.slice_count}};
        e.profile_name = td.profile ? td.profile : "";
        e.schedule = schedule_from(td.schedule);
        s.tenants.push_back(std::move(e));
    }
    for (size_t k = 0; k < d.n_irq_bursts; ++k) {
        const migsim_irq_desc& id = d.irq_bursts[k];
        s.irq_bursts.push_back({id.host, id.core_group, id.extra_noise_ms, schedule_from(id.schedule)});
    }
    const migsim_controller_desc& c = d.controller;
    mgb::ControllerConfig& o = s.controller;
    o.enabled = c.enabled != 0;
    o.enable_mig = c.enable_mig != 0;
    o.enable_placement = c.enable_placement != 0;
    o.enable_guardrails = c.enable_guardrails != 0;
    o.tail_threshold_ms = c.tail_threshold_ms;
    o.persistence_windows = c.persistence_windows;
    o.dwell_obs = c.dwell_obs;
    o.cooldown_obs = c.cooldown_obs;
    o.sample_interval_s = c.sample_interval_s;
    o.warmup_s = c.warmup_s;
    o.move_futility_ratio = c.move_futility_ratio;
    o.throttle_duration_s = c.throttle_duration_s;
    o.quota_duration_s = c.quota_duration_s;
    o.ema_alpha = c.ema_alpha;
    o.hysteresis_clear_ratio = c.hysteresis_clear_ratio;
    o.relax_stability_ratio = c.relax_stability_ratio;
    o.relax_score_threshold = c.relax_score_threshold;
    o.validation_obs = c.validation_obs;
    o.rollback_regress_ratio = c.rollback_regress_ratio;
    o.diag_pcie_util_threshold = c.diag_pcie_util_threshold;
    o.diag_host_io_threshold = c.diag_host_io_threshold;
    o.diag_sm_util_threshold = c.diag_sm_util_threshold;
    o.move_margin = c.move_margin;
    o.admission_queue_timeout_epochs = c.admission_queue_timeout_epochs;
    o.guardrail_io_throttle_Bps = c.guardrail_io_throttle_Bps;
    o.guardrail_mps_quota_pct = c.guardrail_mps_quota_pct;
    o.irq_lookback_s = c.irq_lookback_s;
    o.throughput_floor = c.throughput_floor;
    s.validate();
    return s;
}
}  // namespace

int migsim_gpu_load_spec(migsim_gpu* g, const migsim_scenario_desc* spec, int32_t* scenario_id, char* err,
                         size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!g || !spec || !scenario_id) throw std::runtime_error("null argument");
        g->scenarios.push_back(spec_from(*spec));
        *scenario_id = static_cast<int32_t>(g->scenarios.size() - 1);
    });
}

int migsim_gpu_release_scenario(migsim_gpu* g, int32_t id) {
    if (!g || id < 0 || id >= static_cast<int32_t>(g->scenarios.size())) return MIGSIM_ERR_CONFIG;
    g->scenarios[static_cast<size_t>(id)] = mgb::ScenarioSpec{};
    g->released.resize(g->scenarios.size(), 0);
    g->released[static_cast<size_t>(id)] = 1;
    return MIGSIM_OK;
}

int migsim_gpu_load_scenario_file(migsim_gpu* g, const char* path, int32_t* scenario_id, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        g->scenarios.push_back(mgb::load_scenario(path));
        *scenario_id = static_cast<int32_t>(g->scenarios.size() - 1);
    });
}

int migsim_scenario_n_tenants(migsim_gpu* g, int32_t id) {
    if (!g || id < 0 || id >= static_cast<int32_t>(g->scenarios.size())) return -1;
    return static_cast<int>(g->scenarios[static_cast<size_t>(id)].tenants.size());
}

int migsim_scenario_tenant_id(migsim_gpu* g, int32_t id, int32_t i, char* buf, size_t buflen) {
    if (!g || id < 0 || id >= static_cast<int32_t>(g->scenarios.size())) return MIGSIM_ERR_CONFIG;
    std::vector<std::string> ids;
    for (const auto& t : g->scenarios[static_cast<size_t>(id)].tenants) ids.push_back(t.spec.id);
    std::sort(ids.begin(), ids.end());
    if (i < 0 || i >= static_cast<int32_t>(ids.size())) return MIGSIM_ERR_CONFIG;
    std::snprintf(buf, buflen, "%s", ids[static_cast<size_t>(i)].c_str());
    return MIGSIM_OK;
}

int migsim_gpu_run_batch(migsim_gpu* g, int32_t scenario_id, const migsim_variant* variants, size_t n_variants,
                         const uint64_t* seeds, size_t n_seeds, const migsim_run_opts* opts, migsim_batch_result** out,
                         char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        check_scenario_id(g, scenario_id);
        if (n_seeds == 0) throw mgb::ConfigError("experiment needs at least one seed");
        std::vector<mgb::Variant> vs;
        for (size_t i = 0; i < n_variants; ++i) vs.push_back(to_variant(variants[i]));
        if (vs.empty()) vs.push_back(mgb::Variant{});
        migsim_run_opts o{};
        if (opts) o = *opts;
        auto res = std::make_unique<migsim_batch_result>();
        run_batch_checked(g, g->scenarios[static_cast<size_t>(scenario_id)], vs,
                          std::vector<uint64_t>(seeds, seeds + n_seeds), o, *res);
        *out = res.release();
    });
}

int migsim_gpu_run_scenario(migsim_gpu* g, int32_t scenario_id, const migsim_variant* variant, uint64_t seed,
                            const char* out_dir, int32_t write_traces, char** result_json, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        check_scenario_id(g, scenario_id);
        const std::string dir = out_dir ? out_dir : "";
        std::vector<mgb::Variant> vs(1);
        if (variant) vs[0] = to_variant(*variant);
        migsim_run_opts o{};
        o.write_traces = (write_traces && !dir.empty()) ? 1 : 0;
        auto res = std::make_unique<migsim_batch_result>();
        std::vector<uint64_t> seeds(1, seed);
        run_batch_checked(g, g->scenarios[static_cast<size_t>(scenario_id)], vs, seeds, o, *res);
        std::string js = write_artifacts(*res, dir, o.write_traces != 0);
        if (result_json) *result_json = dup_c(js);
    });
}

}  // extern "C"

namespace {
std::string write_artifacts(const migsim_batch_result& res, const std::string& dir, bool traces) {
    const mgb::RunResult rr = mgb::assemble(res.spec, res.P, res.variants[0].name, res.seeds[0], res.tout.data(),
                                            res.quant.data(), res.actions.data(), static_cast<int>(res.act_off[1]),
                                            res.pauses.data(), static_cast<int>(res.pause_off[1]), res.backlog.data(),
                                            res.rout[0].n_events);
    mgb::write_run_artifacts(dir, res.spec, res.P, rr, traces ? &res.traces[0] : nullptr);
    return mgb::result_to_json(rr);
}
}  // namespace

extern "C" {

size_t migsim_batch_n_runs(const migsim_batch_result* r) { return r ? r->n_runs : 0; }
int migsim_batch_n_tenants(const migsim_batch_result* r) { return r ? r->T : 0; }

int migsim_batch_timing(const migsim_batch_result* r, migsim_timing* t) {
    if (!r || !t) return MIGSIM_ERR_RUNTIME;
    *t = r->timing;
    return MIGSIM_OK;
}

int migsim_batch_tenant_rows(const migsim_batch_result* r, migsim_tenant_row* rows, size_t cap) {
    if (!r || !rows) return MIGSIM_ERR_RUNTIME;
    const double window_s = r->spec.duration_s - r->spec.measure_start_s;
    const size_t n = r->n_runs * static_cast<size_t>(r->T);
    if (cap < n) return MIGSIM_ERR_RUNTIME;
    for (size_t k = 0; k < n; ++k) {
        const mg::TenantOut& o = r->tout[k];
        migsim_tenant_row& w = rows[k];
        w.completed_total = o.completed_total;
        w.completed_window = o.completed_window;
        w.window_misses = o.window_misses;
        const double c = static_cast<double>(o.completed_window);
        w.mean_ms = o.completed_window ? o.sum_total_ms / c : 0.0;
        w.p50_ms = o.completed_window ? r->quant[4 * k + 0] : 0.0;
        w.p95_ms = o.completed_window ? r->quant[4 * k + 1] : 0.0;
        w.p99_ms = o.completed_window ? r->quant[4 * k + 2] : 0.0;
        w.p999_ms = o.completed_window ? r->quant[4 * k + 3] : 0.0;
        w.miss_rate = o.completed_window ? static_cast<double>(o.window_misses) / c : 0.0;
        w.throughput_hz = o.completed_window ? c / window_s : 0.0;
    }
    return MIGSIM_OK;
}

const char* migsim_batch_run_json(migsim_batch_result* r, size_t run) {
    if (!r || run >= r->n_runs) return nullptr;
    if (r->json[run].empty()) {
        const int T = r->T;
        const size_t v = run / r->seeds.size();
        const int64_t a0 = r->act_off[run], a1 = r->act_off[run + 1];
        const int64_t p0 = r->pause_off[run], p1 = r->pause_off[run + 1];
        mgb::RunResult rr = mgb::assemble(r->spec, r->P, r->variants[v].name, r->seeds[run % r->seeds.size()],
                                          r->tout.data() + run * T, r->quant.data() + run * T * 4,
                                          r->actions.data() + a0, static_cast<int>(a1 - a0), r->pauses.data() + p0,
                                          static_cast<int>(p1 - p0), r->backlog.data() + run * r->R * 2,
                                          r->rout[run].n_events);
        r->json[run] = mgb::result_to_json(rr);
    }
    return r->json[run].c_str();
}

int64_t migsim_batch_completions(const migsim_batch_result* r, size_t run, double* out, int64_t cap) {
    if (!r || run >= r->n_runs || r->comp_off.empty()) return -1;
    const int64_t c0 = r->comp_off[run], c1 = r->comp_off[run + 1];
    const int64_t n = c1 - c0;
    if (out) std::memcpy(out, r->comps.data() + 7 * c0, sizeof(double) * 7 * static_cast<size_t>(std::min(n, cap)));
    return n;
}

void migsim_batch_result_free(migsim_batch_result* r) { delete r; }

int64_t migsim_batch_completion_records(const migsim_batch_result* r, size_t run, migsim_completion* out, int64_t cap) {
    if (!r || run >= r->n_runs || r->crec_off.empty()) return -1;
    const int64_t a = r->crec_off[run], b = r->crec_off[run + 1];
    if (!out) return b - a;
    const int64_t n = std::min(cap, b - a);
    if (n > 0) std::memcpy(out, r->crec.data() + a, sizeof(migsim_completion) * static_cast<size_t>(n));
    return b - a;
}

size_t migsim_batch_n_variants(const migsim_batch_result* r) { return r ? r->variants.size() : 0; }

int migsim_batch_latency_hist(const migsim_batch_result* r, uint64_t* out, size_t cap) {
    if (!r || !out || cap < r->hist.size()) return MIGSIM_ERR_RUNTIME;
    std::memcpy(out, r->hist.data(), sizeof(uint64_t) * r->hist.size());
    return MIGSIM_OK;
}

int migsim_batch_tenant_counts(const migsim_batch_result* r, uint64_t* out, size_t cap) {
    if (!r || !out || cap < r->counts.size()) return MIGSIM_ERR_RUNTIME;
    std::memcpy(out, r->counts.data(), sizeof(uint64_t) * r->counts.size());
    return MIGSIM_OK;
}

int migsim_hist_bin_edges(double* lo, size_t n) {
    if (!lo || n < static_cast<size_t>(mg::kHistBins)) return MIGSIM_ERR_RUNTIME;
    for (int b = 0; b < mg::kHistBins; ++b) {
        const uint64_t bits = mg::lat_bin_lo(static_cast<uint32_t>(b)) & ~(1ull << 63);  // positive values
        std::memcpy(lo + b, &bits, 8);
    }
    return MIGSIM_OK;
}

int migsim_gpu_select(migsim_gpu* g, const double* vals, const int64_t* seg_off, size_t n_segments, const double* qs,
                      size_t n_q, double* out, double* device_ms, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        CK(cudaSetDevice(g->device));
        if (device_ms) *device_ms = 0.0;
        if (n_segments == 0 || n_q == 0) return;  // nothing to select: an empty result, no launch
        const int64_t n = seg_off[n_segments];
        DevBuf<double> dv, dq, dout;
        DevBuf<int64_t> doff;
        dv.alloc(static_cast<size_t>(std::max<int64_t>(n, 1)));
        dq.alloc(n_q);
        dout.alloc(n_segments * n_q);
        doff.alloc(n_segments + 1);
        cudaStream_t s = g->stream;
        if (n) CK(cudaMemcpyAsync(dv.p, vals, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dq.p, qs, sizeof(double) * n_q, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(doff.p, seg_off, sizeof(int64_t) * (n_segments + 1), cudaMemcpyHostToDevice, s));
        const size_t sm = mg::select_smem_bytes();
        CK(cudaFuncSetAttribute(mg::select_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        CK(cudaEventRecord(g->ev[4], s));
        mg::select_segments_kernel<<<static_cast<unsigned>(n_segments), mg::select_threads(), sm, s>>>(dv.p, doff.p, static_cast<int>(n_segments),
                                                                                       dq.p, static_cast<int>(n_q), dout.p);
        CK(cudaGetLastError());
        CK(cudaEventRecord(g->ev[5], s));
        CK(cudaMemcpyAsync(out, dout.p, sizeof(double) * n_segments * n_q, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, g->ev[4], g->ev[5]));
        if (device_ms) *device_ms = ms;
    });
}

int migsim_run_plan(migsim_gpu* g, const char* plan, const char* scenario_path, int32_t n_seeds, uint64_t seed_base,
                    const char* focus_tenant, const char* out_dir, char** experiment_json, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto wall0 = std::chrono::steady_clock::now();
        if (n_seeds < 1) throw mgb::ConfigError("experiment needs at least one seed");
        const mgb::ScenarioSpec base = mgb::load_scenario(scenario_path);
        std::string focus = focus_tenant ? focus_tenant : "";
        if (focus.empty()) {  // harness.cpp:80-87: smallest tail SLO, first in file order on ties
            const mgb::TenantEntry* best = nullptr;
            for (const auto& t : base.tenants)
                if (!best || t.spec.slo_tail_ms < best->spec.slo_tail_ms) best = &t;
            focus = best->spec.id;
        }
        base.tenant(focus);
        const std::string p = plan ? plan : "e1";
        std::vector<mgb::Variant> vs;
        auto mk = [](const char* name, int en, int mig, int pl, int gu) {
            mgb::Variant v;
            v.name = name;
            v.enabled = en;
            v.enable_mig = mig;
            v.enable_placement = pl;
            v.enable_guardrails = gu;
            return v;
        };
        if (p == "e1" || p == "llm") {
            vs = {mk("full", 1, 1, 1, 1), mk("static", 0, 0, 0, 0)};
        } else if (p == "e2") {
            vs = {mk("full", 1, 1, 1, 1), mk("mig-only", 1, 1, 0, 0), mk("placement-only", 1, 0, 1, 0),
                  mk("guards-only", 1, 0, 0, 1), mk("static", 0, 0, 0, 0)};
        } else if (p == "e3") {
            char name[48];
            for (double dt : {1.0, 2.0, 5.0}) {
                std::snprintf(name, sizeof(name), "interval=%.0fs", dt);
                mgb::Variant v;
                v.name = name;
                v.sample_interval_s = dt;
                vs.push_back(v);
            }
            for (int y : {2, 3, 5}) {
                std::snprintf(name, sizeof(name), "persistence=%d", y);
                mgb::Variant v;
                v.name = name;
                v.persistence_windows = y;
                vs.push_back(v);
            }
            for (int d : {128, 256, 512}) {
                std::snprintf(name, sizeof(name), "dwell=%d", d);
                mgb::Variant v;
                v.name = name;
                v.dwell_obs = d;
                v.cooldown_obs = d / 2;
                vs.push_back(v);
            }
        } else {
            throw mgb::ConfigError("unknown experiment plan '" + p + "'");
        }
        std::vector<uint64_t> seeds;
        for (int s = 0; s < n_seeds; ++s) seeds.push_back(seed_base + static_cast<uint64_t>(s));
        migsim_batch_result res;
        run_batch_checked(g, base, vs, seeds, migsim_run_opts{}, res);
        int fidx = 0;
        for (int i = 0; i < res.T; ++i)
            if (res.P.tenant_ids[static_cast<size_t>(i)] == focus) fidx = i;
        const double window_s = base.duration_s - base.measure_start_s;
        std::vector<mgb::PlanVariantOut> agg(vs.size());
        for (size_t v = 0; v < vs.size(); ++v) agg[v].name = vs[v].name;
        const std::string dir = out_dir ? out_dir : "";
        for (size_t run = 0; run < res.n_runs; ++run) {
            mgb::PlanVariantOut& a = agg[run / seeds.size()];
            a.seeds.push_back(seeds[run % seeds.size()]);
            const mg::TenantOut& o = res.tout[run * res.T + fidx];
            const double c = static_cast<double>(o.completed_window);
            a.p99_ms.push_back(o.completed_window ? res.quant[(run * res.T + fidx) * 4 + 2] : 0.0);
            a.miss_rate.push_back(o.completed_window ? static_cast<double>(o.window_misses) / c : 0.0);
            double thr = 0.0;
            for (int i = 0; i < res.T; ++i) {
                const mg::TenantOut& x = res.tout[run * res.T + i];
                thr += x.completed_window ? static_cast<double>(x.completed_window) / window_s : 0.0;
            }
            a.throughput_hz.push_back(thr);
            if (!dir.empty()) {  // per-job artifacts, write_traces=false (harness.cpp:131-133,166-171)
                const mgb::RunResult rr = mgb::assemble(
                    res.spec, res.P, a.name, a.seeds.back(), res.tout.data() + run * res.T,
                    res.quant.data() + run * res.T * 4, res.actions.data() + res.act_off[run],
                    static_cast<int>(res.act_off[run + 1] - res.act_off[run]), res.pauses.data() + res.pause_off[run],
                    static_cast<int>(res.pause_off[run + 1] - res.pause_off[run]), res.backlog.data() + run * res.R * 2,
                    res.rout[run].n_events);
                mgb::write_run_artifacts(dir + "/" + a.name + "/seed" + std::to_string(a.seeds.back()), res.spec,
                                         res.P, rr, nullptr);
            }
        }
        for (auto& a : agg) {
            ci(a.p99_ms, a.mean[0], a.half[0]);
            ci(a.miss_rate, a.mean[1], a.half[1]);
            ci(a.throughput_hz, a.mean[2], a.half[2]);
        }
        const double wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
        const std::string j = mgb::experiment_json_text(p, base.name, focus, wall_s, agg);
        if (!dir.empty()) {  // harness.cpp:208-214
            std::filesystem::create_directories(dir);
            mgb::put_text_file(dir + "/experiment.json", j + "\n");
            mgb::put_text_file(dir + "/summary.csv", mgb::experiment_csv_text(agg));
        }
        char* outp = static_cast<char*>(std::malloc(j.size() + 1));
        std::memcpy(outp, j.c_str(), j.size() + 1);
        *experiment_json = outp;
    });
}

void migsim_free(void* p) { std::free(p); }

int migsim_gpu_admit(migsim_gpu* g, int32_t scenario_id, size_t n, const int32_t* tenant, const int32_t* profile,
                     const int32_t* admitted, const int32_t* host, const int32_t* gpu_id, const int32_t* first,
                     const int32_t* count, const double* tenant_pcie_Bps, const double* tenant_host_io_Bps,
                     const uint32_t* irq_recent, int32_t* queue_epochs, migsim_admit_decision* out, double* device_ms,
                     char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        check_scenario_id(g, scenario_id);
        CK(cudaSetDevice(g->device));
        const mgb::ScenarioSpec& spec = g->scenarios[static_cast<size_t>(scenario_id)];
        const mgb::Packed P = mgb::pack(spec, {});
        const int T = P.scen.n_tenants, H = P.scen.n_hosts;
        // (host, gpu id) -> canonical GPU index; validate every case on the host
        std::vector<int32_t> gidx(n * T);
        auto find_gpu = [&](int h, int id) {
            for (int k = 0; k < P.scen.n_gpus; ++k)
                if (P.scen.gpus[k].host == h && P.scen.gpus[k].id == id) return k;
            return -1;
        };
        for (size_t c = 0; c < n; ++c) {
            if (tenant[c] < 0 || tenant[c] >= T) throw mgb::ConfigError("admit: tenant index out of range");
            if (profile[c] < 0 || profile[c] >= mg::kNumProfiles) throw mgb::ConfigError("admit: unknown MIG profile");
            for (int j = 0; j < T; ++j) {
                const size_t x = c * T + j;
                gidx[x] = admitted[x] ? find_gpu(host[x], gpu_id[x]) : 0;
                if (gidx[x] < 0)
                    throw mgb::ConfigError("admit: no GPU " + std::to_string(gpu_id[x]) + " on host " + std::to_string(host[x]));
            }
        }
        DevBuf<mg::PScenario> dS;
        DevBuf<int32_t> dt, dp, da, dh, dg, df, dc, dq;
        DevBuf<double> dpc, dio;
        DevBuf<uint32_t> dirq;
        DevBuf<mg::AdmitOut> dout;
        dS.alloc(1);
        auto up = [&](auto& buf, const auto* src, size_t cnt) {
            buf.alloc(cnt ? cnt : 1);
            if (cnt) CK(cudaMemcpyAsync(buf.p, src, sizeof(*src) * cnt, cudaMemcpyHostToDevice, g->stream));
        };
        cudaStream_t s = g->stream;
        CK(cudaMemcpyAsync(dS.p, &P.scen, sizeof(mg::PScenario), cudaMemcpyHostToDevice, s));
        up(dt, tenant, n);
        up(dp, profile, n);
        up(da, admitted, n * T);
        up(dh, host, n * T);
        up(dg, gidx.data(), n * T);
        up(df, first, n * T);
        up(dc, count, n * T);
        up(dpc, tenant_pcie_Bps, n * T);
        up(dio, tenant_host_io_Bps, n * T);
        up(dirq, irq_recent, n * H);
        if (queue_epochs) up(dq, queue_epochs, n);
        dout.alloc(n ? n : 1);
        mg::AdmitCases C{dt.p, dp.p, da.p, dh.p, dg.p, df.p, dc.p, dpc.p, dio.p, dirq.p, queue_epochs ? dq.p : nullptr};
        CK(cudaEventRecord(g->ev[4], s));
        if (n) mg::admit_kernel<<<static_cast<unsigned>(n), 32, 0, s>>>(dS.p, C, static_cast<int>(n),
                                                                       spec.controller.admission_queue_timeout_epochs, dout.p);
        CK(cudaGetLastError());
        CK(cudaEventRecord(g->ev[5], s));
        std::vector<mg::AdmitOut> h(n);
        if (n) CK(cudaMemcpyAsync(h.data(), dout.p, sizeof(mg::AdmitOut) * n, cudaMemcpyDeviceToHost, s));
        if (n && queue_epochs) CK(cudaMemcpyAsync(queue_epochs, dq.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, g->ev[4], g->ev[5]));
        if (device_ms) *device_ms = ms;
        for (size_t c = 0; c < n; ++c) {
            out[c].outcome = h[c].outcome;
            out[c].host = h[c].host;
            out[c].gpu = h[c].gpu_id;
            out[c].first = h[c].first;
            out[c].count = h[c].count;
            out[c].profile = h[c].profile;
            out[c].reason = h[c].reason;
            out[c].pad = 0;
            out[c].score = h[c].score;
        }
    });
}

int migsim_render_report(const char* experiment_json, char** report, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { *report = dup_c(mgb::render_report_text(experiment_json ? experiment_json : "")); });
}

int migsim_scenario_dump(const char* path, char** json, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const mgb::ScenarioSpec s = mgb::load_scenario(path);
        auto sched = [](const mgb::InterferenceSchedule& x) {
            std::string o = "{\"kind\":\"";
            o += x.kind == mgb::InterferenceSchedule::Kind::always ? "always"
                 : x.kind == mgb::InterferenceSchedule::Kind::square_wave ? "square_wave" : "phases";
            o += "\",\"period_s\":" + num(x.period_s) + ",\"duty\":" + num(x.duty) + ",\"offset_s\":" + num(x.offset_s) +
                 ",\"phases\":[";
            for (size_t i = 0; i < x.phases.size(); ++i)
                o += (i ? "," : "") + std::string("[") + num(x.phases[i].start_s) + "," + num(x.phases[i].end_s) + "]";
            return o + "]}";
        };
        std::string j = "{\"name\":\"" + mgb::json_escape(s.name) + "\",\"duration_s\":" + num(s.duration_s) +
                        ",\"measure_start_s\":" + num(s.measure_start_s) +
                        ",\"fabric_redistribute\":" + (s.fabric_redistribute ? "true" : "false") + ",\"hosts\":[";
        for (size_t h = 0; h < s.topology.hosts.size(); ++h) {
            const auto& H = s.topology.hosts[h];
            j += (h ? "," : "") + std::string("{\"numa_domains\":") + std::to_string(H.numa_domains) +
                 ",\"io_capacity_Bps\":" + num(H.io_capacity_Bps) + ",\"irq_hot_core_groups\":[";
            size_t k = 0;
            for (int c : H.irq_hot_core_groups) j += (k++ ? "," : "") + std::to_string(c);
            j += "],\"pcie_roots\":[";
            for (size_t r = 0; r < H.pcie_roots.size(); ++r)
                j += (r ? "," : "") + std::string("{\"id\":") + std::to_string(H.pcie_roots[r].id) +
                     ",\"capacity_Bps\":" + num(H.pcie_roots[r].capacity_Bps) + "}";
            j += "],\"gpus\":[";
            for (size_t g2 = 0; g2 < H.gpus.size(); ++g2) {
                const auto& G = H.gpus[g2];
                j += (g2 ? "," : "") + std::string("{\"id\":") + std::to_string(G.id) + ",\"pcie_root_id\":" +
                     std::to_string(G.pcie_root_id) + ",\"numa_id\":" + std::to_string(G.numa_id) + ",\"core_group\":" +
                     std::to_string(G.core_group) + ",\"total_slices\":" + std::to_string(G.total_slices) +
                     ",\"mig_enabled\":" + (G.mig_enabled ? "true" : "false") + "}";
            }
            j += "]}";
        }
        j += "],\"tenants\":[";
        for (size_t i = 0; i < s.tenants.size(); ++i) {
            const auto& e = s.tenants[i];
            const auto& t = e.spec;
            j += (i ? "," : "") + std::string("{\"id\":\"") + mgb::json_escape(t.id) + "\",\"class\":\"" +
                 mgb::to_string(t.tclass) + "\",\"arrival_rate_hz\":" + num(t.arrival_rate_hz) + ",\"arrival_cv\":" +
                 num(t.arrival_cv) + ",\"transfer_mix\":[";
            for (size_t m = 0; m < t.transfer_mix.size(); ++m)
                j += (m ? "," : "") + std::string("[") + num(t.transfer_mix[m].bytes) + "," + num(t.transfer_mix[m].weight) + "]";
            j += "],\"base_compute_ms\":" + num(t.base_compute_ms) + ",\"service_cv\":" + num(t.service_cv) +
                 ",\"slo_tail_ms\":" + num(t.slo_tail_ms) + ",\"weight\":" + num(t.weight) + ",\"pcie_cap_Bps\":" +
                 num(t.pcie_cap_Bps) + ",\"host_io_Bps\":" + num(t.host_io_Bps) + ",\"sm_demand\":" + num(t.sm_demand) +
                 ",\"noise_mean_ms\":" + num(t.noise_mean_ms) + ",\"host\":" + std::to_string(e.placement.host) +
                 ",\"gpu\":" + std::to_string(e.placement.gpu) + ",\"first_slice\":" +
                 std::to_string(e.placement.slices.first) + ",\"slice_count\":" + std::to_string(e.placement.slices.count) +
                 ",\"profile\":\"" + e.profile_name + "\",\"schedule\":" + sched(e.schedule) + "}";
        }
        j += "],\"irq_bursts\":[";
        for (size_t b = 0; b < s.irq_bursts.size(); ++b) {
            const auto& q = s.irq_bursts[b];
            j += (b ? "," : "") + std::string("{\"host\":") + std::to_string(q.host) + ",\"core_group\":" +
                 std::to_string(q.core_group) + ",\"extra_noise_ms\":" + num(q.extra_noise_ms) + ",\"schedule\":" +
                 sched(q.schedule) + "}";
        }
        const auto& c = s.controller;
        auto B = [](bool v) { return std::string(v ? "true" : "false"); };
        j += "],\"controller\":{\"enabled\":" + B(c.enabled) + ",\"enable_mig\":" + B(c.enable_mig) +
             ",\"enable_placement\":" + B(c.enable_placement) + ",\"enable_guardrails\":" + B(c.enable_guardrails) +
             ",\"tail_threshold_ms\":" + num(c.tail_threshold_ms) + ",\"persistence_windows\":" +
             std::to_string(c.persistence_windows) + ",\"dwell_obs\":" + std::to_string(c.dwell_obs) +
             ",\"cooldown_obs\":" + std::to_string(c.cooldown_obs) + ",\"sample_interval_s\":" + num(c.sample_interval_s) +
             ",\"warmup_s\":" + num(c.warmup_s) + ",\"move_futility_ratio\":" + num(c.move_futility_ratio) +
             ",\"throttle_duration_s\":" + num(c.throttle_duration_s) + ",\"quota_duration_s\":" +
             num(c.quota_duration_s) + ",\"ema_alpha\":" + num(c.ema_alpha) + ",\"hysteresis_clear_ratio\":" +
             num(c.hysteresis_clear_ratio) + ",\"relax_stability_ratio\":" + num(c.relax_stability_ratio) +
             ",\"relax_score_threshold\":" + num(c.relax_score_threshold) + ",\"validation_obs\":" +
             std::to_string(c.validation_obs) + ",\"rollback_regress_ratio\":" + num(c.rollback_regress_ratio) +
             ",\"diag_pcie_util_threshold\":" + num(c.diag_pcie_util_threshold) + ",\"diag_host_io_threshold\":" +
             num(c.diag_host_io_threshold) + ",\"diag_sm_util_threshold\":" + num(c.diag_sm_util_threshold) +
             ",\"move_margin\":" + num(c.move_margin) + ",\"admission_queue_timeout_epochs\":" +
             std::to_string(c.admission_queue_timeout_epochs) + ",\"guardrail_io_throttle_Bps\":" +
             num(c.guardrail_io_throttle_Bps) + ",\"guardrail_mps_quota_pct\":" + num(c.guardrail_mps_quota_pct) +
             ",\"irq_lookback_s\":" + num(c.irq_lookback_s) + ",\"throughput_floor\":" + num(c.throughput_floor) + "}}";
        char* o = static_cast<char*>(std::malloc(j.size() + 1));
        std::memcpy(o, j.c_str(), j.size() + 1);
        *json = o;
    });
}

int migsim_gpu_libm(migsim_gpu* g, int fn, const double* x, const double* y, double* out, size_t n, char* err,
                    size_t errlen) {
    return guarded(err, errlen, [&] {
        CK(cudaSetDevice(g->device));
        DevBuf<double> dx, dy, dout;
        dx.alloc(n);
        dy.alloc(n);
        dout.alloc(n);
        cudaStream_t s = g->stream;
        CK(cudaMemcpyAsync(dx.p, x, 8 * n, cudaMemcpyHostToDevice, s));
        if (y) CK(cudaMemcpyAsync(dy.p, y, 8 * n, cudaMemcpyHostToDevice, s));
        else CK(cudaMemsetAsync(dy.p, 0, 8 * n, s));
        mg::libm_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(fn, dx.p, dy.p, dout.p,
                                                                               static_cast<int64_t>(n));
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, dout.p, 8 * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

int migsim_gpu_arrivals(migsim_gpu* g, int32_t scenario_id, uint64_t seed, int32_t tenant, double* out, int64_t cap,
                        int64_t* n_out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        check_scenario_id(g, scenario_id);
        CK(cudaSetDevice(g->device));
        const mgb::Packed P = mgb::pack(g->scenarios[static_cast<size_t>(scenario_id)], {});
        const int T = P.scen.n_tenants;
        if (tenant < 0 || tenant >= T) throw mgb::ConfigError("tenant index out of range");
        WaveAlloc A;
        const size_t big = static_cast<size_t>(P.cap_sum);
        A.arr_t.alloc(big);
        A.arr_bytes.alloc(big);
        A.arr_mult.alloc(big);
        A.arr_noise.alloc(big);
        A.irq_e.alloc(big);
        A.t_all.alloc(big);
        A.n_all.alloc(T);
        A.n_kept.alloc(T);
        A.seeds.alloc(1);
        A.gen_overflow.alloc(1);
        A.off.alloc(T);
        A.cap.alloc(T);
        A.scen.alloc(1);
        cudaStream_t s = g->stream;
        CK(cudaMemcpyAsync(A.scen.p, &P.scen, sizeof(mg::PScenario), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(A.off.p, P.off.data(), 8 * T, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(A.cap.p, P.cap.data(), 8 * T, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(A.seeds.p, &seed, 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(A.gen_overflow.p, 0, 4, s));
        mg::WaveBuffers B{};
        B.arr_t = A.arr_t.p;
        B.arr_bytes = A.arr_bytes.p;
        B.arr_mult = A.arr_mult.p;
        B.arr_noise = A.arr_noise.p;
        B.irq_e = A.irq_e.p;
        B.t_all = A.t_all.p;
        B.n_all = A.n_all.p;
        B.n_kept = A.n_kept.p;
        B.seeds = A.seeds.p;
        B.off = A.off.p;
        B.cap = A.cap.p;
        B.gen_overflow = A.gen_overflow.p;
        B.cap_sum = P.cap_sum;
        B.any_irq_noise = P.any_irq_noise;
        mg::gen_times_kernel<<<static_cast<unsigned>(T), 32, mg::gen_times_smem_bytes(), s>>>(A.scen.p, B, 1);
        mg::gen_marks_kernel<<<static_cast<unsigned>(4 * T), 32, 0, s>>>(A.scen.p, B, 1);
        CK(cudaGetLastError());
        std::vector<int32_t> nk(T);
        int32_t overflow = 0;
        CK(cudaMemcpyAsync(nk.data(), A.n_kept.p, 4 * T, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&overflow, A.gen_overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (overflow) throw ParityGuard("arrival-record capacity exceeded");  // never return a truncated list
        const int64_t n = nk[tenant];
        *n_out = n;
        const int64_t m = std::min(n, cap);
        std::vector<double> a(static_cast<size_t>(std::max<int64_t>(m, 1))), b(a), c(a), d(a);
        const int64_t o = P.off[tenant];
        if (m > 0) {
            CK(cudaMemcpy(a.data(), A.arr_t.p + o, 8 * m, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(b.data(), A.arr_bytes.p + o, 8 * m, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(c.data(), A.arr_mult.p + o, 8 * m, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(d.data(), A.arr_noise.p + o, 8 * m, cudaMemcpyDeviceToHost));
        }
        for (int64_t k = 0; k < m; ++k) {
            out[4 * k + 0] = a[k];
            out[4 * k + 1] = b[k];
            out[4 * k + 2] = c[k];
            out[4 * k + 3] = d[k];
        }
    });
}

}  // extern "C"
