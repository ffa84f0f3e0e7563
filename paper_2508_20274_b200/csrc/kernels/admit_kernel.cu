// Batched admission control: Controller::admit (controller.cpp:637-692) over many independent
// cases -- exhaustive placement-candidate scoring, one warp per case, one lane per candidate GPU.
//
// A case = (scenario topology + tenant specs, the cluster state: which tenants are admitted and
// where, the snapshot fields placement_score reads, the request: tenant k at MIG profile p).
//   rate gate     arrival_rate >= effective_service_rate(profile)   (model.cpp:208-212) -> rejected
//   candidates    every (host, gpu) in topology order with a free contiguous slice run
//                 (find_slice_run, controller.cpp:72-99) whose root keeps the summed bandwidth
//                 claims below capacity (controller.cpp:653-660, claims summed in tenant-id order)
//   score         placement_score(...).total() (controller.cpp:101-123): PCIe share of bandwidth-
//                 heavy neighbours on the root + NUMA-local host I/O share + recent IRQ (0/1)
//   choice        minimum score, ties to the smaller (host, gpu id, first)  (controller.cpp:662-668)
//   no slot       queue_epochs_[tenant] += 1; rejected (entry erased) once it exceeds
//                 admission_queue_timeout_epochs, else queued (controller.cpp:677-691); an admitted
//                 request erases the entry (:671).  The per-case epochs are in/out, so a caller can
//                 carry each controller's queue across calls (retry epochs).
// All sums run in the reference's order with IEEE division (no FMA contraction: --fmad=false), so
// outcomes, placements and scores are bit-identical to the reference.
#include "admit_kernel.cuh"

namespace mg {

namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

}  // namespace

__global__ void __launch_bounds__(32) admit_kernel(const PScenario* __restrict__ S, AdmitCases C, int n_cases,
                                                   int queue_timeout_epochs, AdmitOut* __restrict__ out) {
    const int c = blockIdx.x;
    if (c >= n_cases) return;
    const int lane = threadIdx.x;
    const int T = S->n_tenants;
    const int k = C.tenant[c];
    const int prof = C.profile[c];
    const int32_t* adm = C.admitted + static_cast<int64_t>(c) * T;
    const int32_t* th = C.host + static_cast<int64_t>(c) * T;
    const int32_t* tg = C.gpu + static_cast<int64_t>(c) * T;
    const int32_t* tf = C.first + static_cast<int64_t>(c) * T;
    const int32_t* tc = C.count + static_cast<int64_t>(c) * T;
    const double* pcie = C.tenant_pcie + static_cast<int64_t>(c) * T;
    const double* hio = C.tenant_host_io + static_cast<int64_t>(c) * T;
    const uint32_t* irq = C.irq_recent + static_cast<int64_t>(c) * S->n_hosts;
    const PTenant& sp = S->tenants[k];
    AdmitOut o;
    o.outcome = kAdmitRejected;
    o.host = o.gpu_id = o.first = -1;
    o.count = profile_slices(prof);
    o.profile = prof;
    o.reason = kReasonRate;
    o.score = 0.0;
    // rate gate: mu = sm_fraction / (base_ms / 1000)  (model.cpp:208-212, MigProfile::sm_fraction)
    const double frac = ddiv(static_cast<double>(o.count), 7.0);
    const double mu = ddiv(frac, ddiv(sp.base_compute_ms, 1000.0));
    if (sp.arrival_rate_hz >= mu) {
        if (lane == 0) out[c] = o;
        return;
    }
    // lanes walk the GPUs in topology order (host-major); warp-strided for > 32 GPUs
    double best = 0.0;
    int bh = -1, bg = -1, bf = -1, bidx = -1;
    for (int gi = lane; gi < S->n_gpus; gi += 32) {
        const PGpu& g = S->gpus[gi];
        // find_slice_run(gpu, states, host, slices) -- no preference, nothing ignored
        int run = -1;
        if (o.count > 0 && o.count <= g.total_slices) {
            uint64_t used = 0;
            for (int j = 0; j < T; ++j) {
                if (!adm[j] || th[j] != g.host || tg[j] != gi) continue;
                for (int s = tf[j]; s < tf[j] + tc[j]; ++s)
                    if (s >= 0 && s < g.total_slices) used |= 1ull << s;
            }
            for (int f = 0; f + o.count <= g.total_slices && run < 0; ++f) {
                bool ok = true;
                for (int s = f; s < f + o.count; ++s) ok &= !((used >> s) & 1ull);
                if (ok) run = f;
            }
        }
        if (run < 0) continue;
        // claims on this root (controller.cpp:653-659): own claim + admitted others, id order
        double claims = sp.claim;
        for (int j = 0; j < T; ++j) {
            if (!adm[j] || th[j] != g.host) continue;
            if (S->gpus[tg[j]].root != g.root) continue;
            claims = dadd(claims, S->tenants[j].claim);
        }
        if (claims >= S->roots[g.root].capacity) continue;
        // placement_score (controller.cpp:101-123); the request's own id is excluded
        const double root_cap = S->roots[g.root].capacity;
        const double io_cap = S->host_io_capacity[g.host];
        double sp_pcie = 0.0, sp_numa = 0.0, sp_irq = 0.0;
        for (int j = 0; j < T; ++j) {
            if (j == k || !adm[j] || th[j] != g.host) continue;
            const PGpu& og = S->gpus[tg[j]];
            if (S->tenants[j].tclass == kBandwidthHeavy && og.root == g.root) sp_pcie = dadd(sp_pcie, ddiv(pcie[j], root_cap));
            if (og.numa == g.numa) sp_numa = dadd(sp_numa, ddiv(hio[j], io_cap));
        }
        if ((irq[g.host] >> g.core_group) & 1u) sp_irq = 1.0;
        const double score = dadd(dadd(sp_pcie, sp_numa), sp_irq);
        // strict improvement in score, else the smaller (host, gpu id, first)
        const bool better = bidx < 0 || score < best ||
                            (score == best && (g.host < bh || (g.host == bh && (g.id < bg || (g.id == bg && run < bf)))));
        if (better) {
            best = score;
            bh = g.host;
            bg = g.id;
            bf = run;
            bidx = gi;
        }
    }
    // warp reduction with the same order: (score, host, gpu id, first)
    for (int d = 16; d; d >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, best, d);
        const int oh = __shfl_xor_sync(0xffffffffu, bh, d), og = __shfl_xor_sync(0xffffffffu, bg, d),
                  of = __shfl_xor_sync(0xffffffffu, bf, d), oi = __shfl_xor_sync(0xffffffffu, bidx, d);
        const bool take = oi >= 0 && (bidx < 0 || os < best ||
                                      (os == best && (oh < bh || (oh == bh && (og < bg || (og == bg && of < bf))))));
        if (take) {
            best = os;
            bh = oh;
            bg = og;
            bf = of;
            bidx = oi;
        }
    }
    if (lane != 0) return;
    if (bidx >= 0) {
        o.outcome = kAdmitAdmitted;
        o.host = bh;
        o.gpu_id = bg;
        o.first = bf;
        o.score = best;
        o.reason = kReasonNone;
        if (C.queue_epochs) C.queue_epochs[c] = 0;  // queue_epochs_.erase (controller.cpp:671)
    } else {
        int32_t epochs = (C.queue_epochs ? C.queue_epochs[c] : 0) + 1;
        if (epochs > queue_timeout_epochs) {
            o.outcome = kAdmitRejected;
            o.reason = kReasonTimeout;
            epochs = 0;  // erased with the rejection (controller.cpp:680-683)
        } else {
            o.outcome = kAdmitQueued;
            o.reason = kReasonNoSlot;
        }
        if (C.queue_epochs) C.queue_epochs[c] = epochs;
    }
    out[c] = o;
}

}  // namespace mg
