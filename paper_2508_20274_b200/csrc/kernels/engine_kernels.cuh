// sm_100a kernels of the batched controller engine.
//
//  gen_times_kernel   one thread per (replica, tenant): arrival clock stream (gamma renewal) +
//                     schedule thinning                         (workload.cpp:129-136, engine.cpp:435-446)
//  gen_marks_kernel   one thread per (replica, tenant, stream): transfer-size / service / noise
//                     marks and the IRQ exponential stream      (workload.cpp:138-156, engine.cpp:403-404)
//  des_kernel         one warp per replica, state in shared memory: the event loop + controller
//                     (engine.cpp:864-894, controller.cpp:489-603)
//  select_kernel      one CTA per (replica, tenant): nearest-rank p50/p95/p99/p999 of the measurement
//                     window by an 11-bit MSD radix select over the order-preserving bit image of the
//                     FP64 latencies                            (engine.cpp:800-816)
//  compact_kernel     gathers the variable-length action / pause logs into dense host-bound buffers
#pragma once

#include <cuda_runtime.h>

#include "../common/des_core.h"

namespace mg {

struct WaveBuffers {
    // [W][cap_sum] arrays
    double *arr_t, *arr_bytes, *arr_mult, *arr_noise, *irq_e, *t_all, *req_ms, *win_lat;
    double *c_done, *c_total, *c_compute, *c_transfer, *c_noise;  // optional
    int64_t* c_order;                                              // optional, [W][cap_sum]
    uint32_t* win_hist;                                            // [W][T][kHistBins] window-latency bins
    CounterRow* tr_cnt;                                            // optional traces [W][n_ticks][T]
    FabricRow* tr_fab;                                             //                 [W][n_ticks][R]
    TailWin* tr_win;                                               //                 [W][T]
    int32_t *n_all, *n_kept;                                       // [W][T]
    uint64_t* mt_pause;                                            // [W][T][312]
    ActionRec* actions;                                            // [W][action_cap]
    PauseRec* pauses;                                              // [W][pause_cap]
    TenantOut* tout;                                               // [W][T]
    ReplicaOut* rout;                                              // [W]
    double* backlog;                                               // [W][R][2]
    double* quant;                                                 // [W][T][4]
    double* rings;                                                 // [W][T][dwell + validation] when not in smem
    const uint64_t* seeds;                                         // [W]
    const int32_t* variant;                                        // [W]
    const int64_t* off;                                            // [T]
    const int64_t* cap;                                            // [T]
    const int32_t* file_order;                                     // [T]
    const int32_t* sel_order;                                      // [T] tenants by decreasing cap (select LPT order)
    int32_t* gen_overflow;                                         // [1]
    int64_t cap_sum;
    int32_t action_cap, pause_cap;
    int32_t any_irq_noise, rings_in_smem;
    int32_t dwell, validation;  // ring strides (max over variants)
    int32_t n_variants, pad_v;  // PController entries at C
    unsigned long long* prof;   // [6][3] event-loop cycle counters (MG_PROFILE_EVENTS builds only)
};

__global__ void gen_times_kernel(const PScenario* __restrict__ S, WaveBuffers B, int n_rep);
__global__ void gen_marks_kernel(const PScenario* __restrict__ S, WaveBuffers B, int n_rep);
__global__ void des_kernel(const PScenario* __restrict__ S, const PController* __restrict__ C, WaveBuffers B,
                           int n_rep, SimLayout L);
// same, with the event slots in lane registers; for T <= kRegSlotMaxTenants
constexpr int kRegSlotMaxTenants = 10;  // 3T+1 hot slots and 2T rare slots within 32 lanes
__global__ void des_kernel_reg(const PScenario* __restrict__ S, const PController* __restrict__ C, WaveBuffers B,
                               int n_rep, SimLayout L);
// same code capped at 64 registers (32 resident warps/SM instead of 16): the saturated-regime form,
// used when a wave holds more replicas than the uncapped kernel keeps resident
__global__ void des_kernel_reg_occ(const PScenario* __restrict__ S, const PController* __restrict__ C, WaveBuffers B,
                                   int n_rep, SimLayout L);
// SIMT form: one thread per replica, for large waves (see engine_kernels.cu)
constexpr int kSimtMaxTenants = 32;  // 32-bit tenant masks
constexpr int kSimtBlock = 32;       // threads (replicas) per block, at most
struct SimtLayout {
    SimLayout tab;   // block-shared scenario tables (sc_* offsets)
    SimLayout lane;  // per-replica working set, offsets inside one lane's slab
    int64_t ctrl;    // PController[n_variants]
    int64_t lanes;   // first lane slab
    int64_t stride;  // bytes per lane slab (odd multiple of 8)
    int64_t bytes(int lanes_per_block) const { return lanes + stride * lanes_per_block; }
};
SimtLayout simt_layout(int T, int R, int G, int I, int H, int n_variants);
__global__ void des_simt_kernel(const PScenario* __restrict__ S, const PController* __restrict__ C, WaveBuffers B,
                                int n_rep, SimtLayout Y);
__global__ void select_kernel(WaveBuffers B, int T, int n_rep);
// per-(variant, tenant) latency histograms summed over a wave's replicas (int64, persistent)
__global__ void hist_reduce_kernel(const uint32_t* __restrict__ win_hist, const int32_t* __restrict__ variant,
                                   int n_rep, int T, int chunk, unsigned long long* __restrict__ out);
// same results, one HBM pass: 4-CTA cluster per segment, TMA bulk loads, DSMEM histogram/gather
__global__ void select_cluster_kernel(WaveBuffers B, int T, int n_rep);
__global__ void compact_actions_kernel(const ActionRec* __restrict__ src, int cap, const ReplicaOut* __restrict__ rout,
                                       const int64_t* __restrict__ dst_off, ActionRec* __restrict__ dst, int n_rep);
__global__ void compact_pauses_kernel(const PauseRec* __restrict__ src, int cap, const ReplicaOut* __restrict__ rout,
                                      const int64_t* __restrict__ dst_off, PauseRec* __restrict__ dst, int n_rep);

// standalone nearest-rank select over arbitrary segments (C-ABI migsim_gpu_select)
__global__ void select_segments_kernel(const double* __restrict__ vals, const int64_t* __restrict__ seg_off,
                                       int n_seg, const double* __restrict__ qs, int nq, double* __restrict__ out);

}  // namespace mg

namespace mg {
__global__ void libm_kernel(int fn, const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ out,
                            int64_t n);
}
