// Batched admission control (Controller::admit, controller.cpp:637-692): see admit_kernel.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../common/packed.h"

namespace mg {

enum AdmitOutcome : int32_t { kAdmitAdmitted = 0, kAdmitQueued = 1, kAdmitRejected = 2 };  // controller.hpp:121
enum AdmitReason : int32_t { kReasonNone = 0, kReasonRate = 1, kReasonNoSlot = 2, kReasonTimeout = 3 };

// Case arrays, tenants in canonical (lexicographic id) order; gpu = canonical GPU index.
struct AdmitCases {
    const int32_t* tenant;   // [n] request: canonical tenant index
    const int32_t* profile;  // [n] request: lattice index
    const int32_t *admitted, *host, *gpu, *first, *count;  // [n][T] TenantStates
    const double *tenant_pcie, *tenant_host_io;             // [n][T] ClusterSnapshot::tenant_*_Bps
    const uint32_t* irq_recent;                             // [n][H] bit g: (host, core group g) recent
    int32_t* queue_epochs;  // [n] in/out: the controller's queue_epochs_[tenant] (controller.hpp:214),
                            // 0 = no entry; nullptr = a fresh controller
};

struct AdmitOut {
    int32_t outcome, host, gpu_id, first, count, profile, reason, pad;
    double score;
};

__global__ void admit_kernel(const PScenario* __restrict__ S, AdmitCases C, int n_cases, int queue_timeout_epochs,
                             AdmitOut* __restrict__ out);

}  // namespace mg
