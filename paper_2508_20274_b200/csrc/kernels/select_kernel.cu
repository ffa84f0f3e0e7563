// Nearest-rank order statistics on the GPU (engine.cpp:800-816: sort the measurement-window
// latencies, value at rank max(1, ceil(q*n)) - 1; telemetry.cpp:52-55 for the window form).
//
// One CTA per segment; doubles are mapped to order-preserving 64-bit keys.
//  * n <= kSmall: the whole segment is loaded into shared memory once and every quantile is found
//    by an in-smem 8-bit MSD radix select (1 global read).
//  * otherwise the DES hands over each segment's min/max, so the common key prefix is known
//    before the first read:
//      pass 1 (HBM stream, 16-B loads, 4 in flight per thread): 12-bit digit histogram of the
//             bits just below the common prefix, shared by all quantiles;
//      pass 2 (usually L2): the (small) digit groups holding the target ranks are gathered into
//             shared memory and finished by the in-smem radix select.
//    Groups too large for the gather buffer are refined by another digit pass first.
// Every result is an element chosen by exact integer ranks: bit-identical to std::sort + index.
#include "engine_kernels.cuh"

namespace mg {

namespace {

constexpr int kSelThreads = 256;
constexpr int kDigit = 12;
constexpr int kBins = 1 << kDigit;
constexpr int kMaxQ = 4;
constexpr int kCand = 4096;  // shared-memory key buffer (also the small-segment threshold)

__device__ __forceinline__ uint64_t okey(double x) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double kval(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ bool in_group(uint64_t k, uint64_t prefix, int sh) {
    return sh >= 64 || ((k ^ prefix) >> sh) == 0;
}

struct SelSmem {
    uint32_t hist[kBins];
    uint64_t cand[kCand];
    uint32_t wsum[kSelThreads / 32];
    uint64_t qprefix[kMaxQ];
    int64_t qrank[kMaxQ];
    int64_t qgroup[kMaxQ];
    int32_t qshift[kMaxQ];
    int32_t qdone[kMaxQ];
    int32_t qslot[kMaxQ];  // gather slice owner (index of the first quantile of the same group)
    uint32_t qbase[kMaxQ];
    uint32_t qfill[kMaxQ];
    double qresult[kMaxQ];
    uint64_t kmin, kmax;
    uint64_t scr_prefix;
    int64_t scr_rank;
    int32_t fits;
};

template <class F>
__device__ __forceinline__ void stream_keys(const double* __restrict__ v, int64_t n, F&& f) {
    const int tid = threadIdx.x;
    int64_t head = (16 - (reinterpret_cast<uintptr_t>(v) & 15)) / 8 & 1;
    if (head > n) head = n;
    if (tid < head) f(okey(v[tid]));
    const double2* v2 = reinterpret_cast<const double2*>(v + head);
    const int64_t n2 = (n - head) / 2;
    int64_t i = tid;
    for (; i + 3 * kSelThreads < n2; i += 4 * kSelThreads) {
        const double2 a = __ldg(v2 + i), b = __ldg(v2 + i + kSelThreads), c = __ldg(v2 + i + 2 * kSelThreads),
                      d = __ldg(v2 + i + 3 * kSelThreads);
        f(okey(a.x));
        f(okey(a.y));
        f(okey(b.x));
        f(okey(b.y));
        f(okey(c.x));
        f(okey(c.y));
        f(okey(d.x));
        f(okey(d.y));
    }
    for (; i < n2; i += kSelThreads) {
        const double2 a = __ldg(v2 + i);
        f(okey(a.x));
        f(okey(a.y));
    }
    const int64_t tail = head + 2 * n2;
    if (tid < n - tail) f(okey(v[tail + tid]));
}

// Block-wide: given per-thread partial count s, return (exclusive prefix, total) of the block.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t s, uint32_t* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += wsum[w];
    __syncthreads();
    return base + incl - s;
}

// Exact select of the rank-th smallest key among m keys keys[0..m) in shared memory that all
// share `prefix` above bit `sh`: 8-bit MSD radix passes over shared memory.
__device__ uint64_t smem_select(const uint64_t* keys, int m, int64_t rank, uint64_t prefix, int sh, SelSmem& sm) {
    const int tid = threadIdx.x;
    while (sh > 0) {
        const int d = sh < 8 ? sh : 8;
        for (int b = tid; b < 256; b += kSelThreads) sm.hist[b] = 0;
        __syncthreads();
        for (int a = tid; a < m; a += kSelThreads) {
            const uint64_t k = keys[a];
            if (in_group(k, prefix, sh)) atomicAdd(&sm.hist[(k >> (sh - d)) & ((1u << d) - 1)], 1u);
        }
        __syncthreads();
        const uint32_t c = sm.hist[tid];  // 256 threads == 256 bins
        const uint32_t lo = block_excl_scan(c, sm.wsum);
        __syncthreads();
        if (rank >= lo && rank < static_cast<int64_t>(lo) + c) {
            sm.scr_prefix = prefix | (static_cast<uint64_t>(tid) << (sh - d));
            sm.scr_rank = rank - lo;
        }
        __syncthreads();
        prefix = sm.scr_prefix;
        rank = sm.scr_rank;
        sh -= d;
        __syncthreads();
    }
    return prefix;
}

__device__ void block_select(const double* __restrict__ vals, int64_t n, bool have_range, double vmin, double vmax,
                             const double* qs, int nq, double* out, SelSmem& sm) {
    const int tid = threadIdx.x;
    if (n <= 0) {
        if (tid < nq) out[tid] = 0.0;
        return;
    }
    int64_t ranks[kMaxQ];
    for (int q = 0; q < nq; ++q) {
        int64_t r = static_cast<int64_t>(ceil(__dmul_rn(qs[q], static_cast<double>(n))));
        ranks[q] = (r < 1 ? 1 : r > n ? n : r) - 1;
    }
    if (n <= kCand) {
        // small segment: one read into shared memory, then in-smem selects
        for (int64_t i = tid; i < n; i += kSelThreads) sm.cand[i] = okey(vals[i]);
        __syncthreads();
        double res[kMaxQ];
        for (int q = 0; q < nq; ++q) res[q] = kval(smem_select(sm.cand, static_cast<int>(n), ranks[q], 0, 64, sm));
        if (tid < nq) out[tid] = res[tid];
        return;
    }
    // key range (from the producer, else one reduction pass)
    if (tid == 0) {
        sm.kmin = ~0ull;
        sm.kmax = 0;
    }
    __syncthreads();
    if (have_range) {
        if (tid == 0) {
            sm.kmin = okey(vmin);
            sm.kmax = okey(vmax);
        }
    } else {
        uint64_t lo = ~0ull, hi = 0;
        stream_keys(vals, n, [&](uint64_t k) {
            lo = k < lo ? k : lo;
            hi = k > hi ? k : hi;
        });
        for (int o = 16; o; o >>= 1) {
            const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        if ((tid & 31) == 0) {
            atomicMin(reinterpret_cast<unsigned long long*>(&sm.kmin), lo);
            atomicMax(reinterpret_cast<unsigned long long*>(&sm.kmax), hi);
        }
    }
    __syncthreads();
    const uint64_t kmin = sm.kmin, kmax = sm.kmax;
    const int varying = kmin == kmax ? 0 : 64 - __clzll(kmin ^ kmax);
    if (tid < nq) {
        sm.qrank[tid] = ranks[tid];
        sm.qshift[tid] = varying;
        sm.qprefix[tid] = varying >= 64 ? 0 : (kmin >> varying) << varying;
        sm.qgroup[tid] = n;
        sm.qdone[tid] = varying == 0;
        if (varying == 0) sm.qresult[tid] = kval(kmin);
    }
    __syncthreads();
    // digit passes until every group fits the gather buffer together
    for (;;) {
        // owners of distinct groups + gather slices
        if (tid == 0) {
            uint32_t total = 0;
            int widest = -1;
            for (int q = 0; q < nq; ++q) {
                sm.qslot[q] = q;
                if (sm.qdone[q]) continue;
                for (int p = 0; p < q; ++p)
                    if (!sm.qdone[p] && sm.qprefix[p] == sm.qprefix[q] && sm.qshift[p] == sm.qshift[q]) {
                        sm.qslot[q] = sm.qslot[p];
                        break;
                    }
                if (sm.qslot[q] == q) {
                    sm.qbase[q] = total;
                    sm.qfill[q] = 0;
                    total += static_cast<uint32_t>(sm.qgroup[q] > kCand ? kCand + 1 : sm.qgroup[q]);
                    if (widest < 0 || sm.qgroup[q] > sm.qgroup[widest]) widest = q;
                }
            }
            sm.fits = total <= kCand ? -1 : widest;  // -1: gather; else refine this group
        }
        __syncthreads();
        const int refine = sm.fits;
        if (refine < 0) break;
        const uint64_t prefix = sm.qprefix[refine];
        const int sh = sm.qshift[refine];
        const int d = sh < kDigit ? sh : kDigit;
        for (int b = tid; b < kBins; b += kSelThreads) sm.hist[b] = 0;
        __syncthreads();
        stream_keys(vals, n, [&](uint64_t k) {
            if (in_group(k, prefix, sh)) atomicAdd(&sm.hist[static_cast<uint32_t>((k >> (sh - d)) & ((1u << d) - 1))], 1u);
        });
        __syncthreads();
        constexpr int per = kBins / kSelThreads;
        uint32_t s = 0;
        for (int b = 0; b < per; ++b) s += sm.hist[tid * per + b];
        const int64_t lo = block_excl_scan(s, sm.wsum);
        const int64_t hi = lo + s;
        // snapshot the quantile states before any owner rewrites them: a thread must never pair
        // another thread's fresh rank with the stale prefix/shift of the same quantile
        bool member[kMaxQ];
        int64_t rank_of[kMaxQ];
        for (int p = 0; p < nq; ++p) {
            member[p] = !sm.qdone[p] && sm.qprefix[p] == prefix && sm.qshift[p] == sh;
            rank_of[p] = sm.qrank[p];
        }
        __syncthreads();
        for (int p = 0; p < nq; ++p) {
            if (!member[p]) continue;
            const int64_t rk = rank_of[p];
            if (rk >= lo && rk < hi) {
                int64_t acc = lo;
                int bin = tid * per;
                while (acc + sm.hist[bin] <= rk) acc += sm.hist[bin++];
                sm.qprefix[p] = prefix | (static_cast<uint64_t>(bin) << (sh - d));
                sm.qshift[p] = sh - d;
                sm.qrank[p] = rk - acc;
                sm.qgroup[p] = sm.hist[bin];
                if (sh - d == 0) {
                    sm.qdone[p] = 1;
                    sm.qresult[p] = kval(sm.qprefix[p]);
                }
            }
        }
        __syncthreads();
    }
    // gather every open group into its slice of the key buffer (one pass)
    bool any_open = false;
    for (int q = 0; q < nq; ++q) any_open |= !sm.qdone[q];
    if (any_open) {
        uint64_t gp[kMaxQ];
        int gs[kMaxQ], go[kMaxQ];
        int ng = 0;
        for (int q = 0; q < nq; ++q)
            if (!sm.qdone[q] && sm.qslot[q] == q) {
                gp[ng] = sm.qprefix[q];
                gs[ng] = sm.qshift[q];
                go[ng] = q;
                ++ng;
            }
        stream_keys(vals, n, [&](uint64_t k) {
            for (int g = 0; g < ng; ++g)
                if (in_group(k, gp[g], gs[g])) {
                    const uint32_t at = atomicAdd(&sm.qfill[go[g]], 1u);
                    sm.cand[sm.qbase[go[g]] + at] = k;
                }
        });
        __syncthreads();
        for (int q = 0; q < nq; ++q) {
            if (sm.qdone[q]) continue;
            const int o = sm.qslot[q];
            const uint64_t r = smem_select(sm.cand + sm.qbase[o], static_cast<int>(sm.qgroup[o]), sm.qrank[q],
                                           sm.qprefix[q], sm.qshift[q], sm);
            if (tid == 0) sm.qresult[q] = kval(r);
            __syncthreads();
        }
    }
    __syncthreads();
    if (tid < nq) out[tid] = sm.qresult[tid];
}

}  // namespace

__global__ void __launch_bounds__(kSelThreads) select_kernel(WaveBuffers B, int T, int n_rep) {
    extern __shared__ __align__(16) unsigned char smem[];
    SelSmem& sm = *reinterpret_cast<SelSmem*>(smem);
    const int s = blockIdx.x;
    if (s >= n_rep * T) return;
    const int r = s / T, t = s % T;
    const TenantOut& o = B.tout[s];
    const double qs[kMaxQ] = {0.50, 0.95, 0.99, 0.999};
    block_select(B.win_lat + static_cast<int64_t>(r) * B.cap_sum + B.off[t], static_cast<int64_t>(o.completed_window),
                 true, o.win_min, o.win_max, qs, kMaxQ, B.quant + 4ll * s, sm);
}

__global__ void __launch_bounds__(kSelThreads) select_segments_kernel(const double* __restrict__ vals,
                                                                      const int64_t* __restrict__ seg_off, int n_seg,
                                                                      const double* __restrict__ qs, int nq,
                                                                      double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    SelSmem& sm = *reinterpret_cast<SelSmem*>(smem);
    const int s = blockIdx.x;
    if (s >= n_seg) return;
    for (int q0 = 0; q0 < nq; q0 += kMaxQ) {
        const int cnt = nq - q0 < kMaxQ ? nq - q0 : kMaxQ;
        block_select(vals + seg_off[s], seg_off[s + 1] - seg_off[s], false, 0.0, 0.0, qs + q0, cnt,
                     out + static_cast<int64_t>(s) * nq + q0, sm);
        __syncthreads();
    }
}

size_t select_smem_bytes() { return sizeof(SelSmem); }

}  // namespace mg
