// Nearest-rank order statistics on the GPU (engine.cpp:800-816: sort the measurement-window
// latencies, value at rank max(1, ceil(q*n)) - 1; telemetry.cpp:52-55 for the window form).
//
// One CTA per segment; doubles are mapped to order-preserving 64-bit keys.  Every candidate set
// ("group") is a key interval [lo, lo + 2^sh) and digits are taken RELATIVE to lo, so a digit
// pass spreads the keys over the bins even when the range straddles a binary exponent (a
// prefix-based digit of 0.8 .. 19 ms latencies would spend its 12 bits on exponent bits and put
// half the segment in one bin).
//  * n <= kCand: the segment is loaded into shared memory once; every quantile is finished there.
//  * otherwise the DES hands over each segment's min/max, so the first group is known before the
//    first read:
//      pass 1 (HBM stream, 16-B loads, 4 in flight per thread): 12-bit digit histogram of
//             (key - kmin) >> shift, shared by all quantiles (no group test: every key is in);
//      pass 2 (L2): the digit bins holding the target ranks are gathered into shared memory
//             (one digit compare per bin) and finished by the in-smem radix select.
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
// key k in the group [lo, lo + 2^sh)
__device__ __forceinline__ bool in_group(uint64_t k, uint64_t lo, int sh) {
    return sh >= 64 || ((k - lo) >> sh) == 0;
}
__device__ __forceinline__ int bitlen64(uint64_t x) { return x ? 64 - __clzll(static_cast<long long>(x)) : 0; }

struct SelSmem {
    uint32_t hist[kBins];
    uint64_t cand[kCand];
    uint32_t wsum[kSelThreads / 32];
    uint64_t qlo[kMaxQ];
    int64_t qrank[kMaxQ];
    int64_t qgroup[kMaxQ];
    int32_t qshift[kMaxQ];
    int32_t qdone[kMaxQ];
    int32_t qslot[kMaxQ];  // gather slice owner (index of the first quantile of the same group)
    uint32_t qbase[kMaxQ];
    uint32_t qfill[kMaxQ];
    double qresult[kMaxQ];
    uint64_t kmin, kmax;
    uint64_t scr_lo;
    int64_t scr_rank;
    int32_t scr_cnt;
    int32_t fits;
};

// f(key) for every element of v[0..n): 16-B loads, 4 in flight per thread
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

// Block-wide: given per-thread partial count s, return the exclusive prefix of the block.
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
#pragma unroll
    for (int w = 0; w < kSelThreads / 32; ++w) base += w < warp ? wsum[w] : 0u;
    __syncthreads();
    return base + incl - s;
}

// Exact select of the rank-th smallest among the keys of group [lo, lo + 2^sh) found in
// keys[0..m) (shared memory): 8-bit radix steps relative to lo; stops as soon as the rank's bin
// holds a single key.
__device__ uint64_t smem_select(const uint64_t* keys, int m, int64_t rank, uint64_t lo, int sh, SelSmem& sm) {
    const int tid = threadIdx.x;
    while (sh > 0) {
        const int d = sh < 8 ? sh : 8;
        const int s = sh - d;
        sm.hist[tid] = 0;  // 256 threads == 256 bins
        __syncthreads();
        for (int a = tid; a < m; a += kSelThreads) {
            const uint64_t k = keys[a];
            if (in_group(k, lo, sh)) atomicAdd(&sm.hist[static_cast<uint32_t>((k - lo) >> s)], 1u);
        }
        __syncthreads();
        const uint32_t c = sm.hist[tid];
        const uint32_t below = block_excl_scan(c, sm.wsum);
        if (rank >= below && rank < static_cast<int64_t>(below) + c) {
            sm.scr_lo = lo + (static_cast<uint64_t>(tid) << s);
            sm.scr_rank = rank - below;
            sm.scr_cnt = static_cast<int32_t>(c);
        }
        __syncthreads();
        lo = sm.scr_lo;
        rank = sm.scr_rank;
        const int cnt = sm.scr_cnt;
        sh = s;
        __syncthreads();
        if (cnt == 1 && sh > 0) {  // the only key of the bin is the answer
            for (int a = tid; a < m; a += kSelThreads) {
                const uint64_t k = keys[a];
                if (in_group(k, lo, sh)) sm.scr_lo = k;
            }
            __syncthreads();
            lo = sm.scr_lo;
            __syncthreads();
            return lo;
        }
    }
    return lo;
}

// One refinement pass over the keys (source `src`): 12-bit histogram of the group (lo, sh)
// (group test skipped when `all_in`), then every quantile of that group moves to the bin holding
// its rank.
template <class Src>
__device__ void digit_pass(Src&& src, uint64_t lo, int sh, bool all_in, int nq, SelSmem& sm) {
    const int tid = threadIdx.x;
    const int d = sh < kDigit ? sh : kDigit;
    const int s = sh - d;
    for (int b = tid; b < kBins; b += kSelThreads) sm.hist[b] = 0;
    __syncthreads();
    if (all_in)
        src([&](uint64_t k) { atomicAdd(&sm.hist[static_cast<uint32_t>((k - lo) >> s)], 1u); });
    else
        src([&](uint64_t k) {
            if (in_group(k, lo, sh)) atomicAdd(&sm.hist[static_cast<uint32_t>((k - lo) >> s)], 1u);
        });
    __syncthreads();
    constexpr int per = kBins / kSelThreads;
    uint32_t cnt = 0;
    for (int b = 0; b < per; ++b) cnt += sm.hist[tid * per + b];
    const int64_t below = block_excl_scan(cnt, sm.wsum);
    // snapshot the quantile states before any owner rewrites them: a thread must never pair
    // another thread's fresh rank with the stale group of the same quantile
    bool member[kMaxQ];
    int64_t rank_of[kMaxQ];
    for (int p = 0; p < nq; ++p) {
        member[p] = !sm.qdone[p] && sm.qlo[p] == lo && sm.qshift[p] == sh;
        rank_of[p] = sm.qrank[p];
    }
    __syncthreads();
    for (int p = 0; p < nq; ++p) {
        if (!member[p]) continue;
        const int64_t rk = rank_of[p];
        if (rk >= below && rk < below + cnt) {
            int64_t acc = below;
            int bin = tid * per;
            while (acc + sm.hist[bin] <= rk) acc += sm.hist[bin++];
            const uint64_t blo = lo + (static_cast<uint64_t>(bin) << s);
            sm.qlo[p] = blo;
            sm.qshift[p] = s;
            sm.qrank[p] = rk - acc;
            sm.qgroup[p] = sm.hist[bin];
            if (s == 0) {
                sm.qdone[p] = 1;
                sm.qresult[p] = kval(blo);
            }
        }
    }
    __syncthreads();
}

// All quantiles of one large segment.  `src(f)` calls f(key) for every element; kmin/kmax bound
// the keys.
template <class Src>
__device__ void select_in(Src&& src, int64_t n, uint64_t kmin, uint64_t kmax, const int64_t* ranks, int nq,
                          SelSmem& sm) {
    const int tid = threadIdx.x;
    const int sh0 = bitlen64(kmax - kmin);
    if (tid < nq) {
        sm.qrank[tid] = ranks[tid];
        sm.qshift[tid] = sh0;
        sm.qlo[tid] = kmin;
        sm.qgroup[tid] = n;
        sm.qdone[tid] = sh0 == 0;
        sm.qresult[tid] = kval(kmin);
    }
    __syncthreads();
    if (sh0 == 0) return;
    digit_pass(src, kmin, sh0, true, nq, sm);  // pass 1: every key is in the first group
    for (;;) {
        // owners of distinct groups + gather slices
        if (tid == 0) {
            uint32_t total = 0;
            int widest = -1;
            for (int q = 0; q < nq; ++q) {
                sm.qslot[q] = q;
                if (sm.qdone[q]) continue;
                for (int p = 0; p < q; ++p)
                    if (!sm.qdone[p] && sm.qlo[p] == sm.qlo[q] && sm.qshift[p] == sm.qshift[q]) {
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
        digit_pass(src, sm.qlo[refine], sm.qshift[refine], false, nq, sm);
    }
    // gather every open group into its slice of the key buffer (one pass)
    uint64_t glo[kMaxQ];
    int gsh[kMaxQ], go[kMaxQ];
    int ng = 0;
    for (int q = 0; q < nq; ++q)
        if (!sm.qdone[q] && sm.qslot[q] == q) {
            glo[ng] = sm.qlo[q];
            gsh[ng] = sm.qshift[q];
            go[ng] = q;
            ++ng;
        }
    if (ng == 0) return;
    // common case: every open group is a bin of pass 1, [kmin + b*2^s, kmin + (b+1)*2^s) with one
    // s -- then one digit and up to four 32-bit compares per key
    const int s1 = gsh[0];
    bool first_level = s1 < 64 && s1 + kDigit >= sh0;
    for (int g = 0; g < ng && first_level; ++g)
        first_level = gsh[g] == s1 && ((glo[g] - kmin) & ((1ull << s1) - 1)) == 0;
    if (first_level) {
        uint32_t gb[kMaxQ];
        int gof[kMaxQ];
        for (int g = 0; g < kMaxQ; ++g) {
            gb[g] = g < ng ? static_cast<uint32_t>((glo[g] - kmin) >> s1) : 0xffffffffu;
            gof[g] = g < ng ? go[g] : 0;
        }
        src([&](uint64_t k) {
            const uint32_t dg = static_cast<uint32_t>((k - kmin) >> s1);
#pragma unroll
            for (int g = 0; g < kMaxQ; ++g)
                if (dg == gb[g]) {
                    const uint32_t at = atomicAdd(&sm.qfill[gof[g]], 1u);
                    sm.cand[sm.qbase[gof[g]] + at] = k;
                }
        });
    } else {
        src([&](uint64_t k) {
            for (int g = 0; g < ng; ++g)
                if (in_group(k, glo[g], gsh[g])) {
                    const uint32_t at = atomicAdd(&sm.qfill[go[g]], 1u);
                    sm.cand[sm.qbase[go[g]] + at] = k;
                }
        });
    }
    __syncthreads();
    for (int q = 0; q < nq; ++q) {
        if (sm.qdone[q]) continue;
        const int o = sm.qslot[q];
        const uint64_t r = smem_select(sm.cand + sm.qbase[o], static_cast<int>(sm.qgroup[o]), sm.qrank[q], sm.qlo[q],
                                       sm.qshift[q], sm);
        if (tid == 0) sm.qresult[q] = kval(r);
        __syncthreads();
    }
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
    if (tid == 0) {
        sm.kmin = ~0ull;
        sm.kmax = 0;
    }
    __syncthreads();
    const bool small = n <= kCand;
    uint64_t lo = ~0ull, hi = 0;
    auto minmax = [&](uint64_t k) {
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    };
    if (small) {
        // one read into shared memory; the range comes with it
        for (int64_t i = tid; i < n; i += kSelThreads) {
            const uint64_t k = okey(vals[i]);
            sm.cand[i] = k;
            minmax(k);
        }
    } else if (!have_range) {
        stream_keys(vals, n, minmax);
    }
    if (small || !have_range) {
        for (int o = 16; o; o >>= 1) {
            const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        if ((tid & 31) == 0) {
            atomicMin(reinterpret_cast<unsigned long long*>(&sm.kmin), lo);
            atomicMax(reinterpret_cast<unsigned long long*>(&sm.kmax), hi);
        }
    } else if (tid == 0) {
        sm.kmin = okey(vmin);
        sm.kmax = okey(vmax);
    }
    __syncthreads();
    const uint64_t kmin = sm.kmin, kmax = sm.kmax;
    if (small) {
        if (tid < nq) sm.qresult[tid] = kval(kmin);
        __syncthreads();
        if (kmin != kmax) {
            const int sh0 = bitlen64(kmax - kmin);
            for (int q = 0; q < nq; ++q) {
                const uint64_t r = smem_select(sm.cand, static_cast<int>(n), ranks[q], kmin, sh0, sm);
                if (tid == 0) sm.qresult[q] = kval(r);
                __syncthreads();
            }
        }
    } else {
        select_in([&](auto&& f) { stream_keys(vals, n, f); }, n, kmin, kmax, ranks, nq, sm);
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
    // tenant-major, tenants by decreasing record capacity (longest segments first: LPT order over
    // the SMs), replicas of one tenant adjacent
    const int r = s % n_rep, t = B.sel_order[s / n_rep];
    const int so = r * T + t;
    const TenantOut& o = B.tout[so];
    const double qs[kMaxQ] = {0.50, 0.95, 0.99, 0.999};
    block_select(B.win_lat + static_cast<int64_t>(r) * B.cap_sum + B.off[t], static_cast<int64_t>(o.completed_window),
                 true, o.win_min, o.win_max, qs, kMaxQ, B.quant + 4ll * so, sm);
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
