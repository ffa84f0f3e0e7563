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
#include <cooperative_groups.h>

#include "engine_kernels.cuh"

namespace mg {

namespace {

#ifndef MG_SEL_THREADS
#define MG_SEL_THREADS 256
#endif
#ifndef MG_SEL_CAND
#define MG_SEL_CAND 2048
#endif
constexpr int kSelThreads = MG_SEL_THREADS;
#ifndef MG_SEL_MINB
#define MG_SEL_MINB 6  // 6 CTAs x 256 threads per SM: <= 40 registers
#endif
static_assert(kSelThreads / 32 >= 4 && kSelThreads / 32 <= 32, "one warp per quantile, one scan warp");
#ifndef MG_SEL_DIGIT
#define MG_SEL_DIGIT 11
#endif
constexpr int kDigit = MG_SEL_DIGIT;
constexpr int kBins = 1 << kDigit;
static_assert(kBins >= kHistBins, "the producer histogram is staged in the digit histogram");
constexpr int kMaxQ = 4;
constexpr int kCand = MG_SEL_CAND;  // shared-memory key buffer (also the small-segment threshold)

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
    uint32_t wsum[32];
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

// 16-B read-only load with an L2 eviction-priority policy: the first pass over a segment keeps its
// lines (evict_last) for the gather pass that re-reads them, which then releases them (evict_first).
__device__ __forceinline__ double2 ld_hint(const double2* p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
    uint64_t pol;
    if (keep)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// f(key) for every element of v[0..n): 16-B loads, 4 in flight per thread
template <class F>
__device__ __forceinline__ void stream_keys(const double* __restrict__ v, int64_t n, F&& f, bool keep = true) {
    const uint64_t pol = l2_policy(keep);
    const int tid = threadIdx.x;
    int64_t head = (16 - (reinterpret_cast<uintptr_t>(v) & 15)) / 8 & 1;
    if (head > n) head = n;
    if (tid < head) f(okey(v[tid]));
    const double2* v2 = reinterpret_cast<const double2*>(v + head);
    const int64_t n2 = (n - head) / 2;
    int64_t i = tid;
#ifndef MG_SEL_DEPTH
#define MG_SEL_DEPTH 4
#endif
    constexpr int kDepth = MG_SEL_DEPTH;  // 16-B loads in flight per thread (64 B): ~96 KB per SM at 6 CTAs
    const int nthr = blockDim.x;
    for (; i + (kDepth - 1) * nthr < n2; i += kDepth * nthr) {
        double2 x[kDepth];
#pragma unroll
        for (int u = 0; u < kDepth; ++u) x[u] = ld_hint(v2 + i + u * nthr, pol);
#pragma unroll
        for (int u = 0; u < kDepth; ++u) {
            f(okey(x[u].x));
            f(okey(x[u].y));
        }
    }
    for (; i < n2; i += nthr) {
        const double2 a = ld_hint(v2 + i, pol);
        f(okey(a.x));
        f(okey(a.y));
    }
    const int64_t tail = head + 2 * n2;
    if (tid < n - tail) f(okey(v[tail + tid]));
}

// f(x) for every double of v[0..n) (raw values; same access pattern as stream_keys)
template <class F>
__device__ __forceinline__ void stream_raw(const double* __restrict__ v, int64_t n, F&& f, bool keep) {
    const uint64_t pol = l2_policy(keep);
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    int64_t head = (16 - (reinterpret_cast<uintptr_t>(v) & 15)) / 8 & 1;
    if (head > n) head = n;
    if (tid < head) f(v[tid]);
    const double2* v2 = reinterpret_cast<const double2*>(v + head);
    const int64_t n2 = (n - head) / 2;
    int64_t i = tid;
    constexpr int kDepth = MG_SEL_DEPTH;
    for (; i + (kDepth - 1) * nthr < n2; i += kDepth * nthr) {
        double2 x[kDepth];
#pragma unroll
        for (int u = 0; u < kDepth; ++u) x[u] = ld_hint(v2 + i + u * nthr, pol);
#pragma unroll
        for (int u = 0; u < kDepth; ++u) {
            f(x[u].x);
            f(x[u].y);
        }
    }
    for (; i < n2; i += nthr) {
        const double2 a = ld_hint(v2 + i, pol);
        f(a.x);
        f(a.y);
    }
    const int64_t tail = head + 2 * n2;
    if (tid < n - tail) f(v[tail + tid]);
}

// A segment in global memory as a key source: every pass but the last keeps its L2 lines.
struct GlobalSrc {
    const double* v;
    int64_t n;
    template <class F>
    __device__ __forceinline__ void operator()(F&& f) const { stream_keys(v, n, f, true); }
    template <class F>
    __device__ __forceinline__ void last(F&& f) const { stream_keys(v, n, f, false); }
};

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
    if (warp == 0) {  // exclusive scan of the warp totals
        const int kW = static_cast<int>(blockDim.x) / 32;
        const uint32_t w = lane < kW ? wsum[lane] : 0u;
        uint32_t x = w;
        for (int o = 1; o < kW; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < kW) wsum[lane] = x - w;
    }
    __syncthreads();
    const uint32_t base = wsum[warp];
    __syncthreads();
    return base + incl - s;
}

// Exact select of the rank-th smallest among the keys of group [lo, lo + 2^sh) found in
// keys[0..m) (shared memory) by ONE warp, no block barriers: 8-bit radix steps relative to lo
// over a warp-private 256-bin histogram; stops as soon as the rank's bin holds a single key.
// The quantiles of a segment run in parallel, one warp each.
__device__ uint64_t warp_select(const uint64_t* keys, int m, int64_t rank, uint64_t lo, int sh, uint32_t* hist) {
    const int lane = threadIdx.x & 31;
    while (sh > 0) {
        const int d = sh < 8 ? sh : 8;
        const int s = sh - d;
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        for (int a = lane; a < m; a += 32) {
            const uint64_t k = keys[a];
            if (in_group(k, lo, sh)) atomicAdd(&hist[static_cast<uint32_t>((k - lo) >> s)], 1u);
        }
        __syncwarp();
        uint32_t c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = hist[lane * 8 + j];
            tot += c[j];
        }
        uint32_t incl = tot;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int64_t below = static_cast<int64_t>(incl - tot);
        int bin = -1;
        int64_t acc = below;
        uint32_t cnt = 0;
        if (rank >= below && rank < below + tot) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (bin < 0) {
                    if (acc + c[j] > rank) {
                        bin = lane * 8 + j;
                        cnt = c[j];
                    } else {
                        acc += c[j];
                    }
                }
        }
        const int owner = __ffs(__ballot_sync(0xffffffffu, bin >= 0)) - 1;
        bin = __shfl_sync(0xffffffffu, bin, owner);
        acc = __shfl_sync(0xffffffffu, acc, owner);
        cnt = __shfl_sync(0xffffffffu, cnt, owner);
        lo += static_cast<uint64_t>(bin) << s;
        rank -= acc;
        sh = s;
        __syncwarp();
        if (cnt == 1 && sh > 0) {  // the only key of the bin is the answer
            uint64_t hit = 0;
            bool found = false;
            for (int a = lane; a < m && !found; a += 32) {
                const uint64_t k = keys[a];
                if (in_group(k, lo, sh)) {
                    hit = k;
                    found = true;
                }
            }
            const int who = __ffs(__ballot_sync(0xffffffffu, found)) - 1;
            return __shfl_sync(0xffffffffu, hit, who);
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
    for (int b = tid; b < kBins; b += static_cast<int>(blockDim.x)) sm.hist[b] = 0;
    __syncthreads();
    if (all_in)
        src([&](uint64_t k) { atomicAdd(&sm.hist[static_cast<uint32_t>((k - lo) >> s)], 1u); });
    else
        src([&](uint64_t k) {
            if (in_group(k, lo, sh)) atomicAdd(&sm.hist[static_cast<uint32_t>((k - lo) >> s)], 1u);
        });
    __syncthreads();
    const int per = kBins / static_cast<int>(blockDim.x);
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
        src.last([&](uint64_t k) {
            const uint32_t dg = static_cast<uint32_t>((k - kmin) >> s1);
#pragma unroll
            for (int g = 0; g < kMaxQ; ++g)
                if (dg == gb[g]) {
                    const uint32_t at = atomicAdd(&sm.qfill[gof[g]], 1u);
                    sm.cand[sm.qbase[gof[g]] + at] = k;
                }
        });
    } else {
        src.last([&](uint64_t k) {
            for (int g = 0; g < ng; ++g)
                if (in_group(k, glo[g], gsh[g])) {
                    const uint32_t at = atomicAdd(&sm.qfill[go[g]], 1u);
                    sm.cand[sm.qbase[go[g]] + at] = k;
                }
        });
    }
    __syncthreads();
    {
        const int q = tid >> 5;  // warp q finishes quantile q
        if (q < nq && !sm.qdone[q]) {
            const int o = sm.qslot[q];
            const uint64_t r = warp_select(sm.cand + sm.qbase[o], static_cast<int>(sm.qgroup[o]), sm.qrank[q], sm.qlo[q],
                                           sm.qshift[q], sm.hist + 256 * q);
            if ((tid & 31) == 0) sm.qresult[q] = kval(r);
        }
    }
    __syncthreads();
}

// Out of line: the general path's register demand would otherwise cap the one-pass path's
// occupancy (measured: 6 CTAs/SM at 40 registers, 0.080 vs 0.087 ms per C2 wave).
__device__ __noinline__ void block_select(const double* __restrict__ vals, int64_t n, bool have_range, double vmin, double vmax,
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
        for (int64_t i = tid; i < n; i += blockDim.x) {
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
            const int q = tid >> 5;
            if (q < nq) {
                const uint64_t r = warp_select(sm.cand, static_cast<int>(n), ranks[q], kmin, sh0, sm.hist + 256 * q);
                if ((tid & 31) == 0) sm.qresult[q] = kval(r);
            }
            __syncthreads();
        }
    } else {
        select_in(GlobalSrc{vals, n}, n, kmin, kmax, ranks, nq, sm);
    }
    __syncthreads();
    if (tid < nq) out[tid] = sm.qresult[tid];
}


// Producer-histogram form (the default for the per-wave summary): the DES already binned every
// window latency (lat_hist.h), so the target bins are known before the samples are touched and ONE
// streaming pass over HBM gathers the in-bin keys; one warp per quantile finishes.  Falls back to
// the two-pass path when the target bins hold more keys than the gather buffer.
__device__ void hist_select(const double* __restrict__ vals, int64_t n, const uint32_t* __restrict__ hist,
                            double vmin, double vmax, const double* qs, int nq, double* out, SelSmem& sm) {
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const uint64_t kmin = okey(vmin), kmax = okey(vmax);
    if (n <= kCand || kmin == kmax) {  // small or constant segments: the shared-memory path
        block_select(vals, n, true, vmin, vmax, qs, nq, out, sm);
        return;
    }
    int64_t ranks[kMaxQ];
    for (int q = 0; q < nq; ++q) {
        int64_t r = static_cast<int64_t>(ceil(__dmul_rn(qs[q], static_cast<double>(n))));
        ranks[q] = (r < 1 ? 1 : r > n ? n : r) - 1;
    }
    // histogram -> smem (coalesced 16-B loads), locate the rank bins
    {
        const uint4* h4 = reinterpret_cast<const uint4*>(hist);
        uint4* s4 = reinterpret_cast<uint4*>(sm.hist);
        for (int i = tid; i < kHistBins / 4; i += nthr) s4[i] = __ldg(h4 + i);
    }
    __syncthreads();
    const int per = kHistBins / nthr;
    uint32_t cnt = 0;
    for (int b = 0; b < per; ++b) cnt += sm.hist[tid * per + b];
    const int64_t below = block_excl_scan(cnt, sm.wsum);
    for (int q = 0; q < nq; ++q) {
        const int64_t rk = ranks[q];
        if (rk >= below && rk < below + cnt) {
            int64_t acc = below;
            int bin = tid * per;
            while (acc + sm.hist[bin] <= rk) acc += sm.hist[bin++];
            sm.qrank[q] = rk - acc;
            sm.qlo[q] = static_cast<uint64_t>(bin);  // bin index for now
            sm.qgroup[q] = sm.hist[bin];
        }
    }
    __syncthreads();
    if (tid == 0) {  // distinct bins -> slices of the candidate buffer
        uint32_t total = 0;
        for (int q = 0; q < nq; ++q) {
            sm.qslot[q] = q;
            for (int p = 0; p < q; ++p)
                if (sm.qlo[p] == sm.qlo[q]) {
                    sm.qslot[q] = sm.qslot[p];
                    break;
                }
            if (sm.qslot[q] == q) {
                sm.qbase[q] = total;
                sm.qfill[q] = 0;
                total += static_cast<uint32_t>(sm.qgroup[q]);
            }
        }
        sm.fits = total <= static_cast<uint32_t>(kCand);
    }
    __syncthreads();
    if (!sm.fits) {
        __syncthreads();
        block_select(vals, n, true, vmin, vmax, qs, nq, out, sm);
        return;
    }
    uint32_t gb[kMaxQ];
    int gq[kMaxQ];
    for (int g = 0; g < kMaxQ; ++g) {
        const bool own = g < nq && sm.qslot[g] == g;
        gb[g] = own ? static_cast<uint32_t>(sm.qlo[g]) : 0xffffffffu;
        gq[g] = own ? g : 0;
    }
    // the one pass over HBM: the gathered keys are the only reuse, so the lines are not kept
    bool edge = false;
    for (int g = 0; g < kMaxQ; ++g) edge |= gb[g] == 0u || gb[g] == static_cast<uint32_t>(kHistBins - 1);
    if (!edge) {
        // interior target bins of positive values are equal top-18-bit patterns of the raw double
        // (sign, exponent, 6 mantissa bits; lat_hist.h): one shift and four compares per sample,
        // the key is formed only for the few samples that match
        uint32_t tv[kMaxQ];
        for (int g = 0; g < kMaxQ; ++g)
            tv[g] = gb[g] == 0xffffffffu ? 0xffffffffu
                                         : static_cast<uint32_t>(kHistBase + gb[g] - (1ull << (63 - kHistShift)));
        stream_raw(
            vals, n,
            [&](double x) {
                const uint32_t t = static_cast<uint32_t>(__double2hiint(x)) >> (kHistShift - 32);
#pragma unroll
                for (int g = 0; g < kMaxQ; ++g)
                    if (t == tv[g]) {
                        const uint32_t at = atomicAdd(&sm.qfill[gq[g]], 1u);
                        sm.cand[sm.qbase[gq[g]] + at] = okey(x);
                    }
            },
            false);
    } else {
        stream_keys(
            vals, n,
            [&](uint64_t k) {
                const uint32_t b = lat_bin_of_key(k);
#pragma unroll
                for (int g = 0; g < kMaxQ; ++g)
                    if (b == gb[g]) {
                        const uint32_t at = atomicAdd(&sm.qfill[gq[g]], 1u);
                        sm.cand[sm.qbase[gq[g]] + at] = k;
                    }
            },
            false);
    }
    __syncthreads();
    const int q = tid >> 5;  // warp q finishes quantile q
    if (q < nq) {
        const int o = sm.qslot[q];
        const uint32_t b = static_cast<uint32_t>(sm.qlo[q]);
        // interior bins are exact key intervals; the clamped edge bins are bounded by the range
        const bool interior = b > 0 && b < static_cast<uint32_t>(kHistBins - 1);
        const uint64_t lo = interior ? lat_bin_lo(b) : kmin;
        const int sh = interior ? kHistShift : bitlen64(kmax - kmin);
        const uint64_t r = warp_select(sm.cand + sm.qbase[o], static_cast<int>(sm.qgroup[o]), sm.qrank[q], lo, sh,
                                       sm.hist + 256 * q);
        if ((tid & 31) == 0) out[q] = kval(r);
    }
}

// ---------------------------------------------------------------------------------------------
// Cluster form (the per-wave summary select): ONE HBM pass.  A 4-CTA thread-block cluster owns a
// segment; each CTA pulls its quarter into shared memory with a single TMA bulk copy
// (cp.async.bulk, completion on an mbarrier), builds the 12-bit (key - kmin) >> shift histogram
// of its quarter there, and adds it into the leader CTA's histogram through distributed shared
// memory.  The leader locates the bins holding the target ranks; every CTA then copies its
// in-bin keys from its own shared memory into the leader's candidate buffer (DSMEM atomics +
// stores), and the leader finishes each quantile with one warp.  Segments of at most one chunk
// are handled by the leader alone; segments whose target bins overflow the candidate buffer
// (heavy ties) take the two-pass global path above.
namespace cg = cooperative_groups;

constexpr int kCS = 4;          // CTAs per cluster
constexpr int kChunk = 9216;    // doubles per CTA (72 KB of shared memory)
constexpr int kCCand = 2048;    // leader's candidate keys
constexpr int kClThreads = 512;

struct ClSmem {
    double data[kChunk];
    uint32_t hist[kBins];
    uint64_t cand[kCCand];
    unsigned long long mbar;
    int32_t mode;  // 0: gather + finish, 1: two-pass fallback on the leader
    int32_t ng;
    uint32_t gbin[kMaxQ], gbase[kMaxQ], gfill[kMaxQ], gcnt[kMaxQ];
    int32_t qg[kMaxQ];
    int64_t qrank[kMaxQ];
    uint32_t wsum[32];
};
static_assert(sizeof(SelSmem) <= sizeof(ClSmem), "fallback reuses the cluster layout");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// f(key) over the first `len` doubles of shared memory, 16-B loads
template <class F>
__device__ __forceinline__ void smem_keys(const double* data, int len, F&& f) {
    const double2* d2 = reinterpret_cast<const double2*>(data);
    const int n2 = len >> 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const double2 x = d2[i];
        f(okey(x.x));
        f(okey(x.y));
    }
    if ((len & 1) && threadIdx.x == 0) f(okey(data[len - 1]));
}

__device__ void cluster_select(const double* __restrict__ vals, int64_t n, double vmin, double vmax, const double* qs,
                               int nq, double* out, ClSmem& sm) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned crank = cl.block_rank();
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const uint64_t kmin = okey(vmin), kmax = okey(vmax);
    const int sh0 = bitlen64(kmax - kmin);
    const bool aligned = (reinterpret_cast<uintptr_t>(vals) & 15) == 0;
    if (n <= 0 || sh0 == 0 || n > static_cast<int64_t>(kCS) * (kChunk - 2) || !aligned) {
        if (crank == 0)  // trivial or out-of-range segment: the leader alone, global path
            block_select(vals, n, true, vmin, vmax, qs, nq, out, *reinterpret_cast<SelSmem*>(&sm));
        return;
    }
    const bool solo = n <= kChunk;
    if (solo && crank != 0) return;
    const int parts = solo ? 1 : kCS;
    const int me = solo ? 0 : static_cast<int>(crank);
    const int64_t per = ((n + parts - 1) / parts + 1) & ~1ll;
    const int64_t beg = me * per < n ? me * per : n;
    const int64_t end = (me + 1) * per < n ? (me + 1) * per : n;
    const int len = static_cast<int>(end - beg);
    const int len2 = len & ~1;
    const int d = sh0 < kDigit ? sh0 : kDigit;
    const int s1 = sh0 - d;
    // 1. one bulk copy of this CTA's share (16-B aligned, even length) + the odd tail element
    if (tid == 0) {
        mbar_init(&sm.mbar);
        if (len2 > 0) tma_load_1d(sm.data, vals + beg, static_cast<uint32_t>(len2) * 8u, &sm.mbar);
        if (len & 1) sm.data[len - 1] = vals[beg + len - 1];
    }
    for (int b = tid; b < kBins; b += nthr) sm.hist[b] = 0;
    if (tid < kMaxQ) sm.gfill[tid] = 0;
    __syncthreads();
    if (len2 > 0) mbar_wait(&sm.mbar, 0);
    // 2. local histogram of (key - kmin) >> s1
    smem_keys(sm.data, len, [&](uint64_t k) { atomicAdd(&sm.hist[static_cast<uint32_t>((k - kmin) >> s1)], 1u); });
    __syncthreads();
    if (!solo) cl.sync();  // (B) every local histogram is complete
    // 3. the leader folds the other CTAs' histograms into its own (DSMEM reads, all loads of a
    //    thread independent), locates the target bins and publishes the decisions
    if (crank == 0) {
        if (!solo) {
            const uint32_t* hs[kCS - 1];
            for (int c = 1; c < kCS; ++c) hs[c - 1] = cl.map_shared_rank(sm.hist, c);
            for (int b = tid; b < kBins; b += nthr) {
                uint32_t v0 = hs[0][b], v1 = hs[1][b], v2 = hs[2][b];
                sm.hist[b] += v0 + v1 + v2;
            }
            __syncthreads();
        }
        int64_t ranks[kMaxQ];
        for (int q = 0; q < nq; ++q) {
            int64_t r = static_cast<int64_t>(ceil(__dmul_rn(qs[q], static_cast<double>(n))));
            ranks[q] = (r < 1 ? 1 : r > n ? n : r) - 1;
        }
        const int per_t = kBins / nthr;
        uint32_t cnt = 0;
        for (int b = 0; b < per_t; ++b) cnt += sm.hist[tid * per_t + b];
        const int64_t below = block_excl_scan(cnt, sm.wsum);
        for (int q = 0; q < nq; ++q) {
            const int64_t rk = ranks[q];
            if (rk >= below && rk < below + cnt) {
                int64_t acc = below;
                int bin = tid * per_t;
                while (acc + sm.hist[bin] <= rk) acc += sm.hist[bin++];
                sm.qrank[q] = rk - acc;
                sm.gbin[q] = static_cast<uint32_t>(bin);  // per quantile; deduplicated below
                sm.gcnt[q] = sm.hist[bin];
            }
        }
        __syncthreads();
        if (tid == 0) {
            int ng = 0;
            uint32_t total = 0;
            uint32_t qb[kMaxQ], qc[kMaxQ];
            for (int q = 0; q < nq; ++q) {
                qb[q] = sm.gbin[q];
                qc[q] = sm.gcnt[q];
            }
            for (int q = 0; q < nq; ++q) {
                int g = -1;
                for (int p = 0; p < ng; ++p)
                    if (sm.gbin[p] == qb[q]) g = p;
                if (g < 0) {
                    g = ng++;
                    sm.gbin[g] = qb[q];
                    sm.gcnt[g] = qc[q];
                    sm.gbase[g] = total;
                    total += qc[q];
                }
                sm.qg[q] = g;
            }
            for (int g = ng; g < kMaxQ; ++g) sm.gbin[g] = 0xffffffffu;
            sm.ng = ng;
            sm.mode = total <= static_cast<uint32_t>(kCCand) ? 0 : 1;
        }
        __syncthreads();
    }
    if (!solo) cl.sync();  // (C) decisions visible cluster-wide
    ClSmem& L = solo ? sm : *cl.map_shared_rank(&sm, 0);
    const int mode = L.mode;
    if (mode == 0) {
        // 4. every CTA copies its in-bin keys from its own shared memory to the leader's buffer
        uint32_t gb[kMaxQ], gbase[kMaxQ];
        for (int g = 0; g < kMaxQ; ++g) {
            gb[g] = L.gbin[g];
            gbase[g] = L.gbase[g];
        }
        smem_keys(sm.data, len, [&](uint64_t k) {
            const uint32_t dg = static_cast<uint32_t>((k - kmin) >> s1);
#pragma unroll
            for (int g = 0; g < kMaxQ; ++g)
                if (dg == gb[g]) {
                    const uint32_t at = atomicAdd(&L.gfill[g], 1u);
                    L.cand[gbase[g] + at] = k;
                }
        });
    }
    if (!solo) cl.sync();  // (D) candidates complete and no CTA reads a remote histogram any more
    if (crank != 0) return;
    if (mode == 1) {
        block_select(vals, n, true, vmin, vmax, qs, nq, out, *reinterpret_cast<SelSmem*>(&sm));
        return;
    }
    __syncthreads();
    const int q = tid >> 5;  // warp q finishes quantile q
    if (q < nq) {
        const int g = sm.qg[q];
        const uint64_t r = warp_select(sm.cand + sm.gbase[g], static_cast<int>(sm.gcnt[g]), sm.qrank[q],
                                       kmin + (static_cast<uint64_t>(sm.gbin[g]) << s1), s1, sm.hist + 256 * q);
        if ((tid & 31) == 0) out[q] = kval(r);
    }
}
}  // namespace

__global__ void __launch_bounds__(kSelThreads, MG_SEL_MINB) select_kernel(WaveBuffers B, int T, int n_rep) {
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
    const double* vals = B.win_lat + static_cast<int64_t>(r) * B.cap_sum + B.off[t];
    if (B.win_hist)
        hist_select(vals, static_cast<int64_t>(o.completed_window), B.win_hist + static_cast<int64_t>(so) * kHistBins,
                    o.win_min, o.win_max, qs, kMaxQ, B.quant + 4ll * so, sm);
    else
        block_select(vals, static_cast<int64_t>(o.completed_window), true, o.win_min, o.win_max, qs, kMaxQ,
                     B.quant + 4ll * so, sm);
}

__global__ void __launch_bounds__(kSelThreads, MG_SEL_MINB) select_segments_kernel(const double* __restrict__ vals,
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

__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(kClThreads, 2)
    select_cluster_kernel(WaveBuffers B, int T, int n_rep) {
    extern __shared__ __align__(128) unsigned char smem[];
    ClSmem& sm = *reinterpret_cast<ClSmem*>(smem);
    const int s = blockIdx.x / kCS;  // one cluster per segment
    if (s >= n_rep * T) return;
    const int r = s % n_rep, t = B.sel_order[s / n_rep];
    const int so = r * T + t;
    const TenantOut& o = B.tout[so];
    const double qs[kMaxQ] = {0.50, 0.95, 0.99, 0.999};
    cluster_select(B.win_lat + static_cast<int64_t>(r) * B.cap_sum + B.off[t], static_cast<int64_t>(o.completed_window),
                   o.win_min, o.win_max, qs, kMaxQ, B.quant + 4ll * so, sm);
}

size_t select_smem_bytes() { return sizeof(SelSmem); }
size_t select_cluster_smem_bytes() { return sizeof(ClSmem); }
int select_cluster_size() { return kCS; }
int select_cluster_threads() { return kClThreads; }
int select_threads() { return kSelThreads; }

}  // namespace mg
