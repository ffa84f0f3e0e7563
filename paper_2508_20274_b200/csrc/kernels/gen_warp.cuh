// Warp-cooperative arrival-record generation (device only).
//
// Same streams and the same arithmetic as the scalar restatement in common/arrivals.h and
// common/rng.h (ArrivalGen::next, workload.cpp:129-157; libstdc++-13 <random>), reorganised so a
// warp spends its time in parallel work:
//  * mt19937_64 is advanced 312 outputs at a time by the whole warp: the twist of
//    random.tcc:_M_gen_rand has two dependency-free phases (k < 156 reads only old words; k >= 156
//    reads phase-1 words and old words), so each lane twists ~10 words per phase.
//  * uniform-count streams (transfer size, noise, IRQ): one canonical per call, transformed
//    lane-parallel and compacted through the schedule-thinning mask with ballots.
//  * service (lognormal): each call starts with a fresh polar cache and consumes whole pairs, so
//    pairs are aligned on even stream positions; accepted pairs are ranked with ballots.
//  * arrival clock (gamma, Marsaglia-Tsang + pow boost): consumption is irregular, so the warp
//    speculatively evaluates the polar multiplier of the pair at EVERY stream position, then the
//    whole rejection loop of a call starting at every position (lane-parallel; only the number of
//    positions it consumes is kept, plus the length of 4 consecutive calls); lane 0 walks the
//    actual calls through those lengths (one shared-memory load per 4 calls), the walked calls'
//    v and pow(u, 1/alpha) are evaluated lane-parallel, lane 0 accumulates the clock in order
//    (the FP sum order of workload.cpp:135) and the lanes store the arrival times.
#pragma once

#include "../common/arrivals.h"

namespace mg {

// canonical ring (positions): one 312-word block is written per fill, so the scan may look ahead
// kRing - kMtN positions; 512 keeps the block's shared memory at 12.5 KB (17 resident warps/SM)
constexpr int kRing = 512;
static_assert((kRing & (kRing - 1)) == 0, "ring index by mask");
// ring slot of a stream position (positions are >= 0: a mask, not a signed modulo)
__device__ __forceinline__ uint32_t ring_idx(int64_t p) { return static_cast<uint32_t>(p) & (kRing - 1u); }
// a call consuming kLongCall or more positions is marked long and scanned in place by lane 0 (never
// seen at 255; test builds lower it with -DMG_GEN_LONG_CALL to exercise that path)
#ifndef MG_GEN_LONG_CALL
#define MG_GEN_LONG_CALL 255
#endif
constexpr uint32_t kLongCall = MG_GEN_LONG_CALL;
static_assert(kLongCall >= 4 && kLongCall <= 255, "call lengths are stored in one byte");
constexpr int kMaxCallsRound = 80;  // gamma calls walked per round (~one 312-position fill)

struct WarpMtSmem {
    uint64_t x[kMtN];
};

__device__ __forceinline__ void warp_mt_seed(WarpMtSmem& m, uint64_t s, int lane) {
    if (lane == 0) {
        uint64_t prev = s;
        m.x[0] = s;
        for (int i = 1; i < kMtN; ++i) {
            prev = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<uint64_t>(i);
            m.x[i] = prev;
        }
    }
    __syncwarp();
}

// Advance the state by one full twist (random.tcc _M_gen_rand), warp-parallel.
__device__ __forceinline__ void warp_mt_twist(WarpMtSmem& m, int lane) {
    uint64_t v[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int k = lane + 32 * j;
        if (k < kMtN - kMtM) v[j] = mt_twist_one(m.x[k], m.x[k + 1], m.x[k + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int k = lane + 32 * j;
        if (k < kMtN - kMtM) m.x[k] = v[j];
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int k = kMtN - kMtM + lane + 32 * j;
        if (k < kMtN) v[j] = mt_twist_one(m.x[k], k == kMtN - 1 ? m.x[0] : m.x[k + 1], m.x[k - (kMtN - kMtM)]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int k = kMtN - kMtM + lane + 32 * j;
        if (k < kMtN) m.x[k] = v[j];
    }
    __syncwarp();
}

__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// ---------------------------------------------------------------------------------------------
// Uniform-count mark streams: purpose in {kMarkSize, kMarkService, kMarkNoise, kMarkIrq}.
// n_calls: next() calls (or IRQ draws); t_all/thinned: schedule thinning of the calls.
__device__ void warp_gen_marks(WarpMtSmem& m, int purpose, const PTenant& p, uint64_t seed_word, const double* t_all,
                               int32_t n_calls, bool thinned, double* out, int lane) {
    const bool draws = purpose == kMarkIrq || (purpose == kMarkSize && p.n_mix > 0) ||
                       (purpose == kMarkService && p.has_service) || (purpose == kMarkNoise && p.has_noise);
    if (!draws) {
        // no RNG consumption at all: constant marks (workload.cpp:138-156)
        const double v = purpose == kMarkService ? 1.0 : 0.0;
        int64_t kept = 0;
        for (int32_t c0 = 0; c0 < n_calls; c0 += 32) {
            const int32_t c = c0 + lane;
            const bool keep = c < n_calls && (!thinned || sched_active(p.sched, t_all[c]));
            const unsigned mk = __ballot_sync(0xffffffffu, keep);
            if (keep) out[kept + __popc(mk & lanemask_lt(lane))] = v;
            kept += __popc(mk);
        }
        return;
    }
    warp_mt_seed(m, seed_word, lane);
    int64_t call_base = 0, kept = 0;
    while (call_base < n_calls) {
        warp_mt_twist(m, lane);
        if (purpose == kMarkService) {
            // 156 aligned pairs per block; accepted pairs are the calls, in order
            for (int j0 = 0; j0 < kMtN / 2 && call_base < n_calls; j0 += 32) {
                const int j = j0 + lane;
                double x = 0.0, y = 0.0, r2 = 2.0;
                if (j < kMtN / 2) {
                    x = fsub(fmul(2.0, canonical_from(mt_temper(m.x[2 * j]))), 1.0);
                    y = fsub(fmul(2.0, canonical_from(mt_temper(m.x[2 * j + 1]))), 1.0);
                    r2 = fadd(fmul(x, x), fmul(y, y));
                }
                const bool acc = j < kMtN / 2 && !(r2 > 1.0 || r2 == 0.0);
                const unsigned ma = __ballot_sync(0xffffffffu, acc);
                const int64_t call = call_base + __popc(ma & lanemask_lt(lane));
                const bool valid = acc && call < n_calls;
                const bool keep = valid && (!thinned || sched_active(p.sched, t_all[call]));
                const unsigned mk = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const double mult = fsqrt(fdiv_exact(fmul(-2.0, gl_log(r2)), r2));
                    const double n = fadd(fmul(fmul(y, mult), 1.0), 0.0);
                    out[kept + __popc(mk & lanemask_lt(lane))] = gl_exp(fadd(fmul(p.svc_sigma, n), p.svc_mu));
                }
                kept += __popc(mk);
                call_base += __popc(ma);
            }
        } else {
            for (int j0 = 0; j0 < kMtN && call_base < n_calls; j0 += 32) {
                const int j = j0 + lane;
                const int64_t call = call_base + lane;
                const bool valid = j < kMtN && call < n_calls;
                const bool keep = valid && (!thinned || sched_active(p.sched, t_all[call]));
                const unsigned mk = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const double c = canonical_from(mt_temper(m.x[j]));
                    double v;
                    if (purpose == kMarkSize) {
                        const double pick = fadd(fmul(c, fsub(p.mix_cdf[p.n_mix - 1], 0.0)), 0.0);
                        int idx = 0;
                        while (idx + 1 < p.n_mix && pick >= p.mix_cdf[idx]) ++idx;
                        v = p.mix_bytes[idx];
                    } else if (purpose == kMarkNoise) {
                        v = fdiv_exact(-gl_log(fsub(1.0, c)), p.noise_lambda);
                    } else {
                        v = -gl_log(fsub(1.0, c));
                    }
                    out[kept + __popc(mk & lanemask_lt(lane))] = v;
                }
                kept += __popc(mk);
                const int take = kMtN - j0 < 32 ? kMtN - j0 : 32;
                call_base += take;
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Arrival clock stream (gamma renewal).
struct GammaSmem {
    WarpMtSmem mt;
    double c[kRing];    // canonical at position p (ring)
    double pm[kRing];   // polar multiplier of the pair starting at p if it is accepted, NaN if rejected;
                        // the scan forms y*mult / x*mult from c[] with the same two roundings, so the
                        // ring holds one word per position instead of two
    double call_v[kMaxCallsRound];  // the call's gap value, then (in place) its clock
    int16_t call_q[kMaxCallsRound];  // ring index of the call's first position
    uint8_t nxt[kRing];   // positions consumed by a call starting here: 0 = not known yet, kLongCall = long
    uint8_t nxt4[kRing];  // ... by the four calls starting here (0 = not known / too long)
    int32_t n_calls;
    int32_t n_valid;  // calls whose clock is inside the horizon and the capacity (this round)
};

// Generate the next 312 canonicals at positions [gen_end, gen_end+312) and the speculative pair
// transform for positions [gen_end-1, gen_end+311).
__device__ __forceinline__ void gamma_fill(GammaSmem& g, int64_t gen_end, int lane) {
    warp_mt_twist(g.mt, lane);
    for (int j = lane; j < kMtN; j += 32) g.c[ring_idx(gen_end + j)] = canonical_from(mt_temper(g.mt.x[j]));
    __syncwarp();
    for (int j = lane; j < kMtN; j += 32) {
        const int64_t pos = gen_end - 1 + j;
        if (pos < 0) continue;
        const double x = fsub(fmul(2.0, g.c[ring_idx(pos)]), 1.0);
        const double y = fsub(fmul(2.0, g.c[ring_idx(pos + 1)]), 1.0);
        const double r2 = fadd(fmul(x, x), fmul(y, y));
        const bool a = !(r2 > 1.0 || r2 == 0.0);
        // an accepted pair's multiplier is finite
        g.pm[ring_idx(pos)] = a ? fsqrt(fdiv_exact(fmul(-2.0, gl_log(r2)), r2)) : k_nan();
    }
    __syncwarp();
}

// One gamma call's rejection loop (random.tcc:2366-2380) from stream position pos; returns
// false if it would read past `limit` (positions with a complete pair transform).
__device__ __forceinline__ bool gamma_scan_call(const GammaSmem& g, const GammaParams& gp, int64_t& pos, int64_t limit,
                                                double& v_out, int32_t& q_out) {
    int64_t p = pos;
    bool cached = false;
    double cache_m = 0.0, n, v, u;
    uint32_t cache_i = 0;
    for (;;) {
        do {
            if (cached) {
                n = fmul(fsub(fmul(2.0, g.c[cache_i]), 1.0), cache_m);  // x * mult
                cached = false;
            } else {
                double m;
                for (;;) {
                    if (p + 1 >= limit) return false;
                    m = g.pm[ring_idx(p)];
                    if (m == m) break;  // accepted pair
                    p += 2;
                }
                n = fmul(fsub(fmul(2.0, g.c[ring_idx(p + 1)]), 1.0), m);  // y * mult
                cache_m = m;
                cache_i = ring_idx(p);
                cached = true;
                p += 2;
            }
            // (libstdc++'s n*1.0+0.0 scaling is omitted: it only maps -0.0 to +0.0, and n enters
            //  only as 1 + a2*n and through even powers)
            v = fadd(1.0, fmul(gp.a2, n));
        } while (v <= 0.0);
        v = fmul(fmul(v, v), v);
        if (p >= limit) return false;
        u = g.c[ring_idx(p)];
        p += 1;
        const double sq = fsub(1.0, fmul(fmul(fmul(fmul(0.0331, n), n), n), n));
        if (!(u > sq)) break;
        const double rhs = fadd(fmul(fmul(0.5, n), n), fmul(gp.a1, fadd(fsub(1.0, v), gl_log(v))));
        if (!(gl_log(u) > rhs)) break;
    }
    int32_t q = -1;
    if (!(gp.alpha == gp.malpha)) {
        for (;;) {
            if (p >= limit) return false;
            const double u2 = g.c[ring_idx(p)];
            p += 1;
            if (u2 != 0.0) break;
        }
        q = static_cast<int32_t>(ring_idx(p - 1));
    }
    v_out = v;
    q_out = q;
    pos = p;
    return true;
}

// Whole arrival-time stream of one (replica, tenant): t_all / t_kept and counts.
__device__ bool warp_gen_times(GammaSmem& g, const PTenant& p, uint64_t seed_word, double duration, double* t_all,
                               double* t_kept, int64_t cap, int32_t* n_all_out, int32_t* n_kept_out, int lane) {
    int64_t na = 0, nk = 0;
    bool ok = true;
    double clock = 0.0;
    const bool thinned = p.sched.kind != kAlways;
    if (p.deterministic) {
        // clock += 1/lambda (workload.cpp:131-132): no RNG on this stream
        if (lane == 0) {
            for (;;) {
                clock = fadd(clock, p.det_step);
                if (clock >= duration) break;
                if (na >= cap) {
                    ok = false;
                    break;
                }
                if (thinned) {
                    t_all[na] = clock;
                    if (sched_active(p.sched, clock)) t_kept[nk++] = clock;
                } else {
                    t_kept[nk++] = clock;
                }
                ++na;
            }
            *n_all_out = static_cast<int32_t>(na);
            *n_kept_out = static_cast<int32_t>(nk);
        }
        return __shfl_sync(0xffffffffu, ok, 0);
    }
    const GammaParams gp = gamma_params(p);
    warp_mt_seed(g.mt, seed_word, lane);
    int64_t gen_end = 0;  // canonicals known for positions < gen_end
    int64_t pos = 0;      // stream position of the next call
    int64_t evald = 0;    // call lengths (nxt) are known for the positions in [pos, evald)
    gamma_fill(g, gen_end, lane);
    gen_end += kMtN;
    bool done = false;
    while (!done) {
        // fill while the ring has room for a whole block without overwriting positions >= pos - 1
        while (gen_end - pos < kRing - kMtN) {
            gamma_fill(g, gen_end, lane);
            gen_end += kMtN;
        }
        const int64_t limit = gen_end - 1;  // pair transforms exist below gen_end-1
        // speculative scan, lane-parallel: the rejection loop of a call starting at EVERY position
        // not evaluated yet (only the consumption length is kept); evaluations that would read past
        // `limit` stay unknown and are redone after the next fill
        const int64_t ev0 = evald;
        {
            const int64_t from = evald > pos ? evald : pos;
            int64_t first_unknown = limit;
            for (int64_t p0 = from + lane; p0 < limit; p0 += 32) {
                int64_t pp = p0;
                double v;
                int32_t q;
                uint8_t d = 0;
                if (gamma_scan_call(g, gp, pp, limit, v, q)) d = static_cast<uint8_t>(pp - p0 < kLongCall ? pp - p0 : kLongCall);
                else first_unknown = p0 < first_unknown ? p0 : first_unknown;
                g.nxt[ring_idx(p0)] = d;
            }
            // every position below evald has a known length
            const int64_t fu = first_unknown;
            uint32_t hi = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(static_cast<uint64_t>(fu) >> 32));
            uint32_t lo = __reduce_min_sync(0xffffffffu, static_cast<uint32_t>(static_cast<uint64_t>(fu) >> 32) == hi
                                                            ? static_cast<uint32_t>(fu) : 0xffffffffu);
            evald = static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
        }
        __syncwarp();
        // four-call lengths where all four are known (positions below ev0 - 64 kept theirs from
        // earlier rounds; a length still unknown there only costs the walk single steps)
        {
            const int64_t f4 = ev0 - 64 > pos ? ev0 - 64 : pos;
            for (int64_t p0 = f4 + lane; p0 < evald; p0 += 32) {
                uint32_t dsum = 0;
                int j = 0;
                for (; j < 4; ++j) {
                    if (p0 + dsum >= evald) break;
                    const uint32_t d = g.nxt[ring_idx(p0 + dsum)];
                    if (d == kLongCall) break;
                    dsum += d;
                }
                g.nxt4[ring_idx(p0)] = static_cast<uint8_t>(j == 4 && dsum < 255 ? dsum : 0);
            }
        }
        __syncwarp();
        // lane 0: walk the calls through the lengths (one shared-memory load per one or four calls;
        // the starts of jumped-over calls are filled in lane-parallel below, marked -1..-3)
        if (lane == 0) {
            int32_t nc = 0;
            const int64_t stop = evald < limit - 64 ? evald : limit - 64;
            while (nc < kMaxCallsRound && pos < stop) {
                const uint32_t ri = ring_idx(pos);
                const uint32_t d4 = g.nxt4[ri];
                g.call_q[nc] = static_cast<int16_t>(ri);
                if (d4 != 0 && nc + 3 < kMaxCallsRound) {
                    g.call_q[nc + 1] = -1;
                    g.call_q[nc + 2] = -2;
                    g.call_q[nc + 3] = -3;
                    nc += 4;
                    pos += d4;
                    continue;
                }
                const uint32_t d = g.nxt[ri];
                int64_t pp = pos;
                if (d == kLongCall) {  // a long call (never seen at 255): scanned in place
                    double v;
                    int32_t q;
                    if (!gamma_scan_call(g, gp, pp, limit, v, q)) break;
                } else {
                    pp += d;
                }
                ++nc;
                pos = pp;
            }
            g.n_calls = nc;
        }
        __syncwarp();
        pos = __shfl_sync(0xffffffffu, pos, 0);
        const int32_t nc = g.n_calls;
        // lane-parallel: each walked call's v and pow uniform again (the same loop on the same ring
        // words), then its gap value pow(u, 1/alpha) * a1 * v * beta (random.tcc:2382-2392)
        for (int k = lane; k < nc; k += 32) {
            int32_t st = g.call_q[k];
            if (st < 0) {
                const int j = -st;
                st = g.call_q[k - j];
                for (int i = 0; i < j; ++i) st = static_cast<int32_t>(ring_idx(st + g.nxt[st]));
            }
            int64_t pp = st;  // ring index as the position: ring_idx masks the same way
            double v;
            int32_t q;
            gamma_scan_call(g, gp, pp, pp + kRing, v, q);
            if (q < 0) g.call_v[k] = fmul(fmul(gp.a1, v), gp.beta);
            else g.call_v[k] = fmul(fmul(fmul(gl_pow(g.c[q], gp.inv_alpha), gp.a1), v), gp.beta);
        }
        __syncwarp();
        // lane 0: the clock is an ordered FP sum (workload.cpp:135), written over the gap values
        // (only the dependent adds; the horizon and capacity are found lane-parallel after)
        if (lane == 0) {
#pragma unroll 4
            for (int32_t k = 0; k < nc; ++k) {
                clock = fadd(clock, g.call_v[k]);
                g.call_v[k] = clock;
            }
        }
        __syncwarp();
        {
            int32_t kd = nc;  // first call at or past the horizon
            for (int32_t k0 = 0; k0 < nc; k0 += 32) {
                const unsigned m = __ballot_sync(0xffffffffu, k0 + lane < nc && g.call_v[k0 + lane] >= duration);
                if (m) {
                    kd = k0 + __ffs(m) - 1;
                    break;
                }
            }
            const int32_t lim = cap - na < nc ? static_cast<int32_t>(cap - na) : nc;  // capacity left
            if (kd <= lim) {
                if (kd < nc) done = true;
                if (lane == 0) g.n_valid = kd;
            } else {  // the capacity is reached before the horizon
                ok = false;
                done = true;
                if (lane == 0) g.n_valid = lim;
            }
        }
        __syncwarp();
        // the round's arrival times, stored lane-parallel (the unthinned clock is read back only
        // for thinned tenants, by gen_marks)
        const int32_t nv = g.n_valid;
        if (thinned) {
            for (int32_t k0 = 0; k0 < nv; k0 += 32) {
                const int32_t k = k0 + lane;
                const bool valid = k < nv;
                const double c = valid ? g.call_v[k] : 0.0;
                if (valid) t_all[na + k] = c;
                const bool keep = valid && sched_active(p.sched, c);
                const unsigned mk = __ballot_sync(0xffffffffu, keep);
                if (keep) t_kept[nk + __popc(mk & lanemask_lt(lane))] = c;
                nk += __popc(mk);
            }
        } else {
            for (int32_t k = lane; k < nv; k += 32) t_kept[nk + k] = g.call_v[k];
            nk += nv;
        }
        na += nv;
        __syncwarp();
        if (!done && nc == 0) {
            // one call needs more than the lookahead (~10^-200 probability): widen the window
            // while the ring can hold it, otherwise report instead of reading stale positions
            if (gen_end + kMtN - pos > kRing) {
                ok = false;
                done = true;
            } else {
                gamma_fill(g, gen_end, lane);
                gen_end += kMtN;
            }
        }
    }
    if (lane == 0) {
        *n_all_out = static_cast<int32_t>(na);
        *n_kept_out = static_cast<int32_t>(nk);
    }
    return __shfl_sync(0xffffffffu, ok, 0);
}

}  // namespace mg
