// Deterministic random streams, bit-exact with the reference build.
//
// Seeding:   make_substream = mt19937_64(splitmix64(splitmix64(splitmix64(seed) ^ fnv1a(id)) ^ purpose))
//            (/root/reference/proj/src/workload.cpp:24-47)
// Engine:    std::mt19937_64 (n=312, m=156, r=31, a=0xb5026f5aa96619e9, tempering u=29,s=17,t=37,l=43)
// Canonical: libstdc++-13 generate_canonical<double,53> with a 64-bit engine: one draw,
//            double(x) * 2^-64, clamped to nextafter(1,0) (random.tcc:3346-3381)
// Distributions restate libstdc++-13 exactly, operation for operation, with the
// glibc-exact log/exp/pow of glibc_math.h:
//   normal (Marsaglia polar, cached second value)  random.tcc:1811-1845
//   gamma  (Marsaglia-Tsang, pow boost for a<1)    random.tcc:2337-2393
//   lognormal exp(s*N+m)                           random.h:2356-2358
//   exponential -log(1-u)/lambda                   random.h:4899-4905
//   uniform_real u*(b-a)+a                         random.h:1904-1910
#pragma once

#include "glibc_math.h"

namespace mg {

MG_HD uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

inline uint64_t fnv1a(const char* s, size_t n) {
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= static_cast<unsigned char>(s[i]);
        h *= 1099511628211ull;
    }
    return h;
}

enum StreamPurpose : uint64_t { kArrivals = 1, kTransferSize = 2, kService = 3, kNoise = 4, kPause = 5, kIrq = 6 };

// seed of make_substream(seed, name, purpose); `name_hash` = fnv1a(name)
MG_HD uint64_t substream_seed(uint64_t seed, uint64_t name_hash, uint64_t purpose) {
    uint64_t m = splitmix64(seed);
    m = splitmix64(m ^ name_hash);
    return splitmix64(m ^ purpose);
}

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xb5026f5aa96619e9ull;
constexpr uint64_t kMtUpper = 0xffffffff80000000ull;
constexpr uint64_t kMtLower = 0x000000007fffffffull;

MG_HD uint64_t mt_temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    z ^= (z >> 43);
    return z;
}

MG_HD uint64_t mt_twist_one(uint64_t cur, uint64_t next, uint64_t far) {
    const uint64_t y = (cur & kMtUpper) | (next & kMtLower);
    return far ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}

// Sequential mt19937_64 over caller-provided state storage (registers are impossible at 2.5 KB;
// the caller places `x` in local, shared or global memory).
struct Mt64Ref {
    uint64_t* x;
    int p;

    MG_HD void seed(uint64_t s) {
        x[0] = s;
        for (int i = 1; i < kMtN; ++i) {
            const uint64_t prev = x[i - 1];
            x[i] = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<uint64_t>(i);
        }
        p = kMtN;
    }
    MG_HD void twist() {
        for (int k = 0; k < kMtN - kMtM; ++k) x[k] = mt_twist_one(x[k], x[k + 1], x[k + kMtM]);
        for (int k = kMtN - kMtM; k < kMtN - 1; ++k) x[k] = mt_twist_one(x[k], x[k + 1], x[k + kMtM - kMtN]);
        x[kMtN - 1] = mt_twist_one(x[kMtN - 1], x[0], x[kMtM - 1]);
        p = 0;
    }
    MG_HD uint64_t operator()() {
        if (p >= kMtN) twist();
        return mt_temper(x[p++]);
    }
};

// generate_canonical<double, 53>(mt19937_64)
MG_HD double canonical_from(uint64_t v) {
#if defined(__CUDA_ARCH__)
    double d = __ull2double_rn(v);
#else
    double d = static_cast<double>(v);
#endif
    d = fmul(d, as_f64(0x3bf0000000000000ull));  // / 2^64, exact
    if (d >= 1.0) d = as_f64(0x3fefffffffffffffull);  // nextafter(1.0, 0.0)
    return d;
}

template <class G>
MG_HD double canonical(G& g) {
    return canonical_from(g());
}

// std::normal_distribution state (the cached second polar value)
struct NormalCache {
    bool avail = false;
    double saved = 0.0;
};

// One normal_distribution::operator() returning `ret` before `* stddev + mean`.
template <class G>
MG_HD double normal_raw(G& g, NormalCache& c) {
    if (c.avail) {
        c.avail = false;
        return c.saved;
    }
    double x, y, r2;
    do {
        x = fsub(fmul(2.0, canonical(g)), 1.0);
        y = fsub(fmul(2.0, canonical(g)), 1.0);
        r2 = fadd(fmul(x, x), fmul(y, y));
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = fsqrt(fdiv_exact(fmul(-2.0, gl_log(r2)), r2));
    c.saved = fmul(x, mult);
    c.avail = true;
    return fmul(y, mult);
}

// normal_distribution(mean, sd) draw
template <class G>
MG_HD double normal(G& g, NormalCache& c, double mean, double sd) {
    return fadd(fmul(normal_raw(g, c), sd), mean);
}

// Precomputed gamma_distribution::param_type (random.tcc:2337-2345) plus beta.
struct GammaParams {
    double alpha;      // shape
    double beta;       // scale
    double malpha;     // alpha < 1 ? alpha + 1 : alpha
    double a1;         // malpha - 1/3
    double a2;         // 1 / sqrt(9 * a1)
    double inv_alpha;  // 1 / alpha
};

// gamma_distribution(alpha, beta)(g) with a fresh distribution object (fresh normal cache),
// exactly as workload.cpp:134-135 constructs it per call.
template <class G>
MG_HD double gamma_draw(G& g, const GammaParams& p) {
    NormalCache nd;
    double u, v, n;
    for (;;) {
        do {
            n = fadd(fmul(normal_raw(g, nd), 1.0), 0.0);  // _M_nd is normal(0,1)
            v = fadd(1.0, fmul(p.a2, n));
        } while (v <= 0.0);
        v = fmul(fmul(v, v), v);
        u = canonical(g);
        const double sq = fsub(1.0, fmul(fmul(fmul(fmul(0.0331, n), n), n), n));
        if (!(u > sq)) break;
        const double rhs = fadd(fmul(fmul(0.5, n), n), fmul(p.a1, fadd(fsub(1.0, v), gl_log(v))));
        if (!(gl_log(u) > rhs)) break;
    }
    if (p.alpha == p.malpha) return fmul(fmul(p.a1, v), p.beta);
    do {
        u = canonical(g);
    } while (u == 0.0);
    return fmul(fmul(fmul(gl_pow(u, p.inv_alpha), p.a1), v), p.beta);
}

// lognormal_distribution(m, s)(g), fresh object per call (workload.cpp:148-149)
template <class G>
MG_HD double lognormal_draw(G& g, double m, double s) {
    NormalCache nd;
    const double n = fadd(fmul(normal_raw(g, nd), 1.0), 0.0);
    return gl_exp(fadd(fmul(s, n), m));
}

// exponential_distribution(lambda)(g)
template <class G>
MG_HD double exponential_draw(G& g, double lambda) {
    return fdiv_exact(-gl_log(fsub(1.0, canonical(g))), lambda);
}

// uniform_real_distribution(a, b)(g)
template <class G>
MG_HD double uniform_draw(G& g, double a, double b) {
    return fadd(fmul(canonical(g), fsub(b, a)), a);
}

// sample_truncated_normal (engine.cpp:33-39): ONE normal_distribution object per call, so the
// polar cache is reused across rejections.
template <class G>
MG_HD double truncated_normal_draw(G& g, double mean, double sd, double lo, double hi) {
    NormalCache c;
    for (;;) {
        const double v = normal(g, c, mean, sd);
        if (v >= lo && v <= hi) return v;
    }
}

}  // namespace mg
