// Bit-exact restatement of glibc 2.39's x86-64 FMA variants of log, exp and pow.
//
// Why this exists: the reference draws every random quantity through libstdc++ <random>, whose
// gamma/normal/lognormal/exponential distributions call glibc `log`, `exp` and `pow`
// (/usr/include/c++/13/bits/random.tcc:1836,2376-2377,2389; random.h:2358,4904).  On an x86-64
// host with FMA+AVX2 the libm IFUNC resolvers select the FMA-compiled builds of glibc's
// table-driven implementations (sysdeps/ieee754/dbl-64/e_log.c, e_exp.c, e_pow.c; the ARM
// optimized-routines algorithms).  Those are *not* correctly rounded, and CUDA's libdevice
// versions differ from them in the last bit, which would flip gamma accept/reject tests and
// event-time ties.  So the device (and the host test build) evaluates the very same operation
// sequence: every `fma()` below is a `vfmadd*sd` in the FMA build (read from the disassembly of
// __log_fma @0x79d50, __exp_fma @0x79b60, __pow_fma @0x7a1e0 in libm.so.6) and every other
// operation is a plain IEEE add/sub/mul.  Tables/coefficients: libm_tables.inc, extracted
// verbatim from libm's .rodata by tools/gen_libm_tables.py.
//
// Compile device code with --fmad=false and host code with -ffp-contract=off; the explicit
// intrinsics below make these functions independent of that flag anyway.
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define MG_HD __host__ __device__ __forceinline__
// Rare paths.  Kept inline: out-of-line member calls force the simulator object (and every
// member access on the hot path) into local memory, which measured 38% slower.
#define MG_COLD __host__ __device__ __forceinline__
#else
#define MG_HD inline
#define MG_COLD inline
#endif

namespace mg {

// ---- tables (host copy always; device copy when compiled by nvcc) -------------------------
#define MG_TABLE(T, name, N) static const T h_##name[N]
#include "libm_tables.inc"
#undef MG_TABLE
#if defined(__CUDACC__)
#define MG_TABLE(T, name, N) static __device__ const T d_##name[N]
#include "libm_tables.inc"
#undef MG_TABLE
#endif
#if defined(__CUDA_ARCH__)
#define MG_TAB(name) d_##name
#else
#define MG_TAB(name) h_##name
#endif

// ---- exact IEEE primitives ------------------------------------------------------------------
MG_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double d;
    std::memcpy(&d, &u, 8);
    return d;
#endif
}
MG_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
#endif
}
MG_HD double ffma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}
MG_HD double fmul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
MG_HD double fadd(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
MG_HD double fsub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
MG_HD double fdiv_exact(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
// C fmod(x, y) (exact in IEEE arithmetic: the result x - n*y, n = trunc(x/y), is representable),
// without the library's bit-serial loop: n is estimated through a float reciprocal (relative error
// < 2^-22, so off by at most one while |x/y| < 2^20) and corrected until the remainder lies in
// [0, |y|).  For the correct n the FMA computes the exact remainder (representable => no
// rounding); for a wrong n the rounded value still has the right sign / side of |y| (rounding is
// monotone and |y| is representable), so the corrections are exact decisions.  Anything outside
// the fast range (NaN, inf, y outside the float-normal range, huge quotients) takes the library fmod.
MG_HD double fmod_fast(double x, double y) {
    const double ax = fabs(x), ay = fabs(y);
    if (!(ay >= 0x1p-120 && ay <= 0x1p120 && ax < fmul(ay, 0x1p20))) return fmod(x, y);  // float-normal y
#if defined(__CUDA_ARCH__)
    const double inv = static_cast<double>(__frcp_rn(__double2float_rn(ay)));
#else
    const double inv = static_cast<double>(1.0f / static_cast<float>(ay));
#endif
    double n = trunc(fmul(ax, inv));
    double r = ffma(-n, ay, ax);
    while (r < 0.0) {
        n = fsub(n, 1.0);
        r = ffma(-n, ay, ax);
    }
    while (r >= ay) {
        n = fadd(n, 1.0);
        r = ffma(-n, ay, ax);
    }
    return copysign(r, x);
}
MG_HD double fsqrt(double a) {
#if defined(__CUDA_ARCH__)
    return __dsqrt_rn(a);
#else
    return std::sqrt(a);
#endif
}
MG_HD double cvt_i32(int32_t k) { return static_cast<double>(k); }  // vcvtsi2sd: exact

MG_HD double k_inf() { return as_f64(0x7ff0000000000000ull); }
MG_HD double k_nan() { return as_f64(0x7ff8000000000000ull); }

// ---- log (glibc e_log.c, FMA build) -------------------------------------------------------
MG_HD double gl_log(double x) {
    const uint64_t* C = MG_TAB(log_consts);
    const uint64_t* T = MG_TAB(log_tab);
    uint64_t ix = as_u64(x);
    const uint32_t top = static_cast<uint32_t>(ix >> 48);
    // |x - 1| < ~0x1p-4: dedicated polynomial (0x79e50..0x79f22)
    if (ix - 0x3fee000000000000ull < 0x0003090000000000ull) {
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double B0 = as_f64(C[7]), B1 = as_f64(C[8]), B2 = as_f64(C[9]), B3 = as_f64(C[10]);
        const double B4 = as_f64(C[11]), B5 = as_f64(C[12]), B6 = as_f64(C[13]), B7 = as_f64(C[14]);
        const double B8 = as_f64(C[15]), B9 = as_f64(C[16]), B10 = as_f64(C[17]);
        const double r = fsub(x, 1.0);
        const double r2 = fmul(r, r);
        const double r3 = fmul(r, r2);
        const double q3 = ffma(r3, B10, ffma(r2, B9, ffma(r, B8, B7)));
        const double q2 = ffma(q3, r3, ffma(r2, B6, ffma(r, B5, B4)));
        const double p = ffma(q2, r3, ffma(r2, B3, ffma(r, B2, B1)));
        const double t27 = ffma(r, 134217728.0, r);  // r + r*0x1p27, fused
        const double rhi = ffma(-134217728.0, r, t27);
        const double rlo = fsub(r, rhi);
        const double rr = fmul(rhi, rhi);
        const double hi = ffma(rr, B0, r);
        double lo = ffma(rr, B0, fsub(r, hi));
        lo = ffma(fmul(B0, rlo), fadd(r, rhi), lo);
        const double y = ffma(p, r3, lo);
        return fadd(hi, y);
    }
    if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
        // x < 0x1p-1022, negative, inf or nan (0x79f28)
        if ((ix << 1) == 0) return -k_inf();
        if (ix == 0x7ff0000000000000ull) return x;
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return k_nan();
        ix = as_u64(fmul(x, 4503599627370496.0)) - (52ull << 52);  // subnormal: scale by 2^52
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = static_cast<int>((tmp >> 45) & 127u);
    const int32_t k = static_cast<int32_t>(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
    const double invc = as_f64(T[2 * i]);
    const double logc = as_f64(T[2 * i + 1]);
    const double z = as_f64(iz);
    const double kd = cvt_i32(k);
    const double Ln2hi = as_f64(C[0]), Ln2lo = as_f64(C[1]);
    const double A0 = as_f64(C[2]), A1 = as_f64(C[3]), A2 = as_f64(C[4]), A3 = as_f64(C[5]), A4 = as_f64(C[6]);
    const double w = ffma(kd, Ln2hi, logc);
    const double r = ffma(z, invc, -1.0);
    const double t5 = ffma(r, A2, A1);
    const double hi = fadd(r, w);
    const double r2 = fmul(r, r);
    const double lo = ffma(kd, Ln2lo, fadd(fsub(w, hi), r));
    const double r3 = fmul(r, r2);
    double t1 = ffma(r, A4, A3);
    const double t2 = ffma(r2, A0, lo);
    t1 = ffma(t1, r2, t5);
    const double y = ffma(r3, t1, t2);
    return fadd(y, hi);
}

// ---- exp (glibc e_exp.c, FMA build) -------------------------------------------------------
MG_HD double gl_exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;
        const double scale = as_f64(sbits);
        return fmul(ffma(scale, tmp, scale), as_f64(0x7f00000000000000ull));  // * 0x1p1009
    }
    sbits += 1022ull << 52;
    const double scale = as_f64(sbits);
    const double st = fmul(tmp, scale);
    double y = fadd(scale, st);
    if (y < 1.0) {
        double lo = fadd(fsub(scale, y), st);
        const double hi = fadd(y, 1.0);
        lo = fadd(fadd(fsub(1.0, hi), y), lo);
        y = fsub(fadd(lo, hi), 1.0);
        if (y == 0.0) return 0.0;
    }
    return fmul(y, as_f64(0x0010000000000000ull));  // * 0x1p-1022
}

MG_HD double gl_exp(double x) {
    const uint64_t* C = MG_TAB(exp_consts);
    const uint64_t* T = MG_TAB(exp_tab);
    const uint64_t ix = as_u64(x);
    const uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u > 0x3eu) {
        if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return fadd(x, 1.0);  // tiny: 1 + x
        if (abstop <= 0x408u) {
            special = true;  // 512 <= |x| < 1024: scaled evaluation below
        } else {
            if (ix == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ffu) return fadd(x, 1.0);
            return (ix >> 63) ? 0.0 : k_inf();
        }
    }
    const double InvLn2N = as_f64(C[0]), Shift = as_f64(C[1]), NegLn2hiN = as_f64(C[2]), NegLn2loN = as_f64(C[3]);
    const double C2 = as_f64(C[4]), C3 = as_f64(C[5]), C4 = as_f64(C[6]), C5 = as_f64(C[7]);
    double kd = ffma(x, InvLn2N, Shift);
    const uint64_t ki = as_u64(kd);
    kd = fsub(kd, Shift);
    double r = ffma(kd, NegLn2hiN, x);
    r = ffma(kd, NegLn2loN, r);
    double t = ffma(r, C3, C2);
    const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
    const uint64_t top = ki << 45;
    const double u = fadd(r, as_f64(T[idx]));
    const uint64_t sbits = T[idx + 1] + top;
    const double r2 = fmul(r, r);
    const double v = ffma(r, C5, C4);
    t = ffma(t, r2, u);
    const double r4 = fmul(r2, r2);
    const double tmp = ffma(r4, v, t);
    if (special) return gl_exp_specialcase(tmp, sbits, ki);
    const double scale = as_f64(sbits);
    return ffma(scale, tmp, scale);
}

// ---- pow (glibc e_pow.c, FMA build) -------------------------------------------------------
MG_HD double gl_pow_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;
        const double scale = as_f64(sbits);
        return fmul(ffma(scale, tmp, scale), as_f64(0x7f00000000000000ull));
    }
    sbits += 1022ull << 52;
    const double scale = as_f64(sbits);
    const double st = fmul(tmp, scale);
    double y = fadd(scale, st);
    const double ay = as_f64(as_u64(y) & 0x7fffffffffffffffull);
    if (ay < 1.0) {
        const double one = y < 0.0 ? -1.0 : 1.0;
        double lo = fadd(fsub(scale, y), st);
        const double hi = fadd(y, one);
        lo = fadd(fadd(fsub(one, hi), y), lo);
        y = fsub(fadd(lo, hi), one);
        if (y == 0.0) y = as_f64(sbits & 0x8000000000000000ull);
    }
    return fmul(y, as_f64(0x0010000000000000ull));
}

MG_HD double gl_pow_exp_inline(double x, double xtail, uint32_t sign_bias) {
    const uint64_t* C = MG_TAB(exp_consts);
    const uint64_t* T = MG_TAB(exp_tab);
    const uint64_t ix = as_u64(x);
    uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ffu;
    if (abstop - 0x3c9u > 0x3eu) {
        if (static_cast<int32_t>(abstop - 0x3c9u) < 0) {
            const double one = fadd(x, 1.0);
            return sign_bias ? -one : one;
        }
        if (abstop > 0x408u) {
            const double z = (ix >> 63) ? 0.0 : k_inf();
            return sign_bias ? -z : z;
        }
        abstop = 0;
    }
    const double InvLn2N = as_f64(C[0]), Shift = as_f64(C[1]), NegLn2hiN = as_f64(C[2]), NegLn2loN = as_f64(C[3]);
    const double C2 = as_f64(C[4]), C3 = as_f64(C[5]), C4 = as_f64(C[6]), C5 = as_f64(C[7]);
    double kd = ffma(x, InvLn2N, Shift);
    const uint64_t ki = as_u64(kd);
    kd = fsub(kd, Shift);
    double r = ffma(kd, NegLn2hiN, x);
    r = ffma(kd, NegLn2loN, r);
    r = fadd(xtail, r);
    const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
    const uint64_t top = (ki + sign_bias) << 45;
    const uint64_t sbits = T[idx + 1] + top;
    double t = ffma(r, C3, C2);
    const double u = fadd(r, as_f64(T[idx]));
    const double r2 = fmul(r, r);
    const double v = ffma(r, C5, C4);
    t = ffma(t, r2, u);
    const double r4 = fmul(r2, r2);
    const double tmp = ffma(r4, v, t);
    if (abstop == 0) return gl_pow_specialcase(tmp, sbits, ki);
    const double scale = as_f64(sbits);
    return ffma(scale, tmp, scale);
}

// 0: not an integer, 1: odd integer, 2: even integer (e_pow.c checkint)
MG_HD int gl_pow_checkint(uint64_t iy) {
    const int e = static_cast<int>(iy >> 52 & 0x7ff);
    if (e < 0x3ff) return 0;
    if (e > 0x3ff + 52) return 2;
    if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
    if (iy & (1ull << (0x3ff + 52 - e))) return 1;
    return 2;
}

MG_HD bool gl_zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * as_u64(k_inf()) - 1; }

MG_HD double gl_pow(double x, double y) {
    const uint64_t* C = MG_TAB(powlog_consts);
    const uint64_t* T = MG_TAB(powlog_tab);
    uint32_t sign_bias = 0;
    uint64_t ix = as_u64(x);
    const uint64_t iy = as_u64(y);
    uint32_t topx = static_cast<uint32_t>(ix >> 52);
    const uint32_t topy = static_cast<uint32_t>(iy >> 52);
    if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
        if (gl_zeroinfnan(iy)) {
            if (2 * iy == 0) return 1.0;
            if (ix == 0x3ff0000000000000ull) return 1.0;
            if (2 * ix > 2 * as_u64(k_inf()) || 2 * iy > 2 * as_u64(k_inf())) return fadd(x, y);
            if (2 * ix == 2 * 0x3ff0000000000000ull) return 1.0;
            if ((2 * ix < 2 * 0x3ff0000000000000ull) == !(iy >> 63)) return 0.0;
            return fmul(y, y);
        }
        if (gl_zeroinfnan(ix)) {
            double x2 = fmul(x, x);
            if ((ix >> 63) && gl_pow_checkint(iy) == 1) x2 = -x2;
            return (iy >> 63) ? 1.0 / x2 : x2;
        }
        if (ix >> 63) {
            const int yint = gl_pow_checkint(iy);
            if (yint == 0) return k_nan();
            if (yint == 1) sign_bias = 0x800u << 7;
            ix &= 0x7fffffffffffffffull;
            topx &= 0x7ffu;
        }
        if ((topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
            if (ix == 0x3ff0000000000000ull) return 1.0;
            if ((topy & 0x7ffu) < 0x3beu) return ix > 0x3ff0000000000000ull ? fadd(1.0, y) : fsub(1.0, y);
            return ((ix > 0x3ff0000000000000ull) == (topy < 0x800u)) ? k_inf() : 0.0;
        }
        if (topx == 0) {
            ix = as_u64(fmul(x, 4503599627370496.0)) & 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    }
    // log_inline (e_pow.c), double-double result hi + lo
    const uint64_t tmp = ix - 0x3fe6955500000000ull;
    const int i = static_cast<int>((tmp >> 45) & 127u);
    const int32_t k = static_cast<int32_t>(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
    const double z = as_f64(iz);
    const double kd = cvt_i32(k);
    const double invc = as_f64(T[4 * i + 0]);
    const double logc = as_f64(T[4 * i + 2]);
    const double logctail = as_f64(T[4 * i + 3]);
    const double Ln2hi = as_f64(C[0]), Ln2lo = as_f64(C[1]);
    const double A0 = as_f64(C[2]), A1 = as_f64(C[3]), A2 = as_f64(C[4]), A3 = as_f64(C[5]);
    const double A4 = as_f64(C[6]), A5 = as_f64(C[7]), A6 = as_f64(C[8]);
    const double t1 = ffma(kd, Ln2hi, logc);
    const double lo1 = ffma(kd, Ln2lo, logctail);
    const double r = ffma(z, invc, -1.0);
    const double ar = fmul(r, A0);
    const double p1 = ffma(r, A2, A1);
    const double p2 = ffma(r, A4, A3);
    const double t2 = fadd(r, t1);
    const double lo2 = fadd(fsub(t1, t2), r);
    const double ar2 = fmul(r, ar);
    const double ar3 = fmul(r, ar2);
    const double lo3 = ffma(ar, r, -ar2);
    const double hi = fadd(t2, ar2);
    double p3 = ffma(r, A6, A5);
    const double lo4 = fadd(fsub(t2, hi), ar2);
    p3 = ffma(p3, ar2, p2);
    const double p = ffma(ar2, p3, p1);
    double lo = fadd(lo1, lo2);
    lo = fadd(lo, lo3);
    lo = fadd(lo, lo4);
    lo = ffma(ar3, p, lo);
    const double lhi = fadd(hi, lo);
    const double llo = fadd(fsub(hi, lhi), lo);
    const double ehi = fmul(y, lhi);
    double elo = ffma(lhi, y, -ehi);
    elo = ffma(y, llo, elo);
    return gl_pow_exp_inline(ehi, elo, sign_bias);
}

}  // namespace mg
