// exp and log1p with glibc's algorithms, so device values equal the reference's
// std::exp / std::log1p (tensor.hpp:146-154, ssm.cpp:157) bit for bit.
//
// CUDA's exp differs from glibc's in ~6% of arguments and log1p in ~1% (by one
// ulp; scripts/libm_probe.py). An ulp can move a value across a code's rounding
// boundary, and the recurrence then carries the flipped code to the logits. The
// reference links glibc 2.39 on x86-64 with FMA:
//  - exp is the table-driven algorithm of sysdeps/ieee754/dbl-64/e_exp.c (N = 128,
//    degree-5 polynomial), dispatched to its FMA build (x86_64 multiarch
//    e_exp-fma), where the compiler fuses every product that feeds one add;
//  - log1p is the fdlibm algorithm of sysdeps/ieee754/dbl-64/s_log1p.c, also
//    dispatched to an FMA build (Ubuntu's 2.39 libm resolves log1p through an
//    ifunc to it); the fusions below are read off that build's instructions.
// The operation order below is that of those builds. tests/test_glibc_math.py
// checks these functions (compiled for the host) against the live libm on
// millions of arguments.
#pragma once
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define OB_GL_HD __host__ __device__ __forceinline__
#else
#define OB_GL_HD inline
#endif

namespace ob {
namespace gl {

#if defined(__CUDACC__)
static __device__ const unsigned long long kExpTabDev[256] = {
#include "glibc_exp_table.inc"
};
#endif
static const unsigned long long kExpTabHost[256] = {
#include "glibc_exp_table.inc"
};

OB_GL_HD uint64_t tab(unsigned i) {
#if defined(__CUDA_ARCH__)
    return __ldg(&kExpTabDev[i]);
#else
    return kExpTabHost[i];
#endif
}
OB_GL_HD uint64_t as_u64(double x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    return u;
#endif
}
OB_GL_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    std::memcpy(&x, &u, sizeof x);
    return x;
#endif
}
// One rounding each; the host build must not contract (-ffp-contract=off).
OB_GL_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
OB_GL_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
OB_GL_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
OB_GL_HD double div(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
OB_GL_HD double fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return __builtin_fma(a, b, c);
#endif
}

// exp's out-of-range tail (|x| >= 512): scale 2^(k/N) would leave the exponent
// range, so it is applied in two steps (e_exp.c specialcase).
OB_GL_HD double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
    // (the dispatched build fuses the overflow side and not the underflow side;
    // checked against libm over [-760, -512] and [512, 710))
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;
        const double scale = as_f64(sbits);
        return mul(0x1p1009, fma(scale, tmp, scale));
    }
    sbits += 1022ull << 52;
    const double scale = as_f64(sbits);
    double y = add(scale, mul(scale, tmp));
    if (y < 1.0) {  // round to the subnormal precision once
        double lo = add(sub(scale, y), mul(scale, tmp));
        const double hi = add(1.0, y);
        lo = add(add(sub(1.0, hi), y), lo);
        y = sub(add(hi, lo), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return mul(0x1p-1022, y);
}

OB_GL_HD double exp(double x) {
    constexpr double kInvLn2N = 0x1.71547652b82fep0 * 128;
    constexpr double kShift = 0x1.8p52;
    constexpr double kNegLn2HiN = -0x1.62e42fefa0000p-8;
    constexpr double kNegLn2LoN = -0x1.cf79abc9e3b3ap-47;
    constexpr double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    constexpr double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    uint32_t abstop = static_cast<uint32_t>(as_u64(x) >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if (abstop - 0x3c9u >= 0x80000000u) return add(1.0, x);  // |x| < 2^-54
        if (abstop >= 0x409u) {                                   // |x| >= 1024
            if (as_u64(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return add(1.0, x);
            return (as_u64(x) >> 63) ? 0.0 : as_f64(0x7ff0000000000000ull);
        }
        abstop = 0;  // 512 <= |x| < 1024
    }
    const double kd0 = fma(kInvLn2N, x, kShift);
    const uint64_t ki = as_u64(kd0);
    const double kd = sub(kd0, kShift);
    const double r = fma(kd, kNegLn2LoN, fma(kd, kNegLn2HiN, x));
    const unsigned idx = 2u * static_cast<unsigned>(ki % 128u);
    const uint64_t top = ki << 45;
    const double tail = as_f64(tab(idx));
    const uint64_t sbits = tab(idx + 1) + top;
    const double r2 = mul(r, r);
    const double tmp = fma(mul(r2, r2), fma(r, C5, C4), fma(r2, fma(r, C3, C2), add(tail, r)));
    if (abstop == 0) return exp_special(tmp, sbits, ki);
    const double scale = as_f64(sbits);
    return fma(scale, tmp, scale);
}

OB_GL_HD double log1p(double x) {
    const double ln2_hi = as_f64(0x3fe62e42fee00000ull), ln2_lo = as_f64(0x3dea39ef35793c76ull);
    const double Lp1 = as_f64(0x3FE5555555555593ull), Lp2 = as_f64(0x3FD999999997FA04ull),
                 Lp3 = as_f64(0x3FD2492494229359ull), Lp4 = as_f64(0x3FCC71C51D8E78AFull),
                 Lp5 = as_f64(0x3FC7466496CB03DEull), Lp6 = as_f64(0x3FC39A09D078C69Full),
                 Lp7 = as_f64(0x3FC2F112DF3E5244ull);
    const int32_t hx = static_cast<int32_t>(as_u64(x) >> 32);
    const int32_t ax = hx & 0x7fffffff;
    double f = 0.0, c = 0.0;
    int32_t k = 1, hu = 0;
    if (hx < 0x3FDA827A) {  // x < 0.41422
        if (ax >= 0x3ff00000) {  // x <= -1
            if (x == -1.0) return as_f64(0xfff0000000000000ull);
            return as_f64(0x7ff8000000000000ull);
        }
        if (ax < 0x3e200000) {  // |x| < 2^-29
            if (ax < 0x3c900000) return x;
            return fma(-0.5, mul(x, x), x);
        }
        if (hx > 0 || hx <= static_cast<int32_t>(0xbfd2bec3u)) {  // -0.2929 < x < 0.41422
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx >= 0x7ff00000) {
        return add(x, x);
    }
    if (k != 0) {
        double u;
        if (hx < 0x43400000) {
            u = add(1.0, x);
            hu = static_cast<int32_t>(as_u64(u) >> 32);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? sub(1.0, sub(u, x)) : sub(x, sub(u, 1.0));  // correction term
            c = div(c, u);
        } else {
            u = x;
            hu = static_cast<int32_t>(as_u64(u) >> 32);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        const uint64_t lo = as_u64(u) & 0xffffffffull;
        if (hu < 0x6a09e) {  // normalize u
            u = as_f64((static_cast<uint64_t>(static_cast<uint32_t>(hu | 0x3ff00000)) << 32) | lo);
        } else {  // normalize u/2
            k += 1;
            u = as_f64((static_cast<uint64_t>(static_cast<uint32_t>(hu | 0x3fe00000)) << 32) | lo);
            hu = (0x00100000 - hu) >> 2;
        }
        f = sub(u, 1.0);
    }
    const double hfsq = mul(mul(0.5, f), f);
    const double dk = static_cast<double>(k);
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            return fma(dk, ln2_hi, fma(dk, ln2_lo, c));
        }
        const double R = mul(fma(-f, 0.66666666666666666, 1.0), hfsq);
        if (k == 0) return sub(f, R);
        return fma(dk, ln2_hi, -sub(sub(R, fma(dk, ln2_lo, c)), f));
    }
    const double s = div(f, add(2.0, f));
    const double z = mul(s, s);
    const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
    const double z2 = mul(z, z), z4 = mul(z2, z2), z6 = mul(z4, z2);
    const double R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, mul(z2, R2))));
    const double m = mul(add(hfsq, R), s);
    if (k == 0) return sub(f, sub(hfsq, m));
    return fma(dk, ln2_hi, -sub(sub(hfsq, add(fma(dk, ln2_lo, c), m)), f));
}

}  // namespace gl
}  // namespace ob
