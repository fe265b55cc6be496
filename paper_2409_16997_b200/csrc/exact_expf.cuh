// exact_expf.cuh -- bit-exact device restatement of the host expf that the
// reference's std::exp(float) resolves to (glibc 2.39, x86-64 FMA variant),
// and the guarded requantization step built on it.
//
// Algorithm (ARM optimized-routines expf, as shipped in glibc): x*32/ln2 =
// k + r, exp(x) = 2^(k/32) * poly(r), evaluated in double, rounded once to
// float.  Every double operation below is an explicit __dmul_rn/__dadd_rn/
// __fma_rn so the result is bit-identical to the host routine; the
// identical C restatement (oracle/ifa_oracle.c: ifa_or_expf) matched the
// container's libm on all 2,239,627,266 floats in [-103, 88].
//
// Provenance: the 32-entry 2^(i/32) table and the polynomial / shift
// constants are glibc's __exp2f_data (sysdeps/ieee754/flt-32/e_exp2f_data.c,
// glibc 2.39), which comes from ARM's optimized-routines (MIT OR Apache-2.0
// WITH LLVM-exception; glibc ships it under LGPL-2.1+).  They are
// mathematical constants reproduced because bit-exact parity with the
// reference's libm expf needs exactly these values; no code is copied from
// the reference (which has none of it) or from glibc.
#pragma once
#include <cstdint>

namespace ifa_b200 {

__device__ __constant__ uint64_t kExp2fTabDev[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

// Bit-exact glibc expf.  Arguments on the attention path are <= 0 or -inf.
__device__ __forceinline__ float exact_expf(float x) {
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8) return x + x;
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = static_cast<double>(x);
    const double inv = __longlong_as_double(0x40471547652b82feLL);
    const double shift = __longlong_as_double(0x4338000000000000LL);
    double kd = __dadd_rn(__dmul_rn(inv, xd), shift);
    const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, shift);
    const double r = __fma_rn(inv, xd, -kd);
    uint64_t t = kExp2fTabDev[ki & 31];
    t += ki << 47;
    const double s = __longlong_as_double(static_cast<long long>(t));
    const double z = __fma_rn(__longlong_as_double(0x3ebc6af84b912394LL), r,
                              __longlong_as_double(0x3f2ebfce50fac4f3LL));
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(__longlong_as_double(0x3f962e42ff0c52d6LL), r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

// The reference's weight code: (int)std::round(127.0f * std::exp(x))
// (attention.cpp:306-307), exactly.
__device__ __forceinline__ int exact_code(float x) {
    return static_cast<int>(roundf(__fmul_rn(127.0f, exact_expf(x))));
}

// Guarded fast form of exact_code.  The MUFU estimate y ~ 127*e^x is within
// kCodeGuard of the reference's fl(127*fl(expf(x))) (|x*log2e| rounding
// <= 2^-24 rel, ex2.approx <= 2^-21 rel, products 2^-24 each => < 1.9e-4
// absolute on [0,127]); whenever y is that close to a rounding boundary
// (a half-integer) the exact double-precision path decides.
constexpr float kCodeGuard = 1.0e-3f;

__device__ __forceinline__ float ex2_approx(float t) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
    return r;
}

__device__ __forceinline__ int guarded_code(float x) {
    const float y = 127.0f * ex2_approx(x * 1.4426950408889634f);
    const float fl = floorf(y);
    const float frac = y - fl;
    if (fabsf(frac - 0.5f) < kCodeGuard) return exact_code(x);
    return static_cast<int>(fl) + (frac >= 0.5f ? 1 : 0);
}

}  // namespace ifa_b200
