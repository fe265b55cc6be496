// code_bounds.cpp -- host side of the exact requantization (see
// code_bounds.h).  The double-precision steps are written with explicit
// std::fma where glibc's FMA variant contracts and volatile temporaries
// where it does not, so the result does not depend on host compiler flags.
//
// Provenance: the 32-entry 2^(i/32) table and the polynomial / shift
// constants are glibc's __exp2f_data (sysdeps/ieee754/flt-32/e_exp2f_data.c,
// glibc 2.39), which comes from ARM's optimized-routines (MIT OR Apache-2.0
// WITH LLVM-exception; glibc ships it under LGPL-2.1+).  They are
// mathematical constants reproduced because bit-exact parity with the
// reference's libm expf needs exactly these values; no code is copied from
// the reference (which has none of it) or from glibc.
#include "code_bounds.h"

#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>

namespace ifa_b200 {
namespace {

// glibc __exp2f_data (sysdeps/ieee754/flt-32/e_exp2f_data.c): 2^(i/32) with
// the exponent bits pre-subtracted; SHIFT = 0x1.8p52, 32/ln2 and the scaled
// degree-3 polynomial are below.
const uint64_t kTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

double as_d(uint64_t u) {
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}
uint64_t as_u(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

}  // namespace

float host_exact_expf(float x) {
    uint32_t ux;
    std::memcpy(&ux, &x, 4);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8) return x + x;
        if (x > 0x1.62e42ep6f) return std::numeric_limits<float>::infinity();
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = static_cast<double>(x);
    const double inv = as_d(0x40471547652b82feULL);
    const double shift = as_d(0x4338000000000000ULL);
    volatile double prod = inv * xd;  // rounded product, then the shift add
    double kd = prod + shift;
    const uint64_t ki = as_u(kd);
    kd -= shift;
    const double r = std::fma(inv, xd, -kd);
    uint64_t t = kTab[ki % 32];
    t += ki << 47;
    const double s = as_d(t);
    const double z = std::fma(as_d(0x3ebc6af84b912394ULL), r, as_d(0x3f2ebfce50fac4f3ULL));
    volatile double r2 = r * r;
    double y = std::fma(as_d(0x3f962e42ff0c52d6ULL), r, 1.0);
    y = std::fma(z, r2, y);
    volatile double ys = y * s;
    return static_cast<float>(ys);
}

int host_code(float x) {
    volatile float y = 127.0f * host_exact_expf(x);
    return static_cast<int>(std::round(y));
}

const float* code_bounds() {
    static float bounds[128];
    static std::once_flag once;
    std::call_once(once, [] {
        // Negative floats order in reverse of their bit patterns: walk from
        // -0 (0x80000000, code 127) to -104 (0xC2D00000, code 0) and bisect.
        for (int k = 0; k < 127; ++k) {
            uint32_t a = 0x80000000u, b = 0xC2D00000u;  // code(a) >= k+1 > code(b)
            while (b - a > 1) {
                const uint32_t mid = a + (b - a) / 2;
                float xm;
                std::memcpy(&xm, &mid, 4);
                if (host_code(xm) >= k + 1)
                    a = mid;
                else
                    b = mid;
            }
            std::memcpy(&bounds[k], &a, 4);
        }
        bounds[127] = std::numeric_limits<float>::infinity();
    });
    return bounds;
}

}  // namespace ifa_b200
