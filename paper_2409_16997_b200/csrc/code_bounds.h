// code_bounds.h -- exact decision boundaries of the reference's weight code
// (attention.cpp:306-307):  code(x) = (int)std::round(127.0f * std::exp(x)).
//
// code(x) is non-decreasing in x (verified exhaustively over every float in
// [-104, 0] by tests/test_oracle.py::test_code_bounds_exhaustive), so it is
// fully described by 127 thresholds: B[k] = the smallest float x with
// code(x) >= k + 1.  The device kernel's fast MUFU estimate pins a code to
// {k, k+1} whenever it lands near the boundary k + 1/2; one comparison
// x >= B[k] then reproduces the reference bit-exactly.
#pragma once
#include <cstdint>

namespace ifa_b200 {

// Bit-exact host restatement of glibc 2.39 expf (x86-64 FMA variant).
float host_exact_expf(float x);

// code(x) as the reference computes it.
int host_code(float x);

// bounds[0..126] = B[k]; bounds[127] = +inf.  Computed once per process.
const float* code_bounds();

}  // namespace ifa_b200
