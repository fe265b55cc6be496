/*
 * ifa_oracle.h -- CPU restatement of the INT-FlashAttention hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker (never as the measured path).
 *
 * Every function restates the reference algorithm of
 * /root/reference/proj (C++20, CPU) and cites the file:line it follows.
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libifa_ref.so built from the reference's own sources by
 * oracle/Makefile) and against the known-answer hashes of SURVEY.md
 * Appendix A (tests/golden/), see tests/test_oracle.py.
 *
 * Layout contract: all matrices are row-major and
 * contiguous; a batch of (b,h) "slices" is [slices][n][d] with no padding;
 * per-row scales are [slices][n]; the V tensor scale is one float per slice.
 */
#ifndef IFA_ORACLE_H
#define IFA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flags shared with include/ifa_b200.h. */
#define IFA_OR_FLAG_SQRT_D 1u  /* AttentionConfig::apply_sqrt_d_scaling */
#define IFA_OR_FLAG_CAUSAL 2u  /* extension: row i sees keys j <= i      */

typedef struct ifa_or_audit {
    int32_t min_code;               /* PCodeAudit::min_code (attention.hpp:76) */
    int32_t max_code;               /* PCodeAudit::max_code                    */
    int32_t row_max_block_hits_127; /* PCodeAudit::row_max_block_hits_127      */
    int32_t pad_;
    int64_t rows_audited;           /* PCodeAudit::rows_audited                */
} ifa_or_audit;

/* glibc 2.39 expf restated bit-exactly (see ifa_oracle.c). */
float ifa_or_expf(float x);

/* eval.cpp:23-44 stream_seed (mix64/fold). */
uint64_t ifa_or_stream_seed(uint64_t base, int seed_idx, int role, int64_t b, int64_t h);

/* generate.cpp:47-78.  dist 0 = normal(a=mean, b=stddev), 1 = uniform(a=lo, b=hi). */
int ifa_or_generate(int dist, double a, double b, uint64_t seed, int64_t rows, int64_t cols,
                    float *out);

/* quant.cpp:44-57 / :59-69.  Returns 0, or -1 with *bad_index set to the
 * first non-finite element's flat index (quant.cpp:14-22). */
int ifa_or_quantize_per_row(const float *x, int64_t rows, int64_t cols, int8_t *codes,
                            float *scales, int64_t *bad_index);
int ifa_or_quantize_per_tensor(const float *x, int64_t rows, int64_t cols, int8_t *codes,
                               float *scale, int64_t *bad_index);

/* gemm.cpp:32-46: out[m][n] = sum_t a[m][t]*b[n][t], int32. */
void ifa_or_int_gemm_nt(const int8_t *a, const int8_t *b, int64_t m, int64_t n, int64_t k,
                        int32_t *out);

/* attention.cpp:235-357 (one slice) plus the causal extension.
 * Returns 0, -1 (invalid argument) or -2 (depth guard, gemm.cpp:22-28). */
int ifa_or_int_flash_attention(const int8_t *q, const float *sq, const int8_t *k,
                               const float *sk, const int8_t *v, float sv, int64_t n,
                               int64_t d, int64_t br, int64_t bc, uint32_t flags,
                               float *out, ifa_or_audit *audit);

/* ifa_or_int_flash_attention that also records every P code it feeds to
 * P.V (attention.cpp:299-312) into pcodes[n][n] (row i, key j of block j0;
 * masked causal entries 0; entries never visited are left untouched). */
int ifa_or_int_flash_attention_pcodes(const int8_t *q, const float *sq, const int8_t *k,
                                      const float *sk, const int8_t *v, float sv, int64_t n,
                                      int64_t d, int64_t br, int64_t bc, uint32_t flags,
                                      float *out, uint8_t *pcodes);

/* ifa_or_int_flash_attention restricted to the row blocks starting in
 * [row_begin, row_end) (row_begin a multiple of br; row blocks are
 * independent in the reference, attention.cpp:267): writes only those rows
 * of out[n][d].  For spot checks of long sequences (C3 / C5). */
int ifa_or_int_flash_attention_rows(const int8_t *q, const float *sq, const int8_t *k,
                                    const float *sk, const int8_t *v, float sv, int64_t n,
                                    int64_t d, int64_t br, int64_t bc, uint32_t flags,
                                    int64_t row_begin, int64_t row_end, float *out);

/* Batched form over [slices][n][d] using up to `threads` host threads
 * (one slice per task from an atomic queue).  audit may be NULL. */
int ifa_or_int_flash_attention_batched(const int8_t *q, const float *sq, const int8_t *k,
                                       const float *sk, const int8_t *v, const float *sv,
                                       int64_t slices, int64_t n, int64_t d, int64_t br,
                                       int64_t bc, uint32_t flags, float *out, int threads);

/* oracles.cpp:83-134 untiled integer attention (plus causal extension). */
int ifa_or_untiled_int8_attention(const int8_t *q, const float *sq, const int8_t *k,
                                  const float *sk, const int8_t *v, float sv, int64_t n,
                                  int64_t d, uint32_t flags, float *out);

/* attention.cpp:151-192 fp64 ground truth (plus causal extension). */
int ifa_or_half_int8_attention(const int8_t *q, const float *sq, const int8_t *k,
                               const float *sk, const float *v, int64_t n, int64_t d,
                               int64_t br, int64_t bc, uint32_t flags, float *out);
/* fp8.cpp:17-97: e4m3 encode (round half to even on the exact double
 * quotient, saturate at 448, subnormal step 2^-9), decode, and the
 * per-matrix roundtrip (s = 448 / max|x|; x -> decode(encode(x*s)) / s).
 * ifa_or_fp8_roundtrip returns -1 on non-finite input (fp8.cpp:82-84);
 * codes / scale (optional) receive the e4m3 bytes and s (0 for all-zero). */
uint8_t ifa_or_e4m3_encode(float x);
float ifa_or_e4m3_decode(uint8_t bits);
int ifa_or_fp8_roundtrip(const float *x, int64_t count, float *out, uint8_t *codes, float *scale);
/* attention.cpp:401-407 fp8_emulated_attention = flash_attention_float
 * (:194-211, tiled_float_attention :49-80) over the three roundtrips. */
int ifa_or_fp8_attention(const float *q, const float *k, const float *v, int64_t n, int64_t d,
                         int64_t br, int64_t bc, uint32_t flags, float *out);
int ifa_or_reference_attention(const float *q, const float *k, const float *v, int64_t n,
                               int64_t m, int64_t d, int64_t dv, uint32_t flags, float *out);

/* eval.cpp:55-75 ErrorAccum: adds sum|c-r| and sum|r| into num/den. */
void ifa_or_error_accum(const float *reference, const float *candidate, int64_t count,
                        double *num, double *den);

/* Exhaustive scan of code(x) = (int)roundf(127*expf(x)) over every float in
 * [-104, 0] (libm expf, as the reference): writes B[k] = smallest x with
 * code(x) >= k+1 (k = 0..126) into out[0..126] and returns 1 if code is
 * non-decreasing in x, 0 otherwise.  Uses `threads` host threads. */
int ifa_or_code_bounds_exhaustive(float *out, int threads);

/* FNV-1a-64 over raw bytes (SURVEY.md Appendix A hash recipe). */
uint64_t ifa_or_fnv1a64(const void *data, int64_t nbytes);

#ifdef __cplusplus
}
#endif

#endif
