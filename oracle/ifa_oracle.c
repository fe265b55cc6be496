/*
 * ifa_oracle.c -- CPU restatement of the INT-FlashAttention hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see ifa_oracle.h).  Compiled with
 * -ffp-contract=off so every float expression rounds exactly where the
 * reference's does (the reference is built for baseline x86-64 without
 * -march, so GCC cannot contract its float expressions into FMAs).
 *
 * Sources restated (all under /root/reference/proj):
 *   src/generate.cpp:47-78   generate()          (mt19937_64 + Box-Muller)
 *   src/eval.cpp:23-44       stream_seed()
 *   src/quant.cpp:14-69      require_finite / quantize_one / max_abs /
 *                            quantize_per_row / quantize_per_tensor
 *   src/gemm.cpp:22-46       check_int_gemm_depth / int_gemm_nt_strided
 *   src/attention.cpp:213-357 QuantizedAttentionInputs::validate /
 *                            int_flash_attention
 *   src/oracles.cpp:83-134   oracle_untiled_int8_attention
 *   src/attention.cpp:151-192 reference_attention
 *   src/eval.cpp:55-75       ErrorAccum
 * Causal masking is NOT in the reference; the causal
 * branches below are this build's documented extension:
 * row i sees keys j <= i, masked entries are excluded from the row max,
 * from P, from l and from P.V, and a KV block with no visible key for a
 * row leaves that row's state untouched.
 */
#include "ifa_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* glibc 2.39 expf, restated.                                           */
/* ------------------------------------------------------------------ */
/* The reference calls std::exp(float) == glibc expf (attention.cpp:299,
 * :307).  glibc 2.39 implements expf with the published ARM
 * optimized-routines algorithm (sysdeps/ieee754/flt-32/e_expf.c):
 *   x*N/ln2 = k + r, exp(x) = 2^(k/N) * poly(r), N = 32, evaluated in
 *   double and rounded once to float.
 * The constants below are glibc's __exp2f_data (table of 2^(i/32) with the
 * exponent bits pre-subtracted, SHIFT = 0x1.8p52, N/ln2, and the scaled
 * degree-3 polynomial).  On x86-64 glibc selects the FMA variant of expf
 * through an ifunc; the restatement uses fma() for the reduction
 * r = N/ln2*x - kd and for the polynomial.  It was checked exhaustively
 * against the container's libm expf for every float in [-103, 88]
 * (2,239,627,266 inputs, 0 mismatches) and is re-checked on a sample by
 * tests/test_oracle.py.  The device copy lives in csrc/exact_expf.cuh. */
static const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};
static const uint64_t kExp2fShift = 0x4338000000000000ULL;   /* 0x1.8p52        */
static const uint64_t kExp2fInvLn2N = 0x40471547652b82feULL; /* 32/ln2          */
static const uint64_t kExp2fC0 = 0x3ebc6af84b912394ULL;      /* poly_scaled[0]  */
static const uint64_t kExp2fC1 = 0x3f2ebfce50fac4f3ULL;      /* poly_scaled[1]  */
static const uint64_t kExp2fC2 = 0x3f962e42ff0c52d6ULL;      /* poly_scaled[2]  */

static double as_double(uint64_t u) {
    double d;
    memcpy(&d, &u, sizeof d);
    return d;
}
static uint64_t as_u64(double d) {
    uint64_t u;
    memcpy(&u, &d, sizeof u);
    return u;
}

float ifa_or_expf(float x) {
    uint32_t ux;
    memcpy(&ux, &x, sizeof ux);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) { /* |x| >= 88 or nan: e_expf.c special cases */
        if (ux == 0xff800000u) return 0.0f;          /* -inf */
        if (abstop >= 0x7f8) return x + x;           /* nan / +inf */
        if (x > 0x1.62e42ep6f) return (float)INFINITY;
        if (x < -0x1.9fe368p6f) return 0.0f;
        /* the general path below is exact for the rest */
    }
    const double xd = (double)x;
    const double inv = as_double(kExp2fInvLn2N);
    const double shift = as_double(kExp2fShift);
    double kd = inv * xd + shift;
    const uint64_t ki = as_u64(kd);
    kd -= shift;
    const double r = fma(inv, xd, -kd);
    uint64_t t = kExp2fTab[ki % 32];
    t += ki << 47;
    const double s = as_double(t);
    const double z = fma(as_double(kExp2fC0), r, as_double(kExp2fC1));
    const double r2 = r * r;
    double y = fma(as_double(kExp2fC2), r, 1.0);
    y = fma(z, r2, y);
    y = y * s;
    return (float)y;
}

/* ------------------------------------------------------------------ */
/* Seeding and input synthesis                                          */
/* ------------------------------------------------------------------ */
static uint64_t mix64(uint64_t z) { /* eval.cpp:23-28 */
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static uint64_t fold(uint64_t acc, uint64_t v) { /* eval.cpp:30-32 */
    return mix64(acc ^ (v + 0x9e3779b97f4a7c15ull));
}
uint64_t ifa_or_stream_seed(uint64_t base, int seed_idx, int role, int64_t b, int64_t h) {
    uint64_t s = mix64(base); /* eval.cpp:36-44 */
    s = fold(s, (uint64_t)(int64_t)seed_idx);
    s = fold(s, (uint64_t)(int64_t)role);
    s = fold(s, (uint64_t)b);
    s = fold(s, (uint64_t)h);
    return s;
}

/* std::mt19937_64 (parameters fixed by the C++ standard). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;
static void mt64_seed(mt64 *g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(mt64 *g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
static double unit_double(mt64 *g) { /* generate.cpp:19-21 */
    return (double)(mt64_next(g) >> 11) * 0x1.0p-53;
}

int ifa_or_generate(int dist, double a, double b, uint64_t seed, int64_t rows, int64_t cols,
                    float *out) {
    if (rows < 1 || cols < 1) return -1;
    if (dist == 0 ? !(b > 0.0) : !(a < b)) return -1; /* generate.cpp:36-46 */
    mt64 *g = (mt64 *)malloc(sizeof(mt64));
    if (!g) return -1;
    mt64_seed(g, seed);
    const int64_t n = rows * cols;
    if (dist == 1) { /* generate.cpp:59-65 */
        const double range = b - a;
        for (int64_t i = 0; i < n; ++i) out[i] = (float)(a + unit_double(g) * range);
    } else { /* generate.cpp:66-77 */
        const double two_pi = 6.283185307179586476925286766559;
        for (int64_t i = 0; i < n; i += 2) {
            const double u1 = 1.0 - unit_double(g);
            const double u2 = unit_double(g);
            const double r = sqrt(-2.0 * log(u1));
            out[i] = (float)(a + b * r * cos(two_pi * u2));
            if (i + 1 < n) out[i + 1] = (float)(a + b * r * sin(two_pi * u2));
        }
    }
    free(g);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Quantization (quant.cpp)                                             */
/* ------------------------------------------------------------------ */
static int first_nonfinite(const float *x, int64_t count, int64_t *bad_index) {
    for (int64_t i = 0; i < count; ++i) { /* quant.cpp:14-22 */
        if (!isfinite(x[i])) {
            if (bad_index) *bad_index = i;
            return -1;
        }
    }
    return 0;
}
static int8_t quantize_one(float x, float scale) { /* quant.cpp:25-32 */
    if (scale == 0.0f) return 0;
    float q = roundf(x / scale);
    if (q < -127.0f) q = -127.0f;
    if (q > 127.0f) q = 127.0f;
    return (int8_t)q;
}
static float max_abs(const float *p, int64_t n) { /* quant.cpp:34-40 */
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        const float a = fabsf(p[i]);
        m = (m < a) ? a : m; /* std::max(m, a) */
    }
    return m;
}
int ifa_or_quantize_per_row(const float *x, int64_t rows, int64_t cols, int8_t *codes,
                            float *scales, int64_t *bad_index) {
    if (first_nonfinite(x, rows * cols, bad_index)) return -1;
    for (int64_t r = 0; r < rows; ++r) { /* quant.cpp:44-57 */
        const float *src = x + r * cols;
        const float scale = max_abs(src, cols) / 127.0f;
        scales[r] = scale;
        for (int64_t c = 0; c < cols; ++c) codes[r * cols + c] = quantize_one(src[c], scale);
    }
    return 0;
}
int ifa_or_quantize_per_tensor(const float *x, int64_t rows, int64_t cols, int8_t *codes,
                               float *scale, int64_t *bad_index) {
    const int64_t n = rows * cols;
    if (first_nonfinite(x, n, bad_index)) return -1;
    const float s = max_abs(x, n) / 127.0f; /* quant.cpp:59-69 */
    *scale = s;
    for (int64_t i = 0; i < n; ++i) codes[i] = quantize_one(x[i], s);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Integer GEMM (gemm.cpp)                                              */
/* ------------------------------------------------------------------ */
#define IFA_MAX_INT_GEMM_DEPTH (((int64_t)1 << 31) / (127 * 127)) /* gemm.hpp:22 */

void ifa_or_int_gemm_nt(const int8_t *a, const int8_t *b, int64_t m, int64_t n, int64_t k,
                        int32_t *out) {
    for (int64_t i = 0; i < m; ++i) /* gemm.cpp:32-46 */
        for (int64_t j = 0; j < n; ++j) {
            int32_t acc = 0;
            for (int64_t t = 0; t < k; ++t) acc += (int32_t)a[i * k + t] * (int32_t)b[j * k + t];
            out[i * n + j] = acc;
        }
}

/* ------------------------------------------------------------------ */
/* int_flash_attention (attention.cpp:235-357) + causal extension       */
/* ------------------------------------------------------------------ */
static int int_flash_impl(const int8_t *q, const float *sq, const int8_t *k, const float *sk,
                          const int8_t *v, float sv, int64_t n, int64_t d, int64_t br_cfg,
                          int64_t bc_cfg, uint32_t flags, float *out, ifa_or_audit *audit,
                          uint8_t *pdump, int64_t row_begin, int64_t row_end);

int ifa_or_int_flash_attention(const int8_t *q, const float *sq, const int8_t *k,
                               const float *sk, const int8_t *v, float sv, int64_t n,
                               int64_t d, int64_t br_cfg, int64_t bc_cfg, uint32_t flags,
                               float *out, ifa_or_audit *audit) {
    return int_flash_impl(q, sq, k, sk, v, sv, n, d, br_cfg, bc_cfg, flags, out, audit, NULL, 0,
                          n);
}

int ifa_or_int_flash_attention_rows(const int8_t *q, const float *sq, const int8_t *k,
                                    const float *sk, const int8_t *v, float sv, int64_t n,
                                    int64_t d, int64_t br_cfg, int64_t bc_cfg, uint32_t flags,
                                    int64_t row_begin, int64_t row_end, float *out) {
    if (br_cfg < 1 || row_begin < 0 || row_begin % br_cfg != 0 || row_end > n ||
        row_end < row_begin)
        return -1;
    return int_flash_impl(q, sq, k, sk, v, sv, n, d, br_cfg, bc_cfg, flags, out, NULL, NULL,
                          row_begin, row_end);
}

int ifa_or_int_flash_attention_pcodes(const int8_t *q, const float *sq, const int8_t *k,
                                      const float *sk, const int8_t *v, float sv, int64_t n,
                                      int64_t d, int64_t br_cfg, int64_t bc_cfg, uint32_t flags,
                                      float *out, uint8_t *pcodes) {
    return int_flash_impl(q, sq, k, sk, v, sv, n, d, br_cfg, bc_cfg, flags, out, NULL, pcodes, 0,
                          n);
}

static int int_flash_impl(const int8_t *q, const float *sq, const int8_t *k, const float *sk,
                          const int8_t *v, float sv, int64_t n, int64_t d, int64_t br_cfg,
                          int64_t bc_cfg, uint32_t flags, float *out, ifa_or_audit *audit,
                          uint8_t *pdump, int64_t row_begin, int64_t row_end) {
    if (n < 1 || d < 1) return -1;                      /* attention.cpp:215-218 */
    if (!(sv >= 0.0f) || !isfinite(sv)) return -1;      /* attention.cpp:230-232 */
    if (br_cfg < 1 || bc_cfg < 1) return -1;            /* gemm.cpp:16-20 */
    if (d > IFA_MAX_INT_GEMM_DEPTH) return -2;          /* attention.cpp:241 */
    if ((bc_cfg < n ? bc_cfg : n) > IFA_MAX_INT_GEMM_DEPTH) return -2; /* :242 */
    const int causal = (flags & IFA_OR_FLAG_CAUSAL) != 0;
    const float extra = (flags & IFA_OR_FLAG_SQRT_D) ? 1.0f / sqrtf((float)d) : 1.0f;

    const int64_t br_max = br_cfg < n ? br_cfg : n;
    const int64_t bc_max = bc_cfg < n ? bc_cfg : n;
    int32_t *s_int = (int32_t *)malloc(sizeof(int32_t) * br_max * bc_max);
    float *s = (float *)malloc(sizeof(float) * br_max * bc_max);
    int8_t *p = (int8_t *)malloc((size_t)(br_max * bc_max));
    uint8_t *vis = (uint8_t *)malloc((size_t)(br_max * bc_max));
    int32_t *pv = (int32_t *)malloc(sizeof(int32_t) * br_max * d);
    float *acc = (float *)malloc(sizeof(float) * br_max * d);
    float *m = (float *)malloc(sizeof(float) * br_max);
    float *l = (float *)malloc(sizeof(float) * br_max);
    uint8_t *row_hit = (uint8_t *)malloc((size_t)br_max);
    if (!s_int || !s || !p || !vis || !pv || !acc || !m || !l || !row_hit) return -3;

    if (audit) {
        audit->min_code = 127;
        audit->max_code = 0;
        audit->row_max_block_hits_127 = 1;
        audit->rows_audited = 0;
    }
    int32_t code_min = 127, code_max = 0;

    for (int64_t i0 = row_begin; i0 < row_end; i0 += br_cfg) { /* attention.cpp:267 */
        const int64_t br = (br_cfg < n - i0) ? br_cfg : n - i0;
        for (int64_t r = 0; r < br; ++r) {
            m[r] = -INFINITY;
            l[r] = 0.0f;
            row_hit[r] = 0;
        }
        memset(acc, 0, sizeof(float) * br * d);
        /* causal: blocks past the Q block's last row are fully masked (no-op) */
        const int64_t kv_end = causal ? (i0 + br) : n;
        for (int64_t j0 = 0; j0 < kv_end; j0 += bc_cfg) { /* attention.cpp:273 */
            const int64_t bc = (bc_cfg < n - j0) ? bc_cfg : n - j0;
            /* S = Q_i . K_j^T (attention.cpp:275-276, gemm.cpp:32-46) */
            for (int64_t r = 0; r < br; ++r)
                for (int64_t c = 0; c < bc; ++c) {
                    int32_t a = 0;
                    const int8_t *qr = q + (i0 + r) * d;
                    const int8_t *kc = k + (j0 + c) * d;
                    for (int64_t t = 0; t < d; ++t) a += (int32_t)qr[t] * (int32_t)kc[t];
                    s_int[r * bc + c] = a;
                    vis[r * bc + c] = (uint8_t)(!causal || (j0 + c) <= (i0 + r));
                }
            /* dequantize (attention.cpp:277-290): product of scales first */
            for (int64_t r = 0; r < br; ++r) {
                const float sqr = sq[i0 + r];
                for (int64_t c = 0; c < bc; ++c)
                    s[r * bc + c] = (float)s_int[r * bc + c] * (sqr * sk[j0 + c]);
                if (extra != 1.0f)
                    for (int64_t c = 0; c < bc; ++c) s[r * bc + c] *= extra;
            }
            /* online softmax + requantization (attention.cpp:291-327) */
            for (int64_t r = 0; r < br; ++r) {
                const float *srow = s + r * bc;
                const uint8_t *vrow = vis + r * bc;
                float m_loc = -INFINITY;
                for (int64_t c = 0; c < bc; ++c)
                    if (vrow[c] && srow[c] > m_loc) m_loc = srow[c]; /* std::max */
                const float m_new = (m[r] < m_loc) ? m_loc : m[r];
                const float alpha = expf(m[r] - m_new);
                int8_t *prow = p + r * bc;
                int32_t p_sum = 0;
                int has_full = 0;
                for (int64_t c = 0; c < bc; ++c) {
                    if (!vrow[c]) {
                        prow[c] = 0;
                        if (pdump) pdump[(i0 + r) * n + j0 + c] = 0;
                        continue;
                    }
                    const int32_t code = (int32_t)roundf(127.0f * expf(srow[c] - m_new));
                    prow[c] = (int8_t)code;
                    if (pdump) pdump[(i0 + r) * n + j0 + c] = (uint8_t)code;
                    p_sum += code;
                    has_full = has_full || code == 127;
                    if (code < code_min) code_min = code;
                    if (code > code_max) code_max = code;
                }
                l[r] = l[r] * alpha + (float)p_sum;
                float *arow = acc + r * d;
                for (int64_t c = 0; c < d; ++c) arow[c] *= alpha;
                if (m_new > m[r])
                    row_hit[r] = has_full ? 1 : 0;
                else if (m_loc == m_new && has_full)
                    row_hit[r] = 1;
                m[r] = m_new;
            }
            /* PV = P . V_j (attention.cpp:328-329, gemm.cpp:48-63), then acc += float(pv) */
            for (int64_t r = 0; r < br; ++r) {
                int32_t *orow = pv + r * d;
                memset(orow, 0, sizeof(int32_t) * d);
                for (int64_t t = 0; t < bc; ++t) {
                    const int32_t av = p[r * bc + t];
                    const int8_t *vt = v + (j0 + t) * d;
                    for (int64_t c = 0; c < d; ++c) orow[c] += av * (int32_t)vt[c];
                }
            }
            for (int64_t idx = 0; idx < br * d; ++idx) acc[idx] += (float)pv[idx];
        }
        for (int64_t r = 0; r < br; ++r) { /* attention.cpp:335-342 */
            const float lr = l[r];
            for (int64_t c = 0; c < d; ++c) out[(i0 + r) * d + c] = (acc[r * d + c] / lr) * sv;
        }
        if (audit) { /* attention.cpp:343-350 */
            audit->rows_audited += br;
            for (int64_t r = 0; r < br; ++r)
                audit->row_max_block_hits_127 = audit->row_max_block_hits_127 && row_hit[r] != 0;
        }
    }
    if (audit) {
        audit->min_code = code_min;
        audit->max_code = code_max;
    }
    free(s_int);
    free(s);
    free(p);
    free(vis);
    free(pv);
    free(acc);
    free(m);
    free(l);
    free(row_hit);
    return 0;
}

typedef struct {
    const int8_t *q, *k, *v;
    const float *sq, *sk, *sv;
    int64_t slices, n, d, br, bc;
    uint32_t flags;
    float *out;
    int64_t next; /* atomic work counter */
    int status;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *job = (batch_job *)arg;
    const int64_t nd = job->n * job->d;
    for (;;) {
        const int64_t s = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
        if (s >= job->slices) break;
        const int rc = ifa_or_int_flash_attention(
            job->q + s * nd, job->sq + s * job->n, job->k + s * nd, job->sk + s * job->n,
            job->v + s * nd, job->sv[s], job->n, job->d, job->br, job->bc, job->flags,
            job->out + s * nd, NULL);
        if (rc) __atomic_store_n(&job->status, rc, __ATOMIC_RELAXED);
    }
    return NULL;
}

int ifa_or_int_flash_attention_batched(const int8_t *q, const float *sq, const int8_t *k,
                                       const float *sk, const int8_t *v, const float *sv,
                                       int64_t slices, int64_t n, int64_t d, int64_t br,
                                       int64_t bc, uint32_t flags, float *out, int threads) {
    batch_job job = {q, k, v, sq, sk, sv, slices, n, d, br, bc, flags, out, 0, 0};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    int started = 0;
    for (int t = 1; t < threads; ++t)
        if (pthread_create(&tid[started], NULL, batch_worker, &job) == 0) ++started;
    batch_worker(&job);
    for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
    return job.status;
}

/* ------------------------------------------------------------------ */
/* oracles.cpp:83-134 untiled integer attention (+ causal)              */
/* ------------------------------------------------------------------ */
/* half-INT8 attention (attention.cpp:359-399): integer scores scaled by
 * the per-row Q/K scales, then the float tiled flash path
 * (tiled_float_attention :49-80, merge_softmax_state :91-137,
 * finalize_softmax_state :139-149) on float V.  Every float expression in
 * the reference's order; -ffp-contract=off (no FMA), like the reference's
 * build.  No causal mode (the reference has none; this build's GPU
 * half-INT8 kernel refuses it too). */
int ifa_or_half_int8_attention(const int8_t *q, const float *sq, const int8_t *k,
                               const float *sk, const float *v, int64_t n, int64_t d,
                               int64_t br_cfg, int64_t bc_cfg, uint32_t flags, float *out) {
    if (n < 1 || d < 1) return -1;                       /* :372-374 */
    if (br_cfg < 1 || bc_cfg < 1) return -1;             /* cfg.validate() */
    if (d > IFA_MAX_INT_GEMM_DEPTH) return -2;           /* :375 */
    const float extra = (flags & IFA_OR_FLAG_SQRT_D) ? 1.0f / sqrtf((float)d) : 1.0f;
    const int64_t br_max = br_cfg < n ? br_cfg : n;
    const int64_t bc_max = bc_cfg < n ? bc_cfg : n;
    float *s = (float *)malloc(sizeof(float) * br_max * bc_max);
    float *p = (float *)malloc(sizeof(float) * br_max * bc_max);
    float *acc = (float *)malloc(sizeof(float) * br_max * d);
    float *m = (float *)malloc(sizeof(float) * br_max);
    float *l = (float *)malloc(sizeof(float) * br_max);
    if (!s || !p || !acc || !m || !l) return -3;
    for (int64_t i0 = 0; i0 < n; i0 += br_cfg) {
        const int64_t br = (br_cfg < n - i0) ? br_cfg : n - i0;
        for (int64_t r = 0; r < br; ++r) {
            m[r] = -INFINITY;
            l[r] = 0.0f;
        }
        memset(acc, 0, sizeof(float) * br * d);
        for (int64_t j0 = 0; j0 < n; j0 += bc_cfg) {
            const int64_t bc = (bc_cfg < n - j0) ? bc_cfg : n - j0;
            /* fill (:378-394): s = float(S_int) * (sq * sk) [*= extra] */
            for (int64_t r = 0; r < br; ++r) {
                const float sqr = sq[i0 + r];
                for (int64_t c = 0; c < bc; ++c) {
                    int32_t a = 0;
                    const int8_t *qr = q + (i0 + r) * d;
                    const int8_t *kc = k + (j0 + c) * d;
                    for (int64_t t = 0; t < d; ++t) a += (int32_t)qr[t] * (int32_t)kc[t];
                    s[r * bc + c] = (float)a * (sqr * sk[j0 + c]);
                }
                if (extra != 1.0f)
                    for (int64_t c = 0; c < bc; ++c) s[r * bc + c] *= extra;
            }
            /* merge_softmax_state (:114-136) */
            for (int64_t r = 0; r < br; ++r) {
                float m_loc = -INFINITY;
                for (int64_t c = 0; c < bc; ++c)
                    m_loc = (m_loc < s[r * bc + c]) ? s[r * bc + c] : m_loc;
                const float m_new = (m[r] < m_loc) ? m_loc : m[r];
                const float alpha = ifa_or_expf(m[r] - m_new);
                float row_sum = 0.0f;
                for (int64_t c = 0; c < bc; ++c) {
                    const float e = ifa_or_expf(s[r * bc + c] - m_new);
                    p[r * bc + c] = e;
                    row_sum += e;
                }
                l[r] = l[r] * alpha + row_sum;
                for (int64_t c = 0; c < d; ++c) acc[r * d + c] *= alpha;
                m[r] = m_new;
            }
            /* float_gemm_nn_acc_strided (gemm.cpp:80-95) */
            for (int64_t r = 0; r < br; ++r)
                for (int64_t t = 0; t < bc; ++t) {
                    const float av = p[r * bc + t];
                    const float *bt = v + (j0 + t) * d;
                    for (int64_t c = 0; c < d; ++c) acc[r * d + c] += av * bt[c];
                }
        }
        /* finalize_softmax_state (:139-149) */
        for (int64_t r = 0; r < br; ++r) {
            const float inv = 1.0f / l[r];
            for (int64_t c = 0; c < d; ++c) out[(i0 + r) * d + c] = acc[r * d + c] * inv;
        }
    }
    free(s);
    free(p);
    free(acc);
    free(m);
    free(l);
    return 0;
}

int ifa_or_untiled_int8_attention(const int8_t *q, const float *sq, const int8_t *k,
                                  const float *sk, const int8_t *v, float sv, int64_t n,
                                  int64_t d, uint32_t flags, float *out) {
    if (n < 1 || d < 1) return -1;
    if (!(sv >= 0.0f) || !isfinite(sv)) return -1;
    const int causal = (flags & IFA_OR_FLAG_CAUSAL) != 0;
    const float extra = (flags & IFA_OR_FLAG_SQRT_D) ? 1.0f / sqrtf((float)d) : 1.0f;
    float *s = (float *)malloc(sizeof(float) * n);
    int32_t *codes = (int32_t *)malloc(sizeof(int32_t) * n);
    if (!s || !codes) return -3;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t cend = causal ? i + 1 : n;
        const float sqi = sq[i];
        for (int64_t c = 0; c < cend; ++c) {
            int64_t a = 0;
            for (int64_t t = 0; t < d; ++t) a += (int64_t)q[i * d + t] * (int64_t)k[c * d + t];
            s[c] = (float)(int32_t)a * (sqi * sk[c]);
        }
        if (extra != 1.0f)
            for (int64_t c = 0; c < cend; ++c) s[c] *= extra;
        float row_max = -INFINITY;
        for (int64_t c = 0; c < cend; ++c) row_max = (row_max < s[c]) ? s[c] : row_max;
        int32_t l = 0;
        for (int64_t c = 0; c < cend; ++c) {
            codes[c] = (int32_t)roundf(127.0f * expf(s[c] - row_max));
            l += codes[c];
        }
        const float lf = (float)l;
        for (int64_t col = 0; col < d; ++col) {
            int64_t a = 0;
            for (int64_t c = 0; c < cend; ++c) a += (int64_t)codes[c] * (int64_t)v[c * d + col];
            out[i * d + col] = ((float)(int32_t)a / lf) * sv;
        }
    }
    free(s);
    free(codes);
    return 0;
}

/* ------------------------------------------------------------------ */
/* attention.cpp:151-192 fp64 reference (+ causal)                      */
/* ------------------------------------------------------------------ */
int ifa_or_reference_attention(const float *q, const float *k, const float *v, int64_t n,
                               int64_t m, int64_t d, int64_t dv, uint32_t flags, float *out) {
    if (n < 1 || d < 1 || dv < 1) return -1;
    const int causal = (flags & IFA_OR_FLAG_CAUSAL) != 0;
    const double scale = (flags & IFA_OR_FLAG_SQRT_D) ? 1.0 / sqrt((double)d) : 1.0;
    double *s = (double *)malloc(sizeof(double) * m);
    double *acc = (double *)malloc(sizeof(double) * dv);
    if (!s || !acc) return -3;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t jend = causal ? (i + 1 < m ? i + 1 : m) : m;
        double row_max = -INFINITY;
        for (int64_t j = 0; j < jend; ++j) {
            double dot = 0.0;
            for (int64_t t = 0; t < d; ++t) dot += (double)q[i * d + t] * (double)k[j * d + t];
            s[j] = dot * scale;
            row_max = (row_max < s[j]) ? s[j] : row_max;
        }
        for (int64_t c = 0; c < dv; ++c) acc[c] = 0.0;
        double l = 0.0;
        for (int64_t j = 0; j < jend; ++j) {
            const double w = exp(s[j] - row_max);
            l += w;
            for (int64_t c = 0; c < dv; ++c) acc[c] += w * (double)v[j * dv + c];
        }
        for (int64_t c = 0; c < dv; ++c) out[i * dv + c] = (float)(acc[c] / l);
    }
    free(s);
    free(acc);
    return 0;
}

void ifa_or_error_accum(const float *reference, const float *candidate, int64_t count,
                        double *num, double *den) {
    double nu = *num, de = *den; /* eval.cpp:55-75 */
    for (int64_t i = 0; i < count; ++i) {
        nu += fabs((double)candidate[i] - (double)reference[i]);
        de += fabs((double)reference[i]);
    }
    *num = nu;
    *den = de;
}

uint64_t ifa_or_fnv1a64(const void *data, int64_t nbytes) {
    const uint8_t *p = (const uint8_t *)data;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* ------------------------------------------------------------------ */
/* Decision boundaries of the weight code (attention.cpp:306-307)       */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t lo, hi; /* bit-pattern range [lo, hi) of negative floats */
    int first_code, last_code, monotone;
    float bounds[127];
    int have[127];
} code_scan;

static void *code_scan_worker(void *arg) {
    code_scan *cs = (code_scan *)arg;
    int prev = -1;
    cs->monotone = 1;
    for (int k = 0; k < 127; ++k) cs->have[k] = 0;
    /* walk x upwards: bit patterns of negative floats decrease as x grows */
    for (uint32_t b = cs->hi; b-- > cs->lo;) {
        float x;
        memcpy(&x, &b, 4);
        const int code = (int)roundf(127.0f * expf(x));
        if (prev >= 0) {
            if (code < prev) cs->monotone = 0;
            for (int k = prev; k < code; ++k) { /* crossed boundary k -> k+1 */
                cs->bounds[k] = x;
                cs->have[k] = 1;
            }
        } else {
            cs->first_code = code;
        }
        prev = code;
    }
    cs->last_code = prev;
    return NULL;
}

int ifa_or_code_bounds_exhaustive(float *out, int threads) {
    const uint32_t lo = 0x80000000u, hi = 0xC2D00001u; /* -0 .. -104 inclusive */
    if (threads < 1) threads = 1;
    if (threads > 64) threads = 64;
    code_scan *cs = (code_scan *)calloc((size_t)threads, sizeof(code_scan));
    pthread_t tid[64];
    const uint32_t span = (hi - lo + (uint32_t)threads - 1) / (uint32_t)threads;
    for (int t = 0; t < threads; ++t) {
        cs[t].lo = lo + (uint32_t)t * span;
        cs[t].hi = cs[t].lo + span < hi ? cs[t].lo + span : hi;
        pthread_create(&tid[t], NULL, code_scan_worker, &cs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    /* chunk t covers larger (more negative) x for larger t; stitch from the
     * most negative chunk upwards */
    int mono = 1, prev = -1;
    for (int k = 0; k < 127; ++k) out[k] = 0.0f;
    for (int t = threads - 1; t >= 0; --t) {
        if (!cs[t].monotone) mono = 0;
        if (prev >= 0) {
            if (cs[t].first_code < prev) mono = 0;
            /* boundary crossed exactly at this chunk's first (most negative) x */
            float x0;
            uint32_t b0 = cs[t].hi - 1;
            memcpy(&x0, &b0, 4);
            for (int k = prev; k < cs[t].first_code; ++k) out[k] = x0;
        }
        for (int k = 0; k < 127; ++k)
            if (cs[t].have[k]) out[k] = cs[t].bounds[k];
        prev = cs[t].last_code;
    }
    free(cs);
    return mono;
}


/* ------------------------------------------------------------------ fp8 (f3)
 * fp8.cpp:17-24 round_ties_even on an exact double quotient. */
static int64_t or_round_ties_even(double v) {
    const double fl = floor(v);
    const double diff = v - fl;
    const int64_t n = (int64_t)fl;
    if (diff > 0.5) return n + 1;
    if (diff < 0.5) return n;
    return (n % 2 == 0) ? n : n + 1;
}

/* fp8.cpp:28-57 */
uint8_t ifa_or_e4m3_encode(float x) {
    const uint8_t sign = signbit(x) ? 0x80 : 0x00;
    if (isnan(x)) return sign | 0x7f;
    const double a = fabs((double)x);
    if (a == 0.0) return sign;
    if (a > 448.0) return sign | 0x7e;
    int e = ilogb(a);
    if (e < -6) e = -6;
    int64_t q = or_round_ties_even(ldexp(a, -(e - 3)));
    if (e == -6 && q < 8) return sign | (uint8_t)q;
    if (q == 16) {
        e += 1;
        q = 8;
    }
    return sign | (uint8_t)((uint8_t)(e + 7) << 3) | (uint8_t)(q - 8);
}

/* fp8.cpp:59-72 */
float ifa_or_e4m3_decode(uint8_t bits) {
    const int exp_field = (bits >> 3) & 0xf;
    const int mant = bits & 0x7;
    if (exp_field == 0xf && mant == 0x7) return NAN;
    double v;
    if (exp_field == 0)
        v = ldexp((double)mant / 8.0, -6);
    else
        v = ldexp(1.0 + (double)mant / 8.0, exp_field - 7);
    return (float)((bits & 0x80) ? -v : v);
}

/* fp8.cpp:78-97 */
int ifa_or_fp8_roundtrip(const float *x, int64_t count, float *out, uint8_t *codes, float *scale) {
    float max_abs = 0.0f;
    for (int64_t i = 0; i < count; ++i) {
        if (!isfinite(x[i])) return -1;
        const float a = fabsf(x[i]);
        max_abs = max_abs < a ? a : max_abs;
    }
    if (max_abs == 0.0f) {
        for (int64_t i = 0; i < count; ++i) {
            out[i] = 0.0f;
            if (codes) codes[i] = 0;
        }
        if (scale) *scale = 0.0f;
        return 0;
    }
    const float s = 448.0f / max_abs;
    for (int64_t i = 0; i < count; ++i) {
        const uint8_t c = ifa_or_e4m3_encode(x[i] * s);
        out[i] = ifa_or_e4m3_decode(c) / s;
        if (codes) codes[i] = c;
    }
    if (scale) *scale = s;
    return 0;
}

/* attention.cpp:401-407 -> flash_attention_float (:194-211) over the
 * roundtripped matrices; tiled_float_attention / merge_softmax_state /
 * finalize_softmax_state as in ifa_or_half_int8_attention above. */
int ifa_or_fp8_attention(const float *q, const float *k, const float *v, int64_t n, int64_t d,
                         int64_t br_cfg, int64_t bc_cfg, uint32_t flags, float *out) {
    if (n < 1 || d < 1) return -1;
    if (br_cfg < 1 || bc_cfg < 1) return -1;
    const int64_t cnt = n * d;
    float *qr = (float *)malloc(sizeof(float) * cnt);
    float *kr = (float *)malloc(sizeof(float) * cnt);
    float *vr = (float *)malloc(sizeof(float) * cnt);
    if (!qr || !kr || !vr) return -3;
    if (ifa_or_fp8_roundtrip(q, cnt, qr, NULL, NULL) || ifa_or_fp8_roundtrip(k, cnt, kr, NULL, NULL) ||
        ifa_or_fp8_roundtrip(v, cnt, vr, NULL, NULL)) {
        free(qr);
        free(kr);
        free(vr);
        return -1;
    }
    const float extra = (flags & IFA_OR_FLAG_SQRT_D) ? 1.0f / sqrtf((float)d) : 1.0f;
    const int64_t br_max = br_cfg < n ? br_cfg : n;
    const int64_t bc_max = bc_cfg < n ? bc_cfg : n;
    float *s = (float *)malloc(sizeof(float) * br_max * bc_max);
    float *p = (float *)malloc(sizeof(float) * br_max * bc_max);
    float *acc = (float *)malloc(sizeof(float) * br_max * d);
    float *m = (float *)malloc(sizeof(float) * br_max);
    float *l = (float *)malloc(sizeof(float) * br_max);
    if (!s || !p || !acc || !m || !l) return -3;
    for (int64_t i0 = 0; i0 < n; i0 += br_cfg) {
        const int64_t br = (br_cfg < n - i0) ? br_cfg : n - i0;
        for (int64_t r = 0; r < br; ++r) {
            m[r] = -INFINITY;
            l[r] = 0.0f;
        }
        memset(acc, 0, sizeof(float) * br * d);
        for (int64_t j0 = 0; j0 < n; j0 += bc_cfg) {
            const int64_t bc = (bc_cfg < n - j0) ? bc_cfg : n - j0;
            /* fill (:200-210): float_gemm_nt_strided (gemm.cpp:65-78) [*= extra] */
            for (int64_t r = 0; r < br; ++r)
                for (int64_t c = 0; c < bc; ++c) {
                    const float *a = qr + (i0 + r) * d;
                    const float *b = kr + (j0 + c) * d;
                    float accd = 0.0f;
                    for (int64_t t = 0; t < d; ++t) accd += a[t] * b[t];
                    s[r * bc + c] = accd;
                }
            if (extra != 1.0f)
                for (int64_t idx = 0; idx < br * bc; ++idx) s[idx] *= extra;
            for (int64_t r = 0; r < br; ++r) {
                float m_loc = -INFINITY;
                for (int64_t c = 0; c < bc; ++c)
                    m_loc = (m_loc < s[r * bc + c]) ? s[r * bc + c] : m_loc;
                const float m_new = (m[r] < m_loc) ? m_loc : m[r];
                const float alpha = ifa_or_expf(m[r] - m_new);
                float row_sum = 0.0f;
                for (int64_t c = 0; c < bc; ++c) {
                    const float e = ifa_or_expf(s[r * bc + c] - m_new);
                    p[r * bc + c] = e;
                    row_sum += e;
                }
                l[r] = l[r] * alpha + row_sum;
                for (int64_t c = 0; c < d; ++c) acc[r * d + c] *= alpha;
                m[r] = m_new;
            }
            for (int64_t r = 0; r < br; ++r)
                for (int64_t t = 0; t < bc; ++t) {
                    const float av = p[r * bc + t];
                    const float *bt = vr + (j0 + t) * d;
                    for (int64_t c = 0; c < d; ++c) acc[r * d + c] += av * bt[c];
                }
        }
        for (int64_t r = 0; r < br; ++r) {
            const float inv = 1.0f / l[r];
            for (int64_t c = 0; c < d; ++c) out[(i0 + r) * d + c] = acc[r * d + c] * inv;
        }
    }
    free(s);
    free(p);
    free(acc);
    free(m);
    free(l);
    free(qr);
    free(kr);
    free(vr);
    return 0;
}
