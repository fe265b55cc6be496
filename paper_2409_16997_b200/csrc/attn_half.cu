// attn_half.cu -- half-INT8 attention forward for sm_100a (SURVEY.md §8(f)
// row f1; reference ifa::half_int8_attention, attention.cpp:359-399).
//
// Q and K are int8 with per-row scales exactly as in the full-INT8 path, so
// S = Q.K^T is the same exact int32 tcgen05.mma kind::i8 product; V stays a
// float tensor and the attention weights stay float:
//   s = float(S) * (sQ*sK) [* 1/sqrt(d)]   p = exp(s - m')   l = l*alpha + sum p
//   acc = acc*alpha + P.V                   O = acc * (1/l)
// The weights go to the tensor core as fp16 (p in [0,1]) against an fp16
// copy of V (ifa_convert_f16), accumulating in fp32 in TMEM
// (tcgen05.mma kind::f16, A = P from TMEM, B = V from SMEM MN-major, two
// 64-column SW128 halves); l is the tensor core's row sum of the same fp16
// weights (P.1), so numerator and denominator see identical rounding.
// Tolerance semantics (tests/test_gpu_half.py): O within 2e-3 MRE of the
// reference, and its error against fp64 matches the reference's to
// within 1% relative.  The KV block size only changes float rounding
// order here (no requantization), so every Bc maps onto 128-key tiles.
//
// Warp roles as the full-INT8 kernel (attn.cu): 0 TMA producer (Q double-
// buffered, a 3-stage ring of int8 K + fp16 V + K scales), 1 TMEM allocator
// + single-thread MMA issuer (S(i+1) before P.V(i)), 4-19 softmax +
// correction (four threads per row, 32 columns each, f32 accumulator in
// registers).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ifa_internal.h"
#include "ptx.cuh"

namespace ifa_b200 {
namespace halfk {

using namespace ptx;

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int STAGES = 3;
constexpr int SPLIT = 4;
constexpr int NCOL = BN / SPLIT;
constexpr int SOFT_WARP0 = 4;
constexpr int SOFT_WARPS = 4 * SPLIT;
constexpr int NUM_THREADS = 32 * (SOFT_WARP0 + SOFT_WARPS);
constexpr uint32_t kRegsControl = 32;
constexpr uint32_t kRegsSoftmax = 112;
constexpr uint32_t TMEM_COLS = 512;
// S [0,128) | PV [128,128+D) | rowsum [256,272) | P0 [288,352) | P1 [352,416)
constexpr uint32_t T_S = 0, T_PV = 128, T_RS = 256, T_P0 = 288;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct alignas(1024) Smem {
    uint8_t q[2][BM * D];
    uint8_t k[STAGES][BN * D];
    uint8_t v[STAGES][BN * D * 2];  // fp16, [D/64 halves][BN keys][64 columns], SW128
    uint16_t ones[16 * 64];         // fp16 1.0: 16 rows x 128 B (P.1 row sums)
    float sk[STAGES][BN];
    float xmax[2][BM][SPLIT];
    uint64_t q_full[2], q_empty[2];
    uint64_t k_full[STAGES], v_full[STAGES], kv_empty[STAGES];
    uint64_t s_full, s_empty;
    uint64_t p_full[2], p_empty[2];
    uint64_t pv_full, pv_empty;
    uint32_t tmem_base;
};

struct Params {
    const float* sq;  // half-INT8: per row [slices][n]; FP8: per slice [slices]
    const float* sk;  // likewise
    const float* sv;  // FP8: V roundtrip scale per slice (O /= sV); half-INT8: unused
    float* o;
    int32_t n, d;
    float sk_mul;  // log2(e) [* 1/sqrt(d)]: K scales staged pre-multiplied
    int32_t q_tiles, slices, items;
};

template <int N>
struct Ring {
    uint32_t idx = 0, phase = 0;
    __device__ __forceinline__ void advance() {
        if (++idx == N) {
            idx = 0;
            phase ^= 1u;
        }
    }
};

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// Instruction descriptor for kind::f16: D=F32, A=B=F16.
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t m, uint32_t n, bool b_mn_major) {
    return (1u << 4) | ((b_mn_major ? 1u : 0u) << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 2^t on the FMA pipe (degree-5 polynomial, 3.5e-7 relative), t >= -64.
__device__ __forceinline__ float2 exp2_poly2(float2 t) {
    constexpr float kMagic = 12582912.0f;
    t.x = fmaxf(t.x, -64.0f);
    t.y = fmaxf(t.y, -64.0f);
    const float2 r = fadd2(t, f2(kMagic));
    const float2 f = fsub2(t, fsub2(r, f2(kMagic)));
    float2 y = ffma2(f, f2(1.2915651313960552e-3f), f2(9.668535552918911e-3f));
    y = ffma2(y, f, f2(5.5516887456178665e-2f));
    y = ffma2(y, f, f2(2.4022264778614044e-1f));
    y = ffma2(y, f, f2(6.931464672088623e-1f));
    y = ffma2(y, f, f2(1.0f));
    return make_float2(__int_as_float(__float_as_int(y.x) + (__float_as_int(r.x) << 23)),
                       __int_as_float(__float_as_int(y.y) + (__float_as_int(r.y) << 23)));
}

__device__ __forceinline__ float ex2(float t) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
    return r;
}

__device__ __forceinline__ void mma_f8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// FP8 = false: half-INT8 (int8 Q/K codes, per-row scales, S via kind::i8).
// FP8 = true : SURVEY §8(f) f3, fp8_emulated_attention (attention.cpp:401-
// 407): e4m3 Q/K codes with one scale per slice (fp8.cpp:78-97), S via
// tcgen05.mma kind::f8f6f4 (f32 accumulate), V = the decoded e4m3 values as
// fp16 (exact), O divided by the V scale at the end.
template <int D, bool FP8>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    half_int8_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const Params p) {
    constexpr uint32_t kLayout = D == 128 ? kLayoutSw128 : kLayoutSw64;
    constexpr uint32_t kSbo = 8 * D;
    constexpr uint32_t kKBytes = BN * D;
    constexpr uint32_t kVBytes = BN * D * 2;
    // kind::f8f6f4: D = F32 (bit 4), A = B = E4M3 (format fields 0)
    constexpr uint32_t kIdescS =
        FP8 ? ((1u << 4) | ((BN >> 3) << 17) | ((BM >> 4) << 24)) : idesc_i8(BM, BN, false, false);
    constexpr uint32_t kIdescPV = idesc_f16(BM, D, true);
    constexpr uint32_t kIdescSum = idesc_f16(BM, 16, false);
    const float kNegInf = -__int_as_float(0x7f800000);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const int32_t n = p.n;

    const uint32_t b_q_full = smem_u32(&sm.q_full[0]), b_q_empty = smem_u32(&sm.q_empty[0]);
    const uint32_t b_k_full = smem_u32(&sm.k_full[0]), b_v_full = smem_u32(&sm.v_full[0]);
    const uint32_t b_kv_empty = smem_u32(&sm.kv_empty[0]);
    const uint32_t b_s_full = smem_u32(&sm.s_full), b_s_empty = smem_u32(&sm.s_empty);
    const uint32_t b_p_full = smem_u32(&sm.p_full[0]), b_p_empty = smem_u32(&sm.p_empty[0]);
    const uint32_t b_pv_full = smem_u32(&sm.pv_full), b_pv_empty = smem_u32(&sm.pv_empty);

    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023) __trap();
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.q_full[i], 1);
            mbar_init(&sm.q_empty[i], 1);
            mbar_init(&sm.p_full[i], SOFT_WARPS);
            mbar_init(&sm.p_empty[i], 1);
        }
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&sm.k_full[i], 32);
            mbar_init(&sm.v_full[i], 1);
            mbar_init(&sm.kv_empty[i], 1 + SOFT_WARPS);
        }
        mbar_init(&sm.s_full, 1);
        mbar_init(&sm.s_empty, SOFT_WARPS);
        mbar_init(&sm.pv_full, 1);
        mbar_init(&sm.pv_empty, SOFT_WARPS);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) sm.ones[i] = 0x3C00u;  // 1.0h
    fence_proxy_async_shared();
    if (warp == 1) tmem_alloc<TMEM_COLS>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp < SOFT_WARP0) {
        regs_dealloc<kRegsControl>();
        if (warp == 0) {
            // ------------------------------------------------------- producer
            const uint64_t pol_stream = policy_evict_first();
            const uint64_t pol_keep = policy_evict_last();
            Ring<STAGES> kv;
            uint32_t i = 0, wi = 0;
            for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x, ++wi) {
                const int32_t q0 = (idx % p.q_tiles) * BM, slice = idx / p.q_tiles;
                const uint32_t qb = wi & 1;
                if (lane == 0) {
                    if (wi >= 2) bar_wait(b_q_empty + 8 * qb, ((wi >> 1) - 1) & 1);
                    mbar_arrive_expect_tx(&sm.q_full[qb], BM * D);
                    tma_load_3d(sm.q[qb], &tm_q, &sm.q_full[qb], 0, q0, slice, pol_stream);
                }
                const float* sk_slice = p.sk + static_cast<int64_t>(slice) * n;
                // FP8: s = S / (sQ sK) for every key of the slice
                // all-zero Q or K slice: scale 0, codes 0, scores 0 (fp8.cpp:78-97)
                const float sqk = FP8 ? __fmul_rn(p.sq[slice], p.sk[slice]) : 0.0f;
                const float c8 = FP8 && sqk != 0.0f ? __fdiv_rn(p.sk_mul, sqk) : 0.0f;
                for (int32_t key0 = 0; key0 < n; key0 += BN) {
                    const uint32_t st = kv.idx;
                    if (i >= STAGES) bar_wait(b_kv_empty + 8 * st, kv.phase ^ 1u);
                    float4 kv4;
                    const int32_t key = key0 + lane * 4;
                    if constexpr (FP8) {
                        kv4.x = key + 0 < n ? c8 : 0.0f;
                        kv4.y = key + 1 < n ? c8 : 0.0f;
                        kv4.z = key + 2 < n ? c8 : 0.0f;
                        kv4.w = key + 3 < n ? c8 : 0.0f;
                    } else {
                        kv4.x = key + 0 < n ? sk_slice[key + 0] * p.sk_mul : 0.0f;
                        kv4.y = key + 1 < n ? sk_slice[key + 1] * p.sk_mul : 0.0f;
                        kv4.z = key + 2 < n ? sk_slice[key + 2] * p.sk_mul : 0.0f;
                        kv4.w = key + 3 < n ? sk_slice[key + 3] * p.sk_mul : 0.0f;
                    }
                    reinterpret_cast<float4*>(sm.sk[st])[lane] = kv4;
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&sm.k_full[st], kKBytes);
                        tma_load_3d(sm.k[st], &tm_k, &sm.k_full[st], 0, key0, slice, pol_keep);
                        mbar_arrive_expect_tx(&sm.v_full[st], kVBytes);
#pragma unroll
                        for (int h = 0; h < D / 64; ++h)
                            tma_load_3d(sm.v[st] + h * BN * 128, &tm_v, &sm.v_full[st], 64 * h,
                                        key0, slice, pol_keep);
                    } else {
                        bar_arrive(b_k_full + 8 * st);
                    }
                    kv.advance();
                    ++i;
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------------- MMA issuer
            if (lane == 0) {
                const uint64_t odesc = smem_desc(smem_u32(sm.ones), 16, 1024, kLayoutSw128);
                Ring<STAGES> kv;
                uint32_t i = 0, pi = 0, wi = 0;
                bool have_prev = false;
                uint32_t prev_st = 0, prev_ph = 0;
                auto issue_pv = [&](uint32_t st, uint32_t ph, uint32_t pidx) {
                    bar_wait(b_p_full + 8 * (pidx & 1), (pidx >> 1) & 1);
                    bar_wait(b_v_full + 8 * st, ph);
                    if (pidx >= 1) bar_wait(b_pv_empty, (pidx - 1) & 1);
                    tc_fence_after();
                    const uint32_t v_base = smem_u32(sm.v[st]);
                    const uint32_t p_col = T_P0 + 64 * (pidx & 1);
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk) {
                        // B = V, MN-major fp16: 16 keys x D per step; the two
                        // 64-column halves are BN*128 bytes apart (LBO)
                        const uint64_t bdesc =
                            smem_desc(v_base + kk * 16 * 128, BN * 128, 1024, kLayoutSw128);
                        mma_f16_ts(tmem + T_PV, tmem + p_col + kk * 8, bdesc, kIdescPV,
                                   kk > 0 ? 1u : 0u);
                        mma_f16_ts(tmem + T_RS, tmem + p_col + kk * 8, odesc, kIdescSum,
                                   kk > 0 ? 1u : 0u);
                    }
                    mma_commit_u32(b_p_empty + 8 * (pidx & 1));
                    mma_commit_u32(b_kv_empty + 8 * st);
                    mma_commit_u32(b_pv_full);
                };
                for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x, ++wi) {
                    const uint32_t qb = wi & 1;
                    bar_wait(b_q_full + 8 * qb, (wi >> 1) & 1);
                    tc_fence_after();
                    const uint32_t q_base = smem_u32(sm.q[qb]);
                    for (int32_t key0 = 0; key0 < n; key0 += BN) {
                        const uint32_t st = kv.idx, ph = kv.phase;
                        bar_wait(b_k_full + 8 * st, ph);
                        if (i > 0) bar_wait(b_s_empty, (i - 1) & 1);
                        tc_fence_after();
                        const uint32_t k_base = smem_u32(sm.k[st]);
#pragma unroll
                        for (int kk = 0; kk < D / 32; ++kk) {
                            const uint64_t adesc = smem_desc(q_base + kk * 32, 16, kSbo, kLayout);
                            const uint64_t bdesc = smem_desc(k_base + kk * 32, 16, kSbo, kLayout);
                            if constexpr (FP8)
                                mma_f8_ss(tmem + T_S, adesc, bdesc, kIdescS, kk > 0 ? 1u : 0u);
                            else
                                mma_i8_ss(tmem + T_S, adesc, bdesc, kIdescS, kk > 0 ? 1u : 0u);
                        }
                        mma_commit_u32(b_s_full);
                        if (have_prev) issue_pv(prev_st, prev_ph, pi++);
                        have_prev = true;
                        prev_st = st;
                        prev_ph = ph;
                        kv.advance();
                        ++i;
                    }
                    mma_commit_u32(b_q_empty + 8 * qb);
                }
                if (have_prev) issue_pv(prev_st, prev_ph, pi++);
            }
            __syncwarp();
        }
    } else {
        regs_alloc<kRegsSoftmax>();
        // ------------------------------------------------ softmax + correction
        const uint32_t quarter = warp & 3;
        const uint32_t part = (warp - SOFT_WARP0) >> 2;
        const int32_t row = static_cast<int32_t>(quarter * 32 + lane);
        const uint32_t t_lane = tmem + ((quarter * 32) << 16);
        const uint32_t t_s = t_lane + T_S + NCOL * part;
        const uint32_t t_p = t_lane + T_P0 + (NCOL / 2) * part;
        const uint32_t t_pv = t_lane + T_PV + NCOL * part;
        const uint32_t t_rs = t_lane + T_RS;
        const int32_t c_base = NCOL * part;
        const uint32_t bar_id = 1 + quarter;
        float* const xmax_mine = &sm.xmax[0][row][part];
        const float* const xmax_row = &sm.xmax[0][row][0];
        Ring<STAGES> kv;
        uint32_t i = 0, pi = 0, bi = 0;

        for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x) {
            const int32_t q0 = (idx % p.q_tiles) * BM, slice = idx / p.q_tiles;
            const int32_t grow = q0 + row;
            const bool row_ok = grow < n;
            const float sq_r =
                FP8 ? 1.0f : (row_ok ? p.sq[static_cast<int64_t>(slice) * n + grow] : 0.0f);
            float acc[NCOL];
#pragma unroll
            for (int c = 0; c < NCOL; ++c) acc[c] = 0.0f;
            float l = 0.0f, m = kNegInf, pend_alpha = 1.0f;
            bool pend = false;

            auto fold = [&](float alpha) {
                bar_wait(b_pv_full, bi & 1);
                tc_fence_after();
                uint32_t pv[NCOL];
                uint32_t rs;
                tmem_ld32(t_pv, pv);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                             : "=r"(rs)
                             : "r"(t_rs));
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(b_pv_empty);
                ++bi;
                l = __fmaf_rn(l, alpha, __uint_as_float(rs));
#pragma unroll
                for (int c = 0; c < NCOL; c += 2) {
                    const float2 a = ffma2(make_float2(acc[c], acc[c + 1]), f2(alpha),
                                           make_float2(__uint_as_float(pv[c]),
                                                       __uint_as_float(pv[c + 1])));
                    acc[c] = a.x;
                    acc[c + 1] = a.y;
                }
            };

            for (int32_t key0 = 0; key0 < n; key0 += BN) {
                const uint32_t st = kv.idx;
                bar_wait(b_s_full, i & 1);
                tc_fence_after();
                uint32_t sr[NCOL];
                tmem_ld32(t_s, sr);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(b_s_empty);
                bar_wait(b_k_full + 8 * st, kv.phase);
                // u = float(S) * (sK * log2e [* extra])  (log2 domain, before sQ)
                float u[NCOL];
                const float4* sk4 = reinterpret_cast<const float4*>(sm.sk[st] + c_base);
#pragma unroll
                for (int c4 = 0; c4 < NCOL / 4; ++c4) {
                    const float4 k4 = sk4[c4];
                    const int c = 4 * c4;
                    float2 sa, sb;  // S as f32: exact int32 (kind::i8) or f32 (kind::f8f6f4)
                    if constexpr (FP8) {
                        sa = make_float2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
                        sb = make_float2(__uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
                    } else {
                        sa = make_float2(__int2float_rn(static_cast<int32_t>(sr[c])),
                                         __int2float_rn(static_cast<int32_t>(sr[c + 1])));
                        sb = make_float2(__int2float_rn(static_cast<int32_t>(sr[c + 2])),
                                         __int2float_rn(static_cast<int32_t>(sr[c + 3])));
                    }
                    const float2 a = fmul2(sa, make_float2(k4.x, k4.y));
                    const float2 b = fmul2(sb, make_float2(k4.z, k4.w));
                    u[c] = a.x;
                    u[c + 1] = a.y;
                    u[c + 2] = b.x;
                    u[c + 3] = b.y;
                }
                __syncwarp();
                if (lane == 0) bar_arrive(b_kv_empty + 8 * st);
                const int32_t lim = (n - key0 < BN ? n - key0 : BN) - c_base;
                if (lim < NCOL) {
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) u[c] = c < lim ? u[c] : kNegInf;
                }
                float mp = fmaxf(u[0], u[1]);
#pragma unroll
                for (int c = 2; c < NCOL; c += 2) mp = fmax3(mp, u[c], u[c + 1]);
                xmax_mine[(i & 1) * SPLIT * BM] = mp;
                named_bar_sync(bar_id, 32 * SPLIT);
                const float4 x4 = *reinterpret_cast<const float4*>(xmax_row + (i & 1) * SPLIT * BM);
                const float m_loc = fmaxf(fmax3(x4.x, x4.y, x4.z), x4.w);
                const float m_new = (m < m_loc) ? m_loc : m;
                if (pi >= 2) {
                    bar_wait(b_p_empty + 8 * (pi & 1), ((pi - 2) >> 1) & 1);
                    tc_fence_after();
                }
                // p = 2^(sQ*u - sQ*m') = exp(s - m'), as fp16 pairs
                const float2 q2 = f2(sq_r), c2 = f2(-sq_r * m_new);
                uint32_t wd[NCOL / 2];
#pragma unroll
                for (int c = 0; c < NCOL; c += 8) {
                    const float2 ta = ffma2(make_float2(u[c], u[c + 1]), q2, c2);
                    const float2 tb = ffma2(make_float2(u[c + 2], u[c + 3]), q2, c2);
                    const float2 tc = ffma2(make_float2(u[c + 4], u[c + 5]), q2, c2);
                    const float2 td = ffma2(make_float2(u[c + 6], u[c + 7]), q2, c2);
                    float y[8];
                    y[0] = ex2(ta.x);
                    y[1] = ex2(ta.y);
                    y[2] = ex2(tb.x);
                    y[3] = ex2(tb.y);
                    y[4] = ex2(tc.x);
                    y[5] = ex2(tc.y);
                    const float2 yd = exp2_poly2(td);
                    y[6] = yd.x;
                    y[7] = yd.y;
                    if (lim < NCOL) {  // masked keys weigh 0 (also when sQ == 0)
#pragma unroll
                        for (int e = 0; e < 8; ++e) y[e] = c + e < lim ? y[e] : 0.0f;
                    }
#pragma unroll
                    for (int e = 0; e < 8; e += 2) wd[(c + e) >> 1] = pack_h2(y[e], y[e + 1]);
                }
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                    "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                        t_p + 64 * (pi & 1)),
                    "r"(wd[0]), "r"(wd[1]), "r"(wd[2]), "r"(wd[3]), "r"(wd[4]), "r"(wd[5]),
                    "r"(wd[6]), "r"(wd[7]), "r"(wd[8]), "r"(wd[9]), "r"(wd[10]), "r"(wd[11]),
                    "r"(wd[12]), "r"(wd[13]), "r"(wd[14]), "r"(wd[15])
                    : "memory");
                if (pend) fold(pend_alpha);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(b_p_full + 8 * (pi & 1));
                ++pi;
                pend_alpha = (m_new == m) ? 1.0f
                             : (m == kNegInf ? 0.0f : ex2(sq_r * (m - m_new)));
                m = m_new;
                pend = true;
                kv.advance();
                ++i;
            }
            fold(pend_alpha);
            // O = acc * (1/l)  (finalize_softmax_state, attention.cpp:139-149)
            if (row_ok && c_base < p.d) {
                // FP8: V was restored as decode(code) / sV (fp8.cpp:94)
                const float inv =
                    FP8 ? (p.sv[slice] == 0.0f ? 0.0f : __fdiv_rn(__fdiv_rn(1.0f, l), p.sv[slice]))
                        : __fdiv_rn(1.0f, l);
                float* orow = p.o + (static_cast<int64_t>(slice) * n + grow) * p.d + c_base;
                if (p.d % 4 == 0 && c_base + NCOL <= p.d) {
#pragma unroll
                    for (int c = 0; c < NCOL; c += 4)
                        __stcs(reinterpret_cast<float4*>(orow + c),
                               make_float4(acc[c] * inv, acc[c + 1] * inv, acc[c + 2] * inv,
                                           acc[c + 3] * inv));
                } else {
#pragma unroll
                    for (int c = 0; c < NCOL; ++c)
                        if (c_base + c < p.d) orow[c] = acc[c] * inv;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
}

__global__ void convert_f16_kernel(const float* __restrict__ x, int64_t count,
                                   __half* __restrict__ out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += stride)
        out[i] = __float2half_rn(x[i]);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    }
    return fn;
}

// [slices][n][pitch] elements; box = (box0 elements, 128 rows, 1 slice)
static bool make_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize,
                     int64_t slices, int64_t n, int64_t pitch, uint32_t box0,
                     CUtensorMapSwizzle sw) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(slices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch * esize),
                                   static_cast<cuuint64_t>(pitch * esize * n)};
    const cuuint32_t box[3] = {box0, 128u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, bool FP8>
static cudaError_t launch(const uint8_t* q, const float* sq, const uint8_t* k, const float* sk,
                          const uint16_t* v, const float* sv, float* o, int64_t slices,
                          int64_t n, int64_t d, int64_t pitch, bool sqrt_d, cudaStream_t stream) {
    CUtensorMap tq, tk, tv;
    const CUtensorMapSwizzle sw8 = D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    if (!make_map(&tq, q, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, slices, n, pitch, D, sw8) ||
        !make_map(&tk, k, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, slices, n, pitch, D, sw8) ||
        !make_map(&tv, v, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, slices, n, D, 64,
                  CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    Params p;
    p.sq = sq;
    p.sk = sk;
    p.sv = sv;
    p.o = o;
    p.n = static_cast<int32_t>(n);
    p.d = static_cast<int32_t>(d);
    p.sk_mul = kLog2e * (sqrt_d ? 1.0f / sqrtf(static_cast<float>(d)) : 1.0f);
    p.q_tiles = static_cast<int32_t>((n + BM - 1) / BM);
    p.slices = static_cast<int32_t>(slices);
    p.items = p.q_tiles * p.slices;
    const size_t smem = sizeof(Smem<D>) + 1024;
    const cudaError_t e = smem_attr_once<half_int8_fwd_kernel<D, FP8>>(smem);
    if (e != cudaSuccess) return e;
    const int sms = current_device_sms();
    const int grid = p.items < sms ? p.items : sms;
    half_int8_fwd_kernel<D, FP8><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

}  // namespace halfk

cudaError_t launch_half_int8_fwd(const int8_t* q, const float* sq, const int8_t* k,
                                 const float* sk, const uint16_t* v, float* o, int64_t slices,
                                 int64_t n, int64_t d, int64_t pitch, bool sqrt_d,
                                 cudaStream_t stream) {
    const uint8_t* q8 = reinterpret_cast<const uint8_t*>(q);
    const uint8_t* k8 = reinterpret_cast<const uint8_t*>(k);
    if (d == 64)
        return halfk::launch<64, false>(q8, sq, k8, sk, v, nullptr, o, slices, n, d, pitch, sqrt_d,
                                        stream);
    if (d == 128)
        return halfk::launch<128, false>(q8, sq, k8, sk, v, nullptr, o, slices, n, d, pitch,
                                         sqrt_d, stream);
    return cudaErrorInvalidValue;
}

cudaError_t launch_fp8_attention_fwd(const uint8_t* q, const float* q_scales, const uint8_t* k,
                                     const float* k_scales, const uint16_t* v,
                                     const float* v_scales, float* o, int64_t slices, int64_t n,
                                     int64_t d, bool sqrt_d, cudaStream_t stream) {
    if (d == 64)
        return halfk::launch<64, true>(q, q_scales, k, k_scales, v, v_scales, o, slices, n, d, d,
                                       sqrt_d, stream);
    if (d == 128)
        return halfk::launch<128, true>(q, q_scales, k, k_scales, v, v_scales, o, slices, n, d,
                                        d, sqrt_d, stream);
    return cudaErrorInvalidValue;
}

cudaError_t launch_convert_f16(const float* x, int64_t count, uint16_t* out, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    halfk::convert_f16_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        x, count, reinterpret_cast<__half*>(out));
    return cudaGetLastError();
}

}  // namespace ifa_b200
