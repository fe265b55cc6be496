// attn_ws.cu -- full-INT8 tolerance-mode forward (IFA_FLAG_FAST, every KV
// block one 128-key tile), warp-specialised with ONE softmax thread per Q row.
//
// Per block it is the reference's algorithm (attention.cpp:267-351): exact
// int32 S = Q.K^T (tcgen05.mma kind::i8 into TMEM), s = float(S) * sQ * sK,
// running row max, P codes round(127 * exp(s - m)) requantized against the
// running max, O = O * alpha + P.V, l = l * alpha + sum(codes), O * sV / l at
// the end.  As in attn_pp.cu the codes (0..127) and the V codes (-127..127)
// are exact in fp16 and every partial sum of P.V is an exact f32, so P.V runs
// as tcgen05.mma kind::f16 accumulating into an f32 O in TMEM.
//
// What is new against attn_pp.cu is the thread layout (the FlashAttention-4
// pattern on Blackwell):
//   * a CTA holds two 128-row Q tiles (groups g = 0, 1) of one slice;
//   * softmax warpgroup g (warps 4g .. 4g+3) gives each thread ONE row: a
//     32x32b tcgen05.ld hands it the row's 128 int32 scores, so the row max
//     and the row sum need no shuffles and every thread carries 128
//     independent exp2s of instruction-level parallelism;
//   * a correction warpgroup (warps 8-11) rescales the O rows in TMEM when a
//     row's max moved and runs the epilogue (O * sV / l -> HBM), so neither
//     stalls the softmax; the epilogue of item i overlaps the first tile of
//     item i+1;
//   * warp 12 is the TMA producer, warps 13 / 14 issue the MMAs of group 0 /
//     1 (one issuer per group, so neither group waits on the other's
//     progress), warp 15 only donates registers.
// The P codes go to shared memory (fp16 subnormals code * 2^-24, K-major,
// 128B swizzle) so S(j+1) can be issued as soon as the group has read S(j).
//
// TMEM (512 columns): group g has S at [256g, 256g+128) and O at
// [256g+128, 256g+128+D).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "ifa_internal.h"
#include "ptx.cuh"

namespace ifa_b200 {
namespace ws {

using namespace ptx;

constexpr int BM = 128;
constexpr int BN = 128;
#ifndef IFA_WS_KST
#define IFA_WS_KST 2
#endif
#ifndef IFA_WS_VST
#define IFA_WS_VST 2
#endif
constexpr int KST = IFA_WS_KST;  // K tiles (+ K scales) in flight
constexpr int VST = IFA_WS_VST;  // fp16 V tiles in flight
constexpr int NUM_THREADS = 512;
constexpr uint32_t kWarpProducer = 12, kWarpMma = 13;  // correction: warps 8-11
// setmaxnreg inside the 512 x 128 launch pool:
// 2 * 128 * 192 + 128 * 96 + 128 * 32 = 65536
#ifndef IFA_WS_REGS_SOFTMAX
#define IFA_WS_REGS_SOFTMAX 192
#endif
constexpr uint32_t kRegsSoftmax = IFA_WS_REGS_SOFTMAX;
constexpr uint32_t kRegsCtrl = 32;
constexpr uint32_t kRegsCorr = 512 - 2 * kRegsSoftmax - kRegsCtrl;
static_assert(2 * kRegsSoftmax + kRegsCorr + kRegsCtrl == 512, "register pool");
constexpr uint32_t TMEM_COLS = 512;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr float kLog2_127 = 6.9886846867721655f;
// exp2 of every IFA_WS_POLY_EVERY-th key pair on the FMA pipe (0: all MUFU)
#ifndef IFA_WS_POLY_EVERY
#define IFA_WS_POLY_EVERY 0
#endif
constexpr int kPolyEvery = IFA_WS_POLY_EVERY;
// S accumulates onto 0x4B400000 in TMEM: the int32 result's bits are the
// float 1.5 * 2^23 + S, so float(S) is one exact packed subtract (no integer
// add per element).
//   1: the softmax warps write the constant back after reading S (measured
//      slower, C2 1.09 -> 1.38 ms: 64 KiB of tcgen05.st per tile on the math
//      warps);
//   2: the MMA-issuing thread refills the S columns with tcgen05.cp from a
//      4 KiB constant block in shared memory right before the S MMAs (the
//      tensor core's queue runs them in order; no math-warp work).
#ifndef IFA_WS_MAGIC_S
#define IFA_WS_MAGIC_S 0
#endif
constexpr uint32_t kMagicS = IFA_WS_MAGIC_S;
constexpr uint32_t kMagicSoft = kMagicS == 1 ? 1u : 0u;  // softmax-side fill
// float(S) by I2F (quarter-rate pipe of its own) instead of the integer
// magic add + packed subtract
#ifndef IFA_WS_I2F
#define IFA_WS_I2F 0
#endif
// see the code loop: how far (in key pairs) the exp2 run ahead of their use
#ifndef IFA_WS_MUFU_LAG
#define IFA_WS_MUFU_LAG 8
#endif
// softmax -> correction messages through named barriers (a warp blocked in
// bar.sync takes no issue slots; the mbarrier wait of the correction warps
// polls ~170 times per tile, ~870 issue slots) instead of mbarriers.
// Measured: -18% instructions but 1.092 -> 1.130 ms at C2, so off.
#ifndef IFA_WS_NAMED_MSG
#define IFA_WS_NAMED_MSG 0
#endif
constexpr bool kNamedMsg = IFA_WS_NAMED_MSG != 0;
// named barrier ids: 1, 2 group ping-pong; 3 + 2g + slot message full;
// 7 + 2g + slot message empty (softmax warpgroup g + correction warpgroup)
__host__ __device__ constexpr uint32_t msg_full_id(uint32_t g, uint32_t slot) { return 3 + 2 * g + slot; }
__host__ __device__ constexpr uint32_t msg_empty_id(uint32_t g, uint32_t slot) { return 7 + 2 * g + slot; }
// Cold-code skipping (see attn_pp.cu IFA_PP_SPARSE): in the one-row-per-
// thread layout the exp2 phase is MUFU-bound (tools/microbench/code_loop.cu:
// 1194 clk per 128-key row, floor 1024), and a MUFU warp-instruction costs
// its pipe time even with every lane off, so whole 8-key chunks are skipped
// by a warp vote when none of the warp's 32 rows needs a nonzero code
// there.  Used when at most IFA_WS_SPARSE_HOT rows of the warp reach t > -1
// in this block; otherwise the dense loop runs.  Results are identical.
// Measured OFF: C2 1.090 -> 1.225 ms (normal), 1.161 ms (uniform): the exp2
// phase is not what bounds this kernel's period once it runs next to the
// other group's dequant phase.
#ifndef IFA_WS_SPARSE
#define IFA_WS_SPARSE 0
#endif
#ifndef IFA_WS_SPARSE_HOT
#define IFA_WS_SPARSE_HOT 16
#endif
#ifndef IFA_WS_CORR_SLEEP_NS
#define IFA_WS_CORR_SLEEP_NS 0
#endif
#ifndef IFA_WS_G1_DELAY_NS
#define IFA_WS_G1_DELAY_NS 0
#endif

// -DIFA_WS_TRACE=1 (tools/build_variant.sh): clock64 stamps of the pipeline
// events of CTA 0, read back with ifa_ws_trace_read (tools/ws_trace.py).
#ifdef IFA_WS_TRACE
__device__ unsigned long long g_ws_trace[49152];
#define WS_TR(role, g, t, ev)                                                               \
    do {                                                                                   \
        if (blockIdx.x == 0 && (t) < 1024)                                                 \
            g_ws_trace[(role) * 16384 + (g) * 8192 + (t) * 8 + (ev)] = clock64();          \
    } while (0)
#else
#define WS_TR(role, g, t, ev) \
    do {                      \
    } while (0)
#endif

template <int D>
struct alignas(1024) Smem {
    uint8_t q[2][BM * D];        // [group] int8, K-major (SW128 for D = 128, SW64 for 64)
    uint8_t k[KST][BN * D];
    uint8_t v[VST][BN * D * 2];  // fp16 codes: [D/64 column halves][BN keys][64], SW128
    uint8_t p[2][BM * BN * 2];   // [group] fp16 P, K-major SW128: 2 atoms of 64 keys
    float sk[KST][BN];           // K scales * log2(e) [/ sqrt(d)] of the stage
    float msg[2][2][BM];         // [group][slot][row]: alpha of a tile, l at the item end
    uint32_t magic[kMagicS == 2 ? 1024 : 4];  // tcgen05.cp source: 128 rows x 32 B of 0x4B400000
    uint64_t q_full, q_empty;
    uint64_t k_full[KST], k_empty[KST], v_full[VST], v_empty[VST];
    uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2], o_ready[2];
    uint64_t m_full[2][2], m_empty[2][2];
    uint32_t tmem_base;
};

struct Params {
    const float* sq;
    const float* sk;
    const float* sv;
    float* o;
    int32_t* s_dump;  // optional [slices][n][n] int32 S (IFA_FLAG_DUMP_S)
    uint8_t* p_dump;  // optional [slices][n][n] uint8 P codes
    int32_t n, d;
    int32_t n_pad;    // rows per slice of the fp16 V buffer (n rounded up to 128)
    int32_t o_pitch;  // floats per O row
    float sk_mul;     // log2(e) [* 1/sqrt(d)]: scores are kept in the log2 domain
    int32_t pairs, slices, items;
    uint32_t g1_delay_ns;  // start offset of group 1 (IFA_WS_G1_DELAY_NS, env IFA_WS_G1_DELAY)
    uint32_t pingpong;     // the groups take turns in the exp2 phase (env IFA_WS_PINGPONG)
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

// Work item -> (pair of Q tiles, slice, KV tiles the pair reads); as attn_pp.cu.
// Non-causal: the pairs of one slice are adjacent (CTAs running together
// share the slice's K and V in L2).  Causal: longest-processing-time order;
// group g of pair t sees KV tiles 0 .. 2t + g and masks inside tile 2t + g.
struct PWork {
    int32_t pair, slice, jt;
};
__device__ __forceinline__ PWork pwork(int32_t idx, const Params& p, bool causal, int32_t J) {
    PWork w;
    if (causal) {
        w.pair = p.pairs - 1 - idx / p.slices;
        w.slice = idx % p.slices;
        w.jt = 2 * w.pair + 2 < J ? 2 * w.pair + 2 : J;
    } else {
        w.pair = idx % p.pairs;
        w.slice = idx / p.pairs;
        w.jt = J;
    }
    return w;
}
__device__ __forceinline__ int32_t group_tiles(const PWork& w, int g, bool causal, int32_t J) {
    if (!causal) return J;
    const int32_t t = 2 * w.pair + g + 1;
    return t < J ? t : J;
}

__device__ __forceinline__ float ex2(float t) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
    return r;
}

// 2^t on the FMA pipe (degree-5 polynomial, 3.5e-7 relative), t clamped at -64.
__device__ __forceinline__ float2 exp2_poly2(float2 t) {
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

// kind::f16 instruction descriptor: D=F32, A=B=F16, A K-major.
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t m, uint32_t n, bool b_mn_major) {
    return (1u << 4) | ((b_mn_major ? 1u : 0u) << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// tcgen05.st 32x32b.x32 of one value into 32 columns of the warp's lanes.
__device__ __forceinline__ void tmem_fill32(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
        : "memory");
}

// Row max of 128 values: 63 three-input max operations.
__device__ __forceinline__ float row_max128(const float (&u)[128]) {
    float a[43];
#pragma unroll
    for (int i = 0; i < 42; ++i) a[i] = fmax3(u[3 * i], u[3 * i + 1], u[3 * i + 2]);
    a[42] = fmaxf(u[126], u[127]);
    float b[15];
#pragma unroll
    for (int i = 0; i < 14; ++i) b[i] = fmax3(a[3 * i], a[3 * i + 1], a[3 * i + 2]);
    b[14] = a[42];
    float c[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) c[i] = fmax3(b[3 * i], b[3 * i + 1], b[3 * i + 2]);
    return fmax3(fmax3(c[0], c[1], c[2]), c[3], c[4]);
}

// RAGGED: n is not a multiple of 128 (the last KV tile masks missing keys).
// DUMP: write S and / or the P codes to p.s_dump / p.p_dump (a separate
// instantiation, so the product kernel carries no dump code).
template <int D, bool CAUSAL, bool RAGGED, bool DUMP>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    int_flash_ws_kernel(const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const Params p) {
    constexpr uint32_t kLayout = D == 128 ? kLayoutSw128 : kLayoutSw64;
    constexpr uint32_t kSbo = 8 * D;
    constexpr uint32_t kIdescS = idesc_i8(BM, BN, false, false);
    constexpr uint32_t kIdescPV = idesc_f16(BM, D, true);
    constexpr bool causal = CAUSAL;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const int32_t n = p.n;
    const int32_t J = (n + BN - 1) / BN;  // KV tiles of a slice

    const uint32_t b_q_full = smem_u32(&sm.q_full), b_q_empty = smem_u32(&sm.q_empty);
    const uint32_t b_k_full = smem_u32(&sm.k_full[0]), b_k_empty = smem_u32(&sm.k_empty[0]);
    const uint32_t b_v_full = smem_u32(&sm.v_full[0]), b_v_empty = smem_u32(&sm.v_empty[0]);
    const uint32_t b_s_full = smem_u32(&sm.s_full[0]), b_s_empty = smem_u32(&sm.s_empty[0]);
    const uint32_t b_p_full = smem_u32(&sm.p_full[0]), b_p_empty = smem_u32(&sm.p_empty[0]);
    const uint32_t b_o_ready = smem_u32(&sm.o_ready[0]);
    const uint32_t b_m_full = smem_u32(&sm.m_full[0][0]), b_m_empty = smem_u32(&sm.m_empty[0][0]);

    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023) __trap();
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_empty, 2);  // both MMA issuers
        for (int g = 0; g < 2; ++g) {
            mbar_init(&sm.s_full[g], 1);
            mbar_init(&sm.s_empty[g], 4);  // the group's softmax warps
            mbar_init(&sm.p_full[g], 4);
            mbar_init(&sm.p_empty[g], 1);
            mbar_init(&sm.o_ready[g], 4);  // correction warps
            for (int s = 0; s < 2; ++s) {
                mbar_init(&sm.m_full[g][s], 4);
                mbar_init(&sm.m_empty[g][s], 4);
            }
        }
        for (int i = 0; i < KST; ++i) {
            mbar_init(&sm.k_full[i], 32);     // producer lanes (K scales) + TMA bytes
            mbar_init(&sm.k_empty[i], 2 + 8); // 2 MMA issuers + 8 softmax warps (sK read)
        }
        for (int i = 0; i < VST; ++i) {
            mbar_init(&sm.v_full[i], 1);
            mbar_init(&sm.v_empty[i], 2);
        }
        fence_barrier_init();
    }
    if (warp == kWarpMma) tmem_alloc<TMEM_COLS>(&sm.tmem_base);
    if (kMagicS == 2) {
        for (uint32_t i = threadIdx.x; i < 1024; i += NUM_THREADS) sm.magic[i] = 0x4B400000u;
        fence_proxy_async_shared();  // read by the tensor core (tcgen05.cp)
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t wg = warp >> 2;

    if (wg == 3) {
        regs_dealloc<kRegsCtrl>();
        if (warp == kWarpProducer) {
            // ------------------------------------------------------- producer
            const uint64_t pol_stream = policy_evict_first();
            const uint64_t pol_keep = policy_evict_last();
            if (lane == 0) {
                tma_prefetch_desc(&tm_q);
                tma_prefetch_desc(&tm_k);
                tma_prefetch_desc(&tm_v);
            }
            Ring<KST> kr;
            Ring<VST> vr;
            uint32_t i = 0, wi = 0;
            for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x, ++wi) {
                const PWork w = pwork(idx, p, causal, J);
                const int32_t q0 = w.pair * 2 * BM, slice = w.slice;
                if (lane == 0) {
                    if (wi >= 1) bar_wait(b_q_empty, (wi - 1) & 1);
                    mbar_arrive_expect_tx(&sm.q_full, 2 * BM * D);
                    tma_load_3d(sm.q[0], &tm_q, &sm.q_full, 0, q0, slice, pol_stream);
                    tma_load_3d(sm.q[1], &tm_q, &sm.q_full, 0, q0 + BM, slice, pol_stream);
                }
                const float* sk_slice = p.sk + static_cast<int64_t>(slice) * n;
                for (int32_t key0 = 0; key0 < w.jt * BN; key0 += BN) {
                    const uint32_t ks = kr.idx, vs = vr.idx;
                    if (i >= KST) bar_wait(b_k_empty + 8 * ks, kr.phase ^ 1u);
                    float4 k4;
                    const int32_t key = key0 + 4 * lane;
                    if (key + 3 < n && (reinterpret_cast<uintptr_t>(sk_slice + key) & 15) == 0) {
                        k4 = __ldg(reinterpret_cast<const float4*>(sk_slice + key));
                    } else {  // ragged tail (the keys are masked, but stay in bounds)
                        k4.x = key + 0 < n ? sk_slice[key + 0] : 0.0f;
                        k4.y = key + 1 < n ? sk_slice[key + 1] : 0.0f;
                        k4.z = key + 2 < n ? sk_slice[key + 2] : 0.0f;
                        k4.w = key + 3 < n ? sk_slice[key + 3] : 0.0f;
                    }
                    k4.x *= p.sk_mul;
                    k4.y *= p.sk_mul;
                    k4.z *= p.sk_mul;
                    k4.w *= p.sk_mul;
                    reinterpret_cast<float4*>(sm.sk[ks])[lane] = k4;
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&sm.k_full[ks], BN * D);
                        tma_load_3d(sm.k[ks], &tm_k, &sm.k_full[ks], 0, key0, slice, pol_keep);
                        if (i >= VST) bar_wait(b_v_empty + 8 * vs, vr.phase ^ 1u);
                        mbar_arrive_expect_tx(&sm.v_full[vs], BN * D * 2);
#pragma unroll
                        for (int h = 0; h < D / 64; ++h)
                            tma_load_3d(sm.v[vs] + h * BN * 128, &tm_v, &sm.v_full[vs], 64 * h,
                                        key0, slice, pol_keep);
                    } else {
                        bar_arrive(b_k_full + 8 * ks);
                    }
                    kr.advance();
                    vr.advance();
                    ++i;
                }
            }
        } else if (warp == kWarpMma || warp == kWarpMma + 1) {
            // ------------------------------------------- MMA issuers (one per group)
            // Per block j: S(next) as soon as the group has read S(j), then
            // P.V(j) once the group has published P(j) and the correction
            // warps have rescaled O (o_ready).
            if (lane == 0) {
                const int g = static_cast<int>(warp - kWarpMma);
                Ring<KST> kr;
                Ring<VST> vr;
                uint32_t t = 0;  // tiles of this group so far
                uint32_t wi = 0;
                const uint32_t d_s = tmem + 256 * g, d_o = d_s + 128;
                auto issue_s = [&](uint32_t ks, uint32_t kph) {
                    bar_wait(b_k_full + 8 * ks, kph);
                    tc_fence_after();
                    const uint32_t q_base = smem_u32(sm.q[g]);
                    const uint32_t k_base = smem_u32(sm.k[ks]);
                    if (kMagicS == 2) {
                        // no-swizzle K-major 128 x 32 B: 8-row x 16 B core
                        // matrices, LBO 128 B (K), SBO 256 B (8-row groups)
                        const uint64_t cdesc = smem_desc(smem_u32(sm.magic), 128, 256, 0);
#pragma unroll
                        for (int c = 0; c < BN / 8; ++c) tmem_cp_128x256b(d_s + 8 * c, cdesc);
                    }
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk) {
                        const uint64_t adesc = smem_desc(q_base + kk * 32, 16, kSbo, kLayout);
                        const uint64_t bdesc = smem_desc(k_base + kk * 32, 16, kSbo, kLayout);
                        mma_i8_ss(d_s, adesc, bdesc, kIdescS, (kMagicS || kk > 0) ? 1u : 0u);
                    }
                    mma_commit_u32(b_s_full + 8 * g);
                };
                if (blockIdx.x < p.items) {
                    bar_wait(b_q_full, 0);
                    if (kMagicSoft) bar_wait(b_s_empty + 8 * g, 0);  // S filled with the constant
                    issue_s(0, 0);
                }
                const uint32_t p_base = smem_u32(sm.p[g]);
                for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x, ++wi) {
                    const bool has_next_item = idx + static_cast<int32_t>(gridDim.x) < p.items;
                    const PWork w = pwork(idx, p, causal, J);
                    const int32_t jg = group_tiles(w, g, causal, J);
                    for (int32_t j = 0; j < w.jt; ++j) {
                        if (j >= jg) {  // causal: a KV tile only the other group reads
                            bar_wait(b_k_full + 8 * kr.idx, kr.phase);
                            bar_arrive(b_k_empty + 8 * kr.idx);
                            bar_wait(b_v_full + 8 * vr.idx, vr.phase);
                            bar_arrive(b_v_empty + 8 * vr.idx);
                            kr.advance();
                            vr.advance();
                            continue;
                        }
                        const bool last = j == jg - 1;
                        mma_commit_u32(b_k_empty + 8 * kr.idx);  // S(j) issued
                        if (last) {
                            mma_commit_u32(b_q_empty);  // every S of this item issued
                            if (has_next_item) bar_wait(b_q_full, (wi + 1) & 1);
                        }
                        if (!last || has_next_item) {
                            Ring<KST> nk = kr;
                            const int32_t ahead = last ? w.jt - j : 1;
                            for (int32_t a = 0; a < ahead; ++a) nk.advance();
                            bar_wait(b_s_empty + 8 * g, (t + kMagicSoft) & 1);
                            issue_s(nk.idx, nk.phase);
                            WS_TR(1, g, t, 0);
                        }
                        bar_wait(b_v_full + 8 * vr.idx, vr.phase);
                        const uint32_t v_base = smem_u32(sm.v[vr.idx]);
                        bar_wait(b_p_full + 8 * g, t & 1);
                        WS_TR(1, g, t, 1);
                        bar_wait(b_o_ready + 8 * g, t & 1);
                        WS_TR(1, g, t, 2);
                        tc_fence_after();
#pragma unroll
                        for (int kk = 0; kk < BN / 16; ++kk) {
                            const uint64_t adesc = smem_desc(
                                p_base + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16, 1024,
                                kLayoutSw128);
                            const uint64_t bdesc =
                                smem_desc(v_base + kk * 16 * 128, BN * 128, 1024, kLayoutSw128);
                            mma_f16_ss(d_o, adesc, bdesc, kIdescPV, (j == 0 && kk == 0) ? 0u : 1u);
                        }
                        mma_commit_u32(b_p_empty + 8 * g);
                        mma_commit_u32(b_v_empty + 8 * vr.idx);
                        WS_TR(1, g, t, 3);
                        kr.advance();
                        vr.advance();
                        ++t;
                    }
                }
            }
            __syncwarp();
        }
    } else if (wg == 2) {
        // (setmaxnreg: .dec below the 128 of the launch, .inc above it)
        if constexpr (kRegsCorr < 128) regs_dealloc<kRegsCorr>(); else regs_alloc<kRegsCorr>();
        // --------------------------------------------- correction + epilogue
        // Messages of both groups in order (tile j of group 0, tile j of group
        // 1, ...): for a tile, rescale the O rows whose max moved once P.V(j-1)
        // is done and release P.V(j) (o_ready); at the item end (message =
        // l), write O * sV / l.  The wait for P.V(j-1) happens for every tile
        // (also when nothing moves), so o_ready never runs two phases ahead of
        // the MMA issuer that waits on it.
        const uint32_t qw = warp & 3;
        const uint32_t row = 32 * qw + lane;
        const uint32_t t_row = tmem + ((32 * qw) << 16);
        uint32_t mcnt[2] = {0u, 0u}, tcnt[2] = {0u, 0u};
        for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x) {
            const PWork w = pwork(idx, p, causal, J);
            for (int32_t j = 0; j <= w.jt; ++j) {
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    const int32_t jg = group_tiles(w, g, causal, J);
                    if (j > jg) continue;
                    const uint32_t slot = mcnt[g] & 1;
                    // (a poll with a short sleep instead of the suspend-hint wait
                    // saves ~170 issue slots per tile of wake-ups but measured
                    // 3% slower: IFA_WS_CORR_SLEEP_NS)
                    if (kNamedMsg) {
                        named_bar_sync(msg_full_id(g, slot), 256);
                    } else if (IFA_WS_CORR_SLEEP_NS > 0) {
                        const uint32_t bm = b_m_full + 16 * g + 8 * slot, par = (mcnt[g] >> 1) & 1;
                        while (!bar_try(bm, par)) __nanosleep(IFA_WS_CORR_SLEEP_NS);
                    } else {
                        bar_wait(b_m_full + 16 * g + 8 * slot, (mcnt[g] >> 1) & 1);
                    }
                    const float a = sm.msg[g][slot][row];
                    if (warp == 8 && lane == 0) WS_TR(2, g, tcnt[g], 0);
                    if (kNamedMsg) {
                        named_bar_arrive(msg_empty_id(g, slot), 256);
                    } else {
                        __syncwarp();
                        if (lane == 0) bar_arrive(b_m_empty + 16 * g + 8 * slot);
                    }
                    ++mcnt[g];
                    const uint32_t t_o = t_row + 256 * g + 128;
                    if (j < jg) {
                        if (j > 0) {
                            bar_wait(b_p_empty + 8 * g, (tcnt[g] - 1) & 1);  // P.V(j-1) done
                            if (warp == 8 && lane == 0) WS_TR(2, g, tcnt[g], 1);
                            tc_fence_after();
                            if (__any_sync(0xffffffffu, a != 1.0f)) {
#pragma unroll
                                for (int c = 0; c < D / 32; ++c) {
                                    uint32_t o[32];
                                    tmem_ld32(t_o + 32 * c, o);
                                    tmem_wait_ld();
#pragma unroll
                                    for (int k = 0; k < 16; ++k) {
                                        const float2 v = fmul2(make_float2(__uint_as_float(o[2 * k]),
                                                                           __uint_as_float(o[2 * k + 1])),
                                                               f2(a));
                                        o[2 * k] = __float_as_uint(v.x);
                                        o[2 * k + 1] = __float_as_uint(v.y);
                                    }
                                    tmem_st32(t_o + 32 * c, o);
                                }
                                tmem_wait_st();
                            }
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) bar_arrive(b_o_ready + 8 * g);
                        if (warp == 8 && lane == 0) WS_TR(2, g, tcnt[g], 2);
                        ++tcnt[g];
                    } else {
                        // epilogue: O holds 2^-24 * the integer P.V sums
                        const float f = __fdiv_rn(p.sv[w.slice], a) * 16777216.0f;
                        bar_wait(b_p_empty + 8 * g, (tcnt[g] - 1) & 1);  // last P.V done
                        tc_fence_after();
                        const int32_t grow = w.pair * 2 * BM + g * BM + static_cast<int32_t>(row);
                        float* orow = p.o + (static_cast<int64_t>(w.slice) * n + grow) * p.o_pitch;
                        const bool vec = (p.o_pitch & 3) == 0 && p.d == D;
#pragma unroll
                        for (int c = 0; c < D / 32; ++c) {
                            uint32_t o[32];
                            tmem_ld32(t_o + 32 * c, o);
                            tmem_wait_ld();
                            if (grow < n) {
                                if (vec) {
#pragma unroll
                                    for (int k = 0; k < 8; ++k) {
                                        const float2 v0 = fmul2(make_float2(__uint_as_float(o[4 * k]),
                                                                            __uint_as_float(o[4 * k + 1])),
                                                                f2(f));
                                        const float2 v1 = fmul2(make_float2(__uint_as_float(o[4 * k + 2]),
                                                                            __uint_as_float(o[4 * k + 3])),
                                                                f2(f));
                                        __stcs(reinterpret_cast<float4*>(orow + 32 * c + 4 * k),
                                               make_float4(v0.x, v0.y, v1.x, v1.y));
                                    }
                                } else {
#pragma unroll
                                    for (int k = 0; k < 32; ++k)
                                        if (32 * c + k < p.d)
                                            orow[32 * c + k] = __uint_as_float(o[k]) * f;
                                }
                            }
                        }
                        tc_fence_before();
                    }
                }
            }
        }
    } else {
        regs_alloc<kRegsSoftmax>();
        // -------------------------------------------------------- softmax
        const uint32_t g = wg;          // Q tile / group
        const uint32_t qw = warp & 3;   // TMEM lane quarter of this warp
        const uint32_t row = 32 * qw + lane;
        const uint32_t t_s = tmem + ((32 * qw) << 16) + 256 * g;
        const uint32_t bs_full = b_s_full + 8 * g, bs_empty = b_s_empty + 8 * g;
        const uint32_t bp_full = b_p_full + 8 * g, bp_empty = b_p_empty + 8 * g;
        const uint32_t bm_full = b_m_full + 16 * g, bm_empty = b_m_empty + 16 * g;
        // P (fp16, K-major SW128, two 64-key atoms): row r's 16-byte chunk c
        // of an atom sits at r * 128 + ((c ^ (r & 7)) * 16); one store
        // instruction of the warp (32 rows, same c) is 4 conflict-free
        // wavefronts
        const uint32_t p_row = smem_u32(sm.p[g]) + row * 128;
        const uint32_t sw = row & 7;
        Ring<KST> kv;
        uint32_t tc = 0, mc = 0;

        auto post = [&](float value) {  // one message to the correction warps
            const uint32_t slot = mc & 1;
            if (kNamedMsg) {
                if (mc >= 2) named_bar_sync(msg_empty_id(g, slot), 256);
                sm.msg[g][slot][row] = value;
                named_bar_arrive(msg_full_id(g, slot), 256);
            } else {
                if (mc >= 2) bar_wait(bm_empty + 8 * slot, ((mc >> 1) & 1) ^ 1u);
                sm.msg[g][slot][row] = value;
                __syncwarp();
                if (lane == 0) bar_arrive(bm_full + 8 * slot);
            }
            ++mc;
        };

        // group 1 starts later, so the two groups' MUFU-heavy code phases
        // interleave instead of running in lockstep
        if (kMagicSoft) {  // the first S of the kernel accumulates onto the constant
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_fill32(t_s + 32 * c, 0x4B400000u);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(bs_empty);
        }
        if (g == 1 && p.g1_delay_ns > 0) __nanosleep(p.g1_delay_ns);
        // Ping-pong: the exp2 phase (MUFU-bound) of one group runs while the
        // other group loads and dequantizes its next S (ALU/FMA-bound), instead
        // of both groups contending for the MUFU unit at the same time.  Named
        // barrier 1: group 1 -> group 0 ("my exp2 phase is over"), 2: 0 -> 1.
        // Every tile (also a causal skip tile) does one turn per group, so the
        // arrive / sync counts match; group 0 skips its first wait and adds a
        // final one.
        const bool pp = p.pingpong != 0;
        bool first_turn = true;
        auto turn_begin = [&]() {
            if (!pp) return;
            if (g == 0) {
                if (!first_turn) named_bar_sync(1, 256);
            } else {
                named_bar_sync(2, 256);
            }
            first_turn = false;
        };
        auto turn_end = [&]() {
            if (pp) named_bar_arrive(g == 0 ? 2 : 1, 256);
        };
        for (int32_t idx = blockIdx.x; idx < p.items; idx += gridDim.x) {
            const PWork w = pwork(idx, p, causal, J);
            const int32_t jg = group_tiles(w, static_cast<int>(g), causal, J);
            const int32_t diag = causal ? 2 * w.pair + static_cast<int32_t>(g) : -1;
            const int32_t grow = w.pair * 2 * BM + static_cast<int32_t>(g) * BM + static_cast<int32_t>(row);
            const int32_t slice = w.slice;
            const float sq = grow < n ? p.sq[static_cast<int64_t>(slice) * n + grow] : 0.0f;
            float l = 0.0f, m = -__int_as_float(0x7f800000);

            for (int32_t j = 0; j < w.jt; ++j) {
                const uint32_t st = kv.idx;
                if (j >= jg) {  // causal: the other group's diagonal tile
                    bar_wait(b_k_full + 8 * st, kv.phase);
                    __syncwarp();
                    if (lane == 0) bar_arrive(b_k_empty + 8 * st);
                    kv.advance();
                    turn_begin();
                    turn_end();
                    continue;
                }
                bar_wait(bs_full, tc & 1);
                if (qw == 0 && lane == 0) WS_TR(0, g, tc, 0);
                tc_fence_after();
                float u[128];
                {
                    uint32_t s[128];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        tmem_ld32(t_s + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&s[32 * c]));
                    tmem_wait_ld();
                    if (qw == 0 && lane == 0) WS_TR(0, g, tc, 4);
                    if (kMagicSoft) {  // S(j+1) accumulates onto the constant again
#pragma unroll
                        for (int c = 0; c < 4; ++c) tmem_fill32(t_s + 32 * c, 0x4B400000u);
                        tmem_wait_st();
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(bs_empty);
                    if (DUMP && p.s_dump != nullptr && grow < n) {
                        int32_t* dst = p.s_dump + (static_cast<int64_t>(slice) * n + grow) * n + j * BN;
#pragma unroll
                        for (int c = 0; c < 128; ++c)
                            if (j * BN + c < n) dst[c] = static_cast<int32_t>(s[c] - (kMagicS ? 0x4B400000u : 0u));
                    }
                    bar_wait(b_k_full + 8 * st, kv.phase);
                    if (qw == 0 && lane == 0) WS_TR(0, g, tc, 7);
                    // u = float(S) * sK * log2(e).  float(S) without I2F (a
                    // quarter-rate pipe on sm_100): |S| <= 127^2 * 128 < 2^22,
                    // so the bits of S + 0x4B400000 are the float 1.5 * 2^23 + S
                    // and one exact packed subtract leaves float(S)
                    const float4* skv = reinterpret_cast<const float4*>(sm.sk[st]);
                    auto fl2 = [](uint32_t a, uint32_t b) {
#if IFA_WS_I2F
                        return make_float2(__int2float_rn(static_cast<int32_t>(a)),
                                           __int2float_rn(static_cast<int32_t>(b)));
#else
                        const uint32_t add = kMagicS ? 0u : 0x4B400000u;
                        return fsub2(make_float2(__uint_as_float(a + add), __uint_as_float(b + add)),
                                     f2(kMagic));
#endif
                    };
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const float4 k4 = skv[c];
                        const float2 a = fmul2(fl2(s[4 * c], s[4 * c + 1]), make_float2(k4.x, k4.y));
                        const float2 b = fmul2(fl2(s[4 * c + 2], s[4 * c + 3]), make_float2(k4.z, k4.w));
                        u[4 * c] = a.x;
                        u[4 * c + 1] = a.y;
                        u[4 * c + 2] = b.x;
                        u[4 * c + 3] = b.y;
                    }
                }
                if (qw == 0 && lane == 0) WS_TR(0, g, tc, 5);
                __syncwarp();
                if (lane == 0) bar_arrive(b_k_empty + 8 * st);

                auto rest = [&](auto mask_tag) {
                    constexpr bool dmask = decltype(mask_tag)::value;  // keys > kmax masked
                    int32_t kmax = BN - 1;
                    if (dmask) {
                        if (RAGGED && n - j * BN - 1 < kmax) kmax = n - j * BN - 1;
                        if (causal && j == diag && static_cast<int32_t>(row) < kmax)
                            kmax = static_cast<int32_t>(row);
                        // finite: a zero Q row (sQ = 0) must not turn the masked
                        // exponents into 0 * inf = NaN (the exp2 lag chain below
                        // would carry it into the visible codes)
#pragma unroll
                        for (int c = 0; c < 128; ++c)
                            if (c > kmax) u[c] = -3.0e38f;
                    }
                    const float b = row_max128(u);
                    if (qw == 0 && lane == 0) WS_TR(0, g, tc, 6);
                    const float mnew = (m < b) ? b : m;
                    const float cr = kLog2_127 - sq * mnew;
                    const float alpha = (j == 0 || mnew == m) ? 1.0f : ex2(sq * (m - mnew));
                    m = mnew;
                    post(alpha);
                    turn_begin();
                    if (qw == 0 && lane == 0) WS_TR(0, g, tc, 1);
                    // P(j-1) has been read by P.V(j-1): P is stored as it is made
                    if (tc > 0) bar_wait(bp_empty, (tc - 1) & 1);
                    if (qw == 0 && lane == 0) WS_TR(0, g, tc, 2);
                    tc_fence_after();
                    // y + 1.5*2^23 has the code round(y) in its low bits; its
                    // low 16 bits read as fp16 are the subnormal code * 2^-24,
                    // exact, so one PRMT packs two codes.  The row sum adds the
                    // packed words as integers (<= 64 * 127 per half).
                    uint32_t acc = 0u;
                    const float tmax = __fmaf_rn(sq, b, cr);  // the row's largest exponent
                    const bool sparse =
                        IFA_WS_SPARSE &&
                        __popc(__ballot_sync(0xffffffffu, !(tmax < -1.0f))) <= IFA_WS_SPARSE_HOT;
                    auto store_chunk = [&](int ch, const uint32_t (&wd)[4]) {
                        const uint32_t chunk = (static_cast<uint32_t>(ch & 7) ^ sw);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         p_row + (ch >> 3) * (BM * 128) + chunk * 16),
                                     "r"(wd[0]), "r"(wd[1]), "r"(wd[2]), "r"(wd[3])
                                     : "memory");
                        if (DUMP && p.p_dump != nullptr && grow < n) {
                            uint8_t* dst = p.p_dump + (static_cast<int64_t>(slice) * n + grow) * n + j * BN + 8 * ch;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                if (j * BN + 8 * ch + 2 * e < n) dst[2 * e] = static_cast<uint8_t>(wd[e] & 0xffu);
                                if (j * BN + 8 * ch + 2 * e + 1 < n)
                                    dst[2 * e + 1] = static_cast<uint8_t>((wd[e] >> 16) & 0xffu);
                            }
                        }
                    };
                    if (sparse) {
                        // per 8-key chunk: exponents, a warp vote, exp2 only when
                        // some row of the warp has a nonzero code there
#pragma unroll
                        for (int ch = 0; ch < 16; ++ch) {
                            float2 t[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                t[e] = ffma2(make_float2(u[8 * ch + 2 * e], u[8 * ch + 2 * e + 1]), f2(sq),
                                             f2(cr));
                            const float tm = fmaxf(fmax3(t[0].x, t[0].y, t[1].x),
                                                   fmax3(fmax3(t[1].y, t[2].x, t[2].y), t[3].x, t[3].y));
                            uint32_t wd[4] = {0u, 0u, 0u, 0u};
                            if (__any_sync(0xffffffffu, tm >= -1.0f)) {
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    float2 c = fadd2(make_float2(ex2(t[e].x), ex2(t[e].y)), f2(kMagic));
                                    if (dmask) {
                                        if (8 * ch + 2 * e > kmax) c.x = kMagic;
                                        if (8 * ch + 2 * e + 1 > kmax) c.y = kMagic;
                                    }
                                    wd[e] = prmt(__float_as_uint(c.x), __float_as_uint(c.y), 0x5410u);
                                }
                                acc += wd[0] + wd[1];
                                acc += wd[2] + wd[3];
                            }
                            store_chunk(ch, wd);
                        }
                    } else {
                    // all 128 exp2 first (in place of u), then the rounding and
                    // packing, chunk c's magic add made to depend on an exp2
                    // result kLag pairs further on: otherwise ptxas puts each
                    // FADD2 right behind its MUFU pair and the MUFU latency,
                    // not its throughput, sets the pace of the loop
                    float2 y[64];
#pragma unroll
                    for (int k = 0; k < 64; ++k) {
                        const float2 t = ffma2(make_float2(u[2 * k], u[2 * k + 1]), f2(sq), f2(cr));
                        y[k] = (kPolyEvery > 0 && k % (kPolyEvery > 0 ? kPolyEvery : 1) == kPolyEvery - 1)
                                   ? exp2_poly2(t)
                                   : make_float2(ex2(t.x), ex2(t.y));
                    }
#pragma unroll
                    for (int ch = 0; ch < 16; ++ch) {  // 8 keys per 16-byte chunk
                        uint32_t wd[4];
                        constexpr int kLag = IFA_WS_MUFU_LAG;
                        const int dep = 4 * ch + 3 + kLag < 63 ? 4 * ch + 3 + kLag : 63;
                        const float mg = kLag > 0 ? __fmaf_rn(0.0f, y[dep].y, kMagic) : kMagic;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int k = 4 * ch + e;  // key pair
                            float2 c = fadd2(y[k], f2(mg));
                            if (dmask) {  // masked keys are code 0 (also when sQ == 0)
                                if (2 * k > kmax) c.x = kMagic;
                                if (2 * k + 1 > kmax) c.y = kMagic;
                            }
                            wd[e] = prmt(__float_as_uint(c.x), __float_as_uint(c.y), 0x5410u);
                        }
                        acc += wd[0] + wd[1];
                        acc += wd[2] + wd[3];
                        const uint32_t chunk = (static_cast<uint32_t>(ch & 7) ^ sw);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         p_row + (ch >> 3) * (BM * 128) + chunk * 16),
                                     "r"(wd[0]), "r"(wd[1]), "r"(wd[2]), "r"(wd[3])
                                     : "memory");
                        if (DUMP && p.p_dump != nullptr && grow < n) {
                            uint8_t* dst = p.p_dump + (static_cast<int64_t>(slice) * n + grow) * n + j * BN + 8 * ch;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                if (j * BN + 8 * ch + 2 * e < n) dst[2 * e] = static_cast<uint8_t>(wd[e] & 0xffu);
                                if (j * BN + 8 * ch + 2 * e + 1 < n)
                                    dst[2 * e + 1] = static_cast<uint8_t>((wd[e] >> 16) & 0xffu);
                            }
                        }
                    }
                    }
                    fence_proxy_async_shared();  // P is read by the tensor core
                    __syncwarp();
                    if (lane == 0) bar_arrive(bp_full);
                    turn_end();
                    if (qw == 0 && lane == 0) WS_TR(0, g, tc, 3);
                    const float lsum = static_cast<float>(static_cast<int32_t>((acc & 0xffffu) + (acc >> 16)));
                    l = __fmaf_rn(l, alpha, lsum);
                };
                if constexpr (causal || RAGGED) {
                    if ((causal && j == diag) || (RAGGED && (j + 1) * BN > n))
                        rest(std::true_type{});
                    else
                        rest(std::false_type{});
                } else {
                    rest(std::false_type{});
                }
                kv.advance();
                ++tc;
            }
            post(l);  // item end: the correction warps write O * sV / l
        }
        if (pp && g == 0 && !first_turn) named_bar_sync(1, 256);  // group 1's last turn_end
        if (kNamedMsg) {  // complete the correction warps' last releases of both slots
            if (mc >= 2) named_bar_sync(msg_empty_id(g, mc & 1), 256);
            if (mc >= 1) named_bar_sync(msg_empty_id(g, (mc + 1) & 1), 256);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kWarpMma) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
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

// int8 codes [slices][n][pitch], box {D, 128 rows, 1 slice}
static bool make_map_codes(CUtensorMap* map, const int8_t* base, int64_t slices, int64_t n,
                           int64_t pitch, int D) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(slices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch),
                                   static_cast<cuuint64_t>(pitch * n)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(D), 128u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// fp16 V [slices][n_pad][D], box {64 columns, 128 keys, 1 slice}, 128B swizzle:
// keys in natural order (one softmax thread owns a whole row of P).
static bool make_map_v16(CUtensorMap* map, const __half* base, int64_t slices, int64_t n_pad,
                         int D) {
    PFN_encodeTiled enc = get_encode();
    if (!enc || n_pad % 128 != 0) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(n_pad),
                                static_cast<cuuint64_t>(slices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2,
                                   static_cast<cuuint64_t>(D) * 2 * n_pad};
    const cuuint32_t box[3] = {64u, 128u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(base), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

template <int D, bool CAUSAL, bool RAGGED, bool DUMP>
static cudaError_t launch_k(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const Params& p, int dev, int sms, cudaStream_t stream) {
    const size_t smem = sizeof(Smem<D>) + 1024;
    (void)dev;
    const cudaError_t e = smem_attr_once<int_flash_ws_kernel<D, CAUSAL, RAGGED, DUMP>>(smem);
    if (e != cudaSuccess) return e;
    const int grid = p.items < sms ? p.items : sms;
    int_flash_ws_kernel<D, CAUSAL, RAGGED, DUMP><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

template <int D>
static cudaError_t run(const int8_t* q, const int8_t* k, const __half* v16, const Params& p,
                       int64_t pitch, bool causal, cudaStream_t stream) {
    CUtensorMap tq, tk, tv;
    if (!make_map_codes(&tq, q, p.slices, p.n, pitch, D) ||
        !make_map_codes(&tk, k, p.slices, p.n, pitch, D) ||
        !make_map_v16(&tv, v16, p.slices, p.n_pad, D))
        return cudaErrorInvalidValue;
    const int dev = 0;
    const int sms = current_device_sms();
    const bool ragged = p.n % BN != 0;
    if (p.s_dump != nullptr || p.p_dump != nullptr) {  // debug outputs: one generic instantiation
        if (causal) return launch_k<D, true, true, true>(tq, tk, tv, p, dev, sms, stream);
        return launch_k<D, false, true, true>(tq, tk, tv, p, dev, sms, stream);
    }
    if (causal && ragged) return launch_k<D, true, true, false>(tq, tk, tv, p, dev, sms, stream);
    if (causal) return launch_k<D, true, false, false>(tq, tk, tv, p, dev, sms, stream);
    if (ragged) return launch_k<D, false, true, false>(tq, tk, tv, p, dev, sms, stream);
    return launch_k<D, false, false, false>(tq, tk, tv, p, dev, sms, stream);
}

}  // namespace ws

#ifdef IFA_WS_TRACE
extern "C" int ifa_ws_trace_read(unsigned long long* host, int64_t count) {
    return cudaMemcpyFromSymbol(host, ws::g_ws_trace, sizeof(unsigned long long) * count) ==
                   cudaSuccess
               ? 0
               : 1;
}
#endif

// IFA_B200_WS=1 selects this kernel for the full-INT8 tolerance mode (read at
// every call); the default stays attn_pp.cu, which measured faster at C2
// (0.974 vs 1.086 ms).  The S / P dump outputs always run here.
bool int_flash_ws_enabled() {
    const char* e = std::getenv("IFA_B200_WS");
    return e && e[0] == '1';
}

cudaError_t launch_int_flash_ws(const int8_t* q, const float* sq, const int8_t* k,
                                const float* sk, const uint16_t* v16, const float* sv, float* o,
                                int64_t slices, int64_t n, int64_t d, int64_t pitch,
                                int64_t o_pitch, uint32_t flags, const AttnDump* dump,
                                cudaStream_t stream) {
    ws::Params p;
    p.sq = sq;
    p.sk = sk;
    p.sv = sv;
    p.o = o;
    p.s_dump = dump ? dump->s : nullptr;
    p.p_dump = dump ? dump->p : nullptr;
    p.n = static_cast<int32_t>(n);
    p.d = static_cast<int32_t>(d);
    p.n_pad = static_cast<int32_t>((n + ws::BN - 1) / ws::BN * ws::BN);
    p.o_pitch = static_cast<int32_t>(o_pitch);
    p.sk_mul = 1.4426950408889634f *
               ((flags & IFA_FLAG_SQRT_D) ? 1.0f / sqrtf(static_cast<float>(d)) : 1.0f);
    const int32_t q_tiles = static_cast<int32_t>((n + ws::BM - 1) / ws::BM);
    p.pairs = (q_tiles + 1) / 2;
    p.slices = static_cast<int32_t>(slices);
    p.items = p.pairs * p.slices;
    p.g1_delay_ns = IFA_WS_G1_DELAY_NS;
    p.pingpong = 1;
    if (const char* e = std::getenv("IFA_WS_PINGPONG")) p.pingpong = e[0] != '0';
    if (const char* e = std::getenv("IFA_WS_G1_DELAY")) p.g1_delay_ns = static_cast<uint32_t>(std::atoi(e));
    const __half* vh = reinterpret_cast<const __half*>(v16);
    const bool causal = (flags & IFA_FLAG_CAUSAL) != 0;
    if (d <= 64) return ws::run<64>(q, k, vh, p, pitch, causal, stream);
    return ws::run<128>(q, k, vh, p, pitch, causal, stream);
}

}  // namespace ifa_b200
