// attn_pp.cu -- tolerance-mode INT-FlashAttention forward with two Q tiles
// per CTA (IFA_FLAG_FAST, causal or not, every KV block one 128-key tile),
// also instantiated for the half-INT8 and FP8 variants (see
// the MODE comment below).  Same algorithm as attention.cpp:235-357 per block: exact
// int32 S = Q.K^T (tcgen05.mma kind::i8), dequantize, running row max,
// requantize P to integer codes round(127 * exp(s - m)), O = O*alpha + P.V,
// l = l*alpha + sum(codes), O * sV / l at the end.
//
// What differs from the one-tile kernels in attn.cu is where O lives.  The
// P codes (0..127) and V codes (-127..127) are exact in fp16, their products
// (<= 127^2) and 128-key sums (< 2^21) exact in f32, so P.V can run as
// tcgen05.mma kind::f16 accumulating straight into an f32 O in TMEM: the
// tensor core performs the fold's "+ float(PV)".  The softmax warps only
// rescale the O rows whose running max moved (alpha != 1), reading and
// writing TMEM, and no longer hold a 128-column accumulator in registers.
// That frees the register file for a second 128-row Q tile: 16 math warps in
// two groups of 8 (quad layout: 16 TMEM lanes x 128 columns per warp, two
// rows x 32 keys per thread), four math warps per SM sub-partition.
//
// TMEM (512 columns): group g uses S [256g, 256g+128) and O [256g+128,
// 256g+128+D).  S(j+1) of a group is issued as soon as the group has read
// S(j), so the tensor core computes the next scores while the softmax works.
// P goes to shared memory (fp16, K-major, 128B swizzle; 32 KiB per group)
// and P.V(j) reads it from there; the group waits for P.V(j-1) (which also
// makes O(j-1) final) before it rescales O and overwrites P.
//
// Each thread writes its row's 32 keys (8k + 2t0 + e, k = 0..15) as two
// 32-byte runs, MMA keys 64h + 16 t0 + 2k' + e for k = 8h + k' (a layout
// without shared-memory bank conflicts); the fp16 V tile is loaded with its
// rows permuted the same way (smem row 64h + 16t + 2k' + e <- key 64h + 8k' +
// 2t + e) by a 5-D tensor map over a V copy padded to a multiple of 128 rows
// per slice; a ragged last tile masks its missing keys.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "ifa_internal.h"
#include "ptx.cuh"

namespace ifa_b200 {
namespace pp {

using namespace ptx;

constexpr int BM = 128;
constexpr int BN = 128;
#ifndef IFA_PP_KST
#define IFA_PP_KST 2
#endif
constexpr int KST = IFA_PP_KST;  // K tiles (+ K scales) in flight
#ifndef IFA_PP_VST
#define IFA_PP_VST 2
#endif
constexpr int VST = IFA_PP_VST;  // fp16 V tiles in flight
constexpr int CTRL_WARPS = 4;
constexpr int GROUP_WARPS = 8;
// IFA_PP_EPI: a fourth warpgroup (warps 20-23, one per TMEM lane quarter)
// writes each item's O (TMEM -> x sV/l -> global), so the math warps go on
// to the next item without an epilogue; the math warps then run with 104
// registers instead of 112 (the pool is 768 x 80).  Measured slower on the
// non-causal lines (C2 +6%, C5 +5%; C3 -3% with EPI = 2): one warpgroup
// serves both groups in turn, so group 1's next P.V(0) waits for both
// epilogues.  EPI = 2 needs o_pitch * 4 % 16 == 0 (A/B builds only).
#ifndef IFA_PP_EPI
#define IFA_PP_EPI 0
#endif
constexpr bool kEpi = IFA_PP_EPI != 0;
constexpr bool kEpi2 = IFA_PP_EPI == 2;  // O through shared memory + TMA stores
// IFA_PP_CORR: a fourth warpgroup (warps 20-23, one per TMEM lane quarter)
// rescales O by alpha for both groups (FA4's correction warpgroup), so the O
// rescale leaves the math warps' chain: the math warps publish alpha per row
// (smem + alpha_ready), the correction warps rescale once P.V(j-1) is done
// and arrive o_ready, and the MMA issuer waits o_ready before P.V(j).
#ifndef IFA_PP_CORR
#define IFA_PP_CORR 0
#endif
#ifndef IFA_PP_CORR_SLEEP_NS  // back-off between polls of the correction warps
#define IFA_PP_CORR_SLEEP_NS 32
#endif
#ifndef IFA_PP_CORR_COLS  // O columns per TMEM load of a correction warp (8 or 16)
#define IFA_PP_CORR_COLS 16
#endif
constexpr bool kCorr = IFA_PP_CORR != 0;
static_assert(!(kEpi && kCorr), "IFA_PP_EPI and IFA_PP_CORR share the fourth warpgroup");
constexpr int EPI_WARPS = (kEpi || kCorr) ? 4 : 0;
[[maybe_unused]] constexpr int EPI_WARP0 = CTRL_WARPS + 2 * GROUP_WARPS;
constexpr int NUM_THREADS = 32 * (CTRL_WARPS + 2 * GROUP_WARPS + EPI_WARPS);
constexpr int kLaunchRegs = (kEpi || kCorr) ? 80 : 96;  // 65536 / NUM_THREADS, rounded down to 8
#ifndef IFA_PP_REGS_CONTROL
#define IFA_PP_REGS_CONTROL 32
#endif
constexpr uint32_t kRegsControl = IFA_PP_REGS_CONTROL;
constexpr uint32_t kRegsEpi = 32;
// setmaxnreg moves registers inside the CTA pool allocated at launch (640 x 96
// = 61440): 4*32*32 + 16*32*112 = 61440.
#ifndef IFA_PP_REGS_MATH
#define IFA_PP_REGS_MATH ((IFA_PP_EPI || IFA_PP_CORR) ? 104 : 112)
#endif
constexpr uint32_t kRegsMath = IFA_PP_REGS_MATH;
static_assert(4 * kRegsControl + EPI_WARPS * kRegsEpi + 16 * kRegsMath <=
                  NUM_THREADS / 32 * kLaunchRegs,
              "setmaxnreg pool");
constexpr uint32_t TMEM_COLS = 512;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr float kLog2_127 = 6.9886846867721655f;
constexpr float kLog2e = 1.4426950408889634f;
#ifndef IFA_PP_POLY_MASK
#define IFA_PP_POLY_MASK 16
#endif
// key pairs k with (k & mask) == mask take exp2 on the FMA pipe (3: 1 in 4,
// 15: 1 in 16, 16: none).  With four math warps per sub-partition the MUFU
// unit keeps up: C2 0.982 ms at 16 vs 0.989 at 15 and 0.985 at 7 (with the
// groups de-phased; 1.029 at 15 vs 1.034 at 16 before).
constexpr int kPolyMask = IFA_PP_POLY_MASK;
// group 1's start delay (ns): 1000 helped before the warp-wide MMA issue
// (0.994 -> 0.983 ms); since then 0 is best (0.921 vs 0.928 ms at 1000)
#ifndef IFA_PP_G1_DELAY_NS
#define IFA_PP_G1_DELAY_NS 0
#endif
// Cold-code skipping (kModeCodes): a code round(127 * 2^t') is 0 whenever
// t = t' + log2(127) < -1, i.e. when the score is more than ln(254) below the
// running max.  For peaked score distributions (the reference's default:
// N(0,1) activations, no 1/sqrt(d), so s ~ N(0, d)) that is > 99% of the
// codes once the running max has settled.  A MUFU warp-instruction costs its
// full pipe time even with every lane predicated off (tools/microbench/
// mufu_mask.cu), so the skip is warp-uniform: when at most IFA_PP_SPARSE_HOT
// of the warp's lanes hold a row whose block max reaches t > -1, every
// exp2 pair is guarded by a warp vote and skipped (codes 0, exactly what the
// exp2 would round to) when no lane needs it.  Otherwise (flat
// distributions) the dense loop runs unchanged.  Results are identical.
// Measured OFF: C2 0.972 -> 1.100 ms (normal) / 1.181 ms (uniform); this
// kernel is latency- and register-bound, not MUFU-bound, so skipping 90% of
// the MUFU work buys nothing and the second loop costs registers.
#ifndef IFA_PP_SPARSE
#define IFA_PP_SPARSE 0
#endif
#ifndef IFA_PP_SPARSE_HOT
#define IFA_PP_SPARSE_HOT 16
#endif
// float(S) by integer magic add + packed subtract instead of I2F
#ifndef IFA_PP_SPLIT_SLOAD
#define IFA_PP_SPLIT_SLOAD 0
#endif
#ifndef IFA_PP_MAGIC_CVT
#define IFA_PP_MAGIC_CVT 0
#endif
// 0: I2F for every score, 1: magic add for every score, 2: for odd k, 3: for k % 4 == 3;
// 4 / 5 / 6: as 1 / 2 / 3 but the magic add is an IMAD by an opaque 1 (the
// FMA pipe's integer multiply-add instead of the ALU's IADD3)
constexpr int kMagicCvt = IFA_PP_MAGIC_CVT;
// TMA epilogue variants (same-box A/B, attention ms, r2: per-half / per-box /
// per-box + deferred read wait): C2 0.894 / 0.894 / 0.936, C3 1.963 / 1.960 /
// 1.918, C5 55.53 / 55.12 / 57.64.  Deferring the last read wait to the next
// item's first P store helps causal C3 and costs the non-causal lines.
#ifndef IFA_PP_OBOX  // 1 = one bulk group per 32-column box, 0 = per 64-column half
#define IFA_PP_OBOX 1
#endif
#ifndef IFA_PP_OSTG  // 1 = O staged in smem, read back row-contiguously, 16-byte global stores
#define IFA_PP_OSTG 0
#endif
#ifndef IFA_PP_ODEFER  // 1 = the next item's first P stores wait for the O reads
#define IFA_PP_ODEFER 0
#endif
#ifndef IFA_PP_EARLY_P
#define IFA_PP_EARLY_P 1
#endif
static_assert(!kCorr || IFA_PP_EARLY_P, "IFA_PP_CORR publishes alpha after the early P-buffer wait");
// 1: the MMA issuers rebuild the Q / P descriptors at each issue (an opaque
// register copy of the base the compiler cannot hoist), so the 32-register
// control warps do not keep the eight P.V descriptors live across the loop
// and spill them (reloaded between the P-full wait and the first P.V MMA)
#ifndef IFA_PP_LAUNDER
#define IFA_PP_LAUNDER 1
#endif

template <int D>
struct alignas(1024) Smem {
    uint8_t q[2][BM * D];            // [group]
    uint8_t k[KST][BN * D];
    uint8_t v[VST][BN * D * 2];      // fp16 codes: [D/64 halves][BN permuted rows][64]
    uint8_t p[2][BM * BN * 2];       // [group] fp16 P, K-major SW128: 2 K-atoms of 64 keys
    float sk[KST][BN];
    uint64_t q_full, q_empty;
    uint64_t k_full[KST], k_empty[KST], v_full[VST], v_empty[VST];
    uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2], o_full[2], o_free[2];
#if IFA_PP_EPI
    uint64_t epi_ready[2];  // the group's per-row O factors are in epi_f
    float epi_f[2][BM];     // sV / l (or the mode's factor) per row
    // IFA_PP_EPI == 2: per epilogue warp, two 32-row x 16-column f32 staging
    // boxes (SW64) for TMA stores
    alignas(1024) uint8_t epi_stage[kEpi2 ? 4 : 1][2][32 * 64];
#endif
#if IFA_PP_CORR
    float alpha[2][2][BM];     // [group][tile parity][row]
    uint64_t alpha_ready[2];   // the group's alpha of its current tile are in place
    uint64_t o_ready[2];       // O(j-1) rescaled: P.V(j) may accumulate
#endif
    uint32_t tmem_base;
};

struct Params {
    const float* sq;
    const float* sk;
    const float* sv;
    float* o;
    int32_t n, d;
    int32_t n_pad;    // rows per slice of the fp16 V buffer (n rounded up to 128)
    int32_t o_pitch;  // floats per O row (even: the epilogue stores 8-byte pairs)
    int32_t o_tma;    // 1: the epilogue stages O in shared memory and TMA-stores it (tm_o)
    float sk_mul;  // log2(e) [* 1/sqrt(d)]: scores are kept in the log2 domain
    uint32_t flags;
    int32_t pairs, slices, items;
    // streamed step (ifa_int8_attention_step): the inputs of slice s are
    // ready once ready[s] >= ready_target (written by the concurrently
    // running stream quantizer, quant.cu); null = inputs already complete
    const uint32_t* ready;
    uint32_t ready_target;
    int32_t ready_from;  // slices below it were quantized before the launch
    int32_t max_ctas;    // grid cap (SMs left to the quantizer), 0 = all SMs
    // DUMP instantiation only: [slices][n][n] int32 S and uint8 P codes
    int32_t* s_dump;
    uint8_t* p_dump;
};

// -DIFA_PP_TRACE=1 (tools/build_variant.sh): clock64 stamps of CTA 0's
// pipeline events, read back with ifa_pp_trace_read (tools/pp_trace.py).
// role 0 = math warp 4 + 8g (rows 0-15 of group g), role 1 = MMA issuer g.
#ifdef IFA_PP_TRACE
__device__ unsigned long long g_pp_trace[2 * 2 * 1024 * 8];
#define PP_TR(role, g, t, ev)                                                             \
    do {                                                                                 \
        if (blockIdx.x == 0 && (t) < 1024)                                               \
            g_pp_trace[(((role) * 2 + (g)) * 1024 + (t)) * 8 + (ev)] = clock64();        \
    } while (0)
#else
#define PP_TR(role, g, t, ev) \
    do {                      \
    } while (0)
#endif

// Waits until the quantizer has published slice `slice` (acquire), then
// orders this thread's later async-proxy (TMA) reads after it.  Traps after
// ~4 s instead of hanging (a quantizer that cannot make progress).
__device__ __forceinline__ void wait_slice_ready(const Params& p, int32_t slice) {
    if (p.ready == nullptr || slice < p.ready_from) return;
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ready + slice) : "memory");
    if (v < p.ready_target) {
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
            __nanosleep(256);
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ready + slice)
                         : "memory");
            uint64_t t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 4000000000ull) __trap();
        } while (v < p.ready_target);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

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

// Work item -> (pair of Q tiles, slice, KV tiles the pair reads).
// Non-causal: the pairs of one slice are adjacent, so CTAs running together
// share the slice's K and V in L2.  Causal: the pairs nearest the diagonal
// end have the most keys and go first (longest-processing-time order);
// group g of pair t sees KV tiles 0 .. 2t + g and masks inside tile 2t + g.
// (A slice-major causal order measured slower on C3: worse balance.)
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
// The CTA's wi-th work item.  Causal: rounds of gridDim.x items taken in
// alternating directions (snake), so with the longest-first order no CTA gets
// the longest item of every round (C3 1.992 -> 1.875 ms); non-causal items are
// all equal: plain grid stride (the snake measured +0.6% at C2).
template <bool SNAKE>
__device__ __forceinline__ int32_t item_at(uint32_t wi) {
    const int32_t G = static_cast<int32_t>(gridDim.x), c = static_cast<int32_t>(blockIdx.x);
    const int32_t r = static_cast<int32_t>(wi);
    return r * G + ((SNAKE && (r & 1)) ? G - 1 - c : c);
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

__device__ __forceinline__ void ld16x256_x4(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void st16x256_x4(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
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

// MODE: what the weights and S are (the pipeline is the same).
//   kModeCodes (0): full-INT8 tolerance mode -- int8 S (kind::i8), P = the
//                   integer codes round(127 exp(s - m)), O * sV / l.
//   kModeHalf  (1): half-INT8 (attention.cpp:359-399) -- int8 S, float
//                   weights exp(s - m) as fp16, V = fp16 of the float V, O / l.
//   kModeFp8   (2): fp8_emulated_attention (attention.cpp:401-407) -- e4m3 S
//                   (kind::f8f6f4), one scale per slice, V = decoded e4m3,
//                   O / (l sV).
constexpr int kModeCodes = 0, kModeHalf = 1, kModeFp8 = 2;

__device__ __forceinline__ void mma_f8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// RAGGED: n is not a multiple of 128 (the last KV tile masks missing keys);
// a template parameter so the common case carries no masking code.
// STREAMED: the inputs of a slice are waited for per item (streamed step); a
// separate instantiation because the check costs the math warps registers.
// DUMP: also write S and the P codes to p.s_dump / p.p_dump (parity checks;
// a separate instantiation, so the product kernel carries no dump code).
template <int D, bool CAUSAL, int MODE, bool RAGGED, bool STREAMED = false, bool DUMP = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    int_flash_pp_kernel(const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_o, const Params p) {
    constexpr uint32_t kLayout = D == 128 ? kLayoutSw128 : kLayoutSw64;
    constexpr uint32_t kSbo = 8 * D;
    constexpr uint32_t kIdescS = MODE == kModeFp8
                                     ? ((1u << 4) | ((BN >> 3) << 17) | ((BM >> 4) << 24))
                                     : idesc_i8(BM, BN, false, false);
    constexpr uint32_t kIdescPV = idesc_f16(BM, D, true);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const int32_t n = p.n;
    const int32_t J = (n + BN - 1) / BN;  // KV tiles of a slice
    // compile-time: the non-causal instantiation carries no masking or
    // per-group tile-count logic (it measured 20% slower with them at run time)
    constexpr bool causal = CAUSAL;

    const uint32_t b_q_full = smem_u32(&sm.q_full), b_q_empty = smem_u32(&sm.q_empty);
    const uint32_t b_k_full = smem_u32(&sm.k_full[0]), b_k_empty = smem_u32(&sm.k_empty[0]);
    const uint32_t b_v_full = smem_u32(&sm.v_full[0]), b_v_empty = smem_u32(&sm.v_empty[0]);
    const uint32_t b_s_full = smem_u32(&sm.s_full[0]), b_s_empty = smem_u32(&sm.s_empty[0]);
    const uint32_t b_p_full = smem_u32(&sm.p_full[0]), b_p_empty = smem_u32(&sm.p_empty[0]);
    const uint32_t b_o_full = smem_u32(&sm.o_full[0]), b_o_free = smem_u32(&sm.o_free[0]);
#if IFA_PP_EPI
    const uint32_t b_epi_ready = smem_u32(&sm.epi_ready[0]);
#endif

    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023) __trap();
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_empty, 2);  // both MMA issuers
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.s_full[i], 1);
            mbar_init(&sm.s_empty[i], GROUP_WARPS);
            mbar_init(&sm.p_full[i], GROUP_WARPS);
            mbar_init(&sm.p_empty[i], 1);
            mbar_init(&sm.o_full[i], 1);
            mbar_init(&sm.o_free[i], kEpi ? EPI_WARPS : GROUP_WARPS);
#if IFA_PP_EPI
            mbar_init(&sm.epi_ready[i], GROUP_WARPS);
#endif
#if IFA_PP_CORR
            mbar_init(&sm.alpha_ready[i], GROUP_WARPS);
            mbar_init(&sm.o_ready[i], EPI_WARPS);
#endif
        }
        for (int i = 0; i < KST; ++i) {
            mbar_init(&sm.k_full[i], 32);
            mbar_init(&sm.k_empty[i], 2 + 2 * GROUP_WARPS);  // 2 MMA issuers + sK readers
        }
        for (int i = 0; i < VST; ++i) {
            mbar_init(&sm.v_full[i], 1);
            mbar_init(&sm.v_empty[i], 2);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

#if IFA_PP_EPI
    if (warp >= EPI_WARP0) {
        // ----------------------------------------------- epilogue warpgroup
        // Per item and group: O (TMEM, f32) x the group's per-row factor ->
        // global, one row per thread (32x32b loads: lane = row), 16 columns
        // = four 16-byte stores per step.  The math warps only publish the
        // factors (epi_f + epi_ready) and go on to the next item; the group's
        // next P.V(0) waits for o_free as before.
        regs_dealloc<kRegsEpi>();
        const uint32_t quarter = warp & 3;
        const int32_t row = static_cast<int32_t>(quarter * 32 + lane);
        const bool vec4 = p.o_pitch % 4 == 0 && (reinterpret_cast<uintptr_t>(p.o) & 15) == 0;
        uint32_t wi = 0;
        for (int32_t idx = item_at<causal>(wi); idx < p.items; idx = item_at<causal>(++wi)) {
            const PWork w = pwork(idx, p, causal, J);
#pragma unroll 1
            for (int g = 0; g < 2; ++g) {
                bar_wait(b_o_full + 8 * g, wi & 1);
                bar_wait(b_epi_ready + 8 * g, wi & 1);
                tc_fence_after();
                const float f = sm.epi_f[g][row];
                const int32_t grow = w.pair * 2 * BM + g * BM + row;
                const uint32_t t_o = tmem + ((quarter * 32) << 16) + 256 * g + 128;
                float* orow = p.o + (static_cast<int64_t>(w.slice) * n + grow) * p.o_pitch;
#pragma unroll 1
                for (int c = 0; c < D / 16; ++c) {
                    uint32_t o[16];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]),
                          "=r"(o[6]), "=r"(o[7]), "=r"(o[8]), "=r"(o[9]), "=r"(o[10]), "=r"(o[11]),
                          "=r"(o[12]), "=r"(o[13]), "=r"(o[14]), "=r"(o[15])
                        : "r"(t_o + 16 * c));
                    tmem_wait_ld();
                    if (c == D / 16 - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) bar_arrive(b_o_free + 8 * g);
                    }
                    if constexpr (kEpi2) {
                        // 16-byte chunk v of row r at chunk v ^ ((r >> 1) & 3) of
                        // its 64-byte line (SWIZZLE_64B): conflict-free quarter warps
                        const uint32_t buf = smem_u32(sm.epi_stage[quarter][c & 1]);
                        if (c >= 2) {  // box c - 2 (same buffer) has been read
                            if (lane == 0) tma_store_wait_read_but1();
                            __syncwarp();
                        }
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const uint32_t chunk = static_cast<uint32_t>(v) ^ ((lane >> 1) & 3);
                            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                             buf + lane * 64 + chunk * 16),
                                         "f"(__uint_as_float(o[4 * v]) * f),
                                         "f"(__uint_as_float(o[4 * v + 1]) * f),
                                         "f"(__uint_as_float(o[4 * v + 2]) * f),
                                         "f"(__uint_as_float(o[4 * v + 3]) * f)
                                         : "memory");
                        }
                        fence_proxy_async_shared();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_3d(&tm_o, sm.epi_stage[quarter][c & 1], 16 * c,
                                         w.pair * 2 * BM + g * BM + static_cast<int32_t>(quarter) * 32,
                                         w.slice);
                            tma_store_commit();
                        }
                        continue;
                    }
                    if (grow < n) {
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int col = 16 * c + 4 * v;
                            const float4 x = make_float4(__uint_as_float(o[4 * v]) * f,
                                                         __uint_as_float(o[4 * v + 1]) * f,
                                                         __uint_as_float(o[4 * v + 2]) * f,
                                                         __uint_as_float(o[4 * v + 3]) * f);
                            if (vec4 && col + 3 < p.d) {
                                __stcs(reinterpret_cast<float4*>(orow + col), x);
                            } else {
                                if (col < p.d) orow[col] = x.x;
                                if (col + 1 < p.d) orow[col + 1] = x.y;
                                if (col + 2 < p.d) orow[col + 2] = x.z;
                                if (col + 3 < p.d) orow[col + 3] = x.w;
                            }
                        }
                    }
                }
                if constexpr (kEpi2) {  // the next group's boxes reuse the buffers
                    if (lane == 0) tma_store_wait_read();
                    __syncwarp();
                }
            }
        }
        if constexpr (kEpi2) {
            if (lane == 0) tma_store_wait_all();
        }
    } else
#endif
#if IFA_PP_CORR
    if (warp >= EPI_WARP0) {
        // ------------------------------------------------- correction warpgroup
        // Thread = one row of its lane quarter (32x32b loads).  Serves the two
        // groups in whichever order their alpha arrive (non-blocking polls);
        // the math warps publish alpha(t) once P.V(t-1) has completed.
        regs_dealloc<kRegsEpi>();
        const uint32_t quarter = warp & 3;
        const uint32_t row = quarter * 32 + lane;
        uint32_t total[2] = {0u, 0u};
        {
            uint32_t wi = 0;
            for (int32_t idx = item_at<causal>(wi); idx < p.items; idx = item_at<causal>(++wi)) {
                const PWork w = pwork(idx, p, causal, J);
                total[0] += static_cast<uint32_t>(group_tiles(w, 0, causal, J));
                total[1] += static_cast<uint32_t>(group_tiles(w, 1, causal, J));
            }
        }
        const uint32_t b_alpha = smem_u32(&sm.alpha_ready[0]), b_oready = smem_u32(&sm.o_ready[0]);
        uint32_t tcg[2] = {0u, 0u};
        while (tcg[0] < total[0] || tcg[1] < total[1]) {
            bool did = false;
#pragma unroll
            for (int g = 0; g < 2; ++g) {  // unrolled: tcg / total stay in registers
                const uint32_t t = tcg[g];
                if (t >= total[g]) continue;
                int ready = 0;
                if (lane == 0) ready = bar_try(b_alpha + 8 * g, t & 1);  // implies P.V(t-1) done
                if (!__shfl_sync(0xffffffffu, ready, 0)) continue;
                tc_fence_after();
                const float a = sm.alpha[g][t & 1][row];
                if (__any_sync(0xffffffffu, a != 1.0f)) {
                    const uint32_t t_o = tmem + ((quarter * 32) << 16) + 256 * g + 128;
#pragma unroll 1
                    for (int c = 0; c < D / IFA_PP_CORR_COLS; ++c) {
                        uint32_t o[IFA_PP_CORR_COLS];
                        if constexpr (IFA_PP_CORR_COLS == 16) {
                            tmem_ld16(t_o + 16 * c, o);
                        } else {
                            tmem_ld8(t_o + 8 * c, o);
                        }
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < IFA_PP_CORR_COLS; e += 2) {
                            const float2 v = fmul2(make_float2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])),
                                                   f2(a));
                            o[e] = __float_as_uint(v.x);
                            o[e + 1] = __float_as_uint(v.y);
                        }
                        if constexpr (IFA_PP_CORR_COLS == 16) {
                            tmem_st16(t_o + 16 * c, o);
                        } else {
                            tmem_st8(t_o + 8 * c, o);
                        }
                    }
                    tmem_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(b_oready + 8 * g);
                tcg[g] = t + 1;
                did = true;
            }
            if (!did) __nanosleep(IFA_PP_CORR_SLEEP_NS);  // a poll costs the math warps issue slots
        }
    } else
#endif
    if (warp < CTRL_WARPS) {
        regs_dealloc<kRegsControl>();
        if (warp == 0) {
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
            for (int32_t idx = item_at<causal>(wi); idx < p.items; idx = item_at<causal>(++wi)) {
                const PWork w = pwork(idx, p, causal, J);
                const int32_t q0 = w.pair * 2 * BM, slice = w.slice;
                if constexpr (STREAMED) wait_slice_ready(p, slice);  // every lane: sK loads below
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
                    if constexpr (MODE == kModeFp8) {  // s = S / (sQ sK): one constant per slice
                        // an all-zero Q or K slice has scale 0 and zero codes: its
                        // scores are 0 (fp8_e4m3_roundtrip returns zeros, fp8.cpp:78-97)
                        const float sqk = __fmul_rn(p.sq[slice], p.sk[slice]);
                        const float c8 = sqk == 0.0f ? 0.0f : __fdiv_rn(p.sk_mul, sqk);
                        k4 = make_float4(c8, c8, c8, c8);
                    } else {
                        const int32_t key = key0 + 4 * lane;
                        if (key + 3 < n &&
                            (reinterpret_cast<uintptr_t>(sk_slice + key) & 15) == 0) {
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
                    }
                    reinterpret_cast<float4*>(sm.sk[ks])[lane] = k4;
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&sm.k_full[ks], BN * D);
                        tma_load_3d(sm.k[ks], &tm_k, &sm.k_full[ks], 0, key0, slice, pol_keep);
                        if (i >= VST) bar_wait(b_v_empty + 8 * vs, vr.phase ^ 1u);
                        mbar_arrive_expect_tx(&sm.v_full[vs], BN * D * 2);
                        const int32_t tile = (slice * p.n_pad + key0) / 64;  // 64-key halves
#pragma unroll
                        for (int h = 0; h < D / 64; ++h)
                            tma_load_5d(sm.v[vs] + h * BN * 128, &tm_v, &sm.v_full[vs], 64 * h,
                                        0, 0, 0, tile, pol_keep);
                    } else {
                        bar_arrive(b_k_full + 8 * ks);
                    }
                    kr.advance();
                    vr.advance();
                    ++i;
                }
            }
        } else if (warp == 1 || warp == 2) {
            // ------------------------------------------- MMA issuers (one per group)
            // Warp 1 issues group 0's MMAs, warp 2 group 1's, so neither group
            // waits on the other's progress.  Per block j: S(next) as soon as the
            // group has read S(j), then P.V(j) once it has published P(j).
            // The whole warp runs the loop (warp-uniform descriptors live in
            // uniform registers) and one elected lane issues each batch: with
            // only lane 0 running it, every descriptor went through R2UR and an
            // MMA took ~135 cycles to issue (tools/pp_trace.py), twice the
            // tensor core's own 65-90 (tools/microbench/mma_issue.cu).
            {
                const int g = static_cast<int>(warp) - 1;
                Ring<KST> kr;     // K stage of block j
                Ring<VST> vr;     // V stage of block j
                uint32_t t = 0;   // tiles of this group so far
                uint32_t wi = 0;
                const uint32_t d_s = tmem + 256 * g, d_o = d_s + 128;
                // descriptor + (byte offset >> 4) addresses the same layout at an
                // offset (shared memory < 256 KiB: no carry out of the 14-bit field)
                const uint64_t q_desc_base = smem_desc(smem_u32(sm.q[g]), 16, kSbo, kLayout);
                const uint64_t p_desc_base = smem_desc(smem_u32(sm.p[g]), 16, 1024, kLayoutSw128);
                auto launder = [](uint64_t x) {
                    if constexpr (IFA_PP_LAUNDER) asm volatile("mov.b64 %0, %0;" : "+l"(x));
                    return x;
                };
                auto issue_s = [&](uint32_t ks, uint32_t kph) {
                    bar_wait(b_k_full + 8 * ks, kph);
                    tc_fence_after();
                    const uint64_t k_desc = smem_desc(smem_u32(sm.k[ks]), 16, kSbo, kLayout);
                    const uint64_t q_desc = launder(q_desc_base);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < D / 32; ++kk) {
                            if constexpr (MODE == kModeFp8)
                                mma_f8_ss(d_s, q_desc + 2 * kk, k_desc + 2 * kk, kIdescS,
                                          kk > 0 ? 1u : 0u);
                            else
                                mma_i8_ss(d_s, q_desc + 2 * kk, k_desc + 2 * kk, kIdescS,
                                          kk > 0 ? 1u : 0u);
                        }
                        mma_commit_u32(b_s_full + 8 * g);
                    }
                    __syncwarp();
                };
                if (blockIdx.x < p.items) {
                    bar_wait(b_q_full, 0);
                    issue_s(0, 0);
                }
                for (int32_t idx = item_at<causal>(wi); idx < p.items; idx = item_at<causal>(++wi)) {
                    const bool has_next_item = item_at<causal>(wi + 1) < p.items;
                    const PWork w = pwork(idx, p, causal, J);
                    const int32_t jg = group_tiles(w, g, causal, J);
                    for (int32_t j = 0; j < w.jt; ++j) {
                        if (j >= jg) {  // causal: a KV tile only the other group reads
                            bar_wait(b_k_full + 8 * kr.idx, kr.phase);
                            if (elect_one()) bar_arrive(b_k_empty + 8 * kr.idx);
                            __syncwarp();
                            bar_wait(b_v_full + 8 * vr.idx, vr.phase);
                            if (elect_one()) bar_arrive(b_v_empty + 8 * vr.idx);
                            __syncwarp();
                            kr.advance();
                            vr.advance();
                            continue;
                        }
                        const bool last = j == jg - 1;
                        if (elect_one()) {
                            mma_commit_u32(b_k_empty + 8 * kr.idx);  // S(j) issued
                            if (last) mma_commit_u32(b_q_empty);     // every S of this item issued
                        }
                        __syncwarp();
                        // next S: tile j+1 now; tile 0 of the next item (jt - j ring
                        // positions ahead) only after this item's last P.V, which the
                        // epilogue waits for -- not behind the next item's Q load
                        auto next_s = [&]() {
                            Ring<KST> nk = kr;
                            const int32_t ahead = last ? w.jt - j : 1;
                            for (int32_t a = 0; a < ahead; ++a) nk.advance();
                            bar_wait(b_s_empty + 8 * g, t & 1);
                            issue_s(nk.idx, nk.phase);
                            if (lane == 0) PP_TR(1, g, t, 0);
                        };
                        if (!last) next_s();
                        bar_wait(b_v_full + 8 * vr.idx, vr.phase);
                        const uint64_t v_desc =
                            smem_desc(smem_u32(sm.v[vr.idx]), BN * 128, 1024, kLayoutSw128);
                        bar_wait(b_p_full + 8 * g, t & 1);
#if IFA_PP_CORR
                        bar_wait(smem_u32(&sm.o_ready[g]), t & 1);  // O(j-1) rescaled
#endif
                        if (lane == 0) PP_TR(1, g, t, 1);
                        if (j == 0 && wi > 0) bar_wait(b_o_free + 8 * g, (wi - 1) & 1);
                        tc_fence_after();
                        const uint64_t p_desc = launder(p_desc_base);
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < BN / 16; ++kk)
                                mma_f16_ss(d_o, p_desc + (kk >> 2) * (BM * 128 / 16) + (kk & 3) * 2,
                                           v_desc + kk * (16 * 128 / 16), kIdescPV,
                                           (j == 0 && kk == 0) ? 0u : 1u);
                            mma_commit_u32(b_p_empty + 8 * g);
                            if (last) mma_commit_u32(b_o_full + 8 * g);
                            mma_commit_u32(b_v_empty + 8 * vr.idx);
                        }
                        __syncwarp();
                        if (lane == 0) PP_TR(1, g, t, 2);
                        if (last && has_next_item) {
                            bar_wait(b_q_full, (wi + 1) & 1);
                            next_s();
                        }
                        kr.advance();
                        vr.advance();
                        ++t;
                    }
                }
            }
            __syncwarp();
        }
    } else {
        regs_alloc<kRegsMath>();
        // -------------------------------------------- softmax + correction
        const uint32_t mw = warp - CTRL_WARPS;
        const uint32_t g = mw >> 3;                 // Q tile / group
        const uint32_t quarter = warp & 3;          // TMEM lane quarter of this warp
        const uint32_t half = (mw >> 2) & 1;        // which 16 lanes of the quarter
        const uint32_t t0 = lane & 3;
        const uint32_t lane_base = quarter * 32 + half * 16;
        const int32_t row0 = static_cast<int32_t>(lane_base + (lane >> 2));  // and row0 + 8
        const uint32_t t_s = tmem + (lane_base << 16) + 256 * g;  // S
        const uint32_t t_o = t_s + 128;                            // O
        const uint32_t bs_full = b_s_full + 8 * g, bs_empty = b_s_empty + 8 * g;
        const uint32_t bp_full = b_p_full + 8 * g, bp_empty = b_p_empty + 8 * g;
        const uint32_t bo_full = b_o_full + 8 * g, bo_free = b_o_free + 8 * g;
        // P (fp16, K-major SW128, two 64-key atoms): thread t0 of a row owns MMA
        // keys [16 t0, 16 t0 + 16) of each atom = 16-byte chunks 2 t0, 2 t0 + 1,
        // XOR-swizzled by r & 7.  The eight lanes of a quarter warp (two rows x
        // four t0) then hit eight different bank groups: no store conflicts.
        uint32_t p_row[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const uint32_t row = static_cast<uint32_t>(row0) + 8 * r;
            p_row[r] = smem_u32(sm.p[g]) + row * 128;
        }
        const uint32_t sw = static_cast<uint32_t>(row0) & 7;  // same for row0 + 8
        Ring<KST> kv;
        uint32_t tc = 0, wi = 0;
        // the previous item's O boxes (TMA epilogue) may still be reading the
        // P buffer: the first P stores of the next item wait for them
        bool o_pending = false;
        const bool o_issuer = (mw & 7) == 0 && lane == 0;
        auto o_reads_done = [&]() {
            if (o_pending) {
                if (o_issuer) tma_store_wait_read();
                named_bar_sync(1 + g, 256);
                o_pending = false;
            }
        };

        // group 1 starts ~1 us after group 0: started together, the two groups
        // run their MUFU-heavy and barrier-bound phases in lockstep on the same
        // sub-partitions (measured 0.994 -> 0.983 ms at C2, C5 -0.5%; per-item
        // delays hurt)
        if (IFA_PP_G1_DELAY_NS > 0 && g == 1) __nanosleep(IFA_PP_G1_DELAY_NS);
        // sQ of the item's rows and sV of its slice, loaded one item ahead so
        // the global-load latency (~700 cycles each) is not paid at the item
        // boundary (the streamed step loads them after its per-slice wait)
        auto load_scales = [&](int32_t item, float (&q_s)[2], float& v_s) {
            if (item >= p.items) return;
            const PWork nw = pwork(item, p, causal, J);
            const int32_t nq0 = nw.pair * 2 * BM + static_cast<int32_t>(g) * BM;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int32_t gr = nq0 + row0 + 8 * r;
                if constexpr (MODE == kModeFp8)
                    q_s[r] = 1.0f;  // the scales are in the per-key constant
                else
                    q_s[r] = gr < n ? p.sq[static_cast<int64_t>(nw.slice) * n + gr] : 0.0f;
            }
            v_s = MODE == kModeHalf ? 1.0f : p.sv[nw.slice];
        };
        float nsq[2] = {0.0f, 0.0f}, nsv = 0.0f;
        if constexpr (!STREAMED) load_scales(item_at<causal>(wi), nsq, nsv);
        for (int32_t idx = item_at<causal>(wi); idx < p.items; idx = item_at<causal>(++wi)) {
            const PWork w = pwork(idx, p, causal, J);
            const int32_t jg = group_tiles(w, static_cast<int>(g), causal, J);
            const int32_t diag = causal ? 2 * w.pair + static_cast<int32_t>(g) : -1;
            const int32_t q0 = w.pair * 2 * BM + static_cast<int32_t>(g) * BM;
            const int32_t slice = w.slice;
            if constexpr (STREAMED) {
                wait_slice_ready(p, slice);  // sQ, sV of a streamed step
                load_scales(idx, nsq, nsv);
            }
            int32_t grow[2];
            float sq[2] = {nsq[0], nsq[1]};
            const float sv_item = nsv;
#pragma unroll
            for (int r = 0; r < 2; ++r) grow[r] = q0 + row0 + 8 * r;
            if constexpr (!STREAMED) load_scales(item_at<causal>(wi + 1), nsq, nsv);
            float l[2] = {0.0f, 0.0f}, m[2] = {-__int_as_float(0x7f800000), -__int_as_float(0x7f800000)};

            for (int32_t j = 0; j < w.jt; ++j) {
                const uint32_t st = kv.idx;
                if (j >= jg) {  // causal: the other group's diagonal tile
                    bar_wait(b_k_full + 8 * st, kv.phase);
                    __syncwarp();
                    if (lane == 0) bar_arrive(b_k_empty + 8 * st);
                    kv.advance();
                    continue;
                }
                const bool tr = (mw & 7) == 0 && lane == 0;
                if (tr) PP_TR(0, g, tc, 7);
                bar_wait(bs_full, tc & 1);
                if (tr) PP_TR(0, g, tc, 0);
                tc_fence_after();
                uint32_t sr[64];
                // IFA_PP_SPLIT_SLOAD: the second half of S is loaded while the
                // first half is converted (tcgen05.wait::ld waits for every load)
                constexpr bool split_sload = IFA_PP_SPLIT_SLOAD && !DUMP;
#pragma unroll
                for (int c = 0; c < (split_sload ? 2 : 4); ++c) ld16x256_x4(t_s + 32 * c, &sr[16 * c]);
                tmem_wait_ld();
                if constexpr (split_sload) {
#pragma unroll
                    for (int c = 2; c < 4; ++c) ld16x256_x4(t_s + 32 * c, &sr[16 * c]);
                }
                if constexpr (DUMP) {  // sr[4k + 2r + e]: row row0 + 8r, key 8k + 2 t0 + e
                    if (p.s_dump != nullptr) {
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            if (grow[r] >= n) continue;
                            int32_t* dst = p.s_dump + (static_cast<int64_t>(slice) * n + grow[r]) * n;
#pragma unroll
                            for (int k = 0; k < 16; ++k)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int32_t key = j * BN + 8 * k + 2 * static_cast<int32_t>(t0) + e;
                                    if (key < n) dst[key] = static_cast<int32_t>(sr[4 * k + 2 * r + e]);
                                }
                        }
                    }
                }
                if constexpr (!split_sload) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(bs_empty);
                }
                if (tr) PP_TR(0, g, tc, 1);
                bar_wait(b_k_full + 8 * st, kv.phase);
                // u = float(S) * sK * log2(e); sr[4k + {0,1}] row0, [4k + {2,3}] row1,
                // keys 8k + 2*t0 + {0,1}
                float u[64];
                const float* skc = sm.sk[st] + 2 * t0;
                [[maybe_unused]] uint32_t one = 1u;
                if constexpr (kMagicCvt >= 4) asm volatile("mov.b32 %0, %0;" : "+r"(one));
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    if (split_sload && k == 8) {  // the second half of S is in registers
                        tmem_wait_ld();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) bar_arrive(bs_empty);
                    }
                    const float2 s2 = *reinterpret_cast<const float2*>(skc + 8 * k);
                    float2 fa, fb;  // S as f32: exact int32 (kind::i8) or f32 (kind::f8f6f4)
                    if constexpr (MODE == kModeFp8) {
                        fa = make_float2(__uint_as_float(sr[4 * k]), __uint_as_float(sr[4 * k + 1]));
                        fb = make_float2(__uint_as_float(sr[4 * k + 2]), __uint_as_float(sr[4 * k + 3]));
                    } else if (kMagicCvt >= 4 && (kMagicCvt == 4 || (kMagicCvt == 5 && (k & 1)) ||
                                                  (kMagicCvt == 6 && (k & 3) == 3))) {
                        uint32_t x[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x[e])
                                : "r"(sr[4 * k + e]), "r"(one), "r"(0x4B400000u));
                        fa = fsub2(make_float2(__uint_as_float(x[0]), __uint_as_float(x[1])), f2(kMagic));
                        fb = fsub2(make_float2(__uint_as_float(x[2]), __uint_as_float(x[3])), f2(kMagic));
                    } else if (kMagicCvt == 1 || (kMagicCvt == 2 && (k & 1)) ||
                               (kMagicCvt == 3 && (k & 3) == 3)) {
                        // |S| <= 127^2 * 128 < 2^22: the bits of S + 0x4B400000 are
                        // the float 1.5 * 2^23 + S, so one exact packed subtract
                        // leaves float(S) (integer adds on the ALU instead of the
                        // quarter-rate I2F pipe)
                        fa = fsub2(make_float2(__uint_as_float(sr[4 * k] + 0x4B400000u),
                                               __uint_as_float(sr[4 * k + 1] + 0x4B400000u)),
                                   f2(kMagic));
                        fb = fsub2(make_float2(__uint_as_float(sr[4 * k + 2] + 0x4B400000u),
                                               __uint_as_float(sr[4 * k + 3] + 0x4B400000u)),
                                   f2(kMagic));
                    } else {
                        fa = make_float2(__int2float_rn(static_cast<int32_t>(sr[4 * k])),
                                         __int2float_rn(static_cast<int32_t>(sr[4 * k + 1])));
                        fb = make_float2(__int2float_rn(static_cast<int32_t>(sr[4 * k + 2])),
                                         __int2float_rn(static_cast<int32_t>(sr[4 * k + 3])));
                    }
                    const float2 a = fmul2(fa, s2);
                    const float2 b = fmul2(fb, s2);
                    u[4 * k] = a.x;
                    u[4 * k + 1] = a.y;
                    u[4 * k + 2] = b.x;
                    u[4 * k + 3] = b.y;
                }
                __syncwarp();
                if (lane == 0) bar_arrive(b_k_empty + 8 * st);
                // rest of the tile, instantiated twice so the diagonal masking of
                // the causal kernel never becomes per-element predicated code on the
                // other tiles
                auto rest = [&](auto mask_tag) {
                    constexpr bool dmask = decltype(mask_tag)::value;  // keys > kmax masked
                    // last visible key of each row in this tile (masked tiles only):
                    // the causal diagonal and / or the ragged end of the sequence
                    int32_t kmax[2] = {BN - 1, BN - 1};
                    if (dmask) {
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            if (RAGGED && n - j * BN - 1 < kmax[r]) kmax[r] = n - j * BN - 1;
                            if (causal && j == diag && row0 + 8 * r < kmax[r]) kmax[r] = row0 + 8 * r;
                        }
                    }
                    if (dmask) {
    #pragma unroll
                        for (int k = 0; k < 16; ++k)
    #pragma unroll
                            for (int r = 0; r < 2; ++r)
    #pragma unroll
                                for (int e = 0; e < 2; ++e)
                                    if (8 * k + 2 * static_cast<int32_t>(t0) + e > kmax[r])
                                        u[4 * k + 2 * r + e] = -__int_as_float(0x7f800000);
                    }
                    float cr[2], alpha[2], tmax[2];
    #pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        float a[11];
    #pragma unroll
                        for (int jj = 0; jj < 10; ++jj) {
                            const int v0 = 3 * jj, v1 = 3 * jj + 1, v2 = 3 * jj + 2;
                            a[jj] = fmax3(u[4 * (v0 >> 1) + 2 * r + (v0 & 1)],
                                          u[4 * (v1 >> 1) + 2 * r + (v1 & 1)],
                                          u[4 * (v2 >> 1) + 2 * r + (v2 & 1)]);
                        }
                        a[10] = fmaxf(u[4 * 15 + 2 * r], u[4 * 15 + 2 * r + 1]);
                        float b = fmaxf(fmax3(fmax3(a[0], a[1], a[2]), fmax3(a[3], a[4], a[5]),
                                              fmax3(a[6], a[7], a[8])),
                                        fmaxf(a[9], a[10]));
                        b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 1));
                        b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 2));
                        const float mnew = (m[r] < b) ? b : m[r];
                        cr[r] = (MODE == kModeCodes ? kLog2_127 : 0.0f) - sq[r] * mnew;
                        tmax[r] = __fmaf_rn(sq[r], b, cr[r]);  // largest exponent of the row
                        alpha[r] = (j == 0 || mnew == m[r]) ? 1.0f : ex2(sq[r] * (m[r] - mnew));
                        m[r] = mnew;
                    }

                    if (tr) PP_TR(0, g, tc, 2);
                    // weights: 6 of 8 exp2 on MUFU, 2 on the FMA pipe.
                    // wd[r][k] = keys (8k + 2t0, +1) of row r as fp16x2.
                    uint32_t wd[2][16];
                    float lsum[2];
                    // words 4i..4i+3 of row r = pairs k = 4i..4i+3: atom i >> 1,
                    // chunk 2 t0 + (i & 1)
                    auto store_p = [&](int r, int i, const uint32_t (&w)[2][16]) {
                        const uint32_t chunk = (2 * t0 + (i & 1)) ^ sw;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         p_row[r] + (i >> 1) * (BM * 128) + chunk * 16),
                                     "r"(w[r][4 * i]), "r"(w[r][4 * i + 1]),
                                     "r"(w[r][4 * i + 2]), "r"(w[r][4 * i + 3])
                                     : "memory");
                    };
                    constexpr bool early_p = IFA_PP_EARLY_P;
                    if constexpr (early_p) {
                        // P.V(j-1) has long finished by now: P is stored as it is made
                        if (tc > 0) bar_wait(bp_empty, (tc - 1) & 1);
#if IFA_PP_CORR
                        // alpha to the correction warps, after P.V(j-1) is done: so
                        // alpha_ready(j) also says O(j-1) is final, and can never run
                        // two phases ahead of the correction warps (P.V(j) waits for them)
                        if (t0 == 0) {
                            sm.alpha[g][tc & 1][row0] = alpha[0];
                            sm.alpha[g][tc & 1][row0 + 8] = alpha[1];
                        }
                        __syncwarp();
                        if (lane == 0) bar_arrive(smem_u32(&sm.alpha_ready[g]));
#endif
                        o_reads_done();
                        if (tr) PP_TR(0, g, tc, 3);
                        tc_fence_after();
                    }
                    if constexpr (MODE == kModeCodes) {
                        // full-INT8: y + 1.5*2^23 has the code round(y) in its low
                        // bits; its low 16 bits read as fp16 are the subnormal
                        // code * 2^-24, exact, so one PRMT packs two codes (P.V
                        // then accumulates 2^-24 * the integer P.V, undone in the
                        // epilogue).  Row sums add the packed words as integers:
                        // <= 16 * 127 per half, no carry between the halves.
                        uint32_t acc[2] = {0u, 0u};
                        const bool sparse =
                            IFA_PP_SPARSE &&
                            __popc(__ballot_sync(0xffffffffu, !(tmax[0] < -1.0f) || !(tmax[1] < -1.0f))) <=
                                IFA_PP_SPARSE_HOT;
                        auto code_loop = [&](auto sparse_tag) {
                            constexpr bool SP = decltype(sparse_tag)::value;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                float2 t[2];
#pragma unroll
                                for (int r = 0; r < 2; ++r)
                                    t[r] = ffma2(make_float2(u[4 * k + 2 * r], u[4 * k + 2 * r + 1]),
                                                 f2(sq[r]), f2(cr[r]));
                                bool hot = true;
                                if constexpr (SP)  // warp-uniform: skip when every code is 0
                                    hot = __any_sync(0xffffffffu,
                                                     fmaxf(fmaxf(t[0].x, t[0].y), fmaxf(t[1].x, t[1].y)) >= -1.0f);
                                if (!SP || hot) {
#pragma unroll
                                    for (int r = 0; r < 2; ++r) {
                                        const float2 y = (k & kPolyMask) == kPolyMask
                                                             ? exp2_poly2(t[r])
                                                             : make_float2(ex2(t[r].x), ex2(t[r].y));
                                        float2 c = fadd2(y, f2(kMagic));
                                        if (dmask) {  // masked keys are code 0 (also when sQ == 0)
                                            const int32_t key = 8 * k + 2 * static_cast<int32_t>(t0);
                                            if (key > kmax[r]) c.x = kMagic;
                                            if (key + 1 > kmax[r]) c.y = kMagic;
                                        }
                                        wd[r][k] = prmt(__float_as_uint(c.x), __float_as_uint(c.y), 0x5410u);
                                    }
                                } else {
                                    wd[0][k] = 0u;
                                    wd[1][k] = 0u;
                                }
#pragma unroll
                                for (int r = 0; r < 2; ++r)
                                    if (k & 1) acc[r] += wd[r][k - 1] + wd[r][k];
                                if (early_p && (k & 3) == 3) {
                                    store_p(0, k >> 2, wd);
                                    store_p(1, k >> 2, wd);
                                }
                            }
                        };
                        if (sparse)
                            code_loop(std::true_type{});
                        else
                            code_loop(std::false_type{});
#pragma unroll
                        for (int r = 0; r < 2; ++r)
                            lsum[r] = static_cast<float>(static_cast<int32_t>((acc[r] & 0xffffu) + (acc[r] >> 16)));
                        if constexpr (DUMP) {  // wd[r][k]: codes of keys 8k + 2 t0 + {0, 1} (low bytes)
                            if (p.p_dump != nullptr) {
#pragma unroll
                                for (int r = 0; r < 2; ++r) {
                                    if (grow[r] >= n) continue;
                                    uint8_t* dst = p.p_dump + (static_cast<int64_t>(slice) * n + grow[r]) * n;
#pragma unroll
                                    for (int k = 0; k < 16; ++k) {
                                        const int32_t key = j * BN + 8 * k + 2 * static_cast<int32_t>(t0);
                                        if (key < n) dst[key] = static_cast<uint8_t>(wd[r][k] & 0xffu);
                                        if (key + 1 < n) dst[key + 1] = static_cast<uint8_t>((wd[r][k] >> 16) & 0xffu);
                                    }
                                }
                            }
                        }
                    } else {
                        // half-INT8 / FP8: the float weights, rounded to fp16
                        float2 ls[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
#pragma unroll
                            for (int r = 0; r < 2; ++r) {
                                const float2 t = ffma2(make_float2(u[4 * k + 2 * r], u[4 * k + 2 * r + 1]),
                                                       f2(sq[r]), f2(cr[r]));
                                float2 c = (k & kPolyMask) == kPolyMask ? exp2_poly2(t)
                                                         : make_float2(ex2(t.x), ex2(t.y));
                                if (dmask) {  // masked keys weigh 0
                                    const int32_t key = 8 * k + 2 * static_cast<int32_t>(t0);
                                    if (key > kmax[r]) c.x = 0.0f;
                                    if (key + 1 > kmax[r]) c.y = 0.0f;
                                }
                                ls[r] = fadd2(ls[r], c);
                                const __half2 h = __floats2half2_rn(c.x, c.y);
                                wd[r][k] = *reinterpret_cast<const uint32_t*>(&h);
                            }
                            if (early_p && (k & 3) == 3) {
                                store_p(0, k >> 2, wd);
                                store_p(1, k >> 2, wd);
                            }
                        }
#pragma unroll
                        for (int r = 0; r < 2; ++r) lsum[r] = ls[r].x + ls[r].y;
                    }
                    // P.V(j-1) done: the P buffer is free and O(j-1) is final
                    if constexpr (!early_p) {
                        if (tc > 0) bar_wait(bp_empty, (tc - 1) & 1);
                        o_reads_done();
                        tc_fence_after();
                    }
                    if (tr) PP_TR(0, g, tc, 4);
                    const bool need = !kCorr && j > 0 && (alpha[0] != 1.0f || alpha[1] != 1.0f);
                    if (__any_sync(0xffffffffu, need)) {
    #pragma unroll
                        for (int c = 0; c < D / 32; ++c) {
                            uint32_t o[16];
                            ld16x256_x4(t_o + 32 * c, o);
                            tmem_wait_ld();
    #pragma unroll
                            for (int k = 0; k < 4; ++k)
    #pragma unroll
                                for (int r = 0; r < 2; ++r) {
                                    const float2 v = fmul2(make_float2(__uint_as_float(o[4 * k + 2 * r]),
                                                                       __uint_as_float(o[4 * k + 2 * r + 1])),
                                                           f2(alpha[r]));
                                    o[4 * k + 2 * r] = __float_as_uint(v.x);
                                    o[4 * k + 2 * r + 1] = __float_as_uint(v.y);
                                }
                            st16x256_x4(t_o + 32 * c, o);
                        }
                        tmem_wait_st();
                    }
                    if constexpr (!early_p) {
#pragma unroll
                        for (int r = 0; r < 2; ++r)
#pragma unroll
                            for (int i = 0; i < 4; ++i) store_p(r, i, wd);
                    }
                    fence_proxy_async_shared();  // P is read by the tensor core
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(bp_full);
                    if (tr) PP_TR(0, g, tc, 5);

#pragma unroll
                    for (int r = 0; r < 2; ++r) l[r] = __fmaf_rn(l[r], alpha[r], lsum[r]);
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
            // epilogue: O * sV / l, l summed over the quad
            float f[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                float lt = l[r];
                lt += __shfl_xor_sync(0xffffffffu, lt, 1);
                lt += __shfl_xor_sync(0xffffffffu, lt, 2);
                if constexpr (MODE == kModeCodes)
                    f[r] = __fdiv_rn(sv_item, lt);
                else if constexpr (MODE == kModeHalf)
                    f[r] = __fdiv_rn(1.0f, lt);  // finalize_softmax_state (attention.cpp:139-149)
                else
                    // V = decode / sV; an all-zero V slice (sV = 0) gives O = 0
                    f[r] = sv_item == 0.0f ? 0.0f : __fdiv_rn(__fdiv_rn(1.0f, lt), sv_item);
            }
#if IFA_PP_EPI
            {
                // hand the factors to the epilogue warpgroup; it has read the
                // previous item's (o_free), and by induction o_free is at most
                // one phase behind here, so the parity wait is unambiguous
                constexpr float os = MODE == kModeCodes ? 16777216.0f : 1.0f;
                if (wi > 0) bar_wait(bo_free, (wi - 1) & 1);
                if (t0 == 0) {
                    sm.epi_f[g][row0] = f[0] * os;
                    sm.epi_f[g][row0 + 8] = f[1] * os;
                }
                __syncwarp();
                if (lane == 0) bar_arrive(b_epi_ready + 8 * g);
                continue;
            }
#endif
            const bool tre = (mw & 7) == 0 && lane == 0;
            if (tre) PP_TR(1, g, tc - 1, 5);
            bar_wait(bo_full, wi & 1);
            if (tre) PP_TR(1, g, tc - 1, 6);
            tc_fence_after();
            if (p.o_tma) {
                // Stage O through the group's (now idle) P buffer, 64 columns
                // at a time as two 128 x 32 f32 SW128 boxes, and TMA-store it:
                // full-line writes by the TMA engine instead of 8-byte stores
                // scattered over 8 rows per instruction (~6,000 cycles per item
                // epilogue, tools/pp_trace.py).  Rows past n are clipped by TMA.
                constexpr float os = MODE == kModeCodes ? 16777216.0f : 1.0f;
                const uint32_t stage = smem_u32(sm.p[g]);
                [[maybe_unused]] const bool issuer = (mw & 7) == 0 && lane == 0;
if constexpr (IFA_PP_OSTG) {
                // Stage 64 columns at a time in the P buffer (same swizzled
                // boxes), then read them back row-contiguously and store with
                // 16-byte global stores, 512 contiguous bytes per half-warp:
                // no TMA store (its smem reads wait behind the producer's
                // loads of the next item), so the buffer is free as soon as
                // the group has read it back.
#pragma unroll 1
                for (int hh = 0; hh < D / 64; ++hh) {
                    if (hh > 0) named_bar_sync(1 + g, 256);  // the previous half is read back
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int c = 2 * hh + cc;
                        uint32_t o[16];
                        ld16x256_x4(t_o + 32 * c, o);
                        tmem_wait_ld();
                        if (c == D / 32 - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) bar_arrive(bo_free);
                        }
                        const uint32_t box = stage + cc * (BM * 128);
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            const uint32_t row = static_cast<uint32_t>(row0 + 8 * r);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint32_t q16 = (2 * k + (t0 >> 1)) ^ (row & 7);
                                const float vx = __uint_as_float(o[4 * k + 2 * r]) * os * f[r];
                                const float vy = __uint_as_float(o[4 * k + 2 * r + 1]) * os * f[r];
                                asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(
                                                 box + row * 128 + q16 * 16 + (t0 & 1) * 8),
                                             "f"(vx), "f"(vy)
                                             : "memory");
                            }
                        }
                    }
                    named_bar_sync(1 + g, 256);  // the half is staged
                    const uint32_t gw = mw & 7;  // rows [16 gw, 16 gw + 16) of the group
                    const uint32_t col4 = lane & 15, cc = col4 >> 3, q = col4 & 7;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t row = 16 * gw + 2 * i + (lane >> 4);
                        float4 x;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                                     : "r"(stage + cc * (BM * 128) + row * 128 + ((q ^ (row & 7)) * 16)));
                        const int32_t gr = q0 + static_cast<int32_t>(row);
                        const int32_t col = 64 * hh + 4 * static_cast<int32_t>(col4);
                        if (gr < n && col < p.d)
                            __stcs(reinterpret_cast<float4*>(
                                       p.o + (static_cast<int64_t>(slice) * n + gr) * p.o_pitch + col),
                                   x);
                    }
                }
                named_bar_sync(1 + g, 256);  // the next item's P stores reuse the buffer
} else if constexpr (IFA_PP_OBOX) {
                // one bulk group per 128 x 32 box, boxes alternating between
                // the two 16 KiB atoms: box c waits only for box c - 2's read
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    if (c >= 2) {
                        if (issuer) tma_store_wait_read_but1();
                        named_bar_sync(1 + g, 256);
                    }
                    uint32_t o[16];
                    ld16x256_x4(t_o + 32 * c, o);
                    tmem_wait_ld();
                    if (c == D / 32 - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) bar_arrive(bo_free);
                    }
                    const uint32_t box = stage + (c & 1) * (BM * 128);
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const uint32_t row = static_cast<uint32_t>(row0 + 8 * r);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t q16 = (2 * k + (t0 >> 1)) ^ (row & 7);
                            const float vx = __uint_as_float(o[4 * k + 2 * r]) * os * f[r];
                            const float vy = __uint_as_float(o[4 * k + 2 * r + 1]) * os * f[r];
                            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(
                                             box + row * 128 + q16 * 16 + (t0 & 1) * 8),
                                         "f"(vx), "f"(vy)
                                         : "memory");
                        }
                    }
                    fence_proxy_async_shared();
                    named_bar_sync(1 + g, 256);
                    if (issuer) {
                        tma_store_3d(&tm_o, reinterpret_cast<const uint8_t*>(sm.p[g]) + (c & 1) * (BM * 128),
                                     32 * c, q0, slice);
                        tma_store_commit();
                    }
                }
} else {
#pragma unroll
                for (int hh = 0; hh < D / 64; ++hh) {
                    if (hh > 0) {  // the previous half's boxes have been read
                        if (issuer) tma_store_wait_read();
                        named_bar_sync(1 + g, 256);
                    }
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int c = 2 * hh + cc;
                        uint32_t o[16];
                        ld16x256_x4(t_o + 32 * c, o);
                        tmem_wait_ld();
                        if (c == D / 32 - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) bar_arrive(bo_free);
                        }
                        const uint32_t box = stage + cc * (BM * 128);
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            const uint32_t row = static_cast<uint32_t>(row0 + 8 * r);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint32_t q16 = (2 * k + (t0 >> 1)) ^ (row & 7);
                                const float vx = __uint_as_float(o[4 * k + 2 * r]) * os * f[r];
                                const float vy = __uint_as_float(o[4 * k + 2 * r + 1]) * os * f[r];
                                asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(
                                                 box + row * 128 + q16 * 16 + (t0 & 1) * 8),
                                             "f"(vx), "f"(vy)
                                             : "memory");
                            }
                        }
                    }
                    fence_proxy_async_shared();
                    named_bar_sync(1 + g, 256);
                    if (issuer) {
                        tma_store_3d(&tm_o, reinterpret_cast<const void*>(sm.p[g]), 64 * hh, q0, slice);
                        tma_store_3d(&tm_o, reinterpret_cast<const uint8_t*>(sm.p[g]) + BM * 128,
                                     64 * hh + 32, q0, slice);
                        tma_store_commit();
                    }
                }
}
                if constexpr (IFA_PP_OSTG) {
                } else if constexpr (IFA_PP_ODEFER) {
                    o_pending = true;  // the next item's first P stores wait for these reads
                } else {
                    if (issuer) tma_store_wait_read();
                    named_bar_sync(1 + g, 256);
                }
                if (tre) PP_TR(1, g, tc - 1, 7);
                continue;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[16];
                ld16x256_x4(t_o + 32 * c, o);
                tmem_wait_ld();
                if (c == D / 32 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(bo_free);
                }
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if (grow[r] >= n) continue;
                    float* orow = p.o + (static_cast<int64_t>(slice) * n + grow[r]) * p.o_pitch;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int col = 32 * c + 8 * k + 2 * static_cast<int>(t0);
                        // full-INT8: O holds 2^-24 * the integer P.V (exact rescale)
                        constexpr float os = MODE == kModeCodes ? 16777216.0f : 1.0f;
                        const float2 v = make_float2(__uint_as_float(o[4 * k + 2 * r]) * os * f[r],
                                                     __uint_as_float(o[4 * k + 2 * r + 1]) * os * f[r]);
                        if (col + 1 < p.d)
                            __stcs(reinterpret_cast<float2*>(orow + col), v);
                        else if (col < p.d)
                            orow[col] = v.x;
                    }
                }
            }
        }
    }

    if (p.o_tma) tma_store_wait_all();  // the last item's O stores
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// int8 codes [slices][n][pitch] -> fp16 [slices][n_pad][D] (columns >= pitch
// and rows >= n are zero).
__global__ void codes_to_f16_kernel(const int8_t* __restrict__ src, int64_t slices, int64_t n,
                                    int64_t n_pad, int64_t pitch, int dcols,
                                    __half* __restrict__ dst) {
    const int64_t total = slices * n_pad * dcols;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total / 8;
         i += stride) {
        const int64_t e = 8 * i, rp = e / dcols, c = e - rp * dcols;
        const int64_t sl = rp / n_pad, rr = rp - sl * n_pad, r = sl * n + rr;
        __align__(16) __half h[8];
        if (rr >= n) {
#pragma unroll
            for (int t = 0; t < 8; ++t) h[t] = __float2half_rn(0.0f);
        } else if (c + 8 <= pitch && (pitch % 8) == 0) {
            const uint2 w = *reinterpret_cast<const uint2*>(src + r * pitch + c);
            const int8_t* b = reinterpret_cast<const int8_t*>(&w);
#pragma unroll
            for (int t = 0; t < 8; ++t) h[t] = __int2half_rn(b[t]);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t)
                h[t] = __int2half_rn(c + t < pitch ? src[r * pitch + c + t] : 0);
        }
        *reinterpret_cast<uint4*>(dst + e) = *reinterpret_cast<const uint4*>(h);
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

// fp16 V [slices*n][D] viewed as {64 cols, e:2, k':8, t:4, half} so that
// smem row 64h + 16t + 2k' + e holds key 64h + 8k' + 2t + e: the MMA key
// order of the P rows the softmax threads write (thread t0 owns MMA keys
// 64h + 16 t0 + 2k' + e = its keys 8(8h + k') + 2 t0 + e).
static bool make_map_v16(CUtensorMap* map, const __half* base, int64_t slices, int64_t n, int D) {
    PFN_encodeTiled enc = get_encode();
    if (!enc || n % 128 != 0) return false;
    const cuuint64_t row = static_cast<cuuint64_t>(D) * 2;
    const cuuint64_t dims[5] = {static_cast<cuuint64_t>(D), 2, 8, 4,
                                static_cast<cuuint64_t>(slices * n / 64)};
    const cuuint64_t strides[4] = {row, 8 * row, 2 * row, 64 * row};
    const cuuint32_t box[5] = {64u, 2u, 8u, 4u, 2u};
    const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<__half*>(base), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// f32 O [slices][n][o_pitch] (d valid columns), box {32 cols, 128 rows, 1}, SW128
static bool make_map_o(CUtensorMap* map, const float* base, int64_t slices, int64_t n, int64_t d,
                       int64_t o_pitch) {
    PFN_encodeTiled enc = get_encode();
    if (!enc || (o_pitch * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(slices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(o_pitch) * 4,
                                   static_cast<cuuint64_t>(o_pitch) * 4 * n};
    const cuuint32_t box[3] = {32u, 128u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// IFA_PP_EPI == 2: f32 O [slices][n][o_pitch], box {16 cols, 32 rows, 1}, SW64
static bool make_map_o_epi(CUtensorMap* map, const float* base, int64_t slices, int64_t n,
                           int64_t d, int64_t o_pitch) {
    PFN_encodeTiled enc = get_encode();
    if (!enc || (o_pitch * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(slices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(o_pitch) * 4,
                                   static_cast<cuuint64_t>(o_pitch) * 4 * n};
    const cuuint32_t box[3] = {16u, 32u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int MODE>
static cudaError_t run(const void* q, const void* k, const __half* v16, const Params& p_in,
                       int64_t pitch, bool causal, cudaStream_t stream) {
    CUtensorMap tq, tk, tv, to;
    if (!make_map_codes(&tq, static_cast<const int8_t*>(q), p_in.slices, p_in.n, pitch, D) ||
        !make_map_codes(&tk, static_cast<const int8_t*>(k), p_in.slices, p_in.n, pitch, D) ||
        !make_map_v16(&tv, v16, p_in.slices, p_in.n_pad, D))
        return cudaErrorInvalidValue;
    Params p = p_in;
    const char* no_tma = std::getenv("IFA_B200_NO_OTMA");
    p.o_tma = (!kEpi && !(no_tma && no_tma[0] == '1') && p.s_dump == nullptr && p.p_dump == nullptr &&
               make_map_o(&to, p.o, p.slices, p.n, p.d, p.o_pitch))
                  ? 1
                  : 0;
    if (!p.o_tma) to = tq;  // unused
    if (kEpi2 && !make_map_o_epi(&to, p.o, p.slices, p.n, p.d, p.o_pitch))
        return cudaErrorInvalidValue;
    const size_t smem = sizeof(Smem<D>) + 1024;
    cudaError_t e = smem_attr_once<int_flash_pp_kernel<D, false, MODE, false>>(smem);
    if (e == cudaSuccess && MODE == kModeCodes) {
        e = smem_attr_once<int_flash_pp_kernel<D, true, MODE, false>>(smem);
        if (e == cudaSuccess) e = smem_attr_once<int_flash_pp_kernel<D, false, MODE, true>>(smem);
        if (e == cudaSuccess) e = smem_attr_once<int_flash_pp_kernel<D, true, MODE, true>>(smem);
    }
    if (e != cudaSuccess) return e;
    const int sms = current_device_sms();
    const int cap = p.max_ctas > 0 && p.max_ctas < sms ? p.max_ctas : sms;
    const int grid = p.items < cap ? p.items : cap;
    const bool ragged = p.n % BN != 0;
    if constexpr (MODE == kModeCodes) {
        if (p.s_dump != nullptr || p.p_dump != nullptr) {  // parity dumps: the ragged-capable code
            if (causal) {
                e = smem_attr_once<int_flash_pp_kernel<D, true, MODE, true, false, true>>(smem);
                if (e == cudaSuccess)
                    int_flash_pp_kernel<D, true, MODE, true, false, true>
                        <<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
            } else {
                e = smem_attr_once<int_flash_pp_kernel<D, false, MODE, true, false, true>>(smem);
                if (e == cudaSuccess)
                    int_flash_pp_kernel<D, false, MODE, true, false, true>
                        <<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
            }
            if (e != cudaSuccess) return e;
        } else if (p.ready != nullptr) {  // streamed step: non-causal, n % 128 == 0 only
            if (causal || ragged) return cudaErrorInvalidValue;
            e = smem_attr_once<int_flash_pp_kernel<D, false, MODE, false, true>>(smem);
            if (e != cudaSuccess) return e;
            int_flash_pp_kernel<D, false, MODE, false, true><<<grid, NUM_THREADS, smem, stream>>>(
                tq, tk, tv, to, p);
        } else if (causal && ragged)
            int_flash_pp_kernel<D, true, MODE, true><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
        else if (causal)
            int_flash_pp_kernel<D, true, MODE, false><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
        else if (ragged)
            int_flash_pp_kernel<D, false, MODE, true><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
        else
            int_flash_pp_kernel<D, false, MODE, false><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
    } else {  // half-INT8 / FP8: non-causal, n % 128 == 0 (float_weights_pp_eligible)
        int_flash_pp_kernel<D, false, MODE, false><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, to, p);
    }
    return cudaGetLastError();
}

static Params make_params(const float* sq, const float* sk, const float* sv, float* o,
                          int64_t slices, int64_t n, int64_t d, uint32_t flags) {
    Params p;
    p.sq = sq;
    p.sk = sk;
    p.sv = sv;
    p.o = o;
    p.n = static_cast<int32_t>(n);
    p.d = static_cast<int32_t>(d);
    p.o_pitch = static_cast<int32_t>(d);
    p.n_pad = static_cast<int32_t>((n + BN - 1) / BN * BN);
    p.flags = flags;
    p.sk_mul = kLog2e * ((flags & IFA_FLAG_SQRT_D) ? 1.0f / sqrtf(static_cast<float>(d)) : 1.0f);
    const int32_t q_tiles = static_cast<int32_t>((n + BM - 1) / BM);
    p.pairs = (q_tiles + 1) / 2;
    p.slices = static_cast<int32_t>(slices);
    p.items = p.pairs * p.slices;
    p.ready = nullptr;
    p.ready_target = 0;
    p.ready_from = 0;
    p.max_ctas = 0;
    p.s_dump = nullptr;
    p.p_dump = nullptr;
    p.o_tma = 0;
    return p;
}

template <int D>
static cudaError_t launch(const AttnArgs& a, const uint16_t* v16_given, cudaStream_t stream) {
    static std::atomic<uint64_t> pool_kept{0};  // per device
    {  // keep the per-call fp16 V workspace in the stream-ordered pool
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && dev < kMaxDevices &&
            !(pool_kept.load(std::memory_order_relaxed) & (uint64_t{1} << dev)) &&
            cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            pool_kept.fetch_or(uint64_t{1} << dev, std::memory_order_relaxed);
        }
    }
    __half* v16 = const_cast<__half*>(reinterpret_cast<const __half*>(v16_given));
    __half* owned = nullptr;
    const int64_t n_pad = (a.n + BN - 1) / BN * BN;
    const int64_t rows = a.slices * n_pad;
    cudaError_t e = cudaSuccess;
    if (v16 && n_pad != a.n) return cudaErrorInvalidValue;  // a given copy is unpadded
    if (!v16) {  // fp16 copy of the V codes (the caller may pass one: ifa_int_flash_fwd_v16)
        e = cudaMallocAsync(reinterpret_cast<void**>(&owned), rows * D * 2, stream);
        if (e != cudaSuccess) return e;
        v16 = owned;
        int64_t blocks = (rows * D / 8 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        codes_to_f16_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
            a.v, a.slices, a.n, n_pad, a.pitch, D, v16);
    }
    Params p = make_params(a.sq, a.sk, a.sv, a.o, a.slices, a.n, a.d, a.flags);
    float* o_even = nullptr;  // odd d: rows of d + 1 floats, then compacted into a.o
    if (a.d & 1) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&o_even),
                            sizeof(float) * a.slices * a.n * (a.d + 1), stream);
        if (e != cudaSuccess) {
            if (owned) cudaFreeAsync(owned, stream);
            return e;
        }
        p.o = o_even;
        p.o_pitch = static_cast<int32_t>(a.d + 1);
    }
    p.ready = a.ready;
    p.ready_target = a.ready_target;
    p.ready_from = a.ready_from;
    p.max_ctas = a.max_ctas;
    if (a.dump != nullptr && !int_flash_ws_enabled()) {
        p.s_dump = a.dump->s;
        p.p_dump = a.dump->p;
    }
    if ((int_flash_ws_enabled() && a.ready == nullptr) ||
        (a.dump != nullptr && int_flash_ws_enabled()))
        e = launch_int_flash_ws(a.q, a.sq, a.k, a.sk, reinterpret_cast<const uint16_t*>(v16), a.sv,
                                p.o, a.slices, a.n, a.d, a.pitch, p.o_pitch, a.flags, a.dump,
                                stream);
    else
        e = run<D, kModeCodes>(a.q, a.k, v16, p, a.pitch, (a.flags & IFA_FLAG_CAUSAL) != 0, stream);
    if (o_even) {
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(a.o, sizeof(float) * a.d, o_even, sizeof(float) * (a.d + 1),
                                  sizeof(float) * a.d, a.slices * a.n, cudaMemcpyDeviceToDevice,
                                  stream);
        cudaFreeAsync(o_even, stream);
    }
    const cudaError_t e2 = owned ? cudaFreeAsync(owned, stream) : cudaSuccess;
    return e != cudaSuccess ? e : e2;
}

}  // namespace pp

#ifdef IFA_PP_TRACE
extern "C" int ifa_pp_trace_read(unsigned long long* host, int64_t count) {
    return cudaMemcpyFromSymbol(host, pp::g_pp_trace, sizeof(unsigned long long) * count) ==
                   cudaSuccess
               ? 0
               : 1;
}
#endif

bool int_flash_pp_eligible(const AttnArgs& a) {
    const char* off = std::getenv("IFA_B200_NO_PP");
    if (off && off[0] == '1') return false;
    const int64_t bc = a.bc < a.n ? a.bc : a.n;
    const bool tiles_are_blocks = bc == pp::BN || (bc == a.n && a.n <= pp::BN);
    return (a.flags & IFA_FLAG_FAST) &&
           a.audit == nullptr && tiles_are_blocks && a.d <= 128;
}

cudaError_t launch_int_flash_pp(const AttnArgs& a, const uint16_t* v16, cudaStream_t stream) {
    if (a.d <= 64) return pp::launch<64>(a, v16, stream);
    return pp::launch<128>(a, v16, stream);
}

bool float_weights_pp_eligible(int64_t n, int64_t d) {
    const char* off = std::getenv("IFA_B200_NO_PP");
    if (off && off[0] == '1') return false;
    return n % 128 == 0 && (d == 64 || d == 128);
}

cudaError_t launch_half_int8_pp(const int8_t* q, const float* sq, const int8_t* k,
                                const float* sk, const uint16_t* v16, float* o, int64_t slices,
                                int64_t n, int64_t d, uint32_t flags, cudaStream_t stream) {
    const pp::Params p = pp::make_params(sq, sk, nullptr, o, slices, n, d, flags & IFA_FLAG_SQRT_D);
    const __half* vh = reinterpret_cast<const __half*>(v16);
    if (d == 64) return pp::run<64, pp::kModeHalf>(q, k, vh, p, d, false, stream);
    return pp::run<128, pp::kModeHalf>(q, k, vh, p, d, false, stream);
}

cudaError_t launch_fp8_pp(const uint8_t* q, const float* q_scales, const uint8_t* k,
                          const float* k_scales, const uint16_t* v16, const float* v_scales,
                          float* o, int64_t slices, int64_t n, int64_t d, uint32_t flags,
                          cudaStream_t stream) {
    const pp::Params p = pp::make_params(q_scales, k_scales, v_scales, o, slices, n, d,
                                         flags & IFA_FLAG_SQRT_D);
    const __half* vh = reinterpret_cast<const __half*>(v16);
    if (d == 64) return pp::run<64, pp::kModeFp8>(q, k, vh, p, d, false, stream);
    return pp::run<128, pp::kModeFp8>(q, k, vh, p, d, false, stream);
}

}  // namespace ifa_b200
