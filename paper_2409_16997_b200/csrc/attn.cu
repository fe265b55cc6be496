// attn.cu -- fused full-INT8 flash attention forward for sm_100a.
//
// Restates /root/reference/proj/src/attention.cpp:235-357
// (ifa::int_flash_attention) bit-exactly, with the reference's exact float
// expression order:
//   S_int = Q_i . K_j^T                          int32, exact   (:275-276)
//   s     = float(S_int) * (sQ[r] * sK[c]) [* 1/sqrt(d)]       (:277-290)
//   m'    = max(m, rowmax s);  alpha = expf(m - m')             (:291-298)
//   P     = (int) round(127 * expf(s - m'))  in [0,127]         (:299-312)
//   l     = l*alpha + float(sum P);  acc *= alpha               (:313-318)
//   acc  += float(P . V_j)                   int32 per block    (:328-333)
//   O     = (acc / l) * sV                                      (:335-342)
// plus the PCodeAudit bookkeeping (:309-311, :319-326, :343-355) and the
// causal extension (keys j <= row i only).
//
// Persistent kernel: one CTA per SM walks a static list of work items
// (128-row Q tile, (b,h) slice); causal items heaviest first.  Warp roles
// (20 warps = 5 per SM sub-partition; the launch gives each thread 96
// registers, then warps 0-3 drop to 32 and hand theirs to the softmax
// warps, which run with 112):
//   warp 0       TMA producer: Q (double-buffered across work items), then a
//                STAGES-deep ring of K / V tiles (128 keys x D int8, 128B/64B
//                swizzle) + the K scales.
//   warp 1       TMEM allocator + MMA issuer (one thread): S = Q.K^T
//                (tcgen05.mma kind::i8, A and B from SMEM) into TMEM;
//                PV = P.V (A = P from TMEM, B = V from SMEM, MN-major) plus
//                P.1 (a 16-column all-ones B tile: the exact int32 row sum
//                of the codes) into TMEM.
//   warps 2-3    idle.
//   warps 4-19   softmax + correction: four threads per Q row (TMEM lane),
//                each owning 32 of the 128 key columns AND 32 of the output
//                columns.  Per KV tile: tcgen05.ld the int32 S slice,
//                dequantize, exchange the partial row max through SMEM,
//                exact requantization of P (MUFU estimate + rounding guard,
//                exact boundary fallback), tcgen05.st the packed codes.  The
//                PREVIOUS block's P.V (finished while this tile's S was
//                being computed) is folded into the f32 accumulator held in
//                registers -- acc = acc*alpha + float(PV), l = l*alpha +
//                float(rowsum) -- while the row-max exchange completes.
//                Epilogue O = (acc/l)*sV.
// Elementwise math uses sm_100 packed FADD2/FMUL2/FFMA2 (IEEE RN per lane,
// bit-identical to the scalar ops).
// TMEM columns: S [0,128) | PV [128,128+D) | rowsum [256,272) |
// P0 [288,320) | P1 [320,352).
//
// Bc (the reference's KV block size, which changes results) is honoured:
// a block of <= 128 keys is one pipeline item; a larger block is processed
// in two passes over 128-key sub-tiles (pass 1: block row max, pass 2:
// codes + PV accumulated in int32 across the sub-tiles), exactly the
// reference's per-block arithmetic.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "code_bounds.h"
#include "exact_expf.cuh"
#include "ifa_internal.h"
#include "ptx.cuh"

namespace ifa_b200 {

using namespace ptx;

namespace attn {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int STAGES = 4;
constexpr int SPLIT = 4;                 // softmax threads per Q row
constexpr int NCOL = BN / SPLIT;         // key (and output) columns per softmax thread
constexpr int SOFT_WARP0 = 4;
constexpr int SOFT_WARPS = 4 * SPLIT;    // softmax warps (4 lane quarters x SPLIT)
constexpr int NUM_THREADS = 32 * (SOFT_WARP0 + SOFT_WARPS);
// Per sub-partition (16384 registers): 1 control warp x 32 + 4 softmax warps
// x 112 = 15360 = 5 warps x the launch's 96.
constexpr uint32_t kRegsControl = 32;
constexpr uint32_t kRegsSoftmax = 112;
static_assert(kRegsControl + 4 * kRegsSoftmax <= 5 * 96, "register budget");
// quad kernels: 12 warps launch at 168 registers; per sub-partition one
// control warp (32) and two math warps (232): 32 + 2*232 <= 3*168
constexpr uint32_t kRegsControlQuad = 32;
constexpr uint32_t kRegsMathQuad = 232;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t T_S = 0, T_PV = 128, T_RS = 256, T_P0 = 288;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLog2_127 = 6.9886846867721655f;
constexpr float kMagic = 12582912.0f;       // 1.5 * 2^23: rounds to the nearest integer
// The fast estimate y = ex2(s*log2e + c_r), c_r = log2(127) - m*log2e, is
// within  kGuardBase + kGuardScale * (|m*log2e| + |c_r|)  of the reference's
// fl(127*fl(expf(fl(s - m)))): in t, half an ulp of |t| < 8, of m*log2e and
// of c_r, the float log2e / log2(127) constants; then ex2.approx (2^-22.5
// rel) and the reference's own two roundings; times 127*ln2.  Measured
// maxima (tools/microbench/guard.cu, 2^28 points per m) stay below half of
// this bound.  Codes whose estimate lies within that band of a rounding
// boundary (a half-integer) are settled exactly (code_bounds.h).
constexpr float kGuardBase = 1.3e-4f;
constexpr float kGuardScale = 5.5e-6f;
constexpr int kGuardGroup = 16;  // codes checked per branch

enum ItemKind : uint32_t {
    K_MAXONLY = 1u,   // pass-1 sub-tile of a multi-tile block: contributes to the row max
    K_BEGIN = 2u,     // first item of a block
    K_MAXDONE = 4u,   // block max complete after this item
    K_PV = 8u,        // item produces P codes and a P.V product
    K_PV_FIRST = 16u, // first P.V item of the block (fresh int32 accumulator)
    K_END = 32u,      // last item of the block: l / acc update
};

struct Item {
    int32_t key0;
    int32_t width;
    uint32_t kind;
};

// Deterministic KV item sequence of one work item, shared by every warp role.
struct ItemGen {
    int32_t n, bc, kv_limit;
    int32_t b0 = 0;
    int32_t s = 0, pass = 0;

    __device__ ItemGen(int32_t n_, int32_t bc_, int32_t kv_limit_)
        : n(n_), bc(bc_), kv_limit(kv_limit_) {}

    __device__ __forceinline__ bool next(Item& it) {
        if (b0 >= kv_limit) return false;
        const int32_t blk_end = (bc >= n - b0) ? n : b0 + bc;
        const int32_t lim_end = blk_end < kv_limit ? blk_end : kv_limit;
        it.key0 = b0 + BN * s;
        const int32_t rem = lim_end - it.key0;
        it.width = rem < BN ? rem : BN;
        if (lim_end - b0 <= BN) {  // one sub-tile: single pass
            it.kind = K_BEGIN | K_MAXDONE | K_PV | K_PV_FIRST | K_END;
            b0 = blk_end;
            return true;
        }
        const bool last = rem <= BN;
        if (pass == 0) {
            it.kind = K_MAXONLY | (s == 0 ? K_BEGIN : 0u) | (last ? K_MAXDONE : 0u);
            if (last) {
                s = 0;
                pass = 1;
            } else {
                ++s;
            }
        } else {
            it.kind = K_PV | (s == 0 ? K_PV_FIRST : 0u) | (last ? K_END : 0u);
            if (last) {
                b0 = blk_end;
                s = 0;
                pass = 0;
            } else {
                ++s;
            }
        }
        return true;
    }
};

// Fast-path item sequence (Bc == 128 or Bc == n <= 128, non-causal): one
// full block per tile.
struct TileGen {
    int32_t n, kv_limit;
    int32_t key0 = 0;
    __device__ TileGen(int32_t n_, int32_t kv_limit_) : n(n_), kv_limit(kv_limit_) {}
    __device__ __forceinline__ bool next(Item& it) {
        if (key0 >= kv_limit) return false;
        it.key0 = key0;
        it.width = n - key0 < BN ? n - key0 : BN;
        it.kind = K_BEGIN | K_MAXDONE | K_PV | K_PV_FIRST | K_END;
        key0 += BN;
        return true;
    }
};

template <bool GENERIC>
struct GenOf {
    using type = ItemGen;
};
template <>
struct GenOf<false> {
    using type = TileGen;
};
template <bool GENERIC>
__device__ __forceinline__ typename GenOf<GENERIC>::type make_gen(int32_t n, int32_t bc,
                                                                  int32_t kv_limit) {
    if constexpr (GENERIC)
        return ItemGen(n, bc, kv_limit);
    else
        return TileGen(n, kv_limit);
}

template <int D>
struct alignas(1024) Smem {
    uint8_t q[2][BM * D];
    uint8_t k[STAGES][BN * D];
    uint8_t v[STAGES][BN * D];
    uint8_t ones[16 * BN];  // all-ones B tile: P . 1 = exact int32 row sum of the codes
    float sk[STAGES][BN];
    float xmax[2][BM][SPLIT];  // [item parity][row][part]: partial row max exchange
    float alpha[2][BM];        // [block parity][row]: expf(m - m_new), computed by one part
    float bounds[128];         // B[k]: exact code decision boundaries (code_bounds.h)
    uint64_t q_full[2], q_empty[2];
    uint64_t k_full[STAGES], v_full[STAGES], kv_empty[STAGES];
    uint64_t c_full[3], c_empty[3];  // head dims > 128: the (Q, K) depth-chunk ring
    uint64_t s_full, s_empty;
    uint64_t p_full[2], p_empty[2];
    uint64_t pv_full, pv_empty;
    uint32_t tmem_base;
};

struct Params {
    const float* sq;
    const float* sk;
    const float* sv;
    float* o;
    ifa_pcode_audit* audit;
    int32_t n;
    int32_t d;
    int32_t bc;  // clamped to n by the host (any Bc >= n is one block)
    uint32_t flags;
    float extra;  // 1/sqrt(d) when IFA_FLAG_SQRT_D, else 1
    float sk_mul;  // FAST: K scales are staged pre-multiplied by log2(e) [* extra]
    int32_t q_tiles;
    int32_t slices;
    int32_t items;  // q_tiles * slices
    // head dims > 128 (launch_wide): S accumulates over `wide_chunks` 128-column
    // depth chunks of Q and K streamed through a 3-stage ring in the (then
    // unused) Q and K buffers; this launch writes O columns [0, o_cols) of
    // rows o_pitch floats apart (the V map and p.o start at the chunk's column)
    int32_t wide_chunks = 0;
    int32_t o_cols = 0;
    int64_t o_pitch = 0;
    float bounds[128];
};

struct Work {
    int32_t q0, slice, kv_limit;
};

// Work item -> (Q tile, slice).  Non-causal: the Q tiles of one slice are
// adjacent, so CTAs running together share K/V in L2.  Causal: diagonal
// tiles have the most keys, so they go first (longest-processing-time order).
// The CTA's wi-th work item: causal items (longest first) are dealt in
// rounds of gridDim.x taken in alternating directions, so no CTA gets the
// longest item of every round (as attn_pp.cu); otherwise the grid stride.
__device__ __forceinline__ int32_t item_at(uint32_t wi, bool snake) {
    const int32_t G = static_cast<int32_t>(gridDim.x), c = static_cast<int32_t>(blockIdx.x);
    const int32_t r = static_cast<int32_t>(wi);
    return r * G + ((snake && (r & 1)) ? G - 1 - c : c);
}

__device__ __forceinline__ Work work_of(int32_t idx, const Params& p, bool causal) {
    Work w;
    int32_t qt;
    if (causal) {
        qt = p.q_tiles - 1 - idx / p.slices;
        w.slice = idx % p.slices;
    } else {
        qt = idx % p.q_tiles;
        w.slice = idx / p.q_tiles;
    }
    w.q0 = qt * BM;
    w.kv_limit = p.n;
    if (causal && w.q0 + BM < w.kv_limit) w.kv_limit = w.q0 + BM;
    return w;
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// Requantize this thread's NCOL scores to the reference's codes
// (int)round(127*expf(s - m_new)), packed 4 per word.  Fast path: y =
// ex2(s*log2e + c_r) with c_r = log2(127) - m_new*log2e, rounded by the
// magic-number add; every element also measures its distance to that
// integer.  Only when an estimate of a group of kGuardGroup lies within the guard band
// of a rounding boundary k+1/2 (rare) are the ambiguous codes settled exactly by
// one comparison against the precomputed boundary B[k] of the reference's
// code function (code_bounds.h).
__device__ __forceinline__ void codes_part(const float (&s)[NCOL], float m_new, float c_r,
                                           float thresh, const float* bounds,
                                           uint32_t (&w)[NCOL / 4]) {
    const float2 c2 = f2(c_r);
#pragma unroll
    for (int g0 = 0; g0 < NCOL; g0 += kGuardGroup) {
        float df[kGuardGroup];
#pragma unroll
        for (int c = g0; c < g0 + kGuardGroup; c += 4) {
            const float2 ta = ffma2(make_float2(s[c], s[c + 1]), f2(kLog2e), c2);
            const float2 tb = ffma2(make_float2(s[c + 2], s[c + 3]), f2(kLog2e), c2);
            const float2 ya = make_float2(ex2_approx(ta.x), ex2_approx(ta.y));
            const float2 yb = make_float2(ex2_approx(tb.x), ex2_approx(tb.y));
            const float2 ra = fadd2(ya, f2(kMagic));  // bits: magic + nearest integer
            const float2 rb = fadd2(yb, f2(kMagic));
            const float2 da = fsub2(ya, fsub2(ra, f2(kMagic)));  // distance to it
            const float2 db = fsub2(yb, fsub2(rb, f2(kMagic)));
            df[c - g0] = da.x;
            df[c - g0 + 1] = da.y;
            df[c - g0 + 2] = db.x;
            df[c - g0 + 3] = db.y;
            w[c >> 2] = __byte_perm(__byte_perm(__float_as_uint(ra.x), __float_as_uint(ra.y), 0x0040),
                                    __byte_perm(__float_as_uint(rb.x), __float_as_uint(rb.y), 0x0040),
                                    0x5410);
        }
        float g = 0.0f;
#pragma unroll
        for (int e = 0; e < kGuardGroup; e += 2) g = fmax3(g, fabsf(df[e]), fabsf(df[e + 1]));
        if (g > thresh) {  // rare: settle the ambiguous codes exactly
#pragma unroll
            for (int e = 0; e < kGuardGroup; ++e) {
                if (fabsf(df[e]) > thresh) {
                    const int c = g0 + e;
                    const uint32_t sh = 8u * (c & 3);
                    int k = static_cast<int>((w[c >> 2] >> sh) & 0xffu) - (df[e] < 0.0f ? 1 : 0);
                    k = k < 0 ? 0 : (k > 126 ? 126 : k);
                    const int code = k + (__fsub_rn(s[c], m_new) >= bounds[k] ? 1 : 0);
                    w[c >> 2] = (w[c >> 2] & ~(0xffu << sh)) | (static_cast<uint32_t>(code) << sh);
                }
            }
        }
    }
}

// 2^t for a pair on the FMA pipe (tolerance mode): t = j + f, |f| <= 1/2,
// degree-5 polynomial for 2^f (max rel. error 3.5e-7, i.e. < 5e-5 absolute
// on a code <= 127), 2^j added to the exponent bits.  t is clamped at -64
// (any t < -1 gives code 0).  Offloads part of the exp2 work from the MUFU
// unit, which otherwise bounds the requantization phase.
__device__ __forceinline__ float2 exp2_poly2(float2 t) {
    t.x = fmaxf(t.x, -64.0f);
    t.y = fmaxf(t.y, -64.0f);
    const float2 r = fadd2(t, f2(kMagic));           // nearest integer j in the low bits
    const float2 f = fsub2(t, fsub2(r, f2(kMagic)));  // t - j in [-1/2, 1/2]
    float2 y = ffma2(f, f2(1.2915651313960552e-3f), f2(9.668535552918911e-3f));
    y = ffma2(y, f, f2(5.5516887456178665e-2f));
    y = ffma2(y, f, f2(2.4022264778614044e-1f));
    y = ffma2(y, f, f2(6.931464672088623e-1f));
    y = ffma2(y, f, f2(1.0f));
    // bits(r) << 23 == j << 23 (the magic's own bits shift out)
    return make_float2(__int_as_float(__float_as_int(y.x) + (__float_as_int(r.x) << 23)),
                       __int_as_float(__float_as_int(y.y) + (__float_as_int(r.y) << 23)));
}

// Tolerance mode (IFA_FLAG_FAST): u are log2-domain scores; the code is
// rint(2^(u - m + log2 127)), no exactness guard.  Per 8 codes, 6 exp2 run
// on the MUFU unit and 2 on the FMA pipe.
__device__ __forceinline__ void codes_fast(const float (&u)[NCOL], float sq, float c_r,
                                           uint32_t (&w)[NCOL / 4]) {
    const float2 c2 = f2(c_r), q2 = f2(sq);
#pragma unroll
    for (int c = 0; c < NCOL; c += 8) {
        // t = sQ * u + (log2(127) - sQ * m)
        const float2 ta = ffma2(make_float2(u[c], u[c + 1]), q2, c2);
        const float2 tb = ffma2(make_float2(u[c + 2], u[c + 3]), q2, c2);
        const float2 tc = ffma2(make_float2(u[c + 4], u[c + 5]), q2, c2);
        const float2 td = ffma2(make_float2(u[c + 6], u[c + 7]), q2, c2);
        const float2 ra = fadd2(make_float2(ex2_approx(ta.x), ex2_approx(ta.y)), f2(kMagic));
        const float2 rb = fadd2(make_float2(ex2_approx(tb.x), ex2_approx(tb.y)), f2(kMagic));
        const float2 rc = fadd2(make_float2(ex2_approx(tc.x), ex2_approx(tc.y)), f2(kMagic));
        const float2 rd = fadd2(exp2_poly2(td), f2(kMagic));
        w[c >> 2] = __byte_perm(__byte_perm(__float_as_uint(ra.x), __float_as_uint(ra.y), 0x0040),
                                __byte_perm(__float_as_uint(rb.x), __float_as_uint(rb.y), 0x0040),
                                0x5410);
        w[(c >> 2) + 1] =
            __byte_perm(__byte_perm(__float_as_uint(rc.x), __float_as_uint(rc.y), 0x0040),
                        __byte_perm(__float_as_uint(rd.x), __float_as_uint(rd.y), 0x0040), 0x5410);
    }
}

// Max of NCOL floats as a three-input tree.
__device__ __forceinline__ float row_max(const float (&s)[NCOL]) {
    static_assert(NCOL == 32, "tree below is written for 32 columns");
    float a[11];
#pragma unroll
    for (int j = 0; j < 10; ++j) a[j] = fmax3(s[3 * j], s[3 * j + 1], s[3 * j + 2]);
    a[10] = fmaxf(s[30], s[31]);
    const float b0 = fmax3(a[0], a[1], a[2]), b1 = fmax3(a[3], a[4], a[5]);
    const float b2 = fmax3(a[6], a[7], a[8]), b3 = fmaxf(a[9], a[10]);
    return fmaxf(fmax3(b0, b1, b2), b3);
}

// Ring position of a pipelined resource: stage index + phase parity.
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

// ----------------------------------------------------------------------------
// Quad layout (QUAD kernels, 8 math warps): the 16x256b TMEM shape gives the
// four threads of a quad two rows (r, r+8) and 32 of their 128 columns, so a
// row's maximum is combined with two shuffles -- no cross-warp barrier, and
// half the per-tile fixed costs of the 16-warp layout.  The V tile is
// loaded with its rows permuted inside each 32-key group (see
// make_map_vperm) so each thread's packed codes land in whole 32-bit P
// words.
constexpr int QUAD_WARPS = 8;

template <int N>
__device__ __forceinline__ void tmem_ld_16x256b(uint32_t taddr, uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void tmem_ld_16x256b<16>(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld_16x256b<4>(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_16x256b_x4(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

#ifndef IFA_QUAD_POLY
#define IFA_QUAD_POLY 1  // exp2 pairs per 4 evaluated on the FMA pipe
#endif

// Rounds a pair of exp2 estimates to codes: the magic add leaves the integer
// in the low byte of each float's bits.
__device__ __forceinline__ float2 quad_round2(float2 u, float sq, float cr, bool poly) {
    const float2 t = ffma2(u, f2(sq), f2(cr));
    const float2 y = poly ? exp2_poly2(t) : make_float2(ex2_approx(t.x), ex2_approx(t.y));
    return fadd2(y, f2(kMagic));
}
// Low bytes of (a.x, a.y, b.x, b.y) -> one packed P word (three PRMTs).
__device__ __forceinline__ uint32_t pack4(float2 a, float2 b) {
    return __byte_perm(__byte_perm(__float_as_uint(a.x), __float_as_uint(a.y), 0x0040),
                       __byte_perm(__float_as_uint(b.x), __float_as_uint(b.y), 0x0040), 0x5410);
}

template <int D>
__device__ __forceinline__ void softmax_quad(Smem<D>& sm, const Params& p, uint32_t tmem,
                                             uint32_t warp, uint32_t lane, uint32_t b_s_full,
                                             uint32_t b_s_empty, uint32_t b_k_full,
                                             uint32_t b_kv_empty, uint32_t b_p_full,
                                             uint32_t b_p_empty, uint32_t b_pv_full,
                                             uint32_t b_pv_empty) {
    const float kNegInf = -__int_as_float(0x7f800000);
    const bool causal = (p.flags & IFA_FLAG_CAUSAL) != 0;
    const int32_t n = p.n;
    const uint32_t quarter = warp & 3;
    const uint32_t half = (warp - SOFT_WARP0) >> 2;   // which 16 rows of the quarter
    const uint32_t t0 = lane & 3;                      // column pair within an 8-column group
    const uint32_t lane_base = quarter * 32 + half * 16;
    const int32_t row0 = static_cast<int32_t>(lane_base + (lane >> 2));  // and row0 + 8
    const uint32_t t_base = tmem + (lane_base << 16);
    Ring<STAGES> kv;
    uint32_t i = 0, pi = 0, bi = 0;

    uint32_t wn = 0;
    for (int32_t idx = item_at(0, causal); idx < p.items; idx = item_at(++wn, causal)) {
        const Work w = work_of(idx, p, causal);
        int32_t grow[2];
        float sq[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            grow[r] = w.q0 + row0 + 8 * r;
            sq[r] = grow[r] < n ? p.sq[static_cast<int64_t>(w.slice) * n + grow[r]] : 0.0f;
        }
        float acc[2][D / 4];  // [row][column pair k*2 + e over this thread's D/4 columns]
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < D / 4; ++c) acc[r][c] = 0.0f;
        float l[2] = {0.0f, 0.0f}, m[2] = {kNegInf, kNegInf}, alpha[2] = {1.0f, 1.0f};
        bool pend = false;

        // acc = acc*alpha + float(PV), l = l*alpha + rowsum for the finished
        // block: fold_issue() puts every TMEM load in flight, fold_finish()
        // waits once and does the arithmetic.
        uint32_t rs[4];
        uint32_t pv[D / 2];
        auto fold_issue = [&]() {
            bar_wait(b_pv_full, bi & 1);
            tc_fence_after();
            tmem_ld_16x256b<4>(t_base + T_RS, rs);
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch)
                tmem_ld_16x256b<16>(t_base + T_PV + 32 * ch,
                                    *reinterpret_cast<uint32_t(*)[16]>(&pv[16 * ch]));
        };
        auto fold_finish = [&]() {
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(b_pv_empty);
            ++bi;
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch)
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const int a = 8 * ch + 2 * k;  // pair index within acc[r]
                        const uint32_t* q = &pv[16 * ch + 4 * k + 2 * r];
                        const float2 pf = make_float2(__int2float_rn(static_cast<int32_t>(q[0])),
                                                      __int2float_rn(static_cast<int32_t>(q[1])));
                        const float2 o = ffma2(make_float2(acc[r][a], acc[r][a + 1]), f2(alpha[r]), pf);
                        acc[r][a] = o.x;
                        acc[r][a + 1] = o.y;
                    }
#pragma unroll
            for (int r = 0; r < 2; ++r)
                l[r] = __fmaf_rn(l[r], alpha[r], static_cast<float>(static_cast<int32_t>(rs[2 * r])));
        };

        for (int32_t key0 = 0; key0 < w.kv_limit; key0 += BN) {
            const uint32_t st = kv.idx;
            bar_wait(b_s_full, i & 1);
            tc_fence_after();
            uint32_t sr[64];
            {
                uint32_t (&a)[16] = *reinterpret_cast<uint32_t(*)[16]>(&sr[0]);
                uint32_t (&b)[16] = *reinterpret_cast<uint32_t(*)[16]>(&sr[16]);
                uint32_t (&c)[16] = *reinterpret_cast<uint32_t(*)[16]>(&sr[32]);
                uint32_t (&d)[16] = *reinterpret_cast<uint32_t(*)[16]>(&sr[48]);
                tmem_ld_16x256b<16>(t_base + T_S + 0, a);
                tmem_ld_16x256b<16>(t_base + T_S + 32, b);
                tmem_ld_16x256b<16>(t_base + T_S + 64, c);
                tmem_ld_16x256b<16>(t_base + T_S + 96, d);
            }
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(b_s_empty);
            bar_wait(b_k_full + 8 * st, kv.phase);
            // u = float(S) * (sK * log2e [* extra]); sr[4k + {0,1}] row0, [4k + {2,3}] row1,
            // columns 8k + 2*t0 + {0,1}
            float u[64];
            const float* skc = sm.sk[st] + 2 * t0;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const float2 s2 = *reinterpret_cast<const float2*>(skc + 8 * k);
                const float2 a = fmul2(make_float2(__int2float_rn(static_cast<int32_t>(sr[4 * k])),
                                                   __int2float_rn(static_cast<int32_t>(sr[4 * k + 1]))),
                                       s2);
                const float2 b = fmul2(make_float2(__int2float_rn(static_cast<int32_t>(sr[4 * k + 2])),
                                                   __int2float_rn(static_cast<int32_t>(sr[4 * k + 3]))),
                                       s2);
                u[4 * k] = a.x;
                u[4 * k + 1] = a.y;
                u[4 * k + 2] = b.x;
                u[4 * k + 3] = b.y;
            }
            __syncwarp();
            if (lane == 0) bar_arrive(b_kv_empty + 8 * st);
            // causal / ragged tail: keys >= the visible limit of each row
            const int32_t tail = n - key0 < BN ? n - key0 : BN;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                int32_t lim = tail;
                if (causal) {
                    const int32_t vis = grow[r] - key0 + 1;
                    if (vis < lim) lim = vis < 0 ? 0 : vis;
                }
                if (lim < BN) {
#pragma unroll
                    for (int k = 0; k < 16; ++k)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            if (8 * k + 2 * static_cast<int32_t>(t0) + e >= lim)
                                u[4 * k + 2 * r + e] = kNegInf;
                }
            }
            // row maxima: 32 values per thread per row, then the quad
            float mx[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                float a[11];
#pragma unroll
                for (int j = 0; j < 10; ++j) {
                    const int v0 = 3 * j, v1 = 3 * j + 1, v2 = 3 * j + 2;  // value index 2k + e
                    a[j] = fmax3(u[4 * (v0 >> 1) + 2 * r + (v0 & 1)], u[4 * (v1 >> 1) + 2 * r + (v1 & 1)],
                                 u[4 * (v2 >> 1) + 2 * r + (v2 & 1)]);
                }
                a[10] = fmaxf(u[4 * 15 + 2 * r], u[4 * 15 + 2 * r + 1]);
                float b = fmaxf(fmax3(fmax3(a[0], a[1], a[2]), fmax3(a[3], a[4], a[5]),
                                      fmax3(a[6], a[7], a[8])),
                                fmaxf(a[9], a[10]));
                b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 1));
                b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 2));
                mx[r] = b;
            }
            float mnew[2], cr[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                mnew[r] = (m[r] < mx[r]) ? mx[r] : m[r];
                cr[r] = kLog2_127 - sq[r] * mnew[r];
            }
            if (pi >= 2) {
                bar_wait(b_p_empty + 8 * (pi & 1), ((pi - 2) >> 1) & 1);
                tc_fence_after();
            }
            // codes -> P words: st.16x256b rep kp: {row0 word 2kp..., } = columns
            // 8kp + 2t0 + {0,1}; word j0 = codes of k = 4kp + {0,1}, j0+1 = k = 4kp + {2,3}.
            // Per 8 codes, 6 exp2 on the MUFU unit and 2 on the FMA pipe.
            uint32_t wd[16];
#pragma unroll
            for (int kp = 0; kp < 4; ++kp) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int k = 4 * kp;
                    const float2 c0 = quad_round2(make_float2(u[4 * k + 2 * r], u[4 * k + 2 * r + 1]),
                                                  sq[r], cr[r], false);
                    const float2 c1 = quad_round2(make_float2(u[4 * (k + 1) + 2 * r], u[4 * (k + 1) + 2 * r + 1]),
                                                  sq[r], cr[r], IFA_QUAD_POLY >= 3);
                    const float2 c2 = quad_round2(make_float2(u[4 * (k + 2) + 2 * r], u[4 * (k + 2) + 2 * r + 1]),
                                                  sq[r], cr[r], IFA_QUAD_POLY >= 2);
                    const float2 c3 = quad_round2(make_float2(u[4 * (k + 3) + 2 * r], u[4 * (k + 3) + 2 * r + 1]),
                                                  sq[r], cr[r], IFA_QUAD_POLY >= 1);
                    wd[4 * kp + 2 * r] = pack4(c0, c1);
                    wd[4 * kp + 2 * r + 1] = pack4(c2, c3);
                }
            }
            tmem_st_16x256b_x4(t_base + T_P0 + 32 * (pi & 1), wd);
            if (pend) {  // fold the previous block's P.V (loading it before the codes
                         // overlaps the TMEM latency but spills: measured slower)
                fold_issue();
                fold_finish();
                pend = false;
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(b_p_full + 8 * (pi & 1));
            ++pi;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                alpha[r] = (mnew[r] == m[r]) ? 1.0f
                           : (m[r] == kNegInf ? 0.0f : ex2_approx(sq[r] * (m[r] - mnew[r])));
                m[r] = mnew[r];
            }
            pend = true;
            kv.advance();
            ++i;
        }
        // last block's fold, then O = acc * (sV / l)
        fold_issue();
        fold_finish();
        const float sv = p.sv[w.slice];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (grow[r] >= n) continue;
            const float f = __fdiv_rn(sv, l[r]);
            float* orow = p.o + (static_cast<int64_t>(w.slice) * n + grow[r]) * p.d;
#pragma unroll
            for (int k = 0; k < D / 8; ++k) {
                const int col = 8 * k + 2 * static_cast<int>(t0);
                if (col < p.d) {
                    const float2 o = make_float2(acc[r][2 * k] * f, acc[r][2 * k + 1] * f);
                    if (col + 1 < p.d && (p.d & 1) == 0) {  // 8-byte aligned pair
                        __stcs(reinterpret_cast<float2*>(orow + col), o);
                    } else {
                        orow[col] = o.x;
                        if (col + 1 < p.d) orow[col + 1] = o.y;
                    }
                }
            }
        }
    }
}

// GENERIC = false: the benchmark-shaped fast path (non-causal, KV blocks
// equal to the 128-key tiles, no audit, no 1/sqrt(d)); true: every feature,
// selected at run time.
template <int D, bool GENERIC, bool FAST, bool QUAD>
__global__ void __launch_bounds__(QUAD ? 32 * (SOFT_WARP0 + QUAD_WARPS) : NUM_THREADS, 1)
    int_flash_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const Params p) {
    // math warps: 16 (four per row, 32x32b) or 8 (quad layout, 16x256b)
    constexpr int kMathWarps = QUAD ? QUAD_WARPS : SOFT_WARPS;
    constexpr uint32_t kLayout = D == 128 ? kLayoutSw128 : kLayoutSw64;
    constexpr uint32_t kSbo = 8 * D;  // 8 rows of D bytes per swizzle atom
    constexpr uint32_t kTileBytes = BN * D;
    constexpr uint32_t kIdescS = idesc_i8(BM, BN, false, false);
    constexpr uint32_t kIdescPV = idesc_i8(BM, D, false, true);
    constexpr uint32_t kIdescSum = idesc_i8(BM, 16, false, false);
    const float kNegInf = -__int_as_float(0x7f800000);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const bool causal = (GENERIC || QUAD) && (p.flags & IFA_FLAG_CAUSAL) != 0;
    const bool audit = GENERIC && p.audit != nullptr;
    const int32_t n = p.n;

    // shared-window addresses of the barriers
    const uint32_t b_q_full = smem_u32(&sm.q_full[0]), b_q_empty = smem_u32(&sm.q_empty[0]);
    const uint32_t b_k_full = smem_u32(&sm.k_full[0]), b_v_full = smem_u32(&sm.v_full[0]);
    const uint32_t b_kv_empty = smem_u32(&sm.kv_empty[0]);
    const uint32_t b_s_full = smem_u32(&sm.s_full), b_s_empty = smem_u32(&sm.s_empty);
    const uint32_t b_p_full = smem_u32(&sm.p_full[0]), b_p_empty = smem_u32(&sm.p_empty[0]);
    const uint32_t b_pv_full = smem_u32(&sm.pv_full), b_pv_empty = smem_u32(&sm.pv_empty);
    const uint32_t b_c_full = smem_u32(&sm.c_full[0]), b_c_empty = smem_u32(&sm.c_empty[0]);
    // depth-chunk stage cs: (Q, K) in (k[0], k[1]), (k[2], k[3]), (q[0], q[1])
    const bool wide = GENERIC && !QUAD && p.wide_chunks > 0;  // launch_wide uses GENERIC
    auto chunk_q = [&](uint32_t cs) -> uint8_t* { return cs < 2 ? sm.k[2 * cs] : sm.q[0]; };
    auto chunk_k = [&](uint32_t cs) -> uint8_t* { return cs < 2 ? sm.k[2 * cs + 1] : sm.q[1]; };

    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023) __trap();  // SWIZZLE_128B tiles need 1 KiB alignment
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.q_full[i], 1);
            mbar_init(&sm.q_empty[i], 1);
            mbar_init(&sm.p_full[i], kMathWarps);
            mbar_init(&sm.p_empty[i], 1);
        }
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&sm.k_full[i], 32);
            mbar_init(&sm.v_full[i], 1);
            mbar_init(&sm.kv_empty[i], 1 + kMathWarps);
        }
        for (int i = 0; i < 3; ++i) {
            mbar_init(&sm.c_full[i], 1);
            mbar_init(&sm.c_empty[i], 1);
        }
        mbar_init(&sm.s_full, 1);
        mbar_init(&sm.s_empty, kMathWarps);
        mbar_init(&sm.pv_full, 1);
        mbar_init(&sm.pv_empty, kMathWarps);
        fence_barrier_init();
    }
    if (threadIdx.x < 128) sm.bounds[threadIdx.x] = p.bounds[threadIdx.x];
    if (threadIdx.x < 16 * BN / 16)
        reinterpret_cast<uint4*>(sm.ones)[threadIdx.x] = make_uint4(0x01010101u, 0x01010101u,
                                                                    0x01010101u, 0x01010101u);
    fence_proxy_async_shared();  // the all-ones tile is read by the tensor core
    if (warp == 1) tmem_alloc<TMEM_COLS>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp < SOFT_WARP0) {
      if constexpr (QUAD)
          regs_dealloc<kRegsControlQuad>();
      else
          regs_dealloc<kRegsControl>();
      if (warp == 0) {
        // ------------------------------------------------------------ producer
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
        }
        Ring<STAGES> kv;
        uint32_t i = 0, wi = 0, ci = 0;
        for (int32_t idx = item_at(wi, causal); idx < p.items; idx = item_at(++wi, causal)) {
            const Work w = work_of(idx, p, causal);
            const uint32_t qb = wi & 1;
            if (lane == 0 && !wide) {
                if (wi >= 2) bar_wait(b_q_empty + 8 * qb, ((wi >> 1) - 1) & 1);
                mbar_arrive_expect_tx(&sm.q_full[qb], BM * D);
                tma_load_3d(sm.q[qb], &tm_q, &sm.q_full[qb], 0, w.q0, w.slice, pol_stream);
            }
            const float* sk_slice = p.sk + static_cast<int64_t>(w.slice) * n;
            auto gen = make_gen<GENERIC>(n, p.bc, w.kv_limit);
            Item it;
            while (gen.next(it)) {
                const uint32_t st = kv.idx;
                if (i >= STAGES) bar_wait(b_kv_empty + 8 * st, kv.phase ^ 1u);
                float4 kv4;
                const int32_t key = it.key0 + lane * 4;
                if (key + 3 < n && (reinterpret_cast<uintptr_t>(sk_slice + key) & 15) == 0) {
                    kv4 = __ldg(reinterpret_cast<const float4*>(sk_slice + key));
                } else {
                    kv4.x = key + 0 < n ? sk_slice[key + 0] : 0.0f;
                    kv4.y = key + 1 < n ? sk_slice[key + 1] : 0.0f;
                    kv4.z = key + 2 < n ? sk_slice[key + 2] : 0.0f;
                    kv4.w = key + 3 < n ? sk_slice[key + 3] : 0.0f;
                }
                if constexpr (FAST) {
                    kv4.x *= p.sk_mul;
                    kv4.y *= p.sk_mul;
                    kv4.z *= p.sk_mul;
                    kv4.w *= p.sk_mul;
                }
                reinterpret_cast<float4*>(sm.sk[st])[lane] = kv4;
                if (lane == 0) {
                    if (wide) {
                        bar_arrive(b_k_full + 8 * st);  // the K scales only
                        for (int32_t c = 0; c < p.wide_chunks; ++c, ++ci) {
                            const uint32_t cs = ci % 3;
                            if (ci >= 3) bar_wait(b_c_empty + 8 * cs, ((ci / 3) - 1) & 1);
                            mbar_arrive_expect_tx(&sm.c_full[cs], 2 * kTileBytes);
                            tma_load_3d(chunk_q(cs), &tm_q, &sm.c_full[cs], 128 * c, w.q0, w.slice,
                                        pol_keep);
                            tma_load_3d(chunk_k(cs), &tm_k, &sm.c_full[cs], 128 * c, it.key0,
                                        w.slice, pol_keep);
                        }
                    } else {
                        mbar_arrive_expect_tx(&sm.k_full[st], kTileBytes);
                        tma_load_3d(sm.k[st], &tm_k, &sm.k_full[st], 0, it.key0, w.slice, pol_keep);
                    }
                    if (it.kind & K_PV) {
                        mbar_arrive_expect_tx(&sm.v_full[st], kTileBytes);
                        if constexpr (QUAD)
                            tma_load_5d(sm.v[st], &tm_v, &sm.v_full[st], 0, 0, 0, 0,
                                        (w.slice * n + it.key0) / 32, pol_keep);
                        else
                            tma_load_3d(sm.v[st], &tm_v, &sm.v_full[st], 0, it.key0, w.slice,
                                        pol_keep);
                    } else {
                        bar_arrive(b_v_full + 8 * st);
                    }
                } else {
                    bar_arrive(b_k_full + 8 * st);
                }
                kv.advance();
                ++i;
            }
        }
      } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // Warp-wide loop, one elected lane per MMA batch: the descriptors stay
        // in uniform registers (with lane 0 alone every operand went through
        // R2UR and an MMA took ~2x the tensor core's time to issue, attn_pp.cu).
        {
            const uint32_t ones_base = smem_u32(sm.ones);
            Ring<STAGES> kv;
            uint32_t i = 0, pi = 0, bi = 0, wi = 0, ci = 0;
            bool have_prev = false;
            uint32_t prev_st = 0, prev_ph = 0, prev_kind = 0, prev_pi = 0;
            // P.V of a finished softmax item; issued after the next S so the
            // tensor core computes S(i+1) while the softmax works on tile i.
            auto issue_pv = [&](uint32_t st, uint32_t ph, uint32_t kind, uint32_t pidx) {
                bar_wait(b_p_full + 8 * (pidx & 1), (pidx >> 1) & 1);
                bar_wait(b_v_full + 8 * st, ph);
                if ((kind & K_PV_FIRST) && bi >= 1) bar_wait(b_pv_empty, (bi - 1) & 1);
                tc_fence_after();
                const uint64_t v_desc = smem_desc(smem_u32(sm.v[st]), 16, kSbo, kLayout);
                const uint64_t o_desc = smem_desc(ones_base, 16, 1024, kLayoutSw128);
                const uint32_t p_col = T_P0 + 32 * (pidx & 1);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < BN / 32; ++kk) {
                        // B = V tile, MN-major: 32 keys x D per step = 32 rows of D bytes.
                        const uint32_t acc = ((kind & K_PV_FIRST) && kk == 0) ? 0u : 1u;
                        mma_i8_ts(tmem + T_PV, tmem + p_col + kk * 8, v_desc + kk * (32 * D / 16),
                                  kIdescPV, acc);
                        // P . 1 (16 identical columns): the block's exact code row sum.
                        mma_i8_ts(tmem + T_RS, tmem + p_col + kk * 8, o_desc + kk * 2, kIdescSum,
                                  acc);
                    }
                    mma_commit_u32(b_p_empty + 8 * (pidx & 1));
                    mma_commit_u32(b_kv_empty + 8 * st);
                    if (kind & K_END) mma_commit_u32(b_pv_full);
                }
                __syncwarp();
                if (kind & K_END) ++bi;
            };
            for (int32_t idx = item_at(wi, causal); idx < p.items; idx = item_at(++wi, causal)) {
                const Work w = work_of(idx, p, causal);
                const uint32_t qb = wi & 1;
                if (!wide) bar_wait(b_q_full + 8 * qb, (wi >> 1) & 1);
                tc_fence_after();
                const uint32_t q_base = smem_u32(sm.q[qb]);
                auto gen = make_gen<GENERIC>(n, p.bc, w.kv_limit);
                Item it;
                while (gen.next(it)) {
                    const uint32_t st = kv.idx;
                    const uint32_t ph = kv.phase;
                    bar_wait(b_k_full + 8 * st, ph);
                    if (i > 0) bar_wait(b_s_empty, (i - 1) & 1);
                    tc_fence_after();
                    if (wide) {
                        // S = sum over the depth chunks (exact int32 accumulation)
                        for (int32_t c = 0; c < p.wide_chunks; ++c, ++ci) {
                            const uint32_t cs = ci % 3;
                            bar_wait(b_c_full + 8 * cs, (ci / 3) & 1);
                            tc_fence_after();
                            const uint64_t qc = smem_desc(smem_u32(chunk_q(cs)), 16, kSbo, kLayout);
                            const uint64_t kc = smem_desc(smem_u32(chunk_k(cs)), 16, kSbo, kLayout);
                            if (elect_one()) {
#pragma unroll
                                for (int kk = 0; kk < D / 32; ++kk)
                                    mma_i8_ss(tmem + T_S, qc + 2 * kk, kc + 2 * kk, kIdescS,
                                              (c > 0 || kk > 0) ? 1u : 0u);
                                mma_commit_u32(b_c_empty + 8 * cs);
                            }
                            __syncwarp();
                        }
                        if (elect_one()) {
                            mma_commit_u32(b_s_full);
                            if (!(it.kind & K_PV)) mma_commit_u32(b_kv_empty + 8 * st);
                        }
                        __syncwarp();
                    } else {
                    const uint64_t q_desc = smem_desc(q_base, 16, kSbo, kLayout);
                    const uint64_t k_desc = smem_desc(smem_u32(sm.k[st]), 16, kSbo, kLayout);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < D / 32; ++kk)
                            mma_i8_ss(tmem + T_S, q_desc + 2 * kk, k_desc + 2 * kk, kIdescS,
                                      kk > 0 ? 1u : 0u);
                        mma_commit_u32(b_s_full);
                        if (!(it.kind & K_PV)) mma_commit_u32(b_kv_empty + 8 * st);
                    }
                    __syncwarp();
                    }
                    if (have_prev) issue_pv(prev_st, prev_ph, prev_kind, prev_pi);
                    if (it.kind & K_PV) {
                        have_prev = true;
                        prev_st = st;
                        prev_ph = ph;
                        prev_kind = it.kind;
                        prev_pi = pi++;
                    } else {
                        have_prev = false;
                    }
                    kv.advance();
                    ++i;
                }
                // every S MMA reading this Q buffer has been issued
                if (!wide && elect_one()) mma_commit_u32(b_q_empty + 8 * qb);
                __syncwarp();
            }
            if (have_prev) issue_pv(prev_st, prev_ph, prev_kind, prev_pi);
        }
        __syncwarp();
      }
    } else if constexpr (QUAD) {
        regs_alloc<kRegsMathQuad>();
        softmax_quad<D>(sm, p, tmem, warp, lane, b_s_full, b_s_empty, b_k_full, b_kv_empty,
                        b_p_full, b_p_empty, b_pv_full, b_pv_empty);
    } else {
        regs_alloc<kRegsSoftmax>();
        // ------------------------------------------------- softmax + correction
        const uint32_t quarter = warp & 3;
        const uint32_t part = (warp - SOFT_WARP0) >> 2;  // which NCOL-column slice of the row
        const int32_t row = static_cast<int32_t>(quarter * 32 + lane);
        const uint32_t t_lane = tmem + ((quarter * 32) << 16);
        const uint32_t t_s = t_lane + T_S + NCOL * part;
        const uint32_t t_p = t_lane + T_P0 + (NCOL / 4) * part;
        const uint32_t t_pv = t_lane + T_PV + NCOL * part;
        const uint32_t t_rs = t_lane + T_RS;
        const int32_t c_base = NCOL * part;  // first key / output column owned by this thread
        const uint32_t bar_id = 1 + quarter;
        const float extra = p.extra;
        const bool use_extra = GENERIC && (p.flags & IFA_FLAG_SQRT_D) != 0;
        float* const xmax_mine = &sm.xmax[0][row][part];
        const float* const xmax_row = &sm.xmax[0][row][0];
        const float* const sk_part = &sm.sk[0][c_base];
        int32_t cmin = 127, cmax = 0;
        bool all_hit = true;
        int64_t rows_done = 0;
        Ring<STAGES> kv;
        uint32_t i = 0, pi = 0, bi = 0;

        uint32_t wn = 0;
        for (int32_t idx = item_at(0, causal); idx < p.items; idx = item_at(++wn, causal)) {
            const Work w = work_of(idx, p, causal);
            const int32_t grow = w.q0 + row;
            const bool row_ok = grow < n;
            const float sq_r = row_ok ? p.sq[static_cast<int64_t>(w.slice) * n + grow] : 0.0f;
            float acc[NCOL];
#pragma unroll
            for (int c = 0; c < NCOL; ++c) acc[c] = 0.0f;
            float l = 0.0f;
            float m = kNegInf;
            float blk_max = kNegInf, m_new = kNegInf;
            bool has_full = false, row_hit = false;
            bool pend = false;
            float pend_alpha = 1.0f;  // FAST: computed by every thread

            // acc = acc*alpha + float(PV), l = l*alpha + float(rowsum)
            // (attention.cpp:313-318, :330-333) for the finished block bi;
            // alpha was published in SMEM by the block's designated part.
            auto fold_pv = [&](float alpha) {
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
                if constexpr (FAST) {
                    l = __fmaf_rn(l, alpha, static_cast<float>(static_cast<int32_t>(rs)));
#pragma unroll
                    for (int c = 0; c < NCOL; c += 2) {
                        const float2 pf = make_float2(__int2float_rn(static_cast<int32_t>(pv[c])),
                                                      __int2float_rn(static_cast<int32_t>(pv[c + 1])));
                        const float2 a = ffma2(make_float2(acc[c], acc[c + 1]), f2(alpha), pf);
                        acc[c] = a.x;
                        acc[c + 1] = a.y;
                    }
                    return;
                }
                l = __fadd_rn(__fmul_rn(l, alpha), static_cast<float>(static_cast<int32_t>(rs)));
                // acc *= alpha, rounded before the add (no FMA); skipped when
                // alpha == 1 for the whole warp, which leaves acc bit-identical.
                if (!__all_sync(0xffffffffu, alpha == 1.0f)) {
#pragma unroll
                    for (int c = 0; c < NCOL; c += 2) {
                        const float2 a = fmul2_nc(make_float2(acc[c], acc[c + 1]), f2(alpha));
                        acc[c] = a.x;
                        acc[c + 1] = a.y;
                    }
                }
#pragma unroll
                for (int c = 0; c < NCOL; c += 2) {
                    // float(int32) exact here: |PV| < 127*127*Bc < 2^24 for Bc <= 1040;
                    // I2FP rounds to nearest like the reference's cast otherwise.
                    const float2 pf = make_float2(__int2float_rn(static_cast<int32_t>(pv[c])),
                                                  __int2float_rn(static_cast<int32_t>(pv[c + 1])));
                    const float2 a = fadd2(make_float2(acc[c], acc[c + 1]), pf);
                    acc[c] = a.x;
                    acc[c + 1] = a.y;
                }
            };

            auto gen = make_gen<GENERIC>(n, p.bc, w.kv_limit);
            Item it;
            while (gen.next(it)) {
                const uint32_t st = kv.idx;
                bar_wait(b_s_full, i & 1);
                tc_fence_after();
                uint32_t sr[NCOL];
                tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(b_s_empty);

                bar_wait(b_k_full + 8 * st, kv.phase);
                int32_t lim = it.width;
                if (causal) {
                    const int32_t vis = grow - it.key0 + 1;
                    if (vis < lim) lim = vis < 0 ? 0 : vis;
                }
                lim -= c_base;  // columns of this slice still visible
                float s[NCOL];
                const float4* sk4 = reinterpret_cast<const float4*>(sk_part + st * BN);
                if constexpr (FAST) {
                    // u = float(S) * (sK * log2e [* extra]): log2-domain scores
                    // before the per-row factor sQ (>= 0, so the row max
                    // commutes with it; it is applied inside the exp2 FMA)
#pragma unroll
                    for (int c4 = 0; c4 < NCOL / 4; ++c4) {
                        const float4 k4 = sk4[c4];
                        const int c = c4 * 4;
                        const float2 sf01 = make_float2(__int2float_rn(static_cast<int32_t>(sr[c])),
                                                        __int2float_rn(static_cast<int32_t>(sr[c + 1])));
                        const float2 sf23 = make_float2(__int2float_rn(static_cast<int32_t>(sr[c + 2])),
                                                        __int2float_rn(static_cast<int32_t>(sr[c + 3])));
                        const float2 s01 = fmul2(sf01, make_float2(k4.x, k4.y));
                        const float2 s23 = fmul2(sf23, make_float2(k4.z, k4.w));
                        s[c] = s01.x;
                        s[c + 1] = s01.y;
                        s[c + 2] = s23.x;
                        s[c + 3] = s23.y;
                    }
                } else {
                // dequantize: s = float(S) * (sQ * sK) [* extra], product of scales first
#pragma unroll
                for (int c4 = 0; c4 < NCOL / 4; ++c4) {
                    const float4 k4 = sk4[c4];
                    const int c = c4 * 4;
                    // float(S) exact (|S| < 2^24)
                    const float2 sf01 = make_float2(__int2float_rn(static_cast<int32_t>(sr[c])),
                                                    __int2float_rn(static_cast<int32_t>(sr[c + 1])));
                    const float2 sf23 = make_float2(__int2float_rn(static_cast<int32_t>(sr[c + 2])),
                                                    __int2float_rn(static_cast<int32_t>(sr[c + 3])));
                    float2 s01 = fmul2(sf01, fmul2(f2(sq_r), make_float2(k4.x, k4.y)));
                    float2 s23 = fmul2(sf23, fmul2(f2(sq_r), make_float2(k4.z, k4.w)));
                    if (use_extra) {
                        s01 = fmul2(s01, f2(extra));
                        s23 = fmul2(s23, f2(extra));
                    }
                    s[c] = s01.x;
                    s[c + 1] = s01.y;
                    s[c + 2] = s23.x;
                    s[c + 3] = s23.y;
                }
                }
                __syncwarp();
                if (lane == 0) bar_arrive(b_kv_empty + 8 * st);
                if (lim < NCOL) {
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) s[c] = c < lim ? s[c] : kNegInf;
                }
                const float m_part = row_max(s);
                float s_min = -kNegInf;
                if (GENERIC && audit) {
#pragma unroll
                    for (int c = 0; c < NCOL; ++c)
                        if (c < lim) s_min = fminf(s_min, s[c]);
                }
                // partial row max exchange among the SPLIT threads of this row;
                // the previous block's P.V is folded while the others catch up
                xmax_mine[(i & 1) * SPLIT * BM] = m_part;
                named_bar_sync(bar_id, 32 * SPLIT);
                float m_loc;
                {
                    const float4 x4 =
                        *reinterpret_cast<const float4*>(xmax_row + (i & 1) * SPLIT * BM);
                    m_loc = fmaxf(fmax3(x4.x, x4.y, x4.z), x4.w);
                }

                if (it.kind & K_BEGIN) blk_max = kNegInf;
                if (!(it.kind & K_PV) || (it.kind & K_BEGIN)) blk_max = fmaxf(blk_max, m_loc);
                if (it.kind & K_MAXDONE) {
                    m_new = (m < blk_max) ? blk_max : m;  // std::max(m, m_loc)
                    // the block's largest code comes from its largest score
                    if (GENERIC && audit)
                        has_full = blk_max != kNegInf &&
                                   guarded_code(__fsub_rn(blk_max, m_new)) == 127;
                }
                if (it.kind & K_PV) {
                    if (pi >= 2) {
                        bar_wait(b_p_empty + 8 * (pi & 1), ((pi - 2) >> 1) & 1);
                        tc_fence_after();
                    }
                    uint32_t wd[NCOL / 4];
                    if constexpr (FAST) {
                        codes_fast(s, sq_r, kLog2_127 - sq_r * m_new, wd);
                        if (lim < NCOL) {  // masked keys: code 0 even when sQ == 0
#pragma unroll
                            for (int c = 0; c < NCOL; ++c)
                                if (c >= lim) wd[c >> 2] &= ~(0xffu << (8 * (c & 3)));
                        }
                    } else {
                        const float mL = __fmul_rn(m_new, kLog2e);
                        const float c_r = __fsub_rn(kLog2_127, mL);
                        const float thresh =
                            0.5f - (kGuardBase + kGuardScale * (fabsf(mL) + fabsf(c_r)));
                        codes_part(s, m_new, c_r, thresh, sm.bounds, wd);
                    }
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                            t_p + 32 * (pi & 1)),
                        "r"(wd[0]), "r"(wd[1]), "r"(wd[2]), "r"(wd[3]), "r"(wd[4]), "r"(wd[5]),
                        "r"(wd[6]), "r"(wd[7])
                        : "memory");
                    if (GENERIC && audit && row_ok && lim > 0) {
                        cmax = max(cmax, guarded_code(__fsub_rn(m_part, m_new)));
                        cmin = min(cmin, guarded_code(__fsub_rn(s_min, m_new)));
                    }
                    // fold the previous block's P.V (finished long ago) while
                    // the code stores drain; it must precede p_full so the
                    // next P.V may overwrite the single accumulator
                    if (pend) {
                        fold_pv(FAST ? pend_alpha : sm.alpha[bi & 1][row]);
                        pend = false;
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(b_p_full + 8 * (pi & 1));
                    ++pi;
                    if (it.kind & K_END) {
                        // alpha = expf(m - m_new) (attention.cpp:298), exp(0) = 1: one
                        // part per block computes it (rotating) and publishes it;
                        // the fold reads it after the next row-max barrier
                        if constexpr (FAST) {
                            pend_alpha = (m_new == m) ? 1.0f
                                         : (m == kNegInf ? 0.0f : ex2_approx(sq_r * (m - m_new)));
                        } else if (part == (bi & 3)) {
                            const float alpha =
                                (m_new == m) ? 1.0f : exact_expf(__fsub_rn(m, m_new));
                            sm.alpha[bi & 1][row] = alpha;
                        }
                        if (m_new > m)
                            row_hit = has_full;
                        else if (blk_max == m_new && has_full)
                            row_hit = true;
                        m = m_new;
                        pend = true;  // its P.V is folded during the next tile
                    }
                }
                kv.advance();
                ++i;
            }
            if (pend) {
                if (!FAST) named_bar_sync(bar_id, 32 * SPLIT);  // the last alpha is published
                fold_pv(FAST ? pend_alpha : sm.alpha[bi & 1][row]);
            }

            // epilogue: O = (acc / l) * sV (attention.cpp:335-342)
            if (row_ok && c_base < p.o_cols) {
                const float sv = p.sv[w.slice];
                const int32_t d = p.o_cols;
                float* orow = p.o + (static_cast<int64_t>(w.slice) * n + grow) * p.o_pitch + c_base;
                float out[NCOL];
                if constexpr (FAST) {
                    const float f = __fdiv_rn(sv, l);
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) out[c] = acc[c] * f;
                } else {
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) out[c] = __fmul_rn(__fdiv_rn(acc[c], l), sv);
                }
                if (p.o_pitch % 4 == 0 && c_base + NCOL <= d) {
#pragma unroll
                    for (int c = 0; c < NCOL; c += 4)
                        __stcs(reinterpret_cast<float4*>(orow + c),
                               make_float4(out[c], out[c + 1], out[c + 2], out[c + 3]));
                } else {
#pragma unroll
                    for (int c = 0; c < NCOL; ++c)
                        if (c_base + c < d) orow[c] = out[c];
                }
            }
            if (GENERIC && audit && row_ok) {
                all_hit = all_hit && row_hit;
                if (part == 0) ++rows_done;
            }
        }
        if (GENERIC && audit) {
            // rows >= n never emitted a code; only part 0 counts rows
            int32_t my_min = cmin;
            int32_t my_max = cmax;
            int32_t my_hit = all_hit ? 1 : 0;
            unsigned long long my_rows = static_cast<unsigned long long>(rows_done);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                my_min = min(my_min, __shfl_xor_sync(0xffffffffu, my_min, o));
                my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
                my_hit = my_hit & __shfl_xor_sync(0xffffffffu, my_hit, o);
                my_rows += __shfl_xor_sync(0xffffffffu, my_rows, o);
            }
            if (lane == 0) {
                if (my_min < 127) atomicMin(&p.audit->min_code, my_min);
                if (my_max > 0) atomicMax(&p.audit->max_code, my_max);
                if (!my_hit) atomicAnd(&p.audit->row_max_block_hits_127, 0);
                if (my_rows)
                    atomicAdd(reinterpret_cast<unsigned long long*>(&p.audit->rows_audited),
                              my_rows);
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

// ------------------------------------------------------------------ host side
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

// [slices][n][pitch] int8 codes, box = (D, 128 rows, 1 slice)
// (cols = the row extent TMA may read, default the pitch; columns past it load as 0)
static bool make_map(CUtensorMap* map, const int8_t* base, int64_t slices, int64_t n,
                     int64_t pitch, int D, int64_t cols = 0) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols > 0 ? cols : pitch), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(slices)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch),
                                   static_cast<cuuint64_t>(pitch * n)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(D), 128u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// V as a 5-D view [k''][t0][m][e][d] with strides {32, 2, 8, 1} rows: one box
// of 128 keys lands in shared memory with row p = e + 2m + 8t0 + 32k' holding
// key e + 8m + 2t0 + 32k' (a 4x4 transpose of row pairs inside every 32-key
// group), which is the key order of the quad kernel's packed P words.
// Needs n % 32 == 0 (the slices are flattened into the k'' dimension).
static bool make_map_vperm(CUtensorMap* map, const int8_t* base, int64_t slices, int64_t n,
                           int64_t pitch, int D) {
    PFN_encodeTiled enc = get_encode();
    if (!enc || n % 32 != 0) return false;
    const cuuint64_t dims[5] = {static_cast<cuuint64_t>(pitch), 2, 4, 4,
                                static_cast<cuuint64_t>(slices * n / 32)};
    const cuuint64_t strides[4] = {static_cast<cuuint64_t>(pitch),
                                   static_cast<cuuint64_t>(8 * pitch),
                                   static_cast<cuuint64_t>(2 * pitch),
                                   static_cast<cuuint64_t>(32 * pitch)};
    const cuuint32_t box[5] = {static_cast<cuuint32_t>(D), 2u, 4u, 4u, 4u};
    const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<int8_t*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int D, bool GENERIC, bool FAST, bool QUAD = false>
static cudaError_t launch_k(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const Params& p, int64_t slices, cudaStream_t stream) {
    const size_t smem = sizeof(Smem<D>) + 1024;
    const cudaError_t e = smem_attr_once<int_flash_fwd_kernel<D, GENERIC, FAST, QUAD>>(smem);
    if (e != cudaSuccess) return e;
    // persistent: one CTA per SM (the kernel needs the whole SM: 512 TMEM
    // columns, ~170 KB of shared memory)
    const int sms = current_device_sms();
    (void)slices;
    const int grid = p.items < sms ? p.items : sms;
    constexpr int threads = QUAD ? 32 * (SOFT_WARP0 + QUAD_WARPS) : NUM_THREADS;
    int_flash_fwd_kernel<D, GENERIC, FAST, QUAD><<<grid, threads, smem, stream>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

// IFA_B200_NO_QUAD=1 selects the 16-warp tolerance kernel instead (A/B runs;
// read at every call so a test can flip it).
static bool quad_off() {
    const char* e = getenv("IFA_B200_NO_QUAD");
    return e && e[0] == '1';
}

template <int D>
static cudaError_t launch_d(const AttnArgs& a, cudaStream_t stream) {
    CUtensorMap tq, tk, tv;
    if (!make_map(&tq, a.q, a.slices, a.n, a.pitch, D) ||
        !make_map(&tk, a.k, a.slices, a.n, a.pitch, D) ||
        !make_map(&tv, a.v, a.slices, a.n, a.pitch, D))
        return cudaErrorInvalidValue;
    Params p;
    p.sq = a.sq;
    p.sk = a.sk;
    p.sv = a.sv;
    p.o = a.o;
    p.audit = a.audit;
    p.n = static_cast<int32_t>(a.n);
    p.d = static_cast<int32_t>(a.d);
    p.bc = static_cast<int32_t>(a.bc < a.n ? a.bc : a.n);
    p.flags = a.flags;
    p.extra = (a.flags & IFA_FLAG_SQRT_D) ? 1.0f / sqrtf(static_cast<float>(a.d)) : 1.0f;
    p.sk_mul = 1.4426950408889634f * p.extra;
    p.q_tiles = static_cast<int32_t>((a.n + BM - 1) / BM);
    p.slices = static_cast<int32_t>(a.slices);
    p.items = p.q_tiles * p.slices;
    p.o_cols = p.d;
    p.o_pitch = a.d;
    const float* bounds = code_bounds();
    for (int k = 0; k < 128; ++k) p.bounds[k] = bounds[k];
    // the benchmark-shaped fast path, or the fully general kernel
    // (fast path: every KV block is exactly one 128-key tile, or the whole
    // sequence when it is shorter)
    const bool tiles_are_blocks = p.bc == BN || (p.bc == p.n && p.n <= BN);
    const bool generic = a.audit != nullptr || (a.flags & (IFA_FLAG_SQRT_D | IFA_FLAG_CAUSAL)) ||
                         !tiles_are_blocks;
    // tolerance mode (no audit: the audit reports the exact codes); the quad
    // kernel when the V view can be permuted
    if ((a.flags & IFA_FLAG_FAST) && a.audit == nullptr && tiles_are_blocks && !quad_off()) {
        CUtensorMap tvp;
        if (make_map_vperm(&tvp, a.v, a.slices, a.n, a.pitch, D))
            return launch_k<D, false, true, true>(tq, tk, tvp, p, a.slices, stream);
    }
    if ((a.flags & IFA_FLAG_FAST) && a.audit == nullptr)
        return generic ? launch_k<D, true, true>(tq, tk, tv, p, a.slices, stream)
                       : launch_k<D, false, true>(tq, tk, tv, p, a.slices, stream);
    return generic ? launch_k<D, true, false>(tq, tk, tv, p, a.slices, stream)
                   : launch_k<D, false, false>(tq, tk, tv, p, a.slices, stream);
}

// Head dims > 128 (the reference takes any d up to 133144, gemm.hpp:22,
// attention.cpp:241-242): the general 16-warp kernel with S accumulated over
// 128-column depth chunks of Q and K (exact int32 on the tensor core), one
// launch per 128-column chunk of O (V and O offset to the chunk).  P depends on
// S alone, so every launch makes the same codes; the audit is taken from the
// first.
static cudaError_t launch_wide(const AttnArgs& a, cudaStream_t stream) {
    CUtensorMap tq, tk;
    if (!make_map(&tq, a.q, a.slices, a.n, a.pitch, 128) ||
        !make_map(&tk, a.k, a.slices, a.n, a.pitch, 128))
        return cudaErrorInvalidValue;
    Params p;
    p.sq = a.sq;
    p.sk = a.sk;
    p.sv = a.sv;
    p.n = static_cast<int32_t>(a.n);
    p.d = static_cast<int32_t>(a.d);
    p.bc = static_cast<int32_t>(a.bc < a.n ? a.bc : a.n);
    p.flags = a.flags;
    p.extra = (a.flags & IFA_FLAG_SQRT_D) ? 1.0f / sqrtf(static_cast<float>(a.d)) : 1.0f;
    p.sk_mul = 1.4426950408889634f * p.extra;
    p.q_tiles = static_cast<int32_t>((a.n + BM - 1) / BM);
    p.slices = static_cast<int32_t>(a.slices);
    p.items = p.q_tiles * p.slices;
    p.wide_chunks = static_cast<int32_t>((a.d + 127) / 128);
    p.o_pitch = a.d;
    const float* bounds = code_bounds();
    for (int k = 0; k < 128; ++k) p.bounds[k] = bounds[k];
    const bool fast = (a.flags & IFA_FLAG_FAST) && a.audit == nullptr;
    for (int64_t c0 = 0; c0 < a.d; c0 += 128) {
        CUtensorMap tv;
        if (!make_map(&tv, a.v + c0, a.slices, a.n, a.pitch, 128, a.pitch - c0))
            return cudaErrorInvalidValue;
        p.o = a.o + c0;
        p.o_cols = static_cast<int32_t>(a.d - c0 < 128 ? a.d - c0 : 128);
        p.audit = c0 == 0 ? a.audit : nullptr;
        const cudaError_t e = fast ? launch_k<128, true, true>(tq, tk, tv, p, a.slices, stream)
                                   : launch_k<128, true, false>(tq, tk, tv, p, a.slices, stream);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace attn

cudaError_t launch_int_flash_fwd(const AttnArgs& a, cudaStream_t stream) {
    if (a.n > (int64_t{1} << 30) || ((a.n + 127) / 128) * a.slices > INT32_MAX)
        return cudaErrorInvalidValue;
    if (a.d > 128) return attn::launch_wide(a, stream);
    if (int_flash_pp_eligible(a)) return launch_int_flash_pp(a, nullptr, stream);
    if (a.d <= 64) return attn::launch_d<64>(a, stream);
    return attn::launch_d<128>(a, stream);
}

}  // namespace ifa_b200
