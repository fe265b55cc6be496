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
// One CTA owns a 128-row Q tile of one (b,h) slice.  Warp roles:
//   warp 0      TMA producer: Q once, then a STAGES-deep ring of K / V tiles
//               (128 keys x D int8, 128B or 64B swizzle) + the K scales.
//   warp 1      MMA issuer (one thread): S = Q.K^T  (tcgen05.mma kind::i8,
//               A and B from SMEM) into TMEM; PV = P.V (A = P from TMEM,
//               B = V from SMEM, MN-major) into TMEM.
//   warp 2      TMEM allocator.
//   warps 4-7   softmax: thread r owns Q row r (= TMEM lane r); reads the
//               int32 S row with tcgen05.ld, dequantizes, row max, exact
//               expf-based requantization of P to int8, writes P to TMEM.
//   warps 8-11  correction: acc = acc*alpha + float(PV) on the f32
//               accumulator kept in TMEM; final O = (acc/l)*sV epilogue.
// TMEM columns: S [0,128) | PV [128,256) | ACC [256,384) | P0 [384,416) |
// P1 [416,448).
//
// Bc (the reference's KV block size, which changes results) is honoured:
// a block of <= 128 keys is one pipeline item; a larger block is processed
// in two passes over 128-key sub-tiles (pass 1: block row max, pass 2:
// codes + PV accumulated in int32 across the sub-tiles), exactly the
// reference's per-block arithmetic.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "exact_expf.cuh"
#include "ifa_internal.h"
#include "ptx.cuh"

namespace ifa_b200 {

using namespace ptx;

namespace attn {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int STAGES = 3;
constexpr int NUM_THREADS = 384;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t T_S = 0, T_PV = 128, T_ACC = 256, T_P0 = 384;

enum ItemKind : uint32_t {
    K_MAXONLY = 1u,   // pass-1 sub-tile of a multi-tile block: contributes to the row max
    K_BEGIN = 2u,     // first item of a block
    K_MAXDONE = 4u,   // block max complete after this item
    K_PV = 8u,        // item produces P codes and a P.V product
    K_PV_FIRST = 16u, // first P.V item of the block (fresh int32 accumulator)
    K_END = 32u,      // last item of the block: l / acc update
};

struct Item {
    int64_t key0;
    int32_t width;
    uint32_t kind;
};

// Deterministic item sequence shared by every warp role.
struct ItemGen {
    int64_t n, bc, kv_limit;
    int64_t b0 = 0;
    int32_t s = 0, pass = 0;

    __device__ ItemGen(int64_t n_, int64_t bc_, int64_t kv_limit_)
        : n(n_), bc(bc_), kv_limit(kv_limit_) {}

    __device__ bool next(Item& it) {
        if (b0 >= kv_limit) return false;
        const int64_t blk_end = (bc >= n - b0) ? n : b0 + bc;
        const int64_t lim_end = blk_end < kv_limit ? blk_end : kv_limit;
        const int64_t len = lim_end - b0;
        const int32_t nsub = static_cast<int32_t>((len + BN - 1) / BN);
        it.key0 = b0 + static_cast<int64_t>(BN) * s;
        const int64_t rem = lim_end - it.key0;
        it.width = static_cast<int32_t>(rem < BN ? rem : BN);
        if (nsub == 1) {
            it.kind = K_BEGIN | K_MAXDONE | K_PV | K_PV_FIRST | K_END;
            b0 = blk_end;
            s = 0;
            pass = 0;
        } else if (pass == 0) {
            it.kind = K_MAXONLY | (s == 0 ? K_BEGIN : 0u) | (s == nsub - 1 ? K_MAXDONE : 0u);
            if (++s == nsub) {
                s = 0;
                pass = 1;
            }
        } else {
            it.kind = K_PV | (s == 0 ? K_PV_FIRST : 0u) | (s == nsub - 1 ? K_END : 0u);
            if (++s == nsub) {
                b0 = blk_end;
                s = 0;
                pass = 0;
            }
        }
        return true;
    }
};

template <int D>
struct alignas(1024) Smem {
    uint8_t q[BM * D];
    uint8_t k[STAGES][BN * D];
    uint8_t v[STAGES][BN * D];
    float sk[STAGES][BN];
    float alpha[4][BM];
    float lfin[BM];
    uint64_t q_full;
    uint64_t k_full[STAGES], v_full[STAGES], kv_empty[STAGES];
    uint64_t s_full, s_empty;
    uint64_t p_full[2], p_empty[2];
    uint64_t pv_full, pv_empty;
    uint64_t alpha_full[4];
    uint64_t l_full;
    uint32_t tmem_base;
};

struct Params {
    const float* sq;
    const float* sk;
    const float* sv;
    float* o;
    ifa_pcode_audit* audit;
    int64_t n;
    int64_t d;
    int64_t bc;
    uint32_t flags;
    float extra;  // 1/sqrt(d) when IFA_FLAG_SQRT_D, else 1
    int32_t q_tiles;
};

__device__ __forceinline__ float warp_min_i(float v) { return v; }

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    int_flash_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const Params p) {
    constexpr uint32_t kLayout = D == 128 ? kLayoutSw128 : kLayoutSw64;
    constexpr uint32_t kSbo = 8 * D;  // 8 rows of D bytes per swizzle atom
    constexpr uint32_t kTileBytes = BN * D;
    constexpr uint32_t kIdescS = idesc_i8(BM, BN, false, false);
    constexpr uint32_t kIdescPV = idesc_i8(BM, D, false, true);

    extern __shared__ uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const bool causal = (p.flags & IFA_FLAG_CAUSAL) != 0;
    // Heavier causal tiles first (longest-processing-time order).
    const int32_t qt = causal ? (p.q_tiles - 1 - static_cast<int32_t>(blockIdx.x))
                              : static_cast<int32_t>(blockIdx.x);
    const int64_t q0 = static_cast<int64_t>(qt) * BM;
    const int64_t slice = blockIdx.y;
    const int64_t n = p.n;
    int64_t kv_limit = n;
    if (causal && q0 + BM < kv_limit) kv_limit = q0 + BM;

    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&sm.k_full[i], 32);
            mbar_init(&sm.v_full[i], 1);
            mbar_init(&sm.kv_empty[i], 1 + 4);
        }
        mbar_init(&sm.s_full, 1);
        mbar_init(&sm.s_empty, 4);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.p_full[i], 4);
            mbar_init(&sm.p_empty[i], 1);
        }
        mbar_init(&sm.pv_full, 1);
        mbar_init(&sm.pv_empty, 4);
        for (int i = 0; i < 4; ++i) mbar_init(&sm.alpha_full[i], 4);
        mbar_init(&sm.l_full, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<TMEM_COLS>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            mbar_arrive_expect_tx(&sm.q_full, BM * D);
            tma_load_3d(sm.q, &tm_q, &sm.q_full, 0, static_cast<int32_t>(q0),
                        static_cast<int32_t>(slice), pol_stream);
        }
        const float* sk_slice = p.sk + slice * n;
        ItemGen gen(n, p.bc, kv_limit);
        Item it;
        uint32_t i = 0;
        while (gen.next(it)) {
            const uint32_t st = i % STAGES;
            if (i >= STAGES) mbar_wait(&sm.kv_empty[st], ((i / STAGES) - 1) & 1);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t key = it.key0 + lane * 4 + e;
                sm.sk[st][lane * 4 + e] = key < n ? sk_slice[key] : 0.0f;
            }
            if (lane == 0) {
                mbar_arrive_expect_tx(&sm.k_full[st], kTileBytes);
                tma_load_3d(sm.k[st], &tm_k, &sm.k_full[st], 0, static_cast<int32_t>(it.key0),
                            static_cast<int32_t>(slice), pol_keep);
                if (it.kind & K_PV) {
                    mbar_arrive_expect_tx(&sm.v_full[st], kTileBytes);
                    tma_load_3d(sm.v[st], &tm_v, &sm.v_full[st], 0,
                                static_cast<int32_t>(it.key0), static_cast<int32_t>(slice),
                                pol_keep);
                } else {
                    mbar_arrive(&sm.v_full[st]);
                }
            } else {
                mbar_arrive(&sm.k_full[st]);
            }
            ++i;
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            mbar_wait(&sm.q_full, 0);
            tc_fence_after();
            const uint32_t q_base = smem_u32(sm.q);
            ItemGen gen(n, p.bc, kv_limit);
            Item it;
            uint32_t i = 0, pi = 0, bi = 0;
            bool have_prev = false;
            uint32_t prev_st = 0, prev_ph = 0, prev_kind = 0, prev_pi = 0;
            auto issue_pv = [&](uint32_t st, uint32_t ph, uint32_t kind, uint32_t pidx) {
                mbar_wait(&sm.p_full[pidx & 1], (pidx >> 1) & 1);
                mbar_wait(&sm.v_full[st], ph);
                if ((kind & K_PV_FIRST) && bi > 0) mbar_wait(&sm.pv_empty, (bi - 1) & 1);
                tc_fence_after();
                const uint32_t v_base = smem_u32(sm.v[st]);
                const uint32_t p_col = T_P0 + 32 * (pidx & 1);
#pragma unroll
                for (int kk = 0; kk < BN / 32; ++kk) {
                    // B = V tile, MN-major: 32 keys x D per step = 32 rows of D bytes.
                    const uint64_t bdesc = smem_desc(v_base + kk * 32 * D, 16, kSbo, kLayout);
                    const uint32_t acc = ((kind & K_PV_FIRST) && kk == 0) ? 0u : 1u;
                    mma_i8_ts(tmem + T_PV, tmem + p_col + kk * 8, bdesc, kIdescPV, acc);
                }
                mma_commit(&sm.p_empty[pidx & 1]);
                mma_commit(&sm.kv_empty[st]);
                if (kind & K_END) {
                    mma_commit(&sm.pv_full);
                    ++bi;
                }
            };
            while (gen.next(it)) {
                const uint32_t st = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&sm.k_full[st], ph);
                if (i > 0) mbar_wait(&sm.s_empty, (i - 1) & 1);
                tc_fence_after();
                const uint32_t k_base = smem_u32(sm.k[st]);
#pragma unroll
                for (int kk = 0; kk < D / 32; ++kk) {
                    const uint64_t adesc = smem_desc(q_base + kk * 32, 16, kSbo, kLayout);
                    const uint64_t bdesc = smem_desc(k_base + kk * 32, 16, kSbo, kLayout);
                    mma_i8_ss(tmem + T_S, adesc, bdesc, kIdescS, kk > 0 ? 1u : 0u);
                }
                mma_commit(&sm.s_full);
                if (!(it.kind & K_PV)) mma_commit(&sm.kv_empty[st]);
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
                ++i;
            }
            if (have_prev) issue_pv(prev_st, prev_ph, prev_kind, prev_pi);
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------------------ softmax
        const uint32_t quarter = warp - 4;
        const int32_t row = static_cast<int32_t>(quarter * 32 + lane);
        const int64_t grow = q0 + row;
        const bool row_ok = grow < n;
        const float sq_r = row_ok ? p.sq[slice * n + grow] : 0.0f;
        const uint32_t t_lane = tmem + ((quarter * 32) << 16);
        const float extra = p.extra;
        float m = -__int_as_float(0x7f800000);
        float l = 0.0f;
        float blk_max = m, m_new = m, alpha = 0.0f;
        int32_t p_sum = 0;
        bool has_full = false;
        bool row_hit = false;
        int32_t cmin = 127, cmax = 0;
        ItemGen gen(n, p.bc, kv_limit);
        Item it;
        uint32_t i = 0, pi = 0, bi = 0;
        while (gen.next(it)) {
            const uint32_t st = i % STAGES;
            mbar_wait(&sm.s_full, i & 1);
            tc_fence_after();
            uint32_t sr[BN];
#pragma unroll
            for (int c = 0; c < BN; c += 32)
                tmem_ld32(t_lane + T_S + c, *reinterpret_cast<uint32_t(*)[32]>(&sr[c]));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.s_empty);

            mbar_wait(&sm.k_full[st], (i / STAGES) & 1);
            int32_t lim = it.width;
            if (causal) {
                const int64_t vis = grow - it.key0 + 1;
                if (vis < lim) lim = vis < 0 ? 0 : static_cast<int32_t>(vis);
            }
            // dequantize: s = float(S) * (sQ * sK) [* extra], product of scales first
            float m_loc = -__int_as_float(0x7f800000);
            const float4* sk4 = reinterpret_cast<const float4*>(sm.sk[st]);
#pragma unroll
            for (int c4 = 0; c4 < BN / 4; ++c4) {
                const float4 k4 = sk4[c4];
                const float kv[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = c4 * 4 + e;
                    float s = __fmul_rn(__int2float_rn(static_cast<int32_t>(sr[c])),
                                        __fmul_rn(sq_r, kv[e]));
                    if (extra != 1.0f) s = __fmul_rn(s, extra);
                    s = c < lim ? s : -__int_as_float(0x7f800000);
                    m_loc = fmaxf(m_loc, s);
                    sr[c] = __float_as_uint(s);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.kv_empty[st]);

            if (it.kind & K_BEGIN) blk_max = -__int_as_float(0x7f800000);
            if (!(it.kind & K_PV) || (it.kind & K_BEGIN)) blk_max = fmaxf(blk_max, m_loc);
            if (it.kind & K_MAXDONE) {
                m_new = (m < blk_max) ? blk_max : m;  // std::max(m, m_loc)
                alpha = exact_expf(__fsub_rn(m, m_new));
                p_sum = 0;
                has_full = false;
            }
            if (it.kind & K_PV) {
                if (it.kind & K_END) {
                    // l / alpha for the correction warps are final only after the
                    // codes; alpha is already known, publish it first.
                    sm.alpha[bi & 3][row] = alpha;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.alpha_full[bi & 3]);
                }
                if (pi >= 2) {
                    mbar_wait(&sm.p_empty[pi & 1], ((pi - 2) >> 1) & 1);
                    tc_fence_after();
                }
                const uint32_t p_col = T_P0 + 32 * (pi & 1);
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    uint32_t w[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        uint32_t packed = 0;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = c0 + j * 4 + e;
                            int code = 0;
                            if (c < lim) {
                                code = guarded_code(__fsub_rn(__uint_as_float(sr[c]), m_new));
                                p_sum += code;
                                has_full = has_full || code == 127;
                                cmin = min(cmin, code);
                                cmax = max(cmax, code);
                            }
                            packed |= static_cast<uint32_t>(code) << (8 * e);
                        }
                        w[j] = packed;
                    }
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                            t_lane + p_col + c0 / 4),
                        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                        "r"(w[7])
                        : "memory");
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.p_full[pi & 1]);
                if (it.kind & K_END) {
                    l = __fadd_rn(__fmul_rn(l, alpha), static_cast<float>(p_sum));
                    if (m_new > m)
                        row_hit = has_full;
                    else if (blk_max == m_new && has_full)
                        row_hit = true;
                    m = m_new;
                    ++bi;
                }
                ++pi;
            }
            ++i;
        }
        sm.lfin[row] = l;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.l_full);
        if (p.audit != nullptr) {
            // rows >= n and rows with no visible key never emitted a code
            int32_t my_min = row_ok ? cmin : 127;
            int32_t my_max = row_ok ? cmax : 0;
            int32_t my_hit = row_ok ? (row_hit ? 1 : 0) : 1;
            int32_t my_rows = row_ok ? 1 : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                my_min = min(my_min, __shfl_xor_sync(0xffffffffu, my_min, o));
                my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
                my_hit = my_hit & __shfl_xor_sync(0xffffffffu, my_hit, o);
                my_rows += __shfl_xor_sync(0xffffffffu, my_rows, o);
            }
            if (lane == 0 && my_rows > 0) {
                atomicMin(&p.audit->min_code, my_min);
                atomicMax(&p.audit->max_code, my_max);
                if (!my_hit) atomicAnd(&p.audit->row_max_block_hits_127, 0);
                atomicAdd(reinterpret_cast<unsigned long long*>(&p.audit->rows_audited),
                          static_cast<unsigned long long>(my_rows));
            }
        }
    } else if (warp >= 8) {
        // ------------------------------------------------------------ correction
        const uint32_t quarter = warp - 8;
        const int32_t row = static_cast<int32_t>(quarter * 32 + lane);
        const int64_t grow = q0 + row;
        const uint32_t t_lane = tmem + ((quarter * 32) << 16);
        ItemGen gen(n, p.bc, kv_limit);
        Item it;
        uint32_t bi = 0;
        while (gen.next(it)) {
            if (!(it.kind & K_END)) continue;
            mbar_wait(&sm.alpha_full[bi & 3], (bi >> 2) & 1);
            const float alpha = sm.alpha[bi & 3][row];
            mbar_wait(&sm.pv_full, bi & 1);
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
                uint32_t pv[32], acc[32];
                tmem_ld32(t_lane + T_PV + c0, pv);
                if (bi > 0) tmem_ld32(t_lane + T_ACC + c0, acc);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float pf = __int2float_rn(static_cast<int32_t>(pv[j]));
                    const float a = bi > 0 ? __fadd_rn(__fmul_rn(__uint_as_float(acc[j]), alpha), pf)
                                           : pf;
                    acc[j] = __float_as_uint(a);
                }
                tmem_st32(t_lane + T_ACC + c0, acc);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.pv_empty);
            ++bi;
        }
        // epilogue: O = (acc / l) * sV
        mbar_wait(&sm.l_full, 0);
        const float lr = sm.lfin[row];
        const float sv = p.sv[slice];
        tc_fence_after();
        const int64_t d = p.d;
        float* orow = p.o + (slice * n + grow) * d;
        const bool vec = (d % 4 == 0);
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t acc[32];
            tmem_ld32(t_lane + T_ACC + c0, acc);
            tmem_wait_ld();
            if (grow < n && c0 < d) {
                float out[32];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    out[j] = __fmul_rn(__fdiv_rn(__uint_as_float(acc[j]), lr), sv);
                if (vec && c0 + 32 <= d) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        __stcs(reinterpret_cast<float4*>(orow + c0 + j),
                               make_float4(out[j], out[j + 1], out[j + 2], out[j + 3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (c0 + j < d) orow[c0 + j] = out[j];
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
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
static bool make_map(CUtensorMap* map, const int8_t* base, int64_t slices, int64_t n,
                     int64_t pitch, int D) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(n),
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
    p.n = a.n;
    p.d = a.d;
    p.bc = a.bc;
    p.flags = a.flags;
    p.extra = (a.flags & IFA_FLAG_SQRT_D) ? 1.0f / sqrtf(static_cast<float>(a.d)) : 1.0f;
    p.q_tiles = static_cast<int32_t>((a.n + BM - 1) / BM);
    const size_t smem = sizeof(Smem<D>) + 1024;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(int_flash_fwd_kernel<D>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(static_cast<unsigned>(p.q_tiles), static_cast<unsigned>(a.slices));
    int_flash_fwd_kernel<D><<<grid, NUM_THREADS, smem, stream>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

}  // namespace attn

cudaError_t launch_int_flash_fwd(const AttnArgs& a, cudaStream_t stream) {
    if (a.slices > 65535) return cudaErrorInvalidValue;
    if (a.d <= 64) return attn::launch_d<64>(a, stream);
    return attn::launch_d<128>(a, stream);
}

}  // namespace ifa_b200
