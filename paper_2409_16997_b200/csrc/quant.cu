// quant.cu -- bit-exact INT8 quantization kernels (HBM-bandwidth bound).
//
// Reference semantics (/root/reference/proj/src/quant.cpp):
//   scale = max_abs(x) / 127.0f                         (:44-57, :59-69)
//   code  = scale == 0 ? 0 : clamp(round(x / scale), -127, 127)   (:25-32)
//   non-finite input -> error naming the first offending flat index (:14-22)
// round() is roundf (ties away from zero); x/scale is the IEEE quotient
// (nvcc -prec-div=true, no fast-math); max is order independent, so the
// parallel reductions below are bit-identical to the serial loop.
//
// Division: the IEEE quotient is only needed where it decides a rounding.
// Each row (or slice) computes r = RN(1/scale) once; per element q0 =
// RN(x*r) is within 2^-23*|x/scale| <= 1.6e-5 of the exact quotient and so
// within 2.4e-5 of the reference's RN(x/scale).  Whenever q0 is farther than
// kDivGuard from a half-integer, round(q0) IS the reference's code; the
// (rare) others are recomputed with the IEEE division itself.  A scale whose
// reciprocal overflows takes the IEEE path for the whole row.
//
// Per-row (Q, K), cols in {32, 64, 128, 256}: eight lanes per row, four rows
// per warp step, every lane holding its whole share of the row (128-bit
// streaming loads), codes packed four per 32-bit store.  Other shapes: one
// warp per row.  Per-tensor (V, one scale per (b,h) slice): a cluster of 8
// CTAs per slice, partial maxima exchanged through distributed shared memory,
// then the quantize pass re-reads the slice from L2.  Non-finite input is
// detected with a NaN-propagating max, then located exactly (rare path).
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "ifa_internal.h"

namespace ifa_b200 {

__device__ __forceinline__ int8_t quantize_one(float x, float scale) {
    if (scale == 0.0f) return 0;
    float q = roundf(__fdiv_rn(x, scale));
    q = fminf(fmaxf(q, -127.0f), 127.0f);
    return static_cast<int8_t>(static_cast<int>(q));
}

__device__ __forceinline__ uint32_t pack4(float a, float b, float c, float d, float scale) {
    return (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(a, scale)))) |
           (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(b, scale))) << 8) |
           (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(c, scale))) << 16) |
           (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(d, scale))) << 24);
}

__device__ __forceinline__ void note_nonfinite(float v, int64_t idx, int64_t* bad) {
    if (!isfinite(v) && bad != nullptr)
        atomicMin(reinterpret_cast<unsigned long long*>(bad), static_cast<unsigned long long>(idx));
}

constexpr float kDivGuard = 0.5f - 4.0e-5f;
constexpr float kMagicF = 12582912.0f;  // 1.5 * 2^23

// |a| max that propagates NaN (max.NaN.f32), so one check per row finds it.
__device__ __forceinline__ float absmax_nan(float m, float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(m), "f"(fabsf(a)), "f"(fabsf(b)));
    return d;
}

// Codes of 4 values: fast estimate + exact fallback.  Returns the packed word.
__device__ __forceinline__ uint32_t codes4(float4 v, float scale, float rcp, bool exact_row) {
    const float q[4] = {__fmul_rn(v.x, rcp), __fmul_rn(v.y, rcp), __fmul_rn(v.z, rcp),
                        __fmul_rn(v.w, rcp)};
    uint32_t b[4];
    float g = 0.0f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float t = __fadd_rn(q[e], kMagicF);
        g = fmaxf(g, fabsf(__fsub_rn(q[e], __fsub_rn(t, kMagicF))));
        b[e] = __float_as_uint(t);
    }
    uint32_t w = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040),
                             0x5410);
    if (exact_row || !(g <= kDivGuard)) w = pack4(v.x, v.y, v.z, v.w, scale);
    return w;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Vectorised per-row quantizer: cols % 4 == 0, 16-byte aligned rows,
// cols <= 128 * NV.  Each lane keeps its NV float4 in registers (one HBM
// read per element).
template <int NV>
__global__ void __launch_bounds__(256) quantize_rows_vec_kernel(
    const float* __restrict__ x, int64_t rows, int64_t cols, int8_t* __restrict__ codes,
    float* __restrict__ scales, int64_t* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t nvec = cols >> 2;
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         row < rows; row += warps_total) {
        const float4* src = reinterpret_cast<const float4*>(x + row * cols);
        float4 v[NV];
        float m = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t c4 = lane + 32 * i;
            if (c4 < nvec) {
                v[i] = __ldcs(src + c4);
                const int64_t base = row * cols + 4 * c4;
                note_nonfinite(v[i].x, base + 0, bad);
                note_nonfinite(v[i].y, base + 1, bad);
                note_nonfinite(v[i].z, base + 2, bad);
                note_nonfinite(v[i].w, base + 3, bad);
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[i].x), fabsf(v[i].y)),
                                   fmaxf(fabsf(v[i].z), fabsf(v[i].w))));
            }
        }
        m = warp_max(m);
        const float scale = __fdiv_rn(m, 127.0f);
        if (lane == 0) scales[row] = scale;
        uint32_t* dst = reinterpret_cast<uint32_t*>(codes + row * cols);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t c4 = lane + 32 * i;
            if (c4 < nvec) dst[c4] = pack4(v[i].x, v[i].y, v[i].z, v[i].w, scale);
        }
    }
}

// Generic per-row quantizer (any cols / alignment): two passes over the row.
__global__ void __launch_bounds__(256) quantize_rows_generic_kernel(
    const float* __restrict__ x, int64_t rows, int64_t cols, int8_t* __restrict__ codes,
    float* __restrict__ scales, int64_t* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         row < rows; row += warps_total) {
        const float* src = x + row * cols;
        float m = 0.0f;
        for (int64_t c = lane; c < cols; c += 32) {
            const float v = src[c];
            note_nonfinite(v, row * cols + c, bad);
            m = fmaxf(m, fabsf(v));
        }
        m = warp_max(m);
        const float scale = __fdiv_rn(m, 127.0f);
        if (lane == 0) scales[row] = scale;
        for (int64_t c = lane; c < cols; c += 32) codes[row * cols + c] = quantize_one(src[c], scale);
    }
}

// Per-slice absmax: grid (chunks, slices); result as float bits in amax[s].
__global__ void __launch_bounds__(256) slice_absmax_kernel(const float* __restrict__ x,
                                                           int64_t slice_elems,
                                                           uint32_t* __restrict__ amax,
                                                           int64_t* bad, int vec) {
    const int64_t s = blockIdx.y;
    const float* src = x + s * slice_elems;
    float m = 0.0f;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    if (vec) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        const int64_t n4 = slice_elems >> 2;
        for (int64_t i = tid; i < n4; i += stride) {
            const float4 v = s4[i];
            const int64_t base = s * slice_elems + 4 * i;
            note_nonfinite(v.x, base + 0, bad);
            note_nonfinite(v.y, base + 1, bad);
            note_nonfinite(v.z, base + 2, bad);
            note_nonfinite(v.w, base + 3, bad);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    } else {
        for (int64_t i = tid; i < slice_elems; i += stride) {
            const float v = src[i];
            note_nonfinite(v, s * slice_elems + i, bad);
            m = fmaxf(m, fabsf(v));
        }
    }
    m = warp_max(m);
    __shared__ float red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        v = warp_max(v);
        // NaN never reaches here as a max candidate: fmaxf drops NaN, and a
        // non-finite slice is rejected through `bad` anyway.
        if (threadIdx.x == 0) atomicMax(amax + s, __float_as_uint(v));
    }
}

__global__ void __launch_bounds__(256) slice_quantize_kernel(const float* __restrict__ x,
                                                             int64_t slice_elems,
                                                             const uint32_t* __restrict__ amax,
                                                             int8_t* __restrict__ codes,
                                                             float* __restrict__ slice_scales,
                                                             int vec) {
    const int64_t s = blockIdx.y;
    const float scale = __fdiv_rn(__uint_as_float(amax[s]), 127.0f);
    if (blockIdx.x == 0 && threadIdx.x == 0) slice_scales[s] = scale;
    const float* src = x + s * slice_elems;
    int8_t* dst = codes + s * slice_elems;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    if (vec) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
        const int64_t n4 = slice_elems >> 2;
        for (int64_t i = tid; i < n4; i += stride) {
            const float4 v = __ldcs(s4 + i);
            d4[i] = pack4(v.x, v.y, v.z, v.w, scale);
        }
    } else {
        for (int64_t i = tid; i < slice_elems; i += stride) dst[i] = quantize_one(src[i], scale);
    }
}

// FP8 e4m3 per-slice roundtrip codes (fp8.cpp:78-97): s = 448 / max|x|, code
// = e4m3(RN(x * s)) with the hardware's round-to-nearest-even, saturating
// conversion (the reference's e4m3_encode: ties to even, saturate at 448,
// subnormal step 2^-9).  Optionally also the decoded values as fp16 (exact).
__global__ void __launch_bounds__(256) slice_fp8_kernel(const float* __restrict__ x,
                                                        int64_t slice_elems,
                                                        const uint32_t* __restrict__ amax,
                                                        uint8_t* __restrict__ codes,
                                                        __half* __restrict__ decoded,
                                                        float* __restrict__ slice_scales) {
    const int64_t s = blockIdx.y;
    const float mx = __uint_as_float(amax[s]);
    const float scale = mx == 0.0f ? 0.0f : __fdiv_rn(448.0f, mx);
    if (blockIdx.x == 0 && threadIdx.x == 0) slice_scales[s] = scale;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n2 = slice_elems >> 1;  // slice_elems is even (host check)
    const float2* s2 = reinterpret_cast<const float2*>(x + s * slice_elems);
    uint16_t* c2 = reinterpret_cast<uint16_t*>(codes + s * slice_elems);
    __half2* h2 = decoded ? reinterpret_cast<__half2*>(decoded + s * slice_elems) : nullptr;
    for (int64_t i = tid; i < n2; i += stride) {
        const float2 v = __ldcs(s2 + i);
        uint16_t pair;
        // e4m3x2: first operand -> high byte
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;"
            : "=h"(pair)
            : "f"(__fmul_rn(v.y, scale)), "f"(__fmul_rn(v.x, scale)));
        c2[i] = pair;
        if (h2) {
            uint32_t hh;
            asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(hh) : "h"(pair));
            h2[i] = *reinterpret_cast<const __half2*>(&hh);
        }
    }
}

// Eight lanes per row, four rows per warp step: cols == 32 * NV.
template <int NV>
__global__ void __launch_bounds__(256) quantize_rows8_kernel(const float* __restrict__ x,
                                                             int64_t rows,
                                                             int8_t* __restrict__ codes,
                                                             float* __restrict__ scales,
                                                             int64_t* bad) {
    constexpr int64_t kCols = 32 * NV;
    const int lane = threadIdx.x & 31, l8 = lane & 7;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4;
         r0 < rows; r0 += warps_total * 4) {
        const int64_t row = r0 + (lane >> 3);
        const bool ok = row < rows;
        const float4* src = reinterpret_cast<const float4*>(x + row * kCols);
        float4 v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j)
            v[j] = ok ? __ldcs(src + l8 + 8 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
        float m = 0.0f;
#pragma unroll
        for (int j = 0; j < NV; ++j) m = absmax_nan(absmax_nan(m, v[j].x, v[j].y), v[j].z, v[j].w);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            const float other = __shfl_xor_sync(0xffffffffu, m, o);
            asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(other));
        }
        if (!(m <= 3.402823466e38f)) {  // NaN or Inf in the row: locate it exactly
            if (ok) {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int64_t base = row * kCols + 4 * (l8 + 8 * j);
                    note_nonfinite(v[j].x, base + 0, bad);
                    note_nonfinite(v[j].y, base + 1, bad);
                    note_nonfinite(v[j].z, base + 2, bad);
                    note_nonfinite(v[j].w, base + 3, bad);
                }
            }
        }
        const float scale = __fdiv_rn(m, 127.0f);
        if (ok && l8 == 0) scales[row] = scale;
        const float rcp = __frcp_rn(scale);
        const bool exact_row = !(rcp <= 3.402823466e38f);  // scale 0 / denormal / non-finite
        uint32_t* dst = reinterpret_cast<uint32_t*>(codes + row * kCols);
        if (ok) {
#pragma unroll
            for (int j = 0; j < NV; ++j) dst[l8 + 8 * j] = codes4(v[j], scale, rcp, exact_row);
        }
    }
}

// V: clusters of kSliceCluster CTAs, each cluster walking slices (persistent,
// so the slices in flight stay L2-resident).  Pass 1: partial abs max of this
// CTA's chunk; the cluster combines the partials through DSMEM.  Pass 2:
// quantize the chunk, re-read from L2.
constexpr int kSliceCluster = 8;

// Four packed int8 codes -> four fp16 (exact), for the two-Q-tile attention
// kernel's P.V operand.
// Without the quarter-rate I2F.F16 conversions (the V kernel's XU pipe ran at
// 85%): u = c + 128 in [1, 255] (XOR 0x80 per byte) placed under the fp16
// exponent byte 0x66 is the half 1536 + u exactly (ulp 1 in [1024, 2048)), and
// one packed subtract of 1664 leaves c exactly.
__device__ __forceinline__ uint2 codes4_to_f16(uint32_t w) {
    const uint32_t u = w ^ 0x80808080u;
    const uint32_t lo = __byte_perm(u, 0x66666666u, 0x4140);  // halves 1536 + u0, 1536 + u1
    const uint32_t hi = __byte_perm(u, 0x66666666u, 0x4342);
    const __half2 off = __float2half2_rn(1664.0f);
    const __half2 l = __hsub2(*reinterpret_cast<const __half2*>(&lo), off);
    const __half2 h = __hsub2(*reinterpret_cast<const __half2*>(&hi), off);
    return make_uint2(*reinterpret_cast<const uint32_t*>(&l), *reinterpret_cast<const uint32_t*>(&h));
}

// F16: also write the codes as fp16 (codes16, same layout).
template <bool F16>
__global__ void __cluster_dims__(kSliceCluster, 1, 1) __launch_bounds__(512)
    slice_quantize_fused_kernel(const float* __restrict__ x, int64_t slices,
                                int64_t slice_elems, int8_t* __restrict__ codes,
                                float* __restrict__ slice_scales, int64_t* bad,
                                uint16_t* __restrict__ codes16) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ float red[16];
    __shared__ float part[2];  // by iteration parity: a peer may still read the last one
    const int64_t nclusters = gridDim.x / kSliceCluster;
    const int rank = static_cast<int>(cluster.block_rank());
    const int64_t n4 = slice_elems >> 2;
    const int64_t per = (n4 + kSliceCluster - 1) / kSliceCluster;
    const int64_t lo = rank * per;
    const int64_t hi = lo + per < n4 ? lo + per : n4;
    int it = 0;
    for (int64_t slice = blockIdx.x / kSliceCluster; slice < slices; slice += nclusters, ++it) {
        const float4* src = reinterpret_cast<const float4*>(x + slice * slice_elems);
        float m = 0.0f;
        {
            // four loads in flight per thread
            const int64_t stride = blockDim.x;
            int64_t i = lo + threadIdx.x;
            for (; i + 3 * stride < hi; i += 4 * stride) {
                const float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride],
                             d = src[i + 3 * stride];
                m = absmax_nan(absmax_nan(m, a.x, a.y), a.z, a.w);
                m = absmax_nan(absmax_nan(m, b.x, b.y), b.z, b.w);
                m = absmax_nan(absmax_nan(m, c.x, c.y), c.z, c.w);
                m = absmax_nan(absmax_nan(m, d.x, d.y), d.z, d.w);
            }
            for (; i < hi; i += stride) {
                const float4 v = src[i];
                m = absmax_nan(absmax_nan(m, v.x, v.y), v.z, v.w);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float other = __shfl_xor_sync(0xffffffffu, m, o);
            asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(other));
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x < 32) {
            float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float other = __shfl_xor_sync(0xffffffffu, v, o);
                asm("max.NaN.f32 %0, %0, %1;" : "+f"(v) : "f"(other));
            }
            if (threadIdx.x == 0) part[it & 1] = v;
        }
        cluster.sync();
        float smax = 0.0f;
#pragma unroll
        for (int r = 0; r < kSliceCluster; ++r) {
            const float other = *cluster.map_shared_rank(&part[it & 1], r);
            asm("max.NaN.f32 %0, %0, %1;" : "+f"(smax) : "f"(other));
        }
        const float scale = __fdiv_rn(smax, 127.0f);
        if (rank == 0 && threadIdx.x == 0) slice_scales[slice] = scale;
        if (!(smax <= 3.402823466e38f) && !(part[it & 1] <= 3.402823466e38f)) {
            for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {  // locate it exactly
                const float4 v = src[i];
                const int64_t base = slice * slice_elems + 4 * i;
                note_nonfinite(v.x, base + 0, bad);
                note_nonfinite(v.y, base + 1, bad);
                note_nonfinite(v.z, base + 2, bad);
                note_nonfinite(v.w, base + 3, bad);
            }
        }
        const float rcp = __frcp_rn(scale);
        const bool exact_row = !(rcp <= 3.402823466e38f);
        uint32_t* dst = reinterpret_cast<uint32_t*>(codes + slice * slice_elems);
        uint2* dst16 = F16 ? reinterpret_cast<uint2*>(codes16 + slice * slice_elems) : nullptr;
        {
            const int64_t stride = blockDim.x;
            int64_t i = lo + threadIdx.x;
            for (; i + 3 * stride < hi; i += 4 * stride) {
                const float4 a = __ldcs(src + i), b = __ldcs(src + i + stride),
                             c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
                const uint32_t wa = codes4(a, scale, rcp, exact_row);
                const uint32_t wb = codes4(b, scale, rcp, exact_row);
                const uint32_t wc = codes4(c, scale, rcp, exact_row);
                const uint32_t wd = codes4(d, scale, rcp, exact_row);
                dst[i] = wa;
                dst[i + stride] = wb;
                dst[i + 2 * stride] = wc;
                dst[i + 3 * stride] = wd;
                if constexpr (F16) {
                    dst16[i] = codes4_to_f16(wa);
                    dst16[i + stride] = codes4_to_f16(wb);
                    dst16[i + 2 * stride] = codes4_to_f16(wc);
                    dst16[i + 3 * stride] = codes4_to_f16(wd);
                }
            }
            for (; i < hi; i += stride) {
                const uint32_t w = codes4(__ldcs(src + i), scale, rcp, exact_row);
                dst[i] = w;
                if constexpr (F16) dst16[i] = codes4_to_f16(w);
            }
        }
        __syncthreads();  // red[] reuse
    }
    cluster.sync();  // keep `part` alive until every peer has read it
}

// ------------------------------------------------------------------ launchers
static int sm_count() { return current_device_sms(); }

cudaError_t launch_quantize_per_row(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                                    float* scales, int64_t* bad, cudaStream_t stream) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const int threads = 256;
    const int64_t warps_needed = rows;
    int64_t blocks = (warps_needed + 7) / 8;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    const bool vec = (cols % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(codes) % 4 == 0);
    const int64_t blocks8 = std::min<int64_t>((rows + 31) / 32, static_cast<int64_t>(sm_count()) * 8);
    if (vec && (reinterpret_cast<uintptr_t>(codes) % 16 == 0) && cols == 128)
        quantize_rows8_kernel<4><<<blocks8, threads, 0, stream>>>(x, rows, codes, scales, bad);
    else if (vec && (reinterpret_cast<uintptr_t>(codes) % 16 == 0) && cols == 64)
        quantize_rows8_kernel<2><<<blocks8, threads, 0, stream>>>(x, rows, codes, scales, bad);
    else if (vec && (reinterpret_cast<uintptr_t>(codes) % 16 == 0) && cols == 256)
        quantize_rows8_kernel<8><<<blocks8, threads, 0, stream>>>(x, rows, codes, scales, bad);
    else if (vec && cols <= 128)
        quantize_rows_vec_kernel<1><<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    else if (vec && cols <= 256)
        quantize_rows_vec_kernel<2><<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    else if (vec && cols <= 512)
        quantize_rows_vec_kernel<4><<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    else
        quantize_rows_generic_kernel<<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    return cudaGetLastError();
}

__global__ void codes_i8_to_f16_kernel(const int8_t* __restrict__ src, int64_t count,
                                       __half* __restrict__ dst) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += stride)
        dst[i] = __int2half_rn(src[i]);
}

cudaError_t launch_quantize_per_tensor(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                       int8_t* codes, float* slice_scales, uint32_t* amax_ws,
                                       int64_t* bad, cudaStream_t stream, uint16_t* codes_f16) {
    if (slices == 0 || rows == 0 || cols == 0) return cudaSuccess;
    const int64_t elems = rows * cols;
    const int vec = (elems % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(codes) % 4 == 0);
    if (vec && elems % 16 == 0 && slices * kSliceCluster <= INT32_MAX) {
        // clusters in flight: ~48 MB of slices (L2-resident for the second
        // pass), but at least enough CTAs to cover every SM
        const int64_t slice_bytes = elems * 4;
        int64_t nclusters = (64ll << 20) / slice_bytes;
        const int64_t min_clusters = (sm_count() + kSliceCluster - 1) / kSliceCluster + 1;
        if (nclusters < min_clusters) nclusters = min_clusters;
        if (nclusters > slices) nclusters = slices;
        const unsigned grid = static_cast<unsigned>(nclusters * kSliceCluster);
        if (codes_f16 && reinterpret_cast<uintptr_t>(codes_f16) % 8 == 0)
            slice_quantize_fused_kernel<true><<<grid, 512, 0, stream>>>(
                x, slices, elems, codes, slice_scales, bad, codes_f16);
        else
            slice_quantize_fused_kernel<false><<<grid, 512, 0, stream>>>(
                x, slices, elems, codes, slice_scales, bad, nullptr);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess || !codes_f16 || reinterpret_cast<uintptr_t>(codes_f16) % 8 == 0)
            return e;
        codes_i8_to_f16_kernel<<<148 * 8, 256, 0, stream>>>(codes, slices * elems,
                                                             reinterpret_cast<__half*>(codes_f16));
        return cudaGetLastError();
    }
    cudaError_t err = cudaMemsetAsync(amax_ws, 0, sizeof(uint32_t) * slices, stream);
    if (err != cudaSuccess) return err;
    const int threads = 256;
    // Enough CTAs per slice that the whole grid covers the GPU a few times.
    int64_t per_slice = (static_cast<int64_t>(sm_count()) * 8 + slices - 1) / slices;
    const int64_t max_useful = (elems / (vec ? 4 : 1) + threads * 4 - 1) / (threads * 4);
    if (per_slice > max_useful) per_slice = max_useful;
    if (per_slice < 1) per_slice = 1;
    if (slices > 65535) return cudaErrorInvalidValue;
    dim3 grid(static_cast<unsigned>(per_slice), static_cast<unsigned>(slices));
    slice_absmax_kernel<<<grid, threads, 0, stream>>>(x, elems, amax_ws, bad, vec);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    slice_quantize_kernel<<<grid, threads, 0, stream>>>(x, elems, amax_ws, codes, slice_scales, vec);
    err = cudaGetLastError();
    if (err != cudaSuccess || !codes_f16) return err;
    codes_i8_to_f16_kernel<<<148 * 8, 256, 0, stream>>>(codes, slices * elems,
                                                         reinterpret_cast<__half*>(codes_f16));
    return cudaGetLastError();
}

cudaError_t launch_fp8_quantize_per_tensor(const float* x, int64_t slices, int64_t rows,
                                           int64_t cols, uint8_t* codes, uint16_t* decoded,
                                           float* slice_scales, uint32_t* amax_ws, int64_t* bad,
                                           cudaStream_t stream) {
    const int64_t elems = rows * cols;
    if (slices == 0 || elems == 0) return cudaSuccess;
    if (elems % 2 != 0 || slices > 65535 || reinterpret_cast<uintptr_t>(x) % 8 != 0 ||
        reinterpret_cast<uintptr_t>(codes) % 2 != 0 ||
        reinterpret_cast<uintptr_t>(decoded) % 4 != 0)
        return cudaErrorInvalidValue;
    cudaError_t err = cudaMemsetAsync(amax_ws, 0, sizeof(uint32_t) * slices, stream);
    if (err != cudaSuccess) return err;
    const int threads = 256;
    const int vec = (elems % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
    int64_t per_slice = (static_cast<int64_t>(sm_count()) * 8 + slices - 1) / slices;
    const int64_t max_useful = (elems / 2 + threads * 4 - 1) / (threads * 4);
    if (per_slice > max_useful) per_slice = max_useful;
    if (per_slice < 1) per_slice = 1;
    dim3 grid(static_cast<unsigned>(per_slice), static_cast<unsigned>(slices));
    slice_absmax_kernel<<<grid, threads, 0, stream>>>(x, elems, amax_ws, bad, vec);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    slice_fp8_kernel<<<grid, threads, 0, stream>>>(x, elems, amax_ws, codes,
                                                   reinterpret_cast<__half*>(decoded),
                                                   slice_scales);
    return cudaGetLastError();
}

// ------------------------------------------------------ streamed quantizer
// Quantization of slices [s0, slices) on a few SMs next to the attention
// kernel (ifa_int8_attention_step): CTA c owns whole slices s0 + c,
// s0 + c + P, ... and streams each one start to end -- Q rows, K rows (8
// lanes per row, 4 rows per warp step, two steps in flight), then V's abs
// max and V's codes + fp16 codes (the second read hits L2) -- so every
// pass is a long stream that keeps ~128 KB per SM in flight (measured
// ~190 GB/s per SM for plain 128-bit loads, tools/microbench/sm_bw.cu).
// When a slice is complete the CTA publishes ready[s] = epoch (release).
// Arithmetic per element is exactly the per-row / per-tensor kernels'
// (quant.cpp:25-69).
template <int NV>
__global__ void __launch_bounds__(1024, 1) stream_quantize_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    int64_t s0, int64_t slices, int64_t n, int8_t* __restrict__ qc, float* __restrict__ sq,
    int8_t* __restrict__ kc, float* __restrict__ sk, int8_t* __restrict__ vc,
    float* __restrict__ sv, uint16_t* __restrict__ v16, int64_t* bad, uint32_t* ready,
    uint32_t epoch) {
    constexpr int64_t D = 32 * NV;
    const int lane = threadIdx.x & 31, l8 = lane & 7, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    __shared__ float red[32];
    __shared__ float s_max;

    auto rows = [&](const float* x, int8_t* codes, float* scales, int64_t row0) {
        // rows [row0, row0 + n) of x (flat row index, also the index base)
        for (int64_t r0 = warp * 8; r0 < n; r0 += nwarps * 8) {
            float4 val[2][NV];
            int64_t rr[2];
            bool ok[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                rr[h] = r0 + 4 * h + (lane >> 3);
                ok[h] = rr[h] < n;
                const float4* src = reinterpret_cast<const float4*>(x + (row0 + rr[h]) * D);
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    val[h][j] = ok[h] ? __ldcs(src + l8 + 8 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float m = 0.0f;
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    m = absmax_nan(absmax_nan(m, val[h][j].x, val[h][j].y), val[h][j].z,
                                   val[h][j].w);
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    const float other = __shfl_xor_sync(0xffffffffu, m, o);
                    asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(other));
                }
                const int64_t row = row0 + rr[h];
                if (!(m <= 3.402823466e38f) && ok[h]) {  // locate the non-finite input
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        const int64_t b = row * D + 4 * (l8 + 8 * j);
                        note_nonfinite(val[h][j].x, b + 0, bad);
                        note_nonfinite(val[h][j].y, b + 1, bad);
                        note_nonfinite(val[h][j].z, b + 2, bad);
                        note_nonfinite(val[h][j].w, b + 3, bad);
                    }
                }
                const float scale = __fdiv_rn(m, 127.0f);
                const float rcp = __frcp_rn(scale);
                const bool exact_row = !(rcp <= 3.402823466e38f);
                if (ok[h]) {
                    if (l8 == 0) scales[row] = scale;
                    uint32_t* dst = reinterpret_cast<uint32_t*>(codes + row * D);
#pragma unroll
                    for (int j = 0; j < NV; ++j)
                        dst[l8 + 8 * j] = codes4(val[h][j], scale, rcp, exact_row);
                }
            }
        }
    };
    const int64_t E4 = n * D / 4;  // float4 per slice
    for (int64_t s = s0 + blockIdx.x; s < slices; s += gridDim.x) {
        rows(q, qc, sq, s * n);
        rows(k, kc, sk, s * n);
        // V: abs max of the slice
        const float4* src = reinterpret_cast<const float4*>(v + s * n * D);
        float m = 0.0f;
        {
            const int64_t stride = blockDim.x;
            int64_t i = threadIdx.x;
            for (; i + 3 * stride < E4; i += 4 * stride) {
                const float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride],
                             d = src[i + 3 * stride];
                m = absmax_nan(absmax_nan(m, a.x, a.y), a.z, a.w);
                m = absmax_nan(absmax_nan(m, b.x, b.y), b.z, b.w);
                m = absmax_nan(absmax_nan(m, c.x, c.y), c.z, c.w);
                m = absmax_nan(absmax_nan(m, d.x, d.y), d.z, d.w);
            }
            for (; i < E4; i += stride) {
                const float4 a = src[i];
                m = absmax_nan(absmax_nan(m, a.x, a.y), a.z, a.w);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float other = __shfl_xor_sync(0xffffffffu, m, o);
            asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(other));
        }
        if (lane == 0) red[warp] = m;
        __syncthreads();
        if (warp == 0) {
            float x = lane < nwarps ? red[lane] : 0.0f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float other = __shfl_xor_sync(0xffffffffu, x, o);
                asm("max.NaN.f32 %0, %0, %1;" : "+f"(x) : "f"(other));
            }
            if (lane == 0) s_max = x;
        }
        __syncthreads();
        const float smax = s_max;
        const float scale = __fdiv_rn(smax, 127.0f);
        if (threadIdx.x == 0) sv[s] = scale;
        if (!(smax <= 3.402823466e38f)) {
            for (int64_t i = threadIdx.x; i < E4; i += blockDim.x) {
                const float4 a = src[i];
                const int64_t b = s * n * D + 4 * i;
                note_nonfinite(a.x, b + 0, bad);
                note_nonfinite(a.y, b + 1, bad);
                note_nonfinite(a.z, b + 2, bad);
                note_nonfinite(a.w, b + 3, bad);
            }
        }
        const float rcp = __frcp_rn(scale);
        const bool exact_row = !(rcp <= 3.402823466e38f);
        uint32_t* dst = reinterpret_cast<uint32_t*>(vc + s * n * D);
        uint2* dst16 = reinterpret_cast<uint2*>(v16 + s * n * D);
        {
            const int64_t stride = blockDim.x;
            int64_t i = threadIdx.x;
            for (; i + 3 * stride < E4; i += 4 * stride) {
                const float4 a = __ldcs(src + i), b = __ldcs(src + i + stride),
                             c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
                const uint32_t wa = codes4(a, scale, rcp, exact_row);
                const uint32_t wb = codes4(b, scale, rcp, exact_row);
                const uint32_t wc = codes4(c, scale, rcp, exact_row);
                const uint32_t wd = codes4(d, scale, rcp, exact_row);
                dst[i] = wa;
                dst[i + stride] = wb;
                dst[i + 2 * stride] = wc;
                dst[i + 3 * stride] = wd;
                dst16[i] = codes4_to_f16(wa);
                dst16[i + stride] = codes4_to_f16(wb);
                dst16[i + 2 * stride] = codes4_to_f16(wc);
                dst16[i + 3 * stride] = codes4_to_f16(wd);
            }
            for (; i < E4; i += stride) {
                const uint32_t w = codes4(__ldcs(src + i), scale, rcp, exact_row);
                dst[i] = w;
                dst16[i] = codes4_to_f16(w);
            }
        }
        __syncthreads();  // the whole slice is written
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + s), "r"(epoch)
                         : "memory");
        }
    }
}

cudaError_t launch_stream_quantize(const float* q, const float* k, const float* v, int64_t s0,
                                   int64_t slices, int64_t n, int64_t d, int8_t* qc, float* sq,
                                   int8_t* kc, float* sk, int8_t* vc, float* sv, uint16_t* v16,
                                   int64_t* bad, uint32_t* ready, uint32_t epoch, int ctas,
                                   cudaStream_t stream) {
    if (d != 64 && d != 128) return cudaErrorInvalidValue;
    const uintptr_t al = reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                         reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(qc) |
                         reinterpret_cast<uintptr_t>(kc) | reinterpret_cast<uintptr_t>(vc) |
                         reinterpret_cast<uintptr_t>(v16);
    if (al % 16 != 0 || ctas < 1) return cudaErrorInvalidValue;
    if (s0 >= slices) return cudaSuccess;
    if (d == 128)
        stream_quantize_kernel<4><<<ctas, 1024, 0, stream>>>(q, k, v, s0, slices, n, qc, sq, kc,
                                                             sk, vc, sv, v16, bad, ready, epoch);
    else
        stream_quantize_kernel<2><<<ctas, 1024, 0, stream>>>(q, k, v, s0, slices, n, qc, sq, kc,
                                                             sk, vc, sv, v16, bad, ready, epoch);
    return cudaGetLastError();
}

}  // namespace ifa_b200
