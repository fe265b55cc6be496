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
// Per-row (Q, K): one warp per row, 128-bit loads, codes packed four per
// 32-bit store.  Per-tensor (V, one scale per (b,h) slice): slice absmax by
// an unsigned atomicMax on the float bits (all values are >= 0), then a
// quantize pass.
#include <cstdint>
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

// ------------------------------------------------------------------ launchers
static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

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
    if (vec && cols <= 128)
        quantize_rows_vec_kernel<1><<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    else if (vec && cols <= 256)
        quantize_rows_vec_kernel<2><<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    else if (vec && cols <= 512)
        quantize_rows_vec_kernel<4><<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    else
        quantize_rows_generic_kernel<<<blocks, threads, 0, stream>>>(x, rows, cols, codes, scales, bad);
    return cudaGetLastError();
}

cudaError_t launch_quantize_per_tensor(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                       int8_t* codes, float* slice_scales, uint32_t* amax_ws,
                                       int64_t* bad, cudaStream_t stream) {
    if (slices == 0 || rows == 0 || cols == 0) return cudaSuccess;
    const int64_t elems = rows * cols;
    const int vec = (elems % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(codes) % 4 == 0);
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
    return cudaGetLastError();
}

}  // namespace ifa_b200
