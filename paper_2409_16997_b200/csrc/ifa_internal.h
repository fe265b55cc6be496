// ifa_internal.h -- launcher declarations shared by the CUDA translation
// units of libifa_b200.so (not part of the public C-ABI, see
// include/ifa_b200.h for that).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <string>

#include "../../include/ifa_b200.h"

namespace ifa_b200 {

// ---- per-device launch state (a process may drive several GPUs) ----------
constexpr int kMaxDevices = 64;
// SM count of the current device, cached per device id (148 on a B200).
int current_device_sms();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: apply it
// once per (kernel, device).  Idempotent, so a race only repeats the call.
template <auto Kernel>
cudaError_t smem_attr_once(size_t smem) {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev >= 0 && dev < kMaxDevices ? (uint64_t{1} << dev) : 0;
    if (bit && (done.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_relaxed);
    return e;
}

// Sets the thread-local ifa_last_error() message and returns `code`.
int set_error(int code, const std::string& msg);
// ifa_int_flash_fwd's argument checks (status + message), no memory access.
int validate_fwd(int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc, uint32_t flags);

cudaError_t launch_quantize_per_row(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                                    float* scales, int64_t* bad, cudaStream_t stream);
cudaError_t launch_quantize_per_tensor(const float* x, int64_t slices, int64_t rows,
                                       int64_t cols, int8_t* codes, float* slice_scales,
                                       uint32_t* amax_ws, int64_t* bad, cudaStream_t stream,
                                       uint16_t* codes_f16 = nullptr);

// Optional debug outputs of the tolerance-mode kernel (attn_ws.cu):
// s = [slices][n][n] int32 S tiles, p = [slices][n][n] uint8 P codes.
struct AttnDump {
    int32_t* s = nullptr;
    uint8_t* p = nullptr;
};

struct AttnArgs {
    const int8_t* q;
    const float* sq;
    const int8_t* k;
    const float* sk;
    const int8_t* v;
    const float* sv;
    float* o;
    ifa_pcode_audit* audit;  // device pointer or null
    int64_t slices;
    int64_t n;
    int64_t d;       // true head dim (columns of O)
    int64_t pitch;   // row pitch (elements) of the q/k/v code buffers, % 16 == 0
    int64_t bc;
    uint32_t flags;
    const AttnDump* dump = nullptr;  // tolerance-mode kernel only
    // streamed step (attn_pp.cu only): wait for ready[slice] >= ready_target
    // before reading a slice >= ready_from; grid capped at max_ctas (0 = all)
    const uint32_t* ready = nullptr;
    uint32_t ready_target = 0;
    int32_t ready_from = 0;
    int32_t max_ctas = 0;
};

// q/k/v rows have pitch `pitch` >= d with pitch % 16 == 0 (the C-ABI layer
// makes zero-padded copies when d % 16 != 0); columns >= d must be zero.
cudaError_t launch_int_flash_fwd(const AttnArgs& a, cudaStream_t stream);

// attn_pp.cu: tolerance-mode kernel with two Q tiles per CTA (non-causal,
// 128-key blocks, n % 16 == 0); IFA_B200_NO_PP=1 disables it.
bool int_flash_pp_eligible(const AttnArgs& a);
// v16: [slices][n][D] fp16 copy of the V codes (D = 64 for d <= 64, else
// 128), or null to convert a.v internally.
cudaError_t launch_int_flash_pp(const AttnArgs& a, const uint16_t* v16, cudaStream_t stream);
// attn_ws.cu: the full-INT8 tolerance-mode kernel with one softmax thread
// per row (IFA_B200_WS=1 selects it for int_flash_pp_eligible calls and for
// the S / P-code dumps, which otherwise run on attn_pp.cu's DUMP kernel).  v16 = [slices][n_pad][D] fp16 V codes (n_pad = n rounded up
// to 128, zero rows past n), o rows of o_pitch floats.
bool int_flash_ws_enabled();
// quant.cu: Q, K per row and V per slice (+ fp16 V codes) of slices
// [s0, slices), d in {64, 128}, on `ctas` CTAs that each own whole slices;
// ready[s] = epoch (release) once slice s is complete.
cudaError_t launch_stream_quantize(const float* q, const float* k, const float* v, int64_t s0,
                                   int64_t slices, int64_t n, int64_t d, int8_t* qc, float* sq,
                                   int8_t* kc, float* sk, int8_t* vc, float* sv, uint16_t* v16,
                                   int64_t* bad, uint32_t* ready, uint32_t epoch, int ctas,
                                   cudaStream_t stream);
cudaError_t launch_int_flash_ws(const int8_t* q, const float* sq, const int8_t* k,
                                const float* sk, const uint16_t* v16, const float* sv, float* o,
                                int64_t slices, int64_t n, int64_t d, int64_t pitch,
                                int64_t o_pitch, uint32_t flags, const AttnDump* dump,
                                cudaStream_t stream);
// The same two-Q-tile pipeline for the float-weight variants (§8(f) f1, f3):
// n % 128 == 0, d in {64, 128}, non-causal; v16 = fp16 V [slices][n][d].
bool float_weights_pp_eligible(int64_t n, int64_t d);
cudaError_t launch_half_int8_pp(const int8_t* q, const float* sq, const int8_t* k,
                                const float* sk, const uint16_t* v16, float* o, int64_t slices,
                                int64_t n, int64_t d, uint32_t flags, cudaStream_t stream);
cudaError_t launch_fp8_pp(const uint8_t* q, const float* q_scales, const uint8_t* k,
                          const float* k_scales, const uint16_t* v16, const float* v_scales,
                          float* o, int64_t slices, int64_t n, int64_t d, uint32_t flags,
                          cudaStream_t stream);

// attn_half.cu: half-INT8 forward (q/k codes of row pitch `pitch`, v fp16
// [slices][n][d] dense, d in {64, 128}) and the f32 -> fp16 conversion.
cudaError_t launch_half_int8_fwd(const int8_t* q, const float* sq, const int8_t* k,
                                 const float* sk, const uint16_t* v, float* o, int64_t slices,
                                 int64_t n, int64_t d, int64_t pitch, bool sqrt_d,
                                 cudaStream_t stream);
cudaError_t launch_convert_f16(const float* x, int64_t count, uint16_t* out, cudaStream_t stream);
// per-slice e4m3 codes (+ decoded fp16) and the FP8 forward
// (attn_half.cu with S via kind::f8f6f4); d in {64, 128}, V = decoded fp16.
cudaError_t launch_fp8_quantize_per_tensor(const float* x, int64_t slices, int64_t rows,
                                           int64_t cols, uint8_t* codes, uint16_t* decoded,
                                           float* slice_scales, uint32_t* amax_ws, int64_t* bad,
                                           cudaStream_t stream);
cudaError_t launch_fp8_attention_fwd(const uint8_t* q, const float* q_scales, const uint8_t* k,
                                     const float* k_scales, const uint16_t* v,
                                     const float* v_scales, float* o, int64_t slices, int64_t n,
                                     int64_t d, bool sqrt_d, cudaStream_t stream);

}  // namespace ifa_b200
