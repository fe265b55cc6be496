// abi.cu -- the extern "C" boundary (include/ifa_b200.h).
//
// Argument validation mirrors the reference's exception behaviour
// (attention.cpp:213-233 QuantizedAttentionInputs::validate, gemm.cpp:16-20
// BlockSpec::validate, gemm.cpp:22-28 check_int_gemm_depth) as status codes
// plus a thread-local message; the C++ shim (include/ifa_b200.hpp) turns
// them back into the same exception types.  There is no CPU fallback: a
// missing device / CUDA failure is reported as IFA_ECUDA.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "code_bounds.h"
#include "ifa_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    return fail(IFA_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Copies [rows][d] int8 codes into [rows][pitch] with zero columns [d, pitch).
__global__ void pad_codes_kernel(const int8_t* __restrict__ src, int8_t* __restrict__ dst,
                                 int64_t rows, int64_t d, int64_t pitch) {
    const int64_t total = rows * pitch;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / pitch, c = i - r * pitch;
        dst[i] = c < d ? src[r * d + c] : static_cast<int8_t>(0);
    }
}

__global__ void audit_init_kernel(ifa_pcode_audit* a) {
    a->min_code = 127;
    a->max_code = 0;
    a->row_max_block_hits_127 = 1;
    a->reserved = 0;
    a->rows_audited = 0;
}

}  // namespace

namespace ifa_b200 {

int current_device_sms() {
    static std::atomic<int> sms_of[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    int sms = dev >= 0 && dev < kMaxDevices ? sms_of[dev].load(std::memory_order_relaxed) : 0;
    if (sms <= 0) {
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            sms <= 0)
            sms = 148;
        if (dev >= 0 && dev < kMaxDevices) sms_of[dev].store(sms, std::memory_order_relaxed);
    }
    return sms;
}

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// Shape, block and flag checks of ifa_int_flash_fwd, in the reference's
// order (attention.cpp:213-242, gemm.cpp:16-28); touches no memory.
int validate_fwd(int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc, uint32_t flags) {
    if (slices < 0) return fail(IFA_EINVAL, "int_flash_attention: negative slice count");
    // attention.cpp:215-218
    if (n < 1 || d < 1) return fail(IFA_EINVAL, "quantized attention inputs: empty q");
    // gemm.cpp:16-20 (AttentionConfig::validate)
    if (br < 1 || bc < 1) return fail(IFA_EINVAL, "BlockSpec: Br and Bc must be >= 1");
    // attention.cpp:241-242 / gemm.cpp:22-28
    if (d > IFA_MAX_INT_GEMM_DEPTH)
        return fail(IFA_EOVERFLOW, "int gemm depth " + std::to_string(d) +
                                       " exceeds 133144; int32 accumulation could overflow");
    const int64_t kv_depth = bc < n ? bc : n;
    if (kv_depth > IFA_MAX_INT_GEMM_DEPTH)
        return fail(IFA_EOVERFLOW, "int gemm depth " + std::to_string(kv_depth) +
                                       " exceeds 133144; int32 accumulation could overflow");
    if (flags & ~(IFA_FLAG_SQRT_D | IFA_FLAG_CAUSAL | IFA_FLAG_FAST))
        return fail(IFA_EINVAL, "int_flash_attention: unknown flag bits");
    return IFA_OK;
}

}  // namespace ifa_b200

extern "C" {

const char* ifa_last_error(void) { return g_err.c_str(); }

int ifa_code_bounds(float* out128) {
    g_err.clear();
    if (!out128) return fail(IFA_EINVAL, "ifa_code_bounds: null pointer");
    const float* b = ifa_b200::code_bounds();
    for (int k = 0; k < 128; ++k) out128[k] = b[k];
    return IFA_OK;
}

const char* ifa_version(void) { return "ifa_b200 0.1 sm_100a (tcgen05 kind::i8)"; }

int ifa_audit_init(ifa_pcode_audit* audit, void* stream) {
    g_err.clear();
    if (!audit) return fail(IFA_EINVAL, "ifa_audit_init: null audit");
    audit_init_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(audit);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "ifa_audit_init");
}

int ifa_quantize_per_row(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                         float* scales, int64_t* nonfinite_index, void* stream) {
    g_err.clear();
    if (rows < 0 || cols < 0) return fail(IFA_EINVAL, "quantize_per_row: negative matrix extent");
    if (rows == 0 || cols == 0) return IFA_OK;
    if (!x || !codes || !scales) return fail(IFA_EINVAL, "quantize_per_row: null pointer");
    const cudaError_t e = ifa_b200::launch_quantize_per_row(
        x, rows, cols, codes, scales, nonfinite_index, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "quantize_per_row");
}

int ifa_quantize_per_tensor(const float* x, int64_t slices, int64_t rows, int64_t cols,
                            int8_t* codes, float* slice_scales, void* workspace,
                            int64_t* nonfinite_index, void* stream) {
    g_err.clear();
    if (slices < 0 || rows < 0 || cols < 0)
        return fail(IFA_EINVAL, "quantize_per_tensor: negative matrix extent");
    if (slices == 0) return IFA_OK;
    if (!slice_scales || !workspace) return fail(IFA_EINVAL, "quantize_per_tensor: null pointer");
    if (rows == 0 || cols == 0) {
        // max_abs over an empty matrix is 0 -> scale 0 (quant.cpp:34-40, :59-69)
        const cudaError_t e = cudaMemsetAsync(slice_scales, 0, sizeof(float) * slices,
                                              static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? IFA_OK : cuda_fail(e, "quantize_per_tensor");
    }
    if (!x || !codes) return fail(IFA_EINVAL, "quantize_per_tensor: null pointer");
    const cudaError_t e = ifa_b200::launch_quantize_per_tensor(
        x, slices, rows, cols, codes, slice_scales, static_cast<uint32_t*>(workspace),
        nonfinite_index, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "quantize_per_tensor");
}

namespace {

// ifa_int_flash_fwd and ifa_int_flash_fwd_dump after validation: stages
// 16-byte-pitch copies of the codes when TMA needs them, then dispatches.
int fwd_impl(const int8_t* q, const float* sq, const int8_t* k, const float* sk, const int8_t* v,
             const float* sv, float* o, int64_t slices, int64_t n, int64_t d, int64_t bc,
             uint32_t flags, ifa_pcode_audit* audit, const ifa_b200::AttnDump* dump,
             cudaStream_t st) {
    ifa_b200::AttnArgs a{q, sq, k, sk, v, sv, o, audit, slices, n, d, d, bc, flags, dump};
    const bool aligned = (reinterpret_cast<uintptr_t>(q) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(k) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(v) % 16 == 0);
    int8_t* padded = nullptr;
    if (d % 16 != 0 || !aligned) {
        // TMA needs 16-byte row pitches: stage zero-padded copies (exact for
        // the integer dot products, gemm.hpp:12-13).
        const int64_t pitch = (d + 15) / 16 * 16;
        const int64_t per = slices * n * pitch;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&padded), 3 * per, st);
        if (e != cudaSuccess) return cuda_fail(e, "int_flash_attention: workspace");
        const int64_t rows = slices * n;
        const int blocks = static_cast<int>((per + 255) / 256 < 4096 ? (per + 255) / 256 : 4096);
        pad_codes_kernel<<<blocks, 256, 0, st>>>(q, padded, rows, d, pitch);
        pad_codes_kernel<<<blocks, 256, 0, st>>>(k, padded + per, rows, d, pitch);
        pad_codes_kernel<<<blocks, 256, 0, st>>>(v, padded + 2 * per, rows, d, pitch);
        a.q = padded;
        a.k = padded + per;
        a.v = padded + 2 * per;
        a.pitch = pitch;
    }
    cudaError_t e = dump ? ifa_b200::launch_int_flash_pp(a, nullptr, st)
                         : ifa_b200::launch_int_flash_fwd(a, st);
    if (padded) {
        const cudaError_t e2 = cudaFreeAsync(padded, st);
        if (e == cudaSuccess) e = e2;
    }
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "int_flash_attention");
}

}  // namespace

int ifa_int_flash_fwd(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                      const int8_t* v, const float* sv, float* o, int64_t slices, int64_t n,
                      int64_t d, int64_t br, int64_t bc, uint32_t flags,
                      ifa_pcode_audit* audit, void* stream) {
    g_err.clear();
    const int rc = ifa_b200::validate_fwd(slices, n, d, br, bc, flags);
    if (rc != IFA_OK) return rc;
    if (slices == 0) return IFA_OK;
    if (((n + 127) / 128) * slices > INT32_MAX)
        return fail(IFA_ENOTSUP, "int_flash_attention: more than 2^31 (q tile, slice) work items");
    if (!q || !sq || !k || !sk || !v || !sv || !o)
        return fail(IFA_EINVAL, "int_flash_attention: null pointer");
    return fwd_impl(q, sq, k, sk, v, sv, o, slices, n, d, bc, flags, audit, nullptr,
                    static_cast<cudaStream_t>(stream));
}

int ifa_int_flash_fwd_dump(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                           const int8_t* v, const float* sv, float* o, int64_t slices, int64_t n,
                           int64_t d, int64_t br, int64_t bc, uint32_t flags, int32_t* s_out,
                           uint8_t* p_codes, void* stream) {
    g_err.clear();
    flags &= ~IFA_FLAG_DUMP_S;  // implied by this entry point
    const int rc = ifa_b200::validate_fwd(slices, n, d, br, bc, flags);
    if (rc != IFA_OK) return rc;
    if (slices == 0) return IFA_OK;
    if (!(flags & IFA_FLAG_FAST))
        return fail(IFA_EINVAL, "int_flash_attention dump: needs IFA_FLAG_FAST");
    if (d > 128)
        return fail(IFA_ENOTSUP, "int_flash_attention dump: head dim " + std::to_string(d) +
                                     " > 128 (the dump kernel holds one 128-column Q tile)");
    if (!(bc == 128 || (bc >= n && n <= 128)))
        return fail(IFA_ENOTSUP, "int_flash_attention dump: the tolerance kernel's KV block is "
                                 "128 keys (Bc = 128, or Bc >= n <= 128)");
    if (n > 65536 || slices * n * n > (int64_t{1} << 40))
        return fail(IFA_ENOTSUP, "int_flash_attention dump: slice too large for an n x n dump");
    if (((n + 127) / 128) * slices > INT32_MAX)
        return fail(IFA_ENOTSUP, "int_flash_attention: more than 2^31 (q tile, slice) work items");
    if (!q || !sq || !k || !sk || !v || !sv || !o || (!s_out && !p_codes))
        return fail(IFA_EINVAL, "int_flash_attention: null pointer");
    const ifa_b200::AttnDump dump{s_out, p_codes};
    return fwd_impl(q, sq, k, sk, v, sv, o, slices, n, d, bc, flags, nullptr, &dump,
                    static_cast<cudaStream_t>(stream));
}

int ifa_quantize_per_tensor_v16(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                int8_t* codes, uint16_t* codes_f16, float* slice_scales,
                                void* workspace, int64_t* nonfinite_index, void* stream) {
    g_err.clear();
    if (slices < 0 || rows < 0 || cols < 0)
        return fail(IFA_EINVAL, "quantize_per_tensor: negative matrix extent");
    if (slices == 0) return IFA_OK;
    if (!slice_scales || !workspace || !codes_f16)
        return fail(IFA_EINVAL, "quantize_per_tensor: null pointer");
    if (rows == 0 || cols == 0) {
        const cudaError_t e = cudaMemsetAsync(slice_scales, 0, sizeof(float) * slices,
                                              static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? IFA_OK : cuda_fail(e, "quantize_per_tensor");
    }
    if (!x || !codes) return fail(IFA_EINVAL, "quantize_per_tensor: null pointer");
    const cudaError_t e = ifa_b200::launch_quantize_per_tensor(
        x, slices, rows, cols, codes, slice_scales, static_cast<uint32_t*>(workspace),
        nonfinite_index, static_cast<cudaStream_t>(stream), codes_f16);
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "quantize_per_tensor");
}

int ifa_int_flash_fwd_v16(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                          const int8_t* v, const uint16_t* v_f16, const float* sv, float* o,
                          int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc,
                          uint32_t flags, void* stream) {
    g_err.clear();
    const int rc = ifa_b200::validate_fwd(slices, n, d, br, bc, flags);
    if (rc != IFA_OK) return rc;
    if (slices == 0) return IFA_OK;
    if (((n + 127) / 128) * slices > INT32_MAX)
        return fail(IFA_ENOTSUP, "int_flash_attention: more than 2^31 (q tile, slice) work items");
    if (!q || !sq || !k || !sk || !v || !v_f16 || !sv || !o)
        return fail(IFA_EINVAL, "int_flash_attention: null pointer");
    ifa_b200::AttnArgs a{q, sq, k, sk, v, sv, o, nullptr, slices, n, d, d, bc, flags};
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                           reinterpret_cast<uintptr_t>(v_f16)) % 16) == 0;
    if ((d == 64 || d == 128) && n % 128 == 0 && aligned && ifa_b200::int_flash_pp_eligible(a)) {
        const cudaError_t e =
            ifa_b200::launch_int_flash_pp(a, v_f16, static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? IFA_OK : cuda_fail(e, "int_flash_attention");
    }
    return ifa_int_flash_fwd(q, sq, k, sk, v, sv, o, slices, n, d, br, bc, flags, nullptr,
                             stream);
}

namespace {
// Per-device side stream + fork/join events of the streamed step.
struct StepStreams {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t step_streams(StepStreams** out) {
    static StepStreams per_dev[ifa_b200::kMaxDevices];
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= ifa_b200::kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(mu);
    StepStreams& s = per_dev[dev];
    if (!s.side) {
        if ((e = cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming)) != cudaSuccess)
            return e;
    }
    *out = &s;
    return cudaSuccess;
}
}  // namespace

int ifa_int8_attention_step(const float* q, const float* k, const float* v, int8_t* qc,
                            float* sq, int8_t* kc, float* sk, int8_t* vc, float* sv,
                            uint16_t* v16, float* o, int64_t* nonfinite_index,
                            uint32_t* sync_ws, uint32_t epoch, int64_t slices, int64_t n,
                            int64_t d, int64_t br, int64_t bc, uint32_t flags, void* stream) {
    g_err.clear();
    const int rc = ifa_b200::validate_fwd(slices, n, d, br, bc, flags);
    if (rc != IFA_OK) return rc;
    if (slices == 0) return IFA_OK;
    if (!q || !k || !v || !qc || !sq || !kc || !sk || !vc || !sv || !v16 || !o || !sync_ws)
        return fail(IFA_EINVAL, "int8_attention_step: null pointer");
    if (epoch == 0) return fail(IFA_EINVAL, "int8_attention_step: epoch starts at 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int sms = ifa_b200::current_device_sms();
    int qctas = 12;
    if (const char* env = std::getenv("IFA_B200_QUANT_SMS")) qctas = std::atoi(env);
    const int64_t bce = bc < n ? bc : n;
    const bool streamed = (flags & IFA_FLAG_FAST) && !(flags & IFA_FLAG_CAUSAL) &&
                          (bce == 128 || (bce == n && n <= 128)) && n % 128 == 0 &&
                          (d == 64 || d == 128) && qctas >= 1 && qctas <= sms / 4 &&
                          !ifa_b200::int_flash_ws_enabled() && slices <= INT32_MAX / 64;
    if (!streamed) {  // same results, quantize then attention on `stream`
        uint32_t* ws = sync_ws + slices;  // the per-tensor quantizer's scratch
        int r = ifa_quantize_per_row(q, slices * n, d, qc, sq, nonfinite_index, stream);
        if (r == IFA_OK) r = ifa_quantize_per_row(k, slices * n, d, kc, sk, nonfinite_index, stream);
        if (r == IFA_OK)
            r = ifa_quantize_per_tensor_v16(v, slices, n, d, vc, v16, sv, ws, nonfinite_index,
                                            stream);
        if (r != IFA_OK) return r;
        return ifa_int_flash_fwd_v16(qc, sq, kc, sk, vc, v16, sv, o, slices, n, d, br, bc, flags,
                                     stream);
    }
    StepStreams* ss = nullptr;
    cudaError_t e = step_streams(&ss);
    if (e != cudaSuccess) return cuda_fail(e, "int8_attention_step: streams");
    uint32_t* ready = sync_ws;
    const int actas = sms - qctas;
    // The first slices are quantized on the whole GPU before the attention
    // starts (its first wave needs ~actas / pairs slices at once); the
    // streamed quantizer takes the rest, ahead of the attention.
    const int64_t pairs = (n + 255) / 256;
    int64_t s0 = (2 * actas + pairs - 1) / pairs;
    if (s0 < 8) s0 = 8;
    if (s0 > slices) s0 = slices;
    // host order: the streamed quantizer first (it then owns its SMs, and
    // under a serialising profiler it completes before anything waits on it)
    if ((e = cudaEventRecord(ss->fork, st)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(ss->side, ss->fork, 0)) != cudaSuccess)
        return cuda_fail(e, "int8_attention_step: fork");
    e = ifa_b200::launch_stream_quantize(q, k, v, s0, slices, n, d, qc, sq, kc, sk, vc, sv, v16,
                                         nonfinite_index, ready, epoch, qctas, ss->side);
    if (e != cudaSuccess) return cuda_fail(e, "int8_attention_step: quantize");
    {  // slices [0, s0) on `stream`, full GPU
        uint32_t* ws = sync_ws + slices;  // per-tensor quantizer scratch
        int r = ifa_quantize_per_row(q, s0 * n, d, qc, sq, nonfinite_index, stream);
        if (r == IFA_OK) r = ifa_quantize_per_row(k, s0 * n, d, kc, sk, nonfinite_index, stream);
        if (r == IFA_OK)
            r = ifa_quantize_per_tensor_v16(v, s0, n, d, vc, v16, sv, ws, nonfinite_index, stream);
        if (r != IFA_OK) return r;
    }
    ifa_b200::AttnArgs a{qc, sq, kc, sk, vc, sv, o, nullptr, slices, n, d, d, bc, flags};
    a.ready = ready;
    a.ready_target = epoch;
    a.ready_from = static_cast<int32_t>(s0);
    a.max_ctas = actas;
    e = ifa_b200::launch_int_flash_pp(a, v16, st);
    if (e != cudaSuccess) return cuda_fail(e, "int8_attention_step: attention");
    if ((e = cudaEventRecord(ss->join, ss->side)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(st, ss->join, 0)) != cudaSuccess)
        return cuda_fail(e, "int8_attention_step: join");
    return IFA_OK;
}

int ifa_half_int8_fwd(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                      const uint16_t* v_f16, float* o, int64_t slices, int64_t n, int64_t d,
                      int64_t br, int64_t bc, uint32_t flags, void* stream) {
    g_err.clear();
    if (slices < 0) return fail(IFA_EINVAL, "half_int8_attention: negative slice count");
    // attention.cpp:374-376, gemm.cpp:16-20 (tiled_float_attention's cfg.validate)
    if (n < 1 || d < 1) return fail(IFA_EINVAL, "half_int8_attention: empty input");
    if (d > IFA_MAX_INT_GEMM_DEPTH)
        return fail(IFA_EOVERFLOW, "int gemm depth " + std::to_string(d) +
                                       " exceeds 133144; int32 accumulation could overflow");
    if (br < 1 || bc < 1) return fail(IFA_EINVAL, "BlockSpec: Br and Bc must be >= 1");
    if (flags & ~IFA_FLAG_SQRT_D) {
        if (flags & ~(IFA_FLAG_SQRT_D | IFA_FLAG_CAUSAL | IFA_FLAG_FAST))
            return fail(IFA_EINVAL, "half_int8_attention: unknown flag bits");
        return fail(IFA_ENOTSUP, "half_int8_attention: only IFA_FLAG_SQRT_D is supported");
    }
    if (d != 64 && d != 128)
        return fail(IFA_ENOTSUP, "half_int8_attention: head dim " + std::to_string(d) +
                                     " not supported by the sm_100a kernel (64 or 128)");
    if (slices == 0) return IFA_OK;
    if (((n + 127) / 128) * slices > INT32_MAX)
        return fail(IFA_ENOTSUP, "half_int8_attention: more than 2^31 (q tile, slice) work items");
    if (!q || !sq || !k || !sk || !v_f16 || !o)
        return fail(IFA_EINVAL, "half_int8_attention: null pointer");
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
         reinterpret_cast<uintptr_t>(v_f16)) % 16 != 0)
        return fail(IFA_EINVAL, "half_int8_attention: q/k/v must be 16-byte aligned");
    const cudaError_t e =
        ifa_b200::float_weights_pp_eligible(n, d)
            ? ifa_b200::launch_half_int8_pp(q, sq, k, sk, v_f16, o, slices, n, d, flags,
                                            static_cast<cudaStream_t>(stream))
            : ifa_b200::launch_half_int8_fwd(q, sq, k, sk, v_f16, o, slices, n, d, d,
                                             (flags & IFA_FLAG_SQRT_D) != 0,
                                             static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "half_int8_attention");
}

int ifa_fp8_quantize_per_tensor(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                uint8_t* codes, uint16_t* decoded_f16, float* slice_scales,
                                void* workspace, int64_t* nonfinite_index, void* stream) {
    g_err.clear();
    if (slices < 0 || rows < 0 || cols < 0)
        return fail(IFA_EINVAL, "fp8_e4m3_roundtrip: negative matrix extent");
    if (slices == 0) return IFA_OK;
    if (!slice_scales || !workspace) return fail(IFA_EINVAL, "fp8_e4m3_roundtrip: null pointer");
    if (rows == 0 || cols == 0) {
        const cudaError_t e = cudaMemsetAsync(slice_scales, 0, sizeof(float) * slices,
                                              static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? IFA_OK : cuda_fail(e, "fp8_e4m3_roundtrip");
    }
    if (!x || !codes) return fail(IFA_EINVAL, "fp8_e4m3_roundtrip: null pointer");
    if ((rows * cols) % 2 != 0)
        return fail(IFA_ENOTSUP, "fp8_e4m3_roundtrip: odd slice element count");
    const cudaError_t e = ifa_b200::launch_fp8_quantize_per_tensor(
        x, slices, rows, cols, codes, decoded_f16, slice_scales,
        static_cast<uint32_t*>(workspace), nonfinite_index, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "fp8_e4m3_roundtrip");
}

int ifa_fp8_attention_fwd(const uint8_t* q, const float* q_scales, const uint8_t* k,
                          const float* k_scales, const uint16_t* v_f16, const float* v_scales,
                          float* o, int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc,
                          uint32_t flags, void* stream) {
    g_err.clear();
    if (slices < 0) return fail(IFA_EINVAL, "fp8_emulated_attention: negative slice count");
    if (n < 1 || d < 1) return fail(IFA_EINVAL, "fp8_emulated_attention: empty input");
    if (br < 1 || bc < 1) return fail(IFA_EINVAL, "BlockSpec: Br and Bc must be >= 1");
    if (flags & ~IFA_FLAG_SQRT_D) {
        if (flags & ~(IFA_FLAG_SQRT_D | IFA_FLAG_CAUSAL | IFA_FLAG_FAST))
            return fail(IFA_EINVAL, "fp8_emulated_attention: unknown flag bits");
        return fail(IFA_ENOTSUP, "fp8_emulated_attention: only IFA_FLAG_SQRT_D is supported");
    }
    if (d != 64 && d != 128)
        return fail(IFA_ENOTSUP, "fp8_emulated_attention: head dim " + std::to_string(d) +
                                     " not supported by the sm_100a kernel (64 or 128)");
    if (slices == 0) return IFA_OK;
    if (((n + 127) / 128) * slices > INT32_MAX)
        return fail(IFA_ENOTSUP, "fp8_emulated_attention: too many work items");
    if (!q || !q_scales || !k || !k_scales || !v_f16 || !v_scales || !o)
        return fail(IFA_EINVAL, "fp8_emulated_attention: null pointer");
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
         reinterpret_cast<uintptr_t>(v_f16)) % 16 != 0)
        return fail(IFA_EINVAL, "fp8_emulated_attention: q/k/v must be 16-byte aligned");
    const cudaError_t e =
        ifa_b200::float_weights_pp_eligible(n, d)
            ? ifa_b200::launch_fp8_pp(q, q_scales, k, k_scales, v_f16, v_scales, o, slices, n, d,
                                      flags, static_cast<cudaStream_t>(stream))
            : ifa_b200::launch_fp8_attention_fwd(q, q_scales, k, k_scales, v_f16, v_scales, o,
                                                 slices, n, d, (flags & IFA_FLAG_SQRT_D) != 0,
                                                 static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "fp8_emulated_attention");
}

int ifa_convert_f16(const float* x, int64_t count, uint16_t* out, void* stream) {
    g_err.clear();
    if (count < 0) return fail(IFA_EINVAL, "convert_f16: negative count");
    if (count == 0) return IFA_OK;
    if (!x || !out) return fail(IFA_EINVAL, "convert_f16: null pointer");
    const cudaError_t e =
        ifa_b200::launch_convert_f16(x, count, out, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? IFA_OK : cuda_fail(e, "convert_f16");
}

}  // extern "C"
