// host_abi.cu -- host-buffer entry points of the C-ABI (include/ifa_b200.h,
// the *_host functions).
//
// The reference's callers hold their matrices in host memory
// (ifa::Matrix<T>, matrix.hpp:16-64) and call the CPU kernels synchronously
// (eval.cpp:98-102, verify.cpp:187-230).  These entry points keep that
// calling convention for a drop-in: host pointers in and out, the
// host->device copy, the sm_100a kernels and the device->host copy queued on
// one stream, then a synchronize.  Device memory comes from a per-thread,
// grow-only workspace, so repeated calls of one shape do not allocate.
// There is no CPU path: without a usable device every call fails with
// IFA_ECUDA.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "ifa_internal.h"

namespace {

struct Workspace {
    void* ptr = nullptr;
    size_t cap = 0;
    int device = -1;
    ~Workspace() {
        if (ptr) cudaFree(ptr);  // errors at process teardown are irrelevant
    }
    // Returns a device buffer of >= bytes on the current device.
    cudaError_t reserve(size_t bytes) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (ptr && cap >= bytes && dev == device) return cudaSuccess;
        if (ptr) {
            cudaFree(ptr);
            ptr = nullptr;
            cap = 0;
        }
        const size_t want = bytes < (size_t{1} << 20) ? (size_t{1} << 20) : bytes;
        e = cudaMalloc(&ptr, want);
        if (e != cudaSuccess) return e;
        cap = want;
        device = dev;
        return cudaSuccess;
    }
};

thread_local Workspace g_ws;

size_t align256(size_t x) { return (x + 255) & ~size_t{255}; }

// Carves consecutive 256-byte-aligned sub-buffers out of the workspace.
struct Carver {
    char* base;
    size_t off = 0;
    template <typename T>
    T* take(size_t count) {
        T* p = reinterpret_cast<T*>(base + off);
        off += align256(count * sizeof(T));
        return p;
    }
};

int cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return IFA_OK;
    std::string msg = std::string(where) + ": " + cudaGetErrorString(e);
    // route the message through ifa_last_error()
    return ifa_b200::set_error(IFA_ECUDA, msg);
}

constexpr int64_t kNoIndex = INT64_MAX;

}  // namespace

extern "C" {

int ifa_quantize_per_row_host(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                              float* scales, int64_t* nonfinite_index, void* stream) {
    ifa_b200::set_error(IFA_OK, "");
    if (rows < 0 || cols < 0)
        return ifa_b200::set_error(IFA_EINVAL, "quantize_per_row: negative matrix extent");
    if (nonfinite_index) *nonfinite_index = kNoIndex;
    if (rows == 0) return IFA_OK;
    if (!scales) return ifa_b200::set_error(IFA_EINVAL, "quantize_per_row: null pointer");
    if (cols == 0) {
        std::memset(scales, 0, sizeof(float) * rows);
        return IFA_OK;
    }
    if (!x || !codes) return ifa_b200::set_error(IFA_EINVAL, "quantize_per_row: null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t elems = static_cast<size_t>(rows) * cols;
    cudaError_t e = g_ws.reserve(align256(elems * 4) + align256(elems) + align256(rows * 4) + 256);
    if (e != cudaSuccess) return cuda_status(e, "quantize_per_row: workspace");
    Carver c{static_cast<char*>(g_ws.ptr)};
    float* dx = c.take<float>(elems);
    int8_t* dc = c.take<int8_t>(elems);
    float* ds = c.take<float>(rows);
    int64_t* dbad = c.take<int64_t>(1);
    const int64_t no = kNoIndex;
    if ((e = cudaMemcpyAsync(dbad, &no, 8, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dx, x, elems * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_status(e, "quantize_per_row: copy in");
    const int rc = ifa_quantize_per_row(dx, rows, cols, dc, ds, dbad, stream);
    if (rc != IFA_OK) return rc;
    int64_t bad = kNoIndex;
    if ((e = cudaMemcpyAsync(codes, dc, elems, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(scales, ds, rows * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(&bad, dbad, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_status(e, "quantize_per_row: copy out");
    if (nonfinite_index) *nonfinite_index = bad;
    if (bad != kNoIndex)
        return ifa_b200::set_error(IFA_EINVAL, "quantize_per_row: non-finite input at index " +
                                                   std::to_string(bad));
    return IFA_OK;
}

int ifa_quantize_per_tensor_host(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                 int8_t* codes, float* slice_scales, int64_t* nonfinite_index,
                                 void* stream) {
    ifa_b200::set_error(IFA_OK, "");
    if (slices < 0 || rows < 0 || cols < 0)
        return ifa_b200::set_error(IFA_EINVAL, "quantize_per_tensor: negative matrix extent");
    if (nonfinite_index) *nonfinite_index = kNoIndex;
    if (slices == 0) return IFA_OK;
    if (!slice_scales)
        return ifa_b200::set_error(IFA_EINVAL, "quantize_per_tensor: null pointer");
    if (rows == 0 || cols == 0) {
        std::memset(slice_scales, 0, sizeof(float) * slices);
        return IFA_OK;
    }
    if (!x || !codes) return ifa_b200::set_error(IFA_EINVAL, "quantize_per_tensor: null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t elems = static_cast<size_t>(slices) * rows * cols;
    cudaError_t e = g_ws.reserve(align256(elems * 4) + align256(elems) + 2 * align256(slices * 4) +
                                 256);
    if (e != cudaSuccess) return cuda_status(e, "quantize_per_tensor: workspace");
    Carver c{static_cast<char*>(g_ws.ptr)};
    float* dx = c.take<float>(elems);
    int8_t* dc = c.take<int8_t>(elems);
    float* ds = c.take<float>(slices);
    uint32_t* dws = c.take<uint32_t>(slices);
    int64_t* dbad = c.take<int64_t>(1);
    const int64_t no = kNoIndex;
    if ((e = cudaMemcpyAsync(dbad, &no, 8, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dx, x, elems * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_status(e, "quantize_per_tensor: copy in");
    const int rc = ifa_quantize_per_tensor(dx, slices, rows, cols, dc, ds, dws, dbad, stream);
    if (rc != IFA_OK) return rc;
    int64_t bad = kNoIndex;
    if ((e = cudaMemcpyAsync(codes, dc, elems, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(slice_scales, ds, slices * 4, cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(&bad, dbad, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_status(e, "quantize_per_tensor: copy out");
    if (nonfinite_index) *nonfinite_index = bad;
    if (bad != kNoIndex)
        return ifa_b200::set_error(IFA_EINVAL, "quantize_per_tensor: non-finite input at index " +
                                                   std::to_string(bad));
    return IFA_OK;
}

int ifa_int_flash_fwd_host(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                           const int8_t* v, const float* sv, float* o, int64_t slices,
                           int64_t n, int64_t d, int64_t br, int64_t bc, uint32_t flags,
                           ifa_pcode_audit* audit, void* stream) {
    ifa_b200::set_error(IFA_OK, "");
    const int pre = ifa_b200::validate_fwd(slices, n, d, br, bc, flags);
    if (pre != IFA_OK || slices == 0) return pre;
    // attention.cpp:229-232: the V scale must be finite and non-negative.
    if (sv != nullptr) {
        for (int64_t s = 0; s < slices; ++s)
            if (!std::isfinite(sv[s]) || sv[s] < 0.0f)
                return ifa_b200::set_error(
                    IFA_EINVAL, "quantized attention inputs: bad v scale");
    }
    if (!q || !sq || !k || !sk || !v || !sv || !o)
        return ifa_b200::set_error(IFA_EINVAL, "int_flash_attention: null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t elems = static_cast<size_t>(slices) * n * d;
    const size_t rows = static_cast<size_t>(slices) * n;
    cudaError_t e = g_ws.reserve(3 * align256(elems) + 2 * align256(rows * 4) +
                                 align256(slices * 4) + align256(elems * 4) + 256);
    if (e != cudaSuccess) return cuda_status(e, "int_flash_attention: workspace");
    Carver c{static_cast<char*>(g_ws.ptr)};
    int8_t* dq = c.take<int8_t>(elems);
    int8_t* dk = c.take<int8_t>(elems);
    int8_t* dv = c.take<int8_t>(elems);
    float* dsq = c.take<float>(rows);
    float* dsk = c.take<float>(rows);
    float* dsv = c.take<float>(slices);
    float* dout = c.take<float>(elems);
    ifa_pcode_audit* dau = audit ? c.take<ifa_pcode_audit>(1) : nullptr;
    if ((e = cudaMemcpyAsync(dq, q, elems, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dk, k, elems, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dv, v, elems, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dsq, sq, rows * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dsk, sk, rows * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dsv, sv, slices * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_status(e, "int_flash_attention: copy in");
    if (dau) {
        const int rc = ifa_audit_init(dau, stream);
        if (rc != IFA_OK) return rc;
    }
    const int rc = ifa_int_flash_fwd(dq, dsq, dk, dsk, dv, dsv, dout, slices, n, d, br, bc, flags,
                                     dau, stream);
    if (rc != IFA_OK) return rc;
    if ((e = cudaMemcpyAsync(o, dout, elems * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return cuda_status(e, "int_flash_attention: copy out");
    if (dau && (e = cudaMemcpyAsync(audit, dau, sizeof(ifa_pcode_audit), cudaMemcpyDeviceToHost,
                                    st)) != cudaSuccess)
        return cuda_status(e, "int_flash_attention: copy out");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_status(e, "int_flash_attention");
    return IFA_OK;
}

int ifa_half_int8_fwd_host(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                           const float* v, float* o, int64_t slices, int64_t n, int64_t d,
                           int64_t br, int64_t bc, uint32_t flags, void* stream) {
    ifa_b200::set_error(IFA_OK, "");
    if (slices < 0 || n < 1 || d < 1)
        return ifa_b200::set_error(IFA_EINVAL, "half_int8_attention: empty input");
    if (slices == 0) return IFA_OK;
    if (!q || !sq || !k || !sk || !v || !o)
        return ifa_b200::set_error(IFA_EINVAL, "half_int8_attention: null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t elems = static_cast<size_t>(slices) * n * d;
    const size_t rows = static_cast<size_t>(slices) * n;
    cudaError_t e = g_ws.reserve(2 * align256(elems) + 2 * align256(rows * 4) +
                                 2 * align256(elems * 4) + align256(elems * 2) + 256);
    if (e != cudaSuccess) return cuda_status(e, "half_int8_attention: workspace");
    Carver c{static_cast<char*>(g_ws.ptr)};
    int8_t* dq = c.take<int8_t>(elems);
    int8_t* dk = c.take<int8_t>(elems);
    float* dsq = c.take<float>(rows);
    float* dsk = c.take<float>(rows);
    float* dv = c.take<float>(elems);
    uint16_t* dv16 = c.take<uint16_t>(elems);
    float* dout = c.take<float>(elems);
    if ((e = cudaMemcpyAsync(dq, q, elems, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dk, k, elems, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dsq, sq, rows * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dsk, sk, rows * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dv, v, elems * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_status(e, "half_int8_attention: copy in");
    int rc = ifa_convert_f16(dv, static_cast<int64_t>(elems), dv16, stream);
    if (rc != IFA_OK) return rc;
    rc = ifa_half_int8_fwd(dq, dsq, dk, dsk, dv16, dout, slices, n, d, br, bc, flags, stream);
    if (rc != IFA_OK) return rc;
    if ((e = cudaMemcpyAsync(o, dout, elems * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_status(e, "half_int8_attention: copy out");
    return IFA_OK;
}

int ifa_fp8_emulated_attention_host(const float* q, const float* k, const float* v, float* o,
                                    int64_t slices, int64_t n, int64_t d, int64_t br,
                                    int64_t bc, uint32_t flags, void* stream) {
    ifa_b200::set_error(IFA_OK, "");
    if (slices < 0 || n < 1 || d < 1)
        return ifa_b200::set_error(IFA_EINVAL, "fp8_emulated_attention: empty input");
    if (slices == 0) return IFA_OK;
    if (!q || !k || !v || !o)
        return ifa_b200::set_error(IFA_EINVAL, "fp8_emulated_attention: null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t elems = static_cast<size_t>(slices) * n * d;
    cudaError_t e = g_ws.reserve(3 * align256(elems * 4) + 3 * align256(elems) +
                                 align256(elems * 2) + 3 * align256(slices * 4) +
                                 align256(slices * 4) + align256(8) + align256(elems * 4) + 256);
    if (e != cudaSuccess) return cuda_status(e, "fp8_emulated_attention: workspace");
    Carver c{static_cast<char*>(g_ws.ptr)};
    const float* hx[3] = {q, k, v};
    float* dx[3];
    uint8_t* codes[3];
    float* scales[3];
    for (int i = 0; i < 3; ++i) dx[i] = c.take<float>(elems);
    for (int i = 0; i < 3; ++i) codes[i] = c.take<uint8_t>(elems);
    uint16_t* dv16 = c.take<uint16_t>(elems);
    for (int i = 0; i < 3; ++i) scales[i] = c.take<float>(slices);
    uint32_t* ws = c.take<uint32_t>(slices);
    int64_t* bad = c.take<int64_t>(1);
    float* dout = c.take<float>(elems);
    const int64_t none = kNoIndex;
    if ((e = cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_status(e, "fp8_emulated_attention: copy in");
    for (int i = 0; i < 3; ++i) {
        if ((e = cudaMemcpyAsync(dx[i], hx[i], elems * 4, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess)
            return cuda_status(e, "fp8_emulated_attention: copy in");
        const int rc = ifa_fp8_quantize_per_tensor(dx[i], slices, n, d, codes[i],
                                                   i == 2 ? dv16 : nullptr, scales[i], ws, bad,
                                                   stream);
        if (rc != IFA_OK) return rc;
    }
    int64_t hbad = kNoIndex;
    if ((e = cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_status(e, "fp8_emulated_attention");
    if (hbad != kNoIndex)  // fp8.cpp:82-84
        return ifa_b200::set_error(IFA_EINVAL, "fp8_e4m3_roundtrip: non-finite input");
    const int rc = ifa_fp8_attention_fwd(codes[0], scales[0], codes[1], scales[1], dv16,
                                         scales[2], dout, slices, n, d, br, bc, flags, stream);
    if (rc != IFA_OK) return rc;
    if ((e = cudaMemcpyAsync(o, dout, elems * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_status(e, "fp8_emulated_attention: copy out");
    return IFA_OK;
}

}  // extern "C"
