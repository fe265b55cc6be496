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

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

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

// ---------------------------------------------------------------------------
// Chunked host <-> device pipeline for the attention entry points.
//
// The batch of (b,h) slices is cut into chunks; chunk c uses slot c % kSlots
// of a device buffer (and, for pageable caller memory, of a pinned staging
// buffer).  Three streams overlap the host->device copy of chunk c+1, the
// kernels of chunk c and the device->host copy of chunk c-1 (PCIe is full
// duplex).  Caller memory that is already pinned (cudaMallocHost /
// cudaHostRegister) is DMA'd directly; pageable memory is staged through
// pinned buffers with multi-threaded memcpy on the host.
struct InSeg {
    const void* host;
    void* dev;
    size_t bytes;
};
struct OutSeg {
    void* host;
    const void* dev;
    size_t bytes;
};
struct ChunkIO {
    std::vector<InSeg> in;
    std::vector<OutSeg> out;
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kMin = size_t{4} << 20;
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const unsigned parts = bytes < kMin ? 1u : std::min<unsigned>(hw, unsigned(bytes / (kMin / 2)));
    if (parts <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t step = (bytes + parts - 1) / parts;
    std::vector<std::thread> th;
    for (unsigned i = 1; i < parts; ++i) {
        const size_t off = i * step;
        if (off >= bytes) break;
        th.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                        std::min(step, bytes - off));
        });
    }
    std::memcpy(dst, src, std::min(step, bytes));
    for (auto& t : th) t.join();
}

struct Pipe {
    static constexpr int kSlots = 3;
    int device = -1;
    cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // h2d, compute, d2h
    cudaEvent_t in_done[kSlots], comp_done[kSlots], out_done[kSlots];
    void* dev = nullptr;
    size_t dev_cap = 0;
    void* pin = nullptr;
    size_t pin_cap = 0;

    ~Pipe() {
        // process teardown: the driver may already be gone, ignore errors
        if (dev) cudaFree(dev);
        if (pin) cudaFreeHost(pin);
    }
    cudaError_t init() {
        int d = 0;
        cudaError_t e = cudaGetDevice(&d);
        if (e != cudaSuccess) return e;
        if (d == device) return cudaSuccess;
        if (device >= 0) {  // device switched on this thread: drop the old resources
            if (dev) cudaFree(dev);
            dev = nullptr;
            dev_cap = 0;
        }
        for (auto& x : st)
            if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (int i = 0; i < kSlots; ++i) {
            if ((e = cudaEventCreateWithFlags(&in_done[i], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming)) != cudaSuccess)
                return e;
        }
        device = d;
        return cudaSuccess;
    }
    cudaError_t reserve(size_t dev_bytes, size_t pin_bytes) {
        cudaError_t e;
        if (dev_bytes > dev_cap) {
            if (dev) cudaFree(dev);
            dev = nullptr;
            dev_cap = 0;
            if ((e = cudaMalloc(&dev, dev_bytes)) != cudaSuccess) return e;
            dev_cap = dev_bytes;
        }
        if (pin_bytes > pin_cap) {
            if (pin) cudaFreeHost(pin);
            pin = nullptr;
            pin_cap = 0;
            if ((e = cudaMallocHost(&pin, pin_bytes)) != cudaSuccess) return e;
            pin_cap = pin_bytes;
        }
        return cudaSuccess;
    }
};

thread_local Pipe g_pipe;

// Runs `nchunks` chunks through the pipeline.  plan(c, dev_slot, io) names
// the chunk's host <-> device segments (device addresses inside dev_slot);
// compute(c, dev_slot, stream) enqueues its kernels.  slot_dev / slot_in /
// slot_out: bytes per slot of device memory and of pinned in / out staging.
// `prologue` runs once on the compute stream before the first chunk.
int run_pipeline(int64_t nchunks, size_t slot_dev, size_t slot_in, size_t slot_out,
                 const std::function<void(int64_t, char*, ChunkIO&)>& plan,
                 const std::function<int(int64_t, char*, cudaStream_t)>& compute,
                 const char* what, void* caller_stream) {
    Pipe& P = g_pipe;
    cudaError_t e = P.init();
    if (e != cudaSuccess) return cuda_status(e, what);
    const int S = Pipe::kSlots;
    slot_dev = align256(slot_dev);
    slot_in = align256(slot_in);
    slot_out = align256(slot_out);
    if ((e = P.reserve(S * slot_dev, S * (slot_in + slot_out))) != cudaSuccess)
        return cuda_status(e, what);
    cudaStream_t h2d = P.st[0], comp = P.st[1], d2h = P.st[2];
    // order after work the caller queued on its own stream
    {
        cudaEvent_t ev;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_status(e, what);
        cudaEventRecord(ev, static_cast<cudaStream_t>(caller_stream));
        cudaStreamWaitEvent(h2d, ev, 0);
        cudaStreamWaitEvent(comp, ev, 0);
        cudaEventDestroy(ev);
    }
    std::vector<ChunkIO> ios(S);
    std::vector<int64_t> slot_chunk(S, -1);
    auto drain = [&](int slot) -> cudaError_t {  // pageable outputs of the slot's chunk
        if (slot_chunk[slot] < 0) return cudaSuccess;
        bool pageable = false;
        for (const OutSeg& o : ios[slot].out) pageable |= !is_pinned(o.host);
        if (!pageable) return cudaSuccess;
        cudaError_t e2 = cudaEventSynchronize(P.out_done[slot]);
        if (e2 != cudaSuccess) return e2;
        char* stage = static_cast<char*>(P.pin) + S * slot_in + slot * slot_out;
        size_t off = 0;
        for (const OutSeg& o : ios[slot].out) {
            if (!is_pinned(o.host)) par_memcpy(o.host, stage + off, o.bytes);
            off += align256(o.bytes);
        }
        slot_chunk[slot] = -1;
        return cudaSuccess;
    };
    int rc = IFA_OK;
    for (int64_t c = 0; c < nchunks && rc == IFA_OK; ++c) {
        const int slot = static_cast<int>(c % S);
        char* dslot = static_cast<char*>(P.dev) + slot * slot_dev;
        char* in_stage = static_cast<char*>(P.pin) + slot * slot_in;
        char* out_stage = static_cast<char*>(P.pin) + S * slot_in + slot * slot_out;
        if ((e = drain(slot)) != cudaSuccess) return cuda_status(e, what);
        ChunkIO& io = ios[slot];
        io.in.clear();
        io.out.clear();
        plan(c, dslot, io);
        if (c >= S) {
            // the device slot is free once its chunk's output has been copied out
            cudaStreamWaitEvent(h2d, P.out_done[slot], 0);
            // the staging slot is reused only after its last copy finished
            if ((e = cudaEventSynchronize(P.in_done[slot])) != cudaSuccess)
                return cuda_status(e, what);
        }
        size_t off = 0;
        for (const InSeg& s : io.in) {
            const void* src = s.host;
            if (!is_pinned(s.host)) {
                par_memcpy(in_stage + off, s.host, s.bytes);
                src = in_stage + off;
            }
            off += align256(s.bytes);
            if ((e = cudaMemcpyAsync(s.dev, src, s.bytes, cudaMemcpyHostToDevice, h2d)) !=
                cudaSuccess)
                return cuda_status(e, what);
        }
        cudaEventRecord(P.in_done[slot], h2d);
        cudaStreamWaitEvent(comp, P.in_done[slot], 0);
        if (c >= S) cudaStreamWaitEvent(comp, P.out_done[slot], 0);  // output region copied out
        rc = compute(c, dslot, comp);
        cudaEventRecord(P.comp_done[slot], comp);
        cudaStreamWaitEvent(d2h, P.comp_done[slot], 0);
        off = 0;
        for (const OutSeg& o : io.out) {
            void* dst = is_pinned(o.host) ? o.host : out_stage + off;
            off += align256(o.bytes);
            if ((e = cudaMemcpyAsync(dst, o.dev, o.bytes, cudaMemcpyDeviceToHost, d2h)) !=
                cudaSuccess)
                return cuda_status(e, what);
        }
        cudaEventRecord(P.out_done[slot], d2h);
        slot_chunk[slot] = c;
    }
    for (int64_t c = std::max<int64_t>(0, nchunks - S); c < nchunks; ++c)
        if ((e = drain(static_cast<int>(c % S))) != cudaSuccess) return cuda_status(e, what);
    for (auto x : P.st)
        if ((e = cudaStreamSynchronize(x)) != cudaSuccess) return cuda_status(e, what);
    return rc;
}

// slices per chunk: about 16 MiB of f32 output per chunk, but enough
// (q tile pair, slice) work items to fill the GPU
int64_t chunk_slices(int64_t slices, int64_t n, int64_t d) {
    if (const char* env = std::getenv("IFA_B200_HOST_CHUNK")) {  // tests: force many chunks
        const int64_t c = std::atoll(env);
        if (c > 0) return std::min(c, slices);
    }
    const int64_t per_slice_out = n * d * 4;
    int64_t c = std::max<int64_t>(1, (int64_t{16} << 20) / std::max<int64_t>(per_slice_out, 1));
    const int64_t pairs = (n + 255) / 256;
    const int64_t min_items = 2 * ifa_b200::current_device_sms();
    c = std::max<int64_t>(c, (min_items + pairs - 1) / pairs);
    return std::min(c, slices);
}

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
    const int64_t cs = chunk_slices(slices, n, d);
    const int64_t nchunks = (slices + cs - 1) / cs;
    const size_t e1 = static_cast<size_t>(cs) * n * d, r1 = static_cast<size_t>(cs) * n;
    const size_t slot_dev = 3 * align256(e1) + 2 * align256(r1 * 4) + align256(cs * 4) +
                            align256(e1 * 4);
    const size_t slot_in = 3 * align256(e1) + 2 * align256(r1 * 4) + align256(cs * 4);
    const size_t slot_out = align256(e1 * 4);
    // the audit (exact kernel only) folds over every chunk's launch
    cudaError_t e = g_ws.reserve(256);
    if (e != cudaSuccess) return cuda_status(e, "int_flash_attention: workspace");
    ifa_pcode_audit* dau = audit ? static_cast<ifa_pcode_audit*>(g_ws.ptr) : nullptr;
    auto carve = [&](char* dslot, int8_t** dq, int8_t** dk, int8_t** dv, float** dsq,
                     float** dsk, float** dsv, float** dout) {
        Carver c{dslot};
        *dq = c.take<int8_t>(e1);
        *dk = c.take<int8_t>(e1);
        *dv = c.take<int8_t>(e1);
        *dsq = c.take<float>(r1);
        *dsk = c.take<float>(r1);
        *dsv = c.take<float>(cs);
        *dout = c.take<float>(e1);
    };
    auto plan = [&](int64_t ch, char* dslot, ChunkIO& io) {
        const int64_t s0 = ch * cs, ns = std::min(cs, slices - s0);
        const size_t el = static_cast<size_t>(ns) * n * d, rw = static_cast<size_t>(ns) * n;
        const size_t eo = static_cast<size_t>(s0) * n * d, ro = static_cast<size_t>(s0) * n;
        int8_t *dq, *dk, *dv;
        float *dsq, *dsk, *dsv, *dout;
        carve(dslot, &dq, &dk, &dv, &dsq, &dsk, &dsv, &dout);
        io.in = {{q + eo, dq, el}, {k + eo, dk, el}, {v + eo, dv, el},
                 {sq + ro, dsq, rw * 4}, {sk + ro, dsk, rw * 4}, {sv + s0, dsv, size_t(ns) * 4}};
        io.out = {{o + eo, dout, el * 4}};
    };
    bool first = true;
    auto compute = [&](int64_t ch, char* dslot, cudaStream_t st) -> int {
        const int64_t s0 = ch * cs, ns = std::min(cs, slices - s0);
        int8_t *dq, *dk, *dv;
        float *dsq, *dsk, *dsv, *dout;
        carve(dslot, &dq, &dk, &dv, &dsq, &dsk, &dsv, &dout);
        if (dau && first) {
            const int rc = ifa_audit_init(dau, st);
            if (rc != IFA_OK) return rc;
        }
        first = false;
        return ifa_int_flash_fwd(dq, dsq, dk, dsk, dv, dsv, dout, ns, n, d, br, bc, flags, dau,
                                 st);
    };
    const int rc = run_pipeline(nchunks, slot_dev, slot_in, slot_out, plan, compute,
                                "int_flash_attention", stream);
    if (rc != IFA_OK) return rc;
    if (dau && (e = cudaMemcpy(audit, dau, sizeof(ifa_pcode_audit), cudaMemcpyDeviceToHost)) !=
                   cudaSuccess)
        return cuda_status(e, "int_flash_attention: copy out");
    return IFA_OK;
}

int ifa_full_int8_attention_host(const float* q, const float* k, const float* v, float* o,
                                 int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc,
                                 uint32_t flags, void* stream) {
    ifa_b200::set_error(IFA_OK, "");
    const int pre = ifa_b200::validate_fwd(slices, n, d, br, bc, flags);
    if (pre != IFA_OK || slices == 0) return pre;
    if (!q || !k || !v || !o)
        return ifa_b200::set_error(IFA_EINVAL, "full_int8_attention: null pointer");
    const int64_t cs = chunk_slices(slices, n, d);
    const int64_t nchunks = (slices + cs - 1) / cs;
    const size_t e1 = static_cast<size_t>(cs) * n * d, r1 = static_cast<size_t>(cs) * n;
    const size_t slot_dev = 3 * align256(e1 * 4) + 3 * align256(e1) + align256(e1 * 2) +
                            2 * align256(r1 * 4) + 2 * align256(cs * 4);
    const size_t slot_in = 3 * align256(e1 * 4);
    const size_t slot_out = align256(e1 * 4);
    // per chunk and tensor: smallest non-finite flat index inside the chunk
    cudaError_t e = g_ws.reserve(align256(sizeof(int64_t) * 3 * nchunks));
    if (e != cudaSuccess) return cuda_status(e, "full_int8_attention: workspace");
    int64_t* dbad = static_cast<int64_t*>(g_ws.ptr);
    std::vector<int64_t> hbad(3 * nchunks, kNoIndex);
    if ((e = cudaMemcpy(dbad, hbad.data(), 8 * hbad.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_status(e, "full_int8_attention: workspace");
    struct Bufs {
        float *x[3], *sq, *sk, *sv, *out;
        int8_t* c[3];
        uint16_t* v16;
        uint32_t* ws;
    };
    auto carve = [&](char* dslot) {
        Carver c{dslot};
        Bufs b;
        for (auto& x : b.x) x = c.take<float>(e1);
        for (auto& x : b.c) x = c.take<int8_t>(e1);
        b.v16 = c.take<uint16_t>(e1);
        b.sq = c.take<float>(r1);
        b.sk = c.take<float>(r1);
        b.sv = c.take<float>(cs);
        b.ws = c.take<uint32_t>(cs);
        b.out = reinterpret_cast<float*>(b.x[0]);  // Q f32 is dead once quantized
        return b;
    };
    const float* hx[3] = {q, k, v};
    auto plan = [&](int64_t ch, char* dslot, ChunkIO& io) {
        const int64_t s0 = ch * cs, ns = std::min(cs, slices - s0);
        const size_t el = static_cast<size_t>(ns) * n * d, eo = static_cast<size_t>(s0) * n * d;
        const Bufs b = carve(dslot);
        for (int i = 0; i < 3; ++i) io.in.push_back({hx[i] + eo, b.x[i], el * 4});
        io.out = {{o + eo, b.out, el * 4}};
    };
    const bool v16_ok = (n % 128 == 0) && (d == 64 || d == 128);
    auto compute = [&](int64_t ch, char* dslot, cudaStream_t st) -> int {
        const int64_t s0 = ch * cs, ns = std::min(cs, slices - s0);
        const Bufs b = carve(dslot);
        int64_t* bad = dbad + 3 * ch;
        int rc = ifa_quantize_per_row(b.x[0], ns * n, d, b.c[0], b.sq, bad, st);
        if (rc == IFA_OK) rc = ifa_quantize_per_row(b.x[1], ns * n, d, b.c[1], b.sk, bad + 1, st);
        if (rc != IFA_OK) return rc;
        if (v16_ok) {
            rc = ifa_quantize_per_tensor_v16(b.x[2], ns, n, d, b.c[2], b.v16, b.sv, b.ws, bad + 2,
                                             st);
            if (rc == IFA_OK)
                rc = ifa_int_flash_fwd_v16(b.c[0], b.sq, b.c[1], b.sk, b.c[2], b.v16, b.sv, b.out,
                                           ns, n, d, br, bc, flags, st);
        } else {
            rc = ifa_quantize_per_tensor(b.x[2], ns, n, d, b.c[2], b.sv, b.ws, bad + 2, st);
            if (rc == IFA_OK)
                rc = ifa_int_flash_fwd(b.c[0], b.sq, b.c[1], b.sk, b.c[2], b.sv, b.out, ns, n, d,
                                       br, bc, flags, nullptr, st);
        }
        return rc;
    };
    const int rc = run_pipeline(nchunks, slot_dev, slot_in, slot_out, plan, compute,
                                "full_int8_attention", stream);
    if (rc != IFA_OK) return rc;
    if ((e = cudaMemcpy(hbad.data(), dbad, 8 * hbad.size(), cudaMemcpyDeviceToHost)) !=
        cudaSuccess)
        return cuda_status(e, "full_int8_attention: copy out");
    static const char* names[3] = {"q", "k", "v"};
    for (int t = 0; t < 3; ++t)
        for (int64_t ch = 0; ch < nchunks; ++ch)
            if (hbad[3 * ch + t] != kNoIndex) {
                const int64_t idx = ch * cs * n * d + hbad[3 * ch + t];
                return ifa_b200::set_error(IFA_EINVAL, std::string("full_int8_attention: ") +
                                                           names[t] +
                                                           ": non-finite input at index " +
                                                           std::to_string(idx));
            }
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
    {  // V goes to the tensor core as fp16 (include/ifa_b200.h)
        const size_t count = static_cast<size_t>(slices) * n * d;
        for (size_t i = 0; i < count; ++i)
            if (std::fabs(v[i]) > 65504.0f)
                return ifa_b200::set_error(
                    IFA_EINVAL, "half_int8_attention: |v| exceeds the fp16 range (65504) of the "
                                "sm_100a kernel");
    }
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
