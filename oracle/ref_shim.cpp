// ref_shim.cpp -- extern "C" entry points into the UNMODIFIED reference
// library (/root/reference/proj/src, compiled from where it lies by
// oracle/Makefile into oracle/_ref/libifa_ref.so).
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (to pin the C restatement in
// ifa_oracle.c and to check the GPU path) and by bench.py --impl reference /
// the cpu_baseline leg (the reference's own CPU path, timed on host cores).
// Nothing here is part of the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <cmath>
#include <vector>

#include "ifa/attention.hpp"
#include "ifa/fp8.hpp"
#include "ifa/gemm.hpp"
#include "ifa/generate.hpp"
#include "ifa/oracles.hpp"
#include "ifa/quant.hpp"
#include "ifa/tensor_io.hpp"
#include "ifa/verify.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::overflow_error*>(&e)) return -2;
    return -1;
}

ifa::FloatMatrix to_fm(const float* p, int64_t r, int64_t c) {
    return ifa::FloatMatrix(r, c, std::vector<float>(p, p + r * c));
}
ifa::Int8Matrix to_im(const int8_t* p, int64_t r, int64_t c) {
    return ifa::Int8Matrix(r, c, std::vector<int8_t>(p, p + r * c));
}
ifa::QuantizedAttentionInputs make_inputs(const int8_t* q, const float* sq, const int8_t* k,
                                          const float* sk, const int8_t* v, float sv,
                                          int64_t n, int64_t d) {
    ifa::QuantizedAttentionInputs in;
    in.q.values = to_im(q, n, d);
    in.q.scales = ifa::ScaleVector(std::vector<float>(sq, sq + n));
    in.k.values = to_im(k, n, d);
    in.k.scales = ifa::ScaleVector(std::vector<float>(sk, sk + n));
    in.v.values = to_im(v, n, d);
    in.v.scale = sv;
    return in;
}
}  // namespace

extern "C" {

const char* ifa_ref_last_error() { return g_err.c_str(); }

// IFA1 files through the reference's own tensor_io (format cross-checks).
int ifa_ref_save_tensor(const char* path, int dtype, const void* data, int64_t rows,
                        int64_t cols) {
    try {
        if (dtype == 0) {
            const float* p = static_cast<const float*>(data);
            ifa::save_tensor(ifa::FloatMatrix(rows, cols, std::vector<float>(p, p + rows * cols)),
                             path);
        } else if (dtype == 1) {
            const int8_t* p = static_cast<const int8_t*>(data);
            ifa::save_tensor(
                ifa::Int8Matrix(rows, cols, std::vector<int8_t>(p, p + rows * cols)), path);
        } else {
            const int32_t* p = static_cast<const int32_t*>(data);
            ifa::save_tensor(
                ifa::Int32Matrix(rows, cols, std::vector<int32_t>(p, p + rows * cols)), path);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Loads with ifa::load_tensor; fills dtype/rows/cols and copies the payload
// when it fits `capacity` bytes.  On FormatError returns -1 with the message.
int ifa_ref_load_tensor(const char* path, int* dtype, int64_t* rows, int64_t* cols, void* buf,
                        int64_t capacity) {
    try {
        const ifa::LoadedTensor t = ifa::load_tensor(path);
        *dtype = static_cast<int>(ifa::loaded_dtype(t));
        std::visit(
            [&](const auto& m) {
                *rows = m.rows();
                *cols = m.cols();
                const int64_t bytes = m.size() * static_cast<int64_t>(sizeof(m.data()[0]));
                if (buf && bytes <= capacity) std::memcpy(buf, m.data(), static_cast<size_t>(bytes));
            },
            t);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_generate(int dist, double a, double b, uint64_t seed, int64_t rows, int64_t cols,
                     float* out) {
    try {
        const ifa::ActivationSpec spec = dist == 0 ? ifa::ActivationSpec::normal(a, b, seed)
                                                   : ifa::ActivationSpec::uniform(a, b, seed);
        const ifa::FloatMatrix m = ifa::generate(spec, rows, cols);
        std::memcpy(out, m.data(), sizeof(float) * rows * cols);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_quantize_per_row(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                             float* scales) {
    try {
        const ifa::QuantizedRows q = ifa::quantize_per_row(to_fm(x, rows, cols));
        std::memcpy(codes, q.values.data(), rows * cols);
        std::memcpy(scales, q.scales.data(), sizeof(float) * rows);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_quantize_per_tensor(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                                float* scale) {
    try {
        const ifa::QuantizedTensor q = ifa::quantize_per_tensor(to_fm(x, rows, cols));
        std::memcpy(codes, q.values.data(), rows * cols);
        *scale = q.scale;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_int_gemm_nt(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k,
                        int32_t* out) {
    try {
        const ifa::Int32Matrix r = ifa::int_gemm_nt(to_im(a, m, k), to_im(b, n, k));
        std::memcpy(out, r.data(), sizeof(int32_t) * m * n);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// audit4: {min_code, max_code, row_max_block_hits_127, rows_audited} (int64)
int ifa_ref_int_flash_attention(const int8_t* q, const float* sq, const int8_t* k,
                                const float* sk, const int8_t* v, float sv, int64_t n,
                                int64_t d, int64_t br, int64_t bc, int sqrt_d, float* out,
                                int64_t* audit4) {
    try {
        ifa::AttentionConfig cfg;
        cfg.blocks = ifa::BlockSpec{br, bc};
        cfg.apply_sqrt_d_scaling = sqrt_d != 0;
        cfg.variant = ifa::AttentionVariant::kFullInt8;
        ifa::PCodeAudit audit;
        const ifa::FloatMatrix o = ifa::int_flash_attention(
            make_inputs(q, sq, k, sk, v, sv, n, d), cfg, audit4 ? &audit : nullptr);
        std::memcpy(out, o.data(), sizeof(float) * n * d);
        if (audit4) {
            audit4[0] = audit.min_code;
            audit4[1] = audit.max_code;
            audit4[2] = audit.row_max_block_hits_127 ? 1 : 0;
            audit4[3] = audit.rows_audited;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's own CPU path over [slices][n][d], one slice per task from
// an atomic queue on `threads` host threads.
int ifa_ref_int_flash_attention_batched(const int8_t* q, const float* sq, const int8_t* k,
                                        const float* sk, const int8_t* v, const float* sv,
                                        int64_t slices, int64_t n, int64_t d, int64_t br,
                                        int64_t bc, float* out, int threads) {
    std::atomic<int64_t> next{0};
    std::atomic<int> status{0};
    auto work = [&] {
        for (;;) {
            const int64_t s = next.fetch_add(1);
            if (s >= slices) return;
            const int rc = ifa_ref_int_flash_attention(
                q + s * n * d, sq + s * n, k + s * n * d, sk + s * n, v + s * n * d, sv[s], n,
                d, br, bc, 0, out + s * n * d, nullptr);
            if (rc) status = rc;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return status.load();
}

int ifa_ref_untiled_int8_attention(const int8_t* q, const float* sq, const int8_t* k,
                                   const float* sk, const int8_t* v, float sv, int64_t n,
                                   int64_t d, int sqrt_d, float* out) {
    try {
        ifa::AttentionConfig cfg;
        cfg.apply_sqrt_d_scaling = sqrt_d != 0;
        const ifa::FloatMatrix o =
            ifa::oracle_untiled_int8_attention(make_inputs(q, sq, k, sk, v, sv, n, d), cfg);
        std::memcpy(out, o.data(), sizeof(float) * n * d);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_reference_attention(const float* q, const float* k, const float* v, int64_t n,
                                int64_t d, float* out) {
    try {
        const ifa::FloatMatrix o = ifa::reference_attention(to_fm(q, n, d), to_fm(k, n, d),
                                                            to_fm(v, n, d), ifa::AttentionConfig{});
        std::memcpy(out, o.data(), sizeof(float) * n * d);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_half_int8_attention(const int8_t* q, const float* sq, const int8_t* k,
                                const float* sk, const float* v, int64_t n, int64_t d,
                                int64_t br, int64_t bc, int sqrt_d, float* out) {
    try {
        ifa::QuantizedRows qr{to_im(q, n, d), ifa::ScaleVector(std::vector<float>(sq, sq + n))};
        ifa::QuantizedRows kr{to_im(k, n, d), ifa::ScaleVector(std::vector<float>(sk, sk + n))};
        ifa::AttentionConfig cfg;
        cfg.blocks = ifa::BlockSpec{br, bc};
        cfg.apply_sqrt_d_scaling = sqrt_d != 0;
        const ifa::FloatMatrix o = ifa::half_int8_attention(qr, kr, to_fm(v, n, d), cfg);
        std::memcpy(out, o.data(), sizeof(float) * static_cast<size_t>(n * d));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ifa_ref_fp8_roundtrip(const float* x, int64_t rows, int64_t cols, float* out) {
    try {
        const ifa::FloatMatrix o = ifa::fp8_e4m3_roundtrip(to_fm(x, rows, cols));
        std::memcpy(out, o.data(), sizeof(float) * static_cast<size_t>(rows * cols));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

uint8_t ifa_ref_e4m3_encode(float x) { return ifa::e4m3_encode(x); }

int ifa_ref_fp8_attention(const float* q, const float* k, const float* v, int64_t n, int64_t d,
                          int64_t br, int64_t bc, int sqrt_d, float* out) {
    try {
        ifa::AttentionConfig cfg;
        cfg.blocks = ifa::BlockSpec{br, bc};
        cfg.apply_sqrt_d_scaling = sqrt_d != 0;
        const ifa::FloatMatrix o =
            ifa::fp8_emulated_attention(to_fm(q, n, d), to_fm(k, n, d), to_fm(v, n, d), cfg);
        std::memcpy(out, o.data(), sizeof(float) * static_cast<size_t>(n * d));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

float ifa_ref_expf(float x) { return std::exp(x); }

}  // extern "C"
