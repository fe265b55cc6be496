// verify_gpu.cpp -- runs the REFERENCE's own property suites against the
// B200 kernel through the reference's plugin hook.
//
// TEST INFRASTRUCTURE ONLY.  Built by `make -C oracle verify` (links the
// unmodified reference library oracle/_ref/libifa_ref.a and the product
// library paper_2409_16997_b200/lib/libifa_b200.so) into oracle/_ref/, and
// executed on the GPU box by tests/test_gpu_reference_suites.py.
//
//   ifa::VerifyOptions::int_flash (verify.hpp:18-24) = ifa_gpu::int_flash_attention
//   ifa::run_verification(options)                    (verify.cpp:418-450)
//
// Exit status 0 iff every suite passes for every (seed, blocks) option set
// AND a deliberately perturbed GPU kernel is caught (the suites bite), AND
// the shim's quantizers equal ifa::quantize_per_row / _per_tensor bitwise.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ifa/attention.hpp"
#include "ifa/eval.hpp"
#include "ifa/generate.hpp"
#include "ifa/quant.hpp"
#include "ifa/verify.hpp"
#include "ifa_b200.hpp"

namespace {

bool run(const ifa::VerifyOptions& opt, const char* label, bool print) {
    const ifa::VerifyOutcome out = ifa::run_verification(opt);
    for (const ifa::SuiteResult& s : out.suites)
        if (print || !s.passed)
            std::printf("%s %-26s %s%s%s\n", s.passed ? "ok  " : "FAIL", s.name.c_str(), label,
                        s.passed ? "" : "  ", s.detail.c_str());
    return out.passed();
}

bool same_bits(const float* a, const float* b, int64_t n) {
    return std::memcmp(a, b, sizeof(float) * static_cast<size_t>(n)) == 0;
}

}  // namespace

int main() {
    int failures = 0;
    const ifa::BlockSpec blocks[] = {{64, 64}, {128, 128}, {7, 5}, {1, 1}, {33, 200}};
    for (uint64_t seed : {0ull, 1ull, 2ull, 12345ull}) {
        for (const ifa::BlockSpec& b : blocks) {
            ifa::VerifyOptions opt;
            opt.blocks = b;
            opt.seed = seed;
            opt.int_flash = [](const ifa::QuantizedAttentionInputs& in,
                               const ifa::AttentionConfig& cfg, ifa::PCodeAudit* audit) {
                return ifa_gpu::int_flash_attention(in, cfg, audit);
            };
            char label[96];
            std::snprintf(label, sizeof label, "[gpu seed=%llu Br=%lld Bc=%lld]",
                          static_cast<unsigned long long>(seed), static_cast<long long>(b.Br),
                          static_cast<long long>(b.Bc));
            if (!run(opt, label, seed == 0)) ++failures;
        }
    }
    // A perturbed GPU kernel must be rejected (SPEC.md:422 mutation idea).
    {
        ifa::VerifyOptions opt;
        opt.int_flash = [](const ifa::QuantizedAttentionInputs& in,
                           const ifa::AttentionConfig& cfg, ifa::PCodeAudit* audit) {
            ifa::FloatMatrix o = ifa_gpu::int_flash_attention(in, cfg, audit);
            o.data()[0] = std::nextafter(o.data()[0], 1e30f);
            return o;
        };
        if (run(opt, "[mutant: O[0][0] + 1 ulp]", false)) {
            std::printf("FAIL the suites did not catch a perturbed kernel\n");
            ++failures;
        } else {
            std::printf("ok   mutant kernel rejected by the reference suites\n");
        }
    }
    // Quantizer drop-ins vs the reference, on the generator's activations.
    {
        int bad = 0;
        for (int t = 0; t < 24; ++t) {
            const int64_t rows = 1 + 37 * t, cols = (t % 3 == 0) ? 128 : 8 + 13 * t;
            const ifa::FloatMatrix x = ifa::generate(
                t % 2 ? ifa::ActivationSpec::uniform(-0.5, 0.5, 1000 + t)
                      : ifa::ActivationSpec::normal(0.0, 1.0 + t, 1000 + t),
                rows, cols);
            const ifa::QuantizedRows want = ifa::quantize_per_row(x);
            const ifa::QuantizedRows got = ifa_gpu::quantize_per_row(x);
            const ifa::QuantizedTensor want_t = ifa::quantize_per_tensor(x);
            const ifa::QuantizedTensor got_t = ifa_gpu::quantize_per_tensor(x);
            if (!(want.values == got.values) ||
                !same_bits(want.scales.data(), got.scales.data(), rows) ||
                !(want_t.values == got_t.values) || !same_bits(&want_t.scale, &got_t.scale, 1))
                ++bad;
        }
        std::printf("%s quantize_per_row / quantize_per_tensor drop-ins bitwise (24 cases)\n",
                    bad ? "FAIL" : "ok  ");
        failures += bad;
    }
    // §8(f) drop-ins: half_int8_attention and fp8_emulated_attention against the
    // reference library on the same inputs (tolerance: MRE <= 2e-3).
    {
        int bad = 0;
        for (int t = 0; t < 6; ++t) {
            const int64_t n = (t % 2) ? 256 : 200, d = (t % 3 == 0) ? 64 : 128;
            auto gen = [&](int role) {
                return ifa::generate(t % 2 ? ifa::ActivationSpec::uniform(-0.5, 0.5, 77 + 3 * t + role)
                                           : ifa::ActivationSpec::normal(0.0, 1.0, 77 + 3 * t + role),
                                     n, d);
            };
            const ifa::FloatMatrix q = gen(0), k = gen(1), v = gen(2);
            ifa::AttentionConfig cfg;
            cfg.blocks = ifa::BlockSpec{64, t < 3 ? 64 : 128};
            cfg.apply_sqrt_d_scaling = t % 2 == 0;
            const ifa::QuantizedRows qr = ifa::quantize_per_row(q), kr = ifa::quantize_per_row(k);
            const ifa::FloatMatrix h_want = ifa::half_int8_attention(qr, kr, v, cfg);
            const ifa::FloatMatrix h_got = ifa_gpu::half_int8_attention(qr, kr, v, cfg);
            const ifa::FloatMatrix f_want = ifa::fp8_emulated_attention(q, k, v, cfg);
            const ifa::FloatMatrix f_got = ifa_gpu::fp8_emulated_attention(q, k, v, cfg);
            const double e_h = ifa::mre(h_want, h_got), e_f = ifa::mre(f_want, f_got);
            if (!(e_h <= 2e-3) || !(e_f <= 2e-3)) {
                std::printf("FAIL  n=%lld d=%lld half MRE %.3g fp8 MRE %.3g\n",
                            static_cast<long long>(n), static_cast<long long>(d), e_h, e_f);
                ++bad;
            }
        }
        std::printf("%s half_int8_attention / fp8_emulated_attention drop-ins within tolerance\n",
                    bad ? "FAIL" : "ok  ");
        failures += bad;
    }
    // The tolerance kernel through the same plugin signature (IntFlashFn,
    // verify.hpp:15-16) and the full-INT8 step from float matrices
    // (eval.cpp:98-102): vs the reference library on the same inputs.
    {
        int bad = 0;
        const int64_t shapes[][3] = {{1024, 64, 128}, {4096, 128, 128}, {384, 128, 128},
                                     {300, 100, 128}, {96, 64, 300}};
        for (int t = 0; t < 5; ++t) {
            const int64_t n = shapes[t][0], d = shapes[t][1];
            auto gen = [&](int role) {
                return ifa::generate(t % 2 ? ifa::ActivationSpec::uniform(-0.5, 0.5, 501 + 3 * t + role)
                                           : ifa::ActivationSpec::normal(0.0, 1.0, 501 + 3 * t + role),
                                     n, d);
            };
            const ifa::FloatMatrix q = gen(0), k = gen(1), v = gen(2);
            ifa::AttentionConfig cfg;
            cfg.blocks = ifa::BlockSpec{64, shapes[t][2]};
            const ifa::QuantizedAttentionInputs in{ifa::quantize_per_row(q), ifa::quantize_per_row(k),
                                                   ifa::quantize_per_tensor(v)};
            const ifa::FloatMatrix want = ifa::int_flash_attention(in, cfg);
            const double e_fast = ifa::mre(want, ifa_gpu::int_flash_attention_fast(in, cfg));
            const double e_full = ifa::mre(want, ifa_gpu::full_int8_attention(q, k, v, cfg, true));
            const ifa::FloatMatrix exact = ifa_gpu::full_int8_attention(q, k, v, cfg, false);
            const bool bitwise = same_bits(want.data(), exact.data(), n * d);
            if (!(e_fast <= 1e-5) || !(e_full <= 1e-5) || !bitwise) {
                std::printf("FAIL  n=%lld d=%lld fast MRE %.3g full-step MRE %.3g exact bitwise %d\n",
                            static_cast<long long>(n), static_cast<long long>(d), e_fast, e_full,
                            bitwise ? 1 : 0);
                ++bad;
            }
        }
        std::printf("%s int_flash_attention_fast / full_int8_attention drop-ins vs the reference\n",
                    bad ? "FAIL" : "ok  ");
        failures += bad;
    }
    // Exceptions keep the reference's types and messages.
    {
        ifa::QuantizedAttentionInputs in;
        bool ok = false;
        try {
            ifa_gpu::int_flash_attention(in, ifa::AttentionConfig{});
        } catch (const std::invalid_argument& e) {
            ok = std::string(e.what()) == "quantized attention inputs: empty q";
        }
        ifa::FloatMatrix x(1, 3, std::vector<float>{1.0f, std::nanf(""), 2.0f});
        bool ok2 = false;
        try {
            ifa_gpu::quantize_per_row(x);
        } catch (const std::invalid_argument& e) {
            ok2 = std::string(e.what()).find("index 1") != std::string::npos;
        }
        std::printf("%s exception types and messages\n", ok && ok2 ? "ok  " : "FAIL");
        if (!(ok && ok2)) ++failures;
    }
    std::printf("%s\n", failures ? "verify_gpu: FAILED" : "verify_gpu: all passed");
    return failures ? 1 : 0;
}
