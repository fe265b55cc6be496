// ifa_b200_cli.cpp -- command-line front end over the C-ABI for the file
// commands of the reference CLI (proj/tools/ifa_main.cpp):
//
//   ifa_b200 quantize INPUT OUTPUT [--mode per-row|per-tensor]
//       cmd_quantize (ifa_main.cpp:164-197): INPUT f32 IFA1 -> OUTPUT i8 codes
//       and OUTPUT.scales (rows x 1 f32 per-row scales, or 1 x 1 for
//       per-tensor); prints the same two lines (max round-trip error against
//       the dequantized codes, double product rounded once, quant.cpp:71-98).
//       The quantization itself runs on the GPU (ifa_quantize_*_host).
//   ifa_b200 info PATH
//       cmd_info (ifa_main.cpp:198-230): dtype, shape, min and max.
//
// Exit codes as ifa_main.cpp:4: 0 success, 1 runtime or I/O failure,
// 2 usage error.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ifa_b200.h"

namespace {

int usage() {
    std::fprintf(stderr,
                 "usage: ifa_b200 quantize INPUT OUTPUT [--mode per-row|per-tensor]\n"
                 "       ifa_b200 info PATH\n");
    return 2;
}

int fail() {
    std::fprintf(stderr, "error: %s\n", ifa_last_error());
    return 1;
}

int cmd_quantize(const std::string& in_path, const std::string& out_path,
                 const std::string& mode) {
    int32_t dt = 0;
    int64_t rows = 0, cols = 0;
    if (ifa_tensor_info(in_path.c_str(), &dt, &rows, &cols) != IFA_OK) return fail();
    std::vector<float> x(static_cast<size_t>(rows * cols));
    if (ifa_tensor_load(in_path.c_str(), IFA_DT_F32, x.data(), rows, cols) != IFA_OK)
        return fail();
    std::vector<int8_t> codes(x.size());
    std::vector<float> scales;
    double bound = 0.0;
    std::vector<float> restored(x.size());
    if (mode == "per-tensor") {
        scales.assign(1, 0.0f);
        if (ifa_quantize_per_tensor_host(x.data(), 1, rows, cols, codes.data(), scales.data(),
                                         nullptr, nullptr) != IFA_OK)
            return fail();
        const double s = scales[0];
        for (size_t i = 0; i < x.size(); ++i)
            restored[i] = static_cast<float>(static_cast<double>(codes[i]) * s);
        bound = 0.5 * scales[0];
    } else {
        scales.assign(static_cast<size_t>(rows), 0.0f);
        if (rows > 0 && ifa_quantize_per_row_host(x.data(), rows, cols, codes.data(),
                                                  scales.data(), nullptr, nullptr) != IFA_OK)
            return fail();
        for (int64_t r = 0; r < rows; ++r) {
            const double s = scales[static_cast<size_t>(r)];
            for (int64_t c = 0; c < cols; ++c) {
                const size_t i = static_cast<size_t>(r * cols + c);
                restored[i] = static_cast<float>(static_cast<double>(codes[i]) * s);
            }
            bound = std::max(bound, 0.5 * scales[static_cast<size_t>(r)]);
        }
    }
    if (ifa_tensor_save(out_path.c_str(), IFA_DT_I8, codes.data(), rows, cols) != IFA_OK)
        return fail();
    const std::string sc_path = out_path + ".scales";
    if (ifa_tensor_save(sc_path.c_str(), IFA_DT_F32, scales.data(),
                        static_cast<int64_t>(scales.size()), 1) != IFA_OK)
        return fail();
    double worst = 0.0;
    for (size_t i = 0; i < x.size(); ++i)
        worst = std::max(worst, std::fabs(static_cast<double>(restored[i]) -
                                          static_cast<double>(x[i])));
    std::printf("wrote %s (i8 %lldx%lld) and %s.scales\n", out_path.c_str(),
                static_cast<long long>(rows), static_cast<long long>(cols), out_path.c_str());
    std::printf("max round-trip error %.6g (bound scale/2 = %.6g)\n", worst, bound);
    return 0;
}

template <typename T>
void min_max(const std::vector<T>& v, double& lo, double& hi) {
    lo = hi = 0.0;
    if (v.empty()) return;
    lo = hi = static_cast<double>(v[0]);
    for (const T& x : v) {
        lo = std::min(lo, static_cast<double>(x));
        hi = std::max(hi, static_cast<double>(x));
    }
}

int cmd_info(const std::string& path) {
    int32_t dt = 0;
    int64_t rows = 0, cols = 0;
    if (ifa_tensor_info(path.c_str(), &dt, &rows, &cols) != IFA_OK) return fail();
    const size_t n = static_cast<size_t>(rows * cols);
    double lo = 0.0, hi = 0.0;
    const char* name = dt == IFA_DT_F32 ? "f32" : (dt == IFA_DT_I8 ? "i8" : "i32");
    if (dt == IFA_DT_F32) {
        std::vector<float> v(n);
        if (ifa_tensor_load(path.c_str(), dt, v.data(), rows, cols) != IFA_OK) return fail();
        min_max(v, lo, hi);
    } else if (dt == IFA_DT_I8) {
        std::vector<int8_t> v(n);
        if (ifa_tensor_load(path.c_str(), dt, v.data(), rows, cols) != IFA_OK) return fail();
        min_max(v, lo, hi);
    } else {
        std::vector<int32_t> v(n);
        if (ifa_tensor_load(path.c_str(), dt, v.data(), rows, cols) != IFA_OK) return fail();
        min_max(v, lo, hi);
    }
    std::printf("%s: %s %lldx%lld\n", path.c_str(), name, static_cast<long long>(rows),
                static_cast<long long>(cols));
    std::printf("min %.6g max %.6g\n", lo, hi);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    if (cmd == "info") {
        if (argc != 3) return usage();
        return cmd_info(argv[2]);
    }
    if (cmd == "quantize") {
        std::vector<std::string> pos;
        std::string mode = "per-row";
        for (int i = 2; i < argc; ++i) {
            if (std::strcmp(argv[i], "--mode") == 0 && i + 1 < argc) {
                mode = argv[++i];
                if (mode != "per-row" && mode != "per-tensor") return usage();
            } else if (std::strncmp(argv[i], "--mode=", 7) == 0) {
                mode = argv[i] + 7;
                if (mode != "per-row" && mode != "per-tensor") return usage();
            } else {
                pos.push_back(argv[i]);
            }
        }
        if (pos.size() != 2) return usage();
        return cmd_quantize(pos[0], pos[1], mode);
    }
    return usage();
}
