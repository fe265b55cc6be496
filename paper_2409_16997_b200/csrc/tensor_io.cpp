// tensor_io.cpp -- the "IFA1" tensor file format, the
// on-disk interchange for shipping inputs / codes / outputs between the CPU
// reference and the GPU path.
//
// Restates /root/reference/proj/src/tensor_io.cpp:15-178 (format in
// include/ifa/tensor_io.hpp:22-39, proj/README.md "Tensor file format"):
//   magic "IFA1", dtype u8 (0 f32, 1 i8, 2 i32), 3 zero bytes,
//   rows u64 LE, cols u64 LE, row-major little-endian payload.
// Loaders reject the same malformed files with the same messages
// (FormatError there, IFA_EFORMAT + ifa_last_error() here).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ifa_internal.h"

namespace {

constexpr char kMagic[4] = {'I', 'F', 'A', '1'};
constexpr size_t kHeaderSize = 24;
constexpr uint64_t kMaxElems = uint64_t{1} << 33;  // tensor_io.cpp:20

size_t width_of(int32_t dtype) { return dtype == IFA_DT_I8 ? 1 : 4; }

void put_u64_le(uint8_t* dst, uint64_t v) {
    for (int i = 0; i < 8; ++i) dst[i] = static_cast<uint8_t>(v >> (8 * i));
}
uint64_t get_u64_le(const uint8_t* src) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(src[i]) << (8 * i);
    return v;
}

int fmt_error(const std::string& msg) { return ifa_b200::set_error(IFA_EFORMAT, msg); }

// Reads and validates a whole file (tensor_io.cpp:112-152).
int read_checked(const char* path, std::vector<uint8_t>& bytes, int32_t* dtype, int64_t* rows,
                 int64_t* cols) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return fmt_error(std::string("cannot open: ") + path);
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    bytes.resize(size > 0 ? static_cast<size_t>(size) : 0);
    const size_t got = bytes.empty() ? 0 : std::fread(bytes.data(), 1, bytes.size(), f);
    std::fclose(f);
    if (got != bytes.size()) return fmt_error(std::string("cannot read: ") + path);
    if (bytes.size() < kHeaderSize)
        return fmt_error("truncated header: " + std::to_string(bytes.size()) + " bytes");
    if (std::memcmp(bytes.data(), kMagic, 4) != 0) return fmt_error("bad magic");
    const uint8_t dt = bytes[4];
    if (bytes[5] != 0 || bytes[6] != 0 || bytes[7] != 0)
        return fmt_error("nonzero reserved bytes");
    const uint64_t r = get_u64_le(bytes.data() + 8);
    const uint64_t c = get_u64_le(bytes.data() + 16);
    if (r > kMaxElems || c > kMaxElems || (r != 0 && c > kMaxElems / r))
        return fmt_error("header dimensions overflow: " + std::to_string(r) + "x" +
                         std::to_string(c));
    if (dt > IFA_DT_I32) return fmt_error("bad dtype code " + std::to_string(dt));
    const size_t want = static_cast<size_t>(r * c) * width_of(dt);
    const size_t have = bytes.size() - kHeaderSize;
    if (have < want)
        return fmt_error("truncated payload: expected " + std::to_string(want) + " bytes, got " +
                         std::to_string(have));
    if (have > want)
        return fmt_error("oversized payload: expected " + std::to_string(want) + " bytes, got " +
                         std::to_string(have));
    *dtype = dt;
    *rows = static_cast<int64_t>(r);
    *cols = static_cast<int64_t>(c);
    return IFA_OK;
}

}  // namespace

extern "C" {

int ifa_tensor_save(const char* path, int32_t dtype, const void* data, int64_t rows,
                    int64_t cols) {
    ifa_b200::set_error(IFA_OK, "");
    if (!path || dtype < IFA_DT_F32 || dtype > IFA_DT_I32 || rows < 0 || cols < 0 ||
        (rows * cols > 0 && !data))
        return ifa_b200::set_error(IFA_EINVAL, "ifa_tensor_save: bad arguments");
    FILE* f = std::fopen(path, "wb");
    if (!f) return fmt_error(std::string("cannot open for writing: ") + path);
    uint8_t header[kHeaderSize] = {};
    std::memcpy(header, kMagic, 4);
    header[4] = static_cast<uint8_t>(dtype);
    put_u64_le(header + 8, static_cast<uint64_t>(rows));
    put_u64_le(header + 16, static_cast<uint64_t>(cols));
    bool ok = std::fwrite(header, 1, kHeaderSize, f) == kHeaderSize;
    // the payload is little-endian; this host is too (x86-64 / aarch64)
    const size_t bytes = static_cast<size_t>(rows * cols) * width_of(dtype);
    if (ok && bytes) ok = std::fwrite(data, 1, bytes, f) == bytes;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fmt_error(std::string("short write: ") + path);
    return IFA_OK;
}

int ifa_tensor_info(const char* path, int32_t* dtype, int64_t* rows, int64_t* cols) {
    ifa_b200::set_error(IFA_OK, "");
    if (!path || !dtype || !rows || !cols)
        return ifa_b200::set_error(IFA_EINVAL, "ifa_tensor_info: null pointer");
    std::vector<uint8_t> bytes;
    return read_checked(path, bytes, dtype, rows, cols);
}

int ifa_tensor_load(const char* path, int32_t dtype, void* data, int64_t rows, int64_t cols) {
    ifa_b200::set_error(IFA_OK, "");
    if (!path) return ifa_b200::set_error(IFA_EINVAL, "ifa_tensor_load: null path");
    std::vector<uint8_t> bytes;
    int32_t dt = 0;
    int64_t r = 0, c = 0;
    const int rc = read_checked(path, bytes, &dt, &r, &c);
    if (rc != IFA_OK) return rc;
    if (dtype >= 0 && dt != dtype) {  // load_float_tensor / load_int8_tensor
        static const char* names[] = {"f32", "i8", "i32"};
        return fmt_error(std::string("expected ") + names[dtype] + " tensor: " + path);
    }
    if (r != rows || c != cols)
        return ifa_b200::set_error(IFA_EINVAL, "ifa_tensor_load: shape is " + std::to_string(r) +
                                                   "x" + std::to_string(c));
    const size_t n = static_cast<size_t>(r * c) * width_of(dt);
    if (n) {
        if (!data) return ifa_b200::set_error(IFA_EINVAL, "ifa_tensor_load: null buffer");
        std::memcpy(data, bytes.data() + kHeaderSize, n);
    }
    return IFA_OK;
}

}  // extern "C"
