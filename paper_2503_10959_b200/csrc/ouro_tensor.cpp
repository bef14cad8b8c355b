// OURO tensor container on the host side of the B200 path:
// the reference's binary format (tensor_io.hpp:13-19, tensor_io.cpp) —
//
//   "OURO" | u32 version = 1 | u32 rank | u64 dims[rank] | u32 dtype | payload
//
// little-endian, dtype 0 = f64, 1 = i8, 2 = u4 (two's-complement nibbles, element
// i in the low nibble of byte i/2 when i is even, the high nibble when odd; a
// trailing odd element leaves the high nibble 0). The u4 payload of a row-major
// [rows][E] code matrix with E even is exactly the K1 operand's packed device
// layout (kernels.h QAct::packed), so device codes are written without repacking.
// Files are written through a temporary and a rename, like the reference's
// atomic_write_bytes.
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "engine.h"

namespace ob {

namespace fs = std::filesystem;

namespace {
constexpr char kOuroMagic[4] = {'O', 'U', 'R', 'O'};
constexpr uint32_t kOuroVersion = 1;  // tensor_io.hpp:19

template <class T>
void append(std::string& b, T v) {
    b.append(reinterpret_cast<const char*>(&v), sizeof(T));  // little-endian hosts only (x86-64, aarch64)
}
}  // namespace

void atomic_write_bytes(const std::string& path, const std::string& bytes) {
    fs::path tmp = path;
    tmp += ".tmp";
    {
        std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
        if (!f) throw IoError("cannot create file: " + tmp.string());
        f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
        if (!f) throw IoError("short write: " + tmp.string());
    }
    std::error_code ec;
    fs::rename(tmp, path, ec);
    if (ec) throw IoError("rename failed: " + tmp.string() + " -> " + path + ": " + ec.message());
}

std::string read_whole_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open file: " + path);
    return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

size_t ouro_numel(const std::vector<uint64_t>& shape) {
    size_t n = 1;
    for (uint64_t d : shape) n *= static_cast<size_t>(d);
    return n;
}

size_t ouro_payload_bytes(OuroDtype dt, const std::vector<uint64_t>& shape) {
    const size_t n = ouro_numel(shape);
    switch (dt) {
        case OuroDtype::F64: return n * sizeof(double);
        case OuroDtype::I8: return n;
        case OuroDtype::U4: return (n + 1) / 2;
    }
    throw ValidationError("unknown OURO dtype");
}

void pack_nibbles(const int8_t* codes, size_t n, uint8_t* out) {
    std::memset(out, 0, (n + 1) / 2);
    for (size_t i = 0; i < n; ++i) {
        require(codes[i] >= -8 && codes[i] <= 7, "u4 tensor: code " + std::to_string(codes[i]) +
                                                     " at element " + std::to_string(i) + " is outside [-8, 7]");
        const uint8_t nib = static_cast<uint8_t>(codes[i]) & 0x0Fu;
        out[i >> 1] |= (i & 1) ? static_cast<uint8_t>(nib << 4) : nib;
    }
}

void unpack_nibbles(const uint8_t* packed, size_t n, int8_t* out) {
    for (size_t i = 0; i < n; ++i) {
        const unsigned nib = (i & 1) ? (packed[i >> 1] >> 4) : (packed[i >> 1] & 0x0Fu);
        out[i] = static_cast<int8_t>(static_cast<int>(nib << 28) >> 28);  // sign-extend bit 3
    }
}

void ouro_tensor_write(const std::string& path, OuroDtype dt, const std::vector<uint64_t>& shape,
                       const void* payload, size_t bytes) {
    require(shape.size() <= 16, "OURO tensor: rank above 16");
    require(bytes == ouro_payload_bytes(dt, shape), "OURO tensor: payload size does not match the shape");
    std::string b;
    b.reserve(16 + 8 * shape.size() + bytes);
    b.append(kOuroMagic, 4);
    append<uint32_t>(b, kOuroVersion);
    append<uint32_t>(b, static_cast<uint32_t>(shape.size()));
    for (uint64_t d : shape) append<uint64_t>(b, d);
    append<uint32_t>(b, static_cast<uint32_t>(dt));
    b.append(static_cast<const char*>(payload), bytes);
    atomic_write_bytes(path, b);
}

OuroTensor ouro_tensor_read(const std::string& path) {
    const std::string b = read_whole_file(path);
    size_t off = 0;
    auto take = [&](void* dst, size_t n) {
        if (off + n > b.size()) throw IoError(path + ": truncated tensor file");
        std::memcpy(dst, b.data() + off, n);
        off += n;
    };
    char magic[4];
    take(magic, 4);
    if (std::memcmp(magic, kOuroMagic, 4) != 0) throw IoError(path + ": bad magic, not a tensor file");
    uint32_t version = 0, rank = 0, dt = 0;
    take(&version, 4);
    if (version != kOuroVersion) throw IoError(path + ": unsupported tensor format version " + std::to_string(version));
    take(&rank, 4);
    if (rank > 16) throw IoError(path + ": implausible tensor rank " + std::to_string(rank));
    OuroTensor t;
    t.shape.resize(rank);
    for (auto& d : t.shape) take(&d, 8);
    take(&dt, 4);
    if (dt > 2) throw IoError(path + ": unknown dtype tag " + std::to_string(dt));
    t.dtype = static_cast<OuroDtype>(dt);
    const size_t n = ouro_payload_bytes(t.dtype, t.shape);
    t.payload.resize(n);
    take(t.payload.data(), n);
    return t;
}

}  // namespace ob
