// checkpoint.cuh -- FNN1 save / load of a device-resident network.
//
// Byte format of the reference's save_network / load_network (network.hpp:552-607): "FNN1", u32
// layer count, then per spec layer a u32-length tag, a u32 tensor count and per tensor a u32 rank,
// u64 extents and the little-endian f32 values in logical (row-major fastnn) order. Dense layers
// persist {w (out, in), b (out)}, conv layers {kernels (k, c, kh, kw), b (k)}; pooling /
// activations / softmax / flatten persist nothing. The whole parameter set moves in ONE
// device->host copy of the packed buffer (or one host->device copy on load), and the file is
// written / parsed on the host with the reference's checks and messages.
//
// For exact resume the library also writes an optional sidecar `<path>.state` (not read by the
// reference): "B2NS", u32 version 2, u32 optimizer kind, u64 adam step count, f32 lr, momentum,
// weight_decay, u32 buffer count (1 for SGD-momentum / Adagrad, 2 for Adadelta / Adam), then per
// buffer a u32 tensor count and per trainable tensor its rank, extents and values: the momentum
// velocity, or acc [+ acc_update], or m + v (optim.hpp:23-27 OptimizerState::Slot).
#pragma once
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "runtime.cuh"

namespace b2n {
namespace ckpt {

inline void put_u32(std::string& o, uint32_t v) {
    const char b[4] = {(char)(v & 0xff), (char)((v >> 8) & 0xff), (char)((v >> 16) & 0xff), (char)((v >> 24) & 0xff)};
    o.append(b, 4);
}
inline void put_u64(std::string& o, uint64_t v) {
    put_u32(o, (uint32_t)(v & 0xffffffffu));
    put_u32(o, (uint32_t)(v >> 32));
}
inline void put_f32s(std::string& o, const float* p, size_t n) {
    static_assert(sizeof(float) == 4, "f32");
    const size_t at = o.size();
    o.resize(at + n * 4);
    for (size_t i = 0; i < n; ++i) {  // explicit little-endian, like write_f32
        uint32_t v;
        std::memcpy(&v, p + i, 4);
        char* d = &o[at + i * 4];
        d[0] = (char)(v & 0xff);
        d[1] = (char)((v >> 8) & 0xff);
        d[2] = (char)((v >> 16) & 0xff);
        d[3] = (char)((v >> 24) & 0xff);
    }
}

// a bounds-checked reader over the whole file; every short read is LengthError (network.hpp:535)
struct Reader {
    std::string buf;
    size_t pos = 0;
    void need(size_t n) {
        if (buf.size() - pos < n) throw Error(B2N_ELENGTH, "checkpoint truncated");
    }
    uint32_t u32() {
        need(4);
        const unsigned char* b = (const unsigned char*)buf.data() + pos;
        pos += 4;
        return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
    }
    uint64_t u64() {
        const uint64_t lo = u32();
        return lo | ((uint64_t)u32() << 32);
    }
    std::string bytes(size_t n) {
        need(n);
        std::string s = buf.substr(pos, n);
        pos += n;
        return s;
    }
    void f32s(float* out, size_t n) {
        need(n * 4);
        const unsigned char* b = (const unsigned char*)buf.data() + pos;
        for (size_t i = 0; i < n; ++i) {
            const uint32_t v = (uint32_t)b[4 * i] | ((uint32_t)b[4 * i + 1] << 8) | ((uint32_t)b[4 * i + 2] << 16) |
                               ((uint32_t)b[4 * i + 3] << 24);
            std::memcpy(out + i, &v, 4);
        }
        pos += n * 4;
    }
};

inline std::string read_file(const std::string& path, const char* who) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Error(B2N_EIO, std::string(who) + ": cannot open " + path);
    return std::string((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
}

inline void write_file(const std::string& path, const std::string& data, const char* who) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Error(B2N_EIO, std::string(who) + ": cannot open " + path);
    os.write(data.data(), (std::streamsize)data.size());
    if (!os) throw Error(B2N_EIO, std::string(who) + ": write failed for " + path);
}

// tag of a spec layer (the LayerNode::tag() strings, network.hpp:82-180)
inline const char* tag_of(int kind) {
    switch (kind) {
        case B2N_DENSE: return "dense";
        case B2N_CONV: return "conv";
        case B2N_MAXPOOL: return "maxpool";
        case B2N_SIGMOID: return "sigmoid";
        case B2N_RELU: return "relu";
        case B2N_SOFTMAX: return "softmax";
        case B2N_FLATTEN: return "flatten";
        case B2N_DROPOUT: return "dropout";
        case B2N_BATCHNORM: return "batchnorm";
    }
    return "?";
}

}  // namespace ckpt
}  // namespace b2n
