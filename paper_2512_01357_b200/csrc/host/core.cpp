#include "core.hpp"

#include <cstdio>
#include <cstring>

#include "murmur_mix.hpp"

namespace tg {

std::string Key::hex() const {
    char buf[33];
    std::snprintf(buf, sizeof buf, "%016llx%016llx", static_cast<unsigned long long>(hi),
                  static_cast<unsigned long long>(lo));
    return buf;
}

const char* err_name(Err e) {
    static const char* names[] = {"insufficient memory", "pool exhausted",       "infeasible",
                                  "tensor pinned",       "not found",            "overlapping move",
                                  "destination occupied", "out-of-order timestamp", "instance too large",
                                  "invalid argument"};
    const int i = static_cast<int>(e);
    return (i >= 0 && i < 10) ? names[i] : "?";
}

Key murmur3_x64_128(const void* data, std::size_t len, u64 seed) {
    const auto* p = static_cast<const unsigned char*>(data);
    u64 h1 = seed, h2 = seed;
    const std::size_t full = len & ~std::size_t{15};
    for (std::size_t off = 0; off < full; off += 16) {
        u64 k[2];
        std::memcpy(k, p + off, 16);
        mm::body(h1, h2, k[0], k[1]);
    }
    const unsigned rem = static_cast<unsigned>(len & 15);
    u64 t[2] = {0, 0};
    std::memcpy(t, p + full, rem);  // little-endian packing of the tail bytes
    mm::finish(h1, h2, t[0], t[1], rem, len);
    return Key{h1, h2};
}

const char* dtype_name(Dtype d) {
    switch (d) {
        case Dtype::F32: return "f32";
        case Dtype::F16: return "f16";
        case Dtype::BF16: return "bf16";
        case Dtype::I8: return "i8";
    }
    return "?";
}

Key tensor_key(const std::string& model_id, const std::string& name, const std::int64_t* shape, int ndim,
               Dtype dtype) {
    std::string s = model_id;
    s += '\x1f';
    s += name;
    s += '\x1f';
    for (int i = 0; i < ndim; ++i) {
        if (i) s += ',';
        s += std::to_string(shape[i]);
    }
    s += '\x1f';
    s += dtype_name(dtype);
    return murmur3_x64_128(s.data(), s.size(), 0);
}

}  // namespace tg
