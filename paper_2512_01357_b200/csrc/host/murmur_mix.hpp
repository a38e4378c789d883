// MurmurHash3 x64-128 building blocks shared by host code and the sm_100a
// fingerprint kernel, so both sides hash with literally the same arithmetic.
// Algorithm: Austin Appleby's public-domain MurmurHash3_x64_128 (the same
// function the reference calls at types.hpp:77-124).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD inline
#endif

namespace tg {
namespace mm {

constexpr std::uint64_t kC1 = 0x87c37b91114253d5ULL;
constexpr std::uint64_t kC2 = 0x4cf5ad432745937fULL;

TG_HD std::uint64_t rol(std::uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

TG_HD std::uint64_t avalanche(std::uint64_t k) {
    k = (k ^ (k >> 33)) * 0xff51afd7ed558ccdULL;
    k = (k ^ (k >> 33)) * 0xc4ceb9fe1a85ec53ULL;
    return k ^ (k >> 33);
}

TG_HD std::uint64_t scramble1(std::uint64_t k) { return rol(k * kC1, 31) * kC2; }
TG_HD std::uint64_t scramble2(std::uint64_t k) { return rol(k * kC2, 33) * kC1; }

// One 16-byte body block (k1 = bytes 0..7, k2 = bytes 8..15, little endian).
TG_HD void body(std::uint64_t& h1, std::uint64_t& h2, std::uint64_t k1, std::uint64_t k2) {
    h1 ^= scramble1(k1);
    h1 = (rol(h1, 27) + h2) * 5 + 0x52dce729;
    h2 ^= scramble2(k2);
    h2 = (rol(h2, 31) + h1) * 5 + 0x38495ab5;
}

// Tail (len % 16 bytes packed little-endian into t1 | t2) and finalisation.
TG_HD void finish(std::uint64_t& h1, std::uint64_t& h2, std::uint64_t t1, std::uint64_t t2, unsigned rem,
                  std::uint64_t len) {
    if (rem > 8) h2 ^= scramble2(t2);
    if (rem > 0) h1 ^= scramble1(t1);
    h1 ^= len;
    h2 ^= len;
    h1 += h2;
    h2 += h1;
    h1 = avalanche(h1);
    h2 = avalanche(h2);
    h1 += h2;
    h2 += h1;
}

}  // namespace mm
}  // namespace tg
