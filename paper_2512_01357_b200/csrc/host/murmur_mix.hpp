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

#if defined(__CUDACC__)
// Device form of body(): the same arithmetic spelled on 32-bit halves so that
// ptxas emits what the SM executes natively — a 64x64 low multiply by a
// constant as IMAD.WIDE.U32 + 2 IMAD, a 64-bit rotate as 2 funnel shifts
// (SHF), h*5+c as IMAD.WIDE.U32 with a 64-bit addend + IMAD.  The generic u64
// spelling compiles to ~65 instructions per 16-byte block on sm_100a (rotates
// become 4-instruction shift/or chains); this one to ~36.
struct W32 {
    std::uint32_t l, h;
};
__device__ __forceinline__ W32 w_of(std::uint64_t x) { return W32{static_cast<std::uint32_t>(x), static_cast<std::uint32_t>(x >> 32)}; }
__device__ __forceinline__ std::uint64_t u_of(W32 a) { return (static_cast<std::uint64_t>(a.h) << 32) | a.l; }
template <std::uint64_t C>
__device__ __forceinline__ W32 mulc(W32 a) {
    constexpr std::uint32_t cl = static_cast<std::uint32_t>(C), ch = static_cast<std::uint32_t>(C >> 32);
    const std::uint64_t p = static_cast<std::uint64_t>(a.l) * cl;
    return W32{static_cast<std::uint32_t>(p), static_cast<std::uint32_t>(p >> 32) + a.l * ch + a.h * cl};
}
template <int R>  // 0 < R < 32
__device__ __forceinline__ W32 rol32(W32 a) {
    return W32{__funnelshift_l(a.h, a.l, R), __funnelshift_l(a.l, a.h, R)};
}
__device__ __forceinline__ W32 rol33(W32 a) { return W32{__funnelshift_l(a.l, a.h, 1), __funnelshift_l(a.h, a.l, 1)}; }
template <std::uint32_t C>
__device__ __forceinline__ W32 mul5_add(W32 a) {
    const std::uint64_t t = static_cast<std::uint64_t>(a.l) * 5u + C;
    return W32{static_cast<std::uint32_t>(t), static_cast<std::uint32_t>(t >> 32) + a.h * 5u};
}
__device__ __forceinline__ W32 add64(W32 a, W32 b) { return w_of(u_of(a) + u_of(b)); }
__device__ __forceinline__ W32 xor64(W32 a, W32 b) { return W32{a.l ^ b.l, a.h ^ b.h}; }

// body() on halves; k1 = (k1l, k1h), k2 = (k2l, k2h).
__device__ __forceinline__ void body_dev(W32& h1, W32& h2, W32 k1, W32 k2) {
    k1 = mulc<kC2>(rol32<31>(mulc<kC1>(k1)));
    h1 = mul5_add<0x52dce729u>(add64(rol32<27>(xor64(h1, k1)), h2));
    k2 = mulc<kC1>(rol33(mulc<kC2>(k2)));
    h2 = mul5_add<0x38495ab5u>(add64(rol32<31>(xor64(h2, k2)), h1));
}
#endif

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
