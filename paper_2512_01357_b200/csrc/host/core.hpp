// Core value types of the Tangram B200 pool: tensor keys, error codes and a
// small expected-style result.  Semantics follow the reference's types.hpp
// (TensorId 46-60, Error 155-166, Result 197-217) so that every decision the
// control plane takes is bit-identical; the representation is our own.
#pragma once

#include <cstdint>
#include <string>
#include <utility>

namespace tg {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

// 128-bit tensor key.  Ordering is lexicographic (hi, lo), like the
// reference's defaulted operator<=> (types.hpp:51).
struct Key {
    u64 hi = 0;
    u64 lo = 0;
    friend bool operator==(const Key& a, const Key& b) { return a.hi == b.hi && a.lo == b.lo; }
    friend bool operator!=(const Key& a, const Key& b) { return !(a == b); }
    friend bool operator<(const Key& a, const Key& b) { return a.hi != b.hi ? a.hi < b.hi : a.lo < b.lo; }
    std::string hex() const;
};

// Same mixing as TensorIdHash (types.hpp:148-152) so unordered containers see
// the same bucket distribution (iteration order is never relied upon).
struct KeyHash {
    std::size_t operator()(const Key& k) const noexcept {
        return static_cast<std::size_t>(k.hi ^ (k.lo * 0x9e3779b97f4a7c15ULL));
    }
};

// Domain errors; numeric values are the reference's Error ordinals
// (types.hpp:155-166).  The C-ABI reports them as ordinal + 1.
enum class Err : int {
    InsufficientMemory = 0,
    PoolExhausted,
    Infeasible,
    Pinned,
    NotFound,
    OverlapMove,
    DestinationOccupied,
    OrderingError,
    InstanceTooLarge,
    InvalidArgument,
};

const char* err_name(Err e);

// Minimal expected<T, Err>.
template <typename T>
class Res {
public:
    Res(T v) : ok_(true), v_(std::move(v)) {}  // NOLINT
    Res(Err e) : ok_(false), e_(e) {}          // NOLINT
    bool ok() const { return ok_; }
    explicit operator bool() const { return ok_; }
    T& value() { return v_; }
    const T& value() const { return v_; }
    Err error() const { return e_; }

private:
    bool ok_;
    T v_{};
    Err e_ = Err::InvalidArgument;
};

struct Nothing {};
using St = Res<Nothing>;
inline St ok() { return St(Nothing{}); }

// MurmurHash3 x64-128 (Appleby's public algorithm; the reference uses it at
// types.hpp:77-124 for TensorId and we use it as the content-fingerprint
// leaf).  Returns {h1, h2}.
Key murmur3_x64_128(const void* data, std::size_t len, u64 seed);

enum class Dtype : std::uint8_t { F32 = 0, F16 = 1, BF16 = 2, I8 = 3 };
const char* dtype_name(Dtype d);

// Metadata key of a tensor: murmur3 of "model␟name␟d0,d1,…␟dtype"
// (types.hpp:131-146).
Key tensor_key(const std::string& model_id, const std::string& name, const std::int64_t* shape, int ndim,
               Dtype dtype);

}  // namespace tg
