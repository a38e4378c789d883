// Synthetic checkpoint generator (benchmark / test input):
// little-endian u64 word w of tensor (hi, lo) is
// splitmix64(hi ^ rotl(lo, 17) ^ (w * 0x9E3779B97F4A7C15)).
// Used to fill pinned host checkpoints quickly (generate in HBM, one D2H)
// instead of spending minutes on the CPU; the CPU restatement in
// oracle/cpu_oracle.c checks it.
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace tg {
namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ u64 splitmix(u64 z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void synth_kernel(u64 seed, u64 begin, u64 len, std::uint8_t* __restrict__ dst) {
    const u64 w0 = begin >> 3, w1 = (begin + len + 7) >> 3;
    const bool aligned = ((reinterpret_cast<std::uintptr_t>(dst) - begin) & 7) == 0;
    for (u64 w = w0 + static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; w < w1;
         w += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 v = splitmix(seed ^ (w * 0x9E3779B97F4A7C15ULL));
        const u64 a = w << 3;
        if (aligned && a >= begin && a + 8 <= begin + len) {
            *reinterpret_cast<u64*>(dst + (a - begin)) = v;
            continue;
        }
        for (int b = 0; b < 8; ++b) {
            const u64 pos = a + b;
            if (pos >= begin && pos < begin + len) dst[pos - begin] = static_cast<std::uint8_t>(v >> (8 * b));
        }
    }
}

}  // namespace

void synth_launch(u64 hi, u64 lo, u64 begin, u64 len, std::uint8_t* dst, cudaStream_t s) {
    if (len == 0) return;
    const u64 seed = hi ^ ((lo << 17) | (lo >> 47));
    synth_kernel<<<148 * 8, 256, 0, s>>>(seed, begin, len, dst);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

std::atomic<std::uint64_t> g_kernel_launches{0};

}  // namespace tg
