// K6: batch lookup through the device tensor index with the
// consumer-side probe of include/tangram_index.cuh.
#include "../../../include/tangram_index.cuh"
#include "kernels.hpp"

namespace tg {
namespace {

__global__ void index_lookup_kernel(const tg_index_slot* __restrict__ table, std::uint64_t capacity,
                                    const std::uint64_t* __restrict__ keys, std::uint32_t n,
                                    std::uint64_t* __restrict__ out) {
    const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const tg_index_slot* s = tg_index_find(table, capacity, keys[2 * i], keys[2 * i + 1]);
    out[3 * i] = s ? s->offset : ~std::uint64_t{0};
    out[3 * i + 1] = s ? s->size : 0;
    out[3 * i + 2] = s ? (1ull | (static_cast<std::uint64_t>(s->flags) << 32)) : 0;
}

}  // namespace

void index_lookup_launch(const void* table, std::uint64_t capacity, const std::uint64_t* d_keys, std::uint32_t n,
                         std::uint64_t* d_out, cudaStream_t s) {
    if (!n) return;
    index_lookup_kernel<<<(n + 127) / 128, 128, 0, s>>>(static_cast<const tg_index_slot*>(table), capacity, d_keys,
                                                        n, d_out);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace tg
