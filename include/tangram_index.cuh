/* Device-side probe of the pool's tensor index (tg_pool_device_index).
 * Header-only, for consumer kernels: resolves a TensorId to its arena offset
 * without a host round trip. */
#pragma once

#include "tangram.h"

#ifdef __CUDACC__
/* Returns the slot holding (hi, lo), or nullptr.  Linear probing from
 * lo & (capacity - 1); an unoccupied slot ends the probe. */
__device__ __forceinline__ const tg_index_slot* tg_index_find(const tg_index_slot* table, uint64_t capacity,
                                                              uint64_t hi, uint64_t lo) {
    const uint64_t mask = capacity - 1;
    for (uint64_t i = lo & mask, n = 0; n < capacity; i = (i + 1) & mask, ++n) {
        const tg_index_slot* s = table + i;
        if (!(s->flags & TG_INDEX_OCCUPIED)) return nullptr;
        if (s->key_lo == lo && s->key_hi == hi) return s;
    }
    return nullptr;
}
#endif
