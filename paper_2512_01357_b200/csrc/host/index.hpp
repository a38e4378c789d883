// Tensor index image for the device: the store's tensor map
// (reuse_store.hpp:338, TensorEntry :26-32) as an open-addressing table.
#pragma once

#include <vector>

#include "store.hpp"

namespace tg {

// Layout-identical to tg_index_slot (include/tangram.h).
struct IndexSlot {
    u64 key_hi, key_lo;
    u64 off, size;
    double last_access;
    u64 model;
    u32 flags;
    u32 reserved0;
    u64 reserved1;
};
static_assert(sizeof(IndexSlot) == 64, "one 64-byte slot per probe");
constexpr u32 kIndexOccupied = 1u, kIndexPinned = 2u;

// Capacity = max(1024, next power of two >= 2 x entries); entries are inserted
// in offset order, so the image is a pure function of the store's state.
std::vector<IndexSlot> build_index_image(const Store& store);

}  // namespace tg
