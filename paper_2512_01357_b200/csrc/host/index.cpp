#include "index.hpp"

#include <algorithm>

namespace tg {

std::vector<IndexSlot> build_index_image(const Store& store) {
    const auto& map = store.tensors();
    u64 cap = 1024;
    while (cap < 2 * static_cast<u64>(map.size())) cap <<= 1;
    std::vector<const std::pair<const Key, Entry>*> order;
    order.reserve(map.size());
    for (const auto& kv : map) order.push_back(&kv);
    std::sort(order.begin(), order.end(), [](auto* a, auto* b) { return a->second.off < b->second.off; });
    std::vector<IndexSlot> t(cap, IndexSlot{});
    for (const auto* kv : order) {
        const Key& k = kv->first;
        const Entry& e = kv->second;
        u64 i = k.lo & (cap - 1);
        while (t[i].flags & kIndexOccupied) i = (i + 1) & (cap - 1);
        t[i] = IndexSlot{k.hi, k.lo, e.off, e.size, e.last_access,
                         murmur3_x64_128(e.model.data(), e.model.size(), 0).lo,
                         kIndexOccupied | (e.pinned ? kIndexPinned : 0u), 0, 0};
    }
    return t;
}

}  // namespace tg
