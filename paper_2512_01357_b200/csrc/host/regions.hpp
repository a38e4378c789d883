// Address-ordered extent map of one device arena (the "unified pool").
//
// Semantics are those of the reference RegionList (region_pool.hpp:41-222):
// extents tile [0, pool) exactly, free extents are eagerly coalesced, a free
// index ordered by (size, offset) serves best-fit.  Two representation
// changes make the B200 control plane cheaper without changing any decision:
//   * KV blocks carved back-to-back by one allocation batch are stored as a
//     single "block run" extent (n equal blocks with consecutive block ids);
//     the reference stores one region per block.  Every query that could
//     observe the difference (region dumps, counts, find/release/move of one
//     block) expands or splits the run on demand, so the observable region
//     chain is identical.
//   * The free byte total is maintained incrementally (region_pool.hpp:52-56
//     recomputes it per call; the planner's Stage-1 loop calls it per
//     eviction, packing.hpp:348).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <utility>
#include <vector>

#include "core.hpp"

namespace tg {

enum class Kind : std::uint8_t { Free = 0, Tensor = 1, Kv = 2 };

struct Extent {
    u64 off = 0;
    u64 len = 0;  // bytes of the whole extent
    Kind kind = Kind::Free;
    Key tensor;        // Kind::Tensor
    u64 block0 = 0;    // Kind::Kv: block id of the first block
    u64 nblocks = 1;   // Kind::Kv: equal blocks in this run
    u64 end() const { return off + len; }
    u64 block_len() const { return len / nblocks; }
};

// One region of the expanded (reference-visible) chain.
struct Region {
    u64 off = 0;
    u64 len = 0;
    Kind kind = Kind::Free;
    Key tensor;
    u64 block = 0;
};

class PoolMap {
public:
    PoolMap() = default;
    explicit PoolMap(u64 pool_size);

    u64 pool_size() const { return pool_; }
    u64 free_total() const { return free_bytes_; }
    u64 largest_free() const { return free_.empty() ? 0 : free_.rbegin()->first; }
    u64 region_count() const { return expanded_count_; }
    std::size_t extent_count() const { return map_.size(); }

    // allocate_at (region_pool.hpp:95-113).  For Kind::Kv, `nblocks` equal
    // blocks with ids block0.. are carved as one run.
    Res<u64> carve(u64 off, u64 len, Kind kind, Key tensor, u64 block0, u64 nblocks = 1);
    // allocate_best_fit (region_pool.hpp:117-123).
    Res<u64> carve_best_fit(u64 len, Kind kind, Key tensor, u64 block0);
    // release + eager coalescing (region_pool.hpp:126-152); `off` must start
    // a (possibly run-embedded) allocated region.
    St release(u64 off);
    // Release a whole extent (all blocks of a KV run at once).  Same final
    // state as releasing its blocks one by one.
    St release_extent(u64 off);
    // move (region_pool.hpp:157-167): disjoint destination inside free space.
    St move(u64 from, u64 to);

    bool is_free_range(u64 off, u64 len) const;
    // Region starting exactly at `off` (expanded view), if any.
    bool region_at(u64 off, Region* out) const;

    // Maximal free runs in address order (region_pool.hpp:66-71).
    template <typename F>
    void for_each_free(F&& f) const {
        for (const auto& [o, e] : map_)
            if (e.kind == Kind::Free) f(e);
    }
    // Free runs intersecting [lo, hi) in address order.
    template <typename F>
    void for_each_free_in(u64 lo, u64 hi, F&& f) const {
        auto it = map_.upper_bound(lo);
        if (it != map_.begin()) --it;
        for (; it != map_.end() && it->first < hi; ++it)
            if (it->second.kind == Kind::Free) f(it->second);
    }
    // Free runs of at least `min_len` bytes in ascending (size, offset) order.
    template <typename F>
    void for_each_free_by_size(u64 min_len, F&& f) const {
        for (auto it = free_.lower_bound({min_len, 0}); it != free_.end(); ++it) f(it->second, it->first);
    }
    // Smallest free run of at least `len` bytes, lowest offset on ties.
    bool best_fit(u64 len, u64* off, u64* flen) const {
        auto it = free_.lower_bound({len, 0});
        if (it == free_.end()) return false;
        *off = it->second;
        *flen = it->first;
        return true;
    }
    const std::map<u64, Extent>& extents() const { return map_; }

    std::vector<Region> expanded() const;
    St validate() const;
    // Rebuild from an address-ordered tiling (RegionList::from_snapshot,
    // region_pool.hpp:176-184); no coalescing is applied.
    static PoolMap from_regions(u64 pool_size, const std::vector<Region>& regs);

private:
    using It = std::map<u64, Extent>::iterator;
    void put(const Extent& e);
    void drop(It it);
    // If `off` is a block boundary inside a KV run, split the run so that a
    // single-block extent starts at `off`.  Returns map_.end() when `off`
    // does not start a region.
    It isolate(u64 off);

    u64 pool_ = 0;
    u64 free_bytes_ = 0;
    u64 expanded_count_ = 0;
    std::map<u64, Extent> map_;
    std::set<std::pair<u64, u64>> free_;  // (len, off)
};

}  // namespace tg
