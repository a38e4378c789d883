#include "regions.hpp"

namespace tg {

PoolMap::PoolMap(u64 pool_size) : pool_(pool_size) {
    if (pool_size > 0) put(Extent{0, pool_size, Kind::Free, {}, 0, 1});
}

void PoolMap::put(const Extent& e) {
    map_.emplace(e.off, e);
    expanded_count_ += e.kind == Kind::Kv ? e.nblocks : 1;
    if (e.kind == Kind::Free) {
        free_.insert({e.len, e.off});
        free_bytes_ += e.len;
    }
}

void PoolMap::drop(It it) {
    const Extent& e = it->second;
    expanded_count_ -= e.kind == Kind::Kv ? e.nblocks : 1;
    if (e.kind == Kind::Free) {
        free_.erase({e.len, e.off});
        free_bytes_ -= e.len;
    }
    map_.erase(it);
}

PoolMap::It PoolMap::isolate(u64 off) {
    auto it = map_.upper_bound(off);
    if (it == map_.begin()) return map_.end();
    --it;
    Extent e = it->second;
    if (e.off == off && (e.kind != Kind::Kv || e.nblocks == 1)) return it;
    if (e.kind != Kind::Kv) return e.off == off ? it : map_.end();
    const u64 blk = e.block_len();
    if ((off - e.off) % blk != 0 || off >= e.end()) return map_.end();
    const u64 idx = (off - e.off) / blk;
    drop(it);
    if (idx > 0) put(Extent{e.off, idx * blk, Kind::Kv, {}, e.block0, idx});
    put(Extent{off, blk, Kind::Kv, {}, e.block0 + idx, 1});
    const u64 rest = e.nblocks - idx - 1;
    if (rest > 0) put(Extent{off + blk, rest * blk, Kind::Kv, {}, e.block0 + idx + 1, rest});
    return map_.find(off);
}

Res<u64> PoolMap::carve(u64 off, u64 len, Kind kind, Key tensor, u64 block0, u64 nblocks) {
    if (len == 0 || off > pool_ || len > pool_ - off) return Err::InvalidArgument;
    auto it = map_.upper_bound(off);
    if (it == map_.begin()) return Err::InvalidArgument;
    --it;
    const Extent host = it->second;
    if (host.kind != Kind::Free || off + len > host.end()) return Err::DestinationOccupied;
    drop(it);
    if (off > host.off) put(Extent{host.off, off - host.off, Kind::Free, {}, 0, 1});
    put(Extent{off, len, kind, tensor, block0, kind == Kind::Kv ? nblocks : 1});
    if (host.end() > off + len) put(Extent{off + len, host.end() - (off + len), Kind::Free, {}, 0, 1});
    return off;
}

Res<u64> PoolMap::carve_best_fit(u64 len, Kind kind, Key tensor, u64 block0) {
    if (len == 0) return Err::InvalidArgument;
    auto f = free_.lower_bound({len, 0});
    if (f == free_.end()) return Err::InsufficientMemory;
    return carve(f->second, len, kind, tensor, block0, 1);
}

St PoolMap::release_extent(u64 off) {
    auto it = map_.find(off);
    if (it == map_.end() || it->second.kind == Kind::Free) return Err::NotFound;
    u64 lo = it->second.off, hi = it->second.end();
    drop(it);
    auto prev = map_.lower_bound(lo);
    if (prev != map_.begin()) {
        --prev;
        if (prev->second.kind == Kind::Free && prev->second.end() == lo) {
            lo = prev->second.off;
            drop(prev);
        }
    }
    auto next = map_.find(hi);
    if (next != map_.end() && next->second.kind == Kind::Free) {
        hi = next->second.end();
        drop(next);
    }
    put(Extent{lo, hi - lo, Kind::Free, {}, 0, 1});
    return ok();
}

St PoolMap::release(u64 off) {
    auto it = isolate(off);
    if (it == map_.end() || it->second.kind == Kind::Free) return Err::NotFound;
    return release_extent(off);
}

St PoolMap::move(u64 from, u64 to) {
    auto it = isolate(from);
    if (it == map_.end() || it->second.kind == Kind::Free) return Err::NotFound;
    const Extent r = it->second;
    if (to == from) return Err::OverlapMove;
    if (to < from + r.len && from < to + r.len) return Err::OverlapMove;
    auto placed = carve(to, r.len, r.kind, r.tensor, r.block0, r.nblocks);
    if (!placed) return placed.error();
    return release_extent(from);
}

bool PoolMap::is_free_range(u64 off, u64 len) const {
    if (off >= pool_) return false;
    auto it = map_.upper_bound(off);
    --it;
    return it->second.kind == Kind::Free && off + len <= it->second.end();
}

bool PoolMap::region_at(u64 off, Region* out) const {
    auto it = map_.upper_bound(off);
    if (it == map_.begin()) return false;
    --it;
    const Extent& e = it->second;
    if (e.kind == Kind::Kv) {
        const u64 blk = e.block_len();
        if (off >= e.end() || (off - e.off) % blk != 0) return false;
        if (out) *out = Region{off, blk, Kind::Kv, {}, e.block0 + (off - e.off) / blk};
        return true;
    }
    if (e.off != off) return false;
    if (out) *out = Region{e.off, e.len, e.kind, e.tensor, 0};
    return true;
}

std::vector<Region> PoolMap::expanded() const {
    std::vector<Region> out;
    out.reserve(expanded_count_);
    for (const auto& [o, e] : map_) {
        if (e.kind != Kind::Kv) {
            out.push_back(Region{e.off, e.len, e.kind, e.tensor, 0});
            continue;
        }
        const u64 blk = e.block_len();
        for (u64 i = 0; i < e.nblocks; ++i) out.push_back(Region{e.off + i * blk, blk, Kind::Kv, {}, e.block0 + i});
    }
    return out;
}

PoolMap PoolMap::from_regions(u64 pool_size, const std::vector<Region>& regs) {
    PoolMap m;
    m.pool_ = pool_size;
    for (const Region& r : regs) m.put(Extent{r.off, r.len, r.kind, r.tensor, r.block, 1});
    return m;
}

St PoolMap::validate() const {
    u64 cursor = 0, free_sum = 0, count = 0;
    bool prev_free = false;
    std::set<std::pair<u64, u64>> seen;
    for (const auto& [o, e] : map_) {
        if (o != cursor || e.off != o || e.len == 0) return Err::Infeasible;
        const bool is_free = e.kind == Kind::Free;
        if (is_free && prev_free) return Err::Infeasible;
        if (e.kind == Kind::Kv && (e.nblocks == 0 || e.len % e.nblocks != 0)) return Err::Infeasible;
        if (is_free) {
            seen.insert({e.len, e.off});
            free_sum += e.len;
        }
        count += e.kind == Kind::Kv ? e.nblocks : 1;
        prev_free = is_free;
        cursor += e.len;
    }
    if (cursor != pool_ || seen != free_ || free_sum != free_bytes_ || count != expanded_count_)
        return Err::Infeasible;
    return ok();
}

}  // namespace tg
