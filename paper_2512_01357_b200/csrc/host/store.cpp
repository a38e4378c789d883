#include "store.hpp"

#include <algorithm>
#include <atomic>
#include <cstdio>

#include "json_out.hpp"

namespace tg {

void Store::lookup(const ModelDesc& m, std::vector<u32>* hits, std::vector<u32>* misses) const {
    for (u32 i = 0; i < m.tensors.size(); ++i) (tensors_.count(m.tensors[i].id) ? hits : misses)->push_back(i);
}

u64 Store::reuse_size(const ModelDesc& m) const {
    u64 s = 0;
    for (const auto& t : m.tensors)
        if (auto it = tensors_.find(t.id); it != tensors_.end()) s += it->second.size;
    return s;
}

std::vector<Candidate> Store::candidates(const StatsView& stats, const std::string& exclude) const {
    std::vector<Candidate> out;
    out.reserve(tensors_.size());
    for (const auto& [k, e] : tensors_) {
        if (e.pinned || e.model == exclude) continue;
        const double p = stats.miss_probability(e.model);
        const double bw = stats.load_bandwidth_or(e.model, gpu_.pcie_bw);
        out.push_back(Candidate{k, e.size, eviction_cost(e.size, p, bw, alpha_of(e.model)), e.last_access, e.model});
    }
    std::sort(out.begin(), out.end(), [](const Candidate& a, const Candidate& b) { return a.tensor < b.tensor; });
    return out;
}

Res<LoadDecision> Store::decide(const ModelDesc& m, const StatsView& stats, const LoadOptions& opt) {
    set_alpha(m.model_id, m.alpha);
    u64 pinned_self = 0;  // an already-active model reloading itself stays idempotent
    for (const auto& t : m.tensors)
        if (auto it = tensors_.find(t.id); it != tensors_.end() && it->second.pinned) pinned_self += it->second.size;
    const u64 pinned_other = pinned_bytes() - pinned_self;
    if (m.total_size > gpu_.pool_size || m.total_size > gpu_.pool_size - pinned_other)
        return Err::InsufficientMemory;

    LoadDecision d;
    lookup(m, &d.hits, &d.misses);
    for (u32 i : d.hits) d.hit_keys.push_back(m.tensors[i].id);
    for (u32 i : d.misses) {
        d.miss_desc.push_back(m.tensors[i]);
        d.bytes_transferred += m.tensors[i].size;
    }
    if (d.misses.empty()) return d;

    PlanInput in;
    in.pool = &map_;
    in.tensors = &d.miss_desc;
    in.candidates = candidates(stats, m.model_id);
    if (opt.random_eviction && opt.rng) {
        auto& c = in.candidates;
        for (std::size_t i = c.size(); i > 1; --i) std::swap(c[i - 1], c[opt.rng->uniform_below(i)]);
        in.keep_candidate_order = true;
    }
    for (const auto& [k, e] : tensors_)
        if (e.pinned) in.immovable.insert(k);
    in.strictness = opt.strictness;
    in.merge = opt.merge;
    auto plan = make_plan(in, &d.after);
    if (!plan) return plan.error();
    d.plan = std::move(plan.value());
    return d;
}

void Store::touch() {
    static std::atomic<u64> next{0};
    epoch_ = ++next;
}

void Store::commit(const ModelDesc& m, LoadDecision& d, double clock) {
    touch();
    if (!d.misses.empty()) {
        for (const auto& ev : d.plan.evictions) {
            tensors_.erase(ev.tensor);
            ++evictions_total_;
        }
        for (const auto& mv : d.plan.relocations) {
            tensors_.at(mv.tensor).off = mv.to;
            merged_total_ += mv.size;
        }
        for (const auto& pl : d.plan.placements) {
            const TensorDesc& t = d.miss_desc[pl.tensor];
            Entry e;
            e.off = pl.off;
            e.size = t.size;
            e.model = t.model_id;
            e.last_access = clock;
            tensors_.emplace(t.id, std::move(e));
        }
        map_ = std::move(d.after);
    }
    for (const auto& t : m.tensors) {
        Entry& e = tensors_.at(t.id);
        e.last_access = clock;
        if (!e.pinned) {
            e.pinned = true;
            pinned_tensor_bytes_ += e.size;
        }
    }
    transferred_total_ += d.bytes_transferred;
}

void Store::end_instance(const std::string& model) {
    touch();
    for (auto& [k, e] : tensors_)
        if (e.model == model && e.pinned) {
            e.pinned = false;
            pinned_tensor_bytes_ -= e.size;
        }
}

St Store::evict_tensor(const Key& k) {
    auto it = tensors_.find(k);
    if (it == tensors_.end()) return Err::NotFound;
    if (it->second.pinned) return Err::Pinned;
    map_.release(it->second.off);
    tensors_.erase(it);
    ++evictions_total_;
    touch();
    return ok();
}

void Store::evict_model(const std::string& model) {
    touch();
    std::vector<Key> ids;
    for (const auto& [k, e] : tensors_)
        if (e.model == model) ids.push_back(k);
    std::sort(ids.begin(), ids.end());
    for (const Key& k : ids) {
        Entry& e = tensors_.at(k);
        if (e.pinned) {
            e.pinned = false;
            pinned_tensor_bytes_ -= e.size;
        }
        evict_tensor(k);
    }
}

St Store::move_tensor(const Key& k, u64 to) {
    auto it = tensors_.find(k);
    if (it == tensors_.end()) return Err::NotFound;
    if (it->second.pinned) return Err::Pinned;
    auto st = map_.move(it->second.off, to);
    if (!st) return st;
    it->second.off = to;
    merged_total_ += it->second.size;
    touch();
    return ok();
}

Res<u64> Store::alloc_kv_region(u64 size, u64 block_id) {
    auto r = map_.carve_best_fit(size, Kind::Kv, {}, block_id);
    if (r) kv_bytes_ += size;
    return r;
}

St Store::free_kv_region(u64 off) {
    Region r;
    if (!map_.region_at(off, &r) || r.kind != Kind::Kv) return Err::NotFound;
    kv_bytes_ -= r.len;
    return map_.release(off);
}

void Store::carve_kv_run(u64 off, u64 nblocks, u64 block_len, u64 first_block) {
    if (!map_.carve(off, nblocks * block_len, Kind::Kv, {}, first_block, nblocks))
        throw DeviceError(106, "kv: run [" + std::to_string(off) + ", +" + std::to_string(nblocks * block_len) +
                                   ") is not free in this pool");
    kv_bytes_ += nblocks * block_len;
}

void Store::release_kv_range(u64 off, u64 bytes) {
    std::vector<std::pair<u64, u64>> kv;
    const auto& ex = map_.extents();
    for (auto it = ex.lower_bound(off); it != ex.end() && it->first < off + bytes; ++it)
        if (it->second.kind == Kind::Kv) kv.push_back({it->first, it->second.len});
    for (const auto& [o, len] : kv) {
        map_.release_extent(o);
        kv_bytes_ -= len;
    }
}

St Store::validate() const {
    if (auto st = map_.validate(); !st) return st;
    u64 n_tensor_regions = 0, free = 0, tensor_bytes = 0, kv = 0;
    for (const auto& [o, e] : map_.extents()) {
        switch (e.kind) {
            case Kind::Free: free += e.len; break;
            case Kind::Kv: kv += e.len; break;
            case Kind::Tensor: {
                ++n_tensor_regions;
                tensor_bytes += e.len;
                auto it = tensors_.find(e.tensor);
                if (it == tensors_.end() || it->second.off != e.off || it->second.size != e.len)
                    return Err::Infeasible;
                break;
            }
        }
    }
    if (n_tensor_regions != tensors_.size()) return Err::Infeasible;
    if (free + tensor_bytes + kv != gpu_.pool_size) return Err::Infeasible;
    if (kv != kv_bytes_) return Err::Infeasible;
    u64 pinned = 0;
    for (const auto& [k, e] : tensors_)
        if (e.pinned) pinned += e.size;
    if (pinned != pinned_tensor_bytes_) return Err::Infeasible;
    return ok();
}

// Same document as ReuseStore::dump (reuse_store.hpp:270-308); keys are
// emitted in sorted order like nlohmann::json objects.
std::string Store::dump_json() const {
    JsonOut j;
    j.raw("{\"format_version\":1,\"gpu_id\":");
    j.str(gpu_.gpu_id);
    j.raw(",\"pool_size\":");
    j.num(gpu_.pool_size);
    j.raw(",\"regions\":[");
    bool first = true;
    for (const Region& r : map_.expanded()) {
        if (!first) j.raw(",");
        first = false;
        j.raw("{");
        if (r.kind == Kind::Kv) {
            j.raw("\"block\":");
            j.num(r.block);
            j.raw(",");
        } else if (r.kind == Kind::Tensor) {
            j.raw("\"model\":");
            j.str(tensors_.at(r.tensor).model);
            j.raw(",");
        }
        j.raw("\"offset\":");
        j.num(r.off);
        j.raw(",\"size\":");
        j.num(r.len);
        j.raw(",\"state\":");
        j.str(r.kind == Kind::Free ? "free" : r.kind == Kind::Tensor ? "tensor" : "kv_block");
        if (r.kind == Kind::Tensor) {
            j.raw(",\"tensor\":");
            j.str(r.tensor.hex());
        }
        j.raw("}");
    }
    j.raw("],\"tensor_map\":[");
    std::vector<std::pair<u64, Key>> order;
    order.reserve(tensors_.size());
    for (const auto& [k, e] : tensors_) order.push_back({e.off, k});
    std::sort(order.begin(), order.end(), [](const auto& a, const auto& b) {
        return a.first != b.first ? a.first < b.first : a.second < b.second;
    });
    first = true;
    for (const auto& [off, k] : order) {
        const Entry& e = tensors_.at(k);
        if (!first) j.raw(",");
        first = false;
        j.raw("{\"last_access\":");
        j.dbl(e.last_access);
        j.raw(",\"model\":");
        j.str(e.model);
        j.raw(",\"offset\":");
        j.num(e.off);
        j.raw(",\"pinned\":");
        j.raw(e.pinned ? "true" : "false");
        j.raw(",\"size\":");
        j.num(e.size);
        j.raw(",\"tensor\":");
        j.str(k.hex());
        j.raw("}");
    }
    j.raw("]}");
    return j.take();
}

}  // namespace tg
