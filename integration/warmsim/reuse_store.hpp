// Drop-in binding: warmsim::ReuseStore backed by the B200 pool (libtangram.so).
//
// Put this directory before the reference's include directory
// (-I<repo>/integration -I<reference>/proj/include) and the unmodified
// reference code (simulator.hpp, kv_engine users, ...) compiles against the
// B200 implementation: every "warmsim/reuse_store.hpp" include resolves here
// while types.hpp / model.hpp / packing.hpp / region_pool.hpp / rng.hpp stay
// the reference's.  Declarations mirror reuse_store.hpp:26-345; bodies are
// thin calls through include/tangram.h.
//
// Device selection (env TANGRAM_DEVICE): "auto" (default) maps gpu_id "gpuN"
// to CUDA device N when it exists, otherwise the pool is control-plane only;
// "none" forces control-plane-only pools; an integer pins every pool to that
// device.  Value semantics as in the reference (reuse_store.hpp:336-344),
// copy-on-write over one device pool:
//  * a copy shares the pool until either side mutates;
//  * the store that owns the device (the one that created it, or whoever
//    holds it once the owner is gone) keeps it: when it mutates while shared,
//    the sharers are first switched to a control-plane snapshot of the state
//    they saw (tg_pool_clone); when a non-owner mutates while shared, it
//    detaches to such a snapshot itself (bytes never travel);
//  * assigning a store into one holding a device (the reference's rollback
//    idiom, kv_engine.hpp:146-158: `store = std::move(store_copy)`) keeps the
//    target's arena and adopts the metadata (tg_pool_assign: tensors the
//    arena does not hold at their adopted offsets become suspect and are
//    re-sent on their next reuse).
// So `ReuseStore backup = s; s.load_model(...)` leaves backup the old state
// and s on the GPU, and containers that copy stores on reallocation keep the
// device with the surviving copy.
//
// Trace replay at full speed (§8(f) row 1):
//  * TANGRAM_ASYNC_LOADS=1: loads return once the decision is committed
//    (TG_LOAD_ASYNC) — the simulator only reads the decision — and each
//    pool's data plane finishes in the background until that pool's next
//    operation, so loads on different GPUs overlap;
//  * TANGRAM_PEER_SCHEDULE=<GB/s> (warmsim/scheduler.hpp): every device pool
//    is an NVLink peer of every other and loads with TG_LOAD_PEER, misses
//    resident on another pool are pulled from it instead of over PCIe.
#pragma once

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "json.hpp"
#include "tangram.h"
#include "warmsim/model.hpp"
#include "warmsim/packing.hpp"
#include "warmsim/region_pool.hpp"
#include "warmsim/rng.hpp"
#include "warmsim/scheduler.hpp"  // the binding's (live device pools, peer term)
#include "warmsim/types.hpp"

namespace warmsim {

struct TensorEntry {
    Bytes offset = 0;
    Bytes size = 0;
    std::string model_id;
    Seconds last_access = 0;
    bool pinned = false;
};

struct LoadOutcome {
    std::vector<TensorId> hit_tensors;
    std::vector<TensorSpec> missed_tensors;
    Bytes bytes_transferred = 0;
    Bytes bytes_merged = 0;
    Seconds eviction_cost_total = 0;
    AllocationPlan plan;
    tg_load_outcome device{};  // measured data plane of this load
};

struct LoadPolicy {
    MergePolicy merge = MergePolicy::PartitionedGain;
    PackingStrictness strictness = PackingStrictness::Functional;
    bool random_eviction = false;
    Rng* rng = nullptr;
};

namespace tgb {

inline tg_tensor_id cid(const TensorId& t) { return tg_tensor_id{t.hi, t.lo}; }
inline TensorId wid(const tg_tensor_id& t) { return TensorId{t.hi, t.lo}; }

[[noreturn]] inline void fail(int rc, const char* where) {
    throw std::runtime_error(std::string("tangram: ") + where + ": " + tg_error_string(rc) + " " +
                             tg_last_error_detail());
}
// 0 → ok; 1..10 → the reference's Error; anything else is a runtime failure.
inline int domain(int rc, const char* where) {
    if (rc >= 100) fail(rc, where);
    return rc;
}

// ModelSpec → tg_model_spec (views into the spec's own strings).
struct ModelView {
    std::vector<tg_tensor_spec> t;
    tg_model_spec spec{};
    explicit ModelView(const ModelSpec& m) {
        t.reserve(m.tensors.size());
        for (const auto& x : m.tensors) t.push_back(tg_tensor_spec{cid(x.id), x.name.c_str(), x.size, x.model_id.c_str()});
        spec = tg_model_spec{m.model_id.c_str(), t.data(), static_cast<uint32_t>(t.size()), m.total_size,
                             m.latency_sensitivity, m.location == ModelLocation::ModelStore ? 1 : 0,
                             m.bytes_per_token};
    }
};

// The caller's ModelStatsTable, read through callbacks.
struct StatsHandle {
    tg_stats* h = nullptr;
    explicit StatsHandle(const ModelStatsTable& s) {
        tg_stats_create_external(
            const_cast<ModelStatsTable*>(&s),
            [](void* c, const char* m) { return static_cast<const ModelStatsTable*>(c)->miss_probability(m); },
            [](void* c, const char* m, double f) {
                return static_cast<const ModelStatsTable*>(c)->load_bandwidth_or(m, f);
            },
            &h);
    }
    ~StatsHandle() { tg_stats_destroy(h); }
    StatsHandle(const StatsHandle&) = delete;
    StatsHandle& operator=(const StatsHandle&) = delete;
};

inline bool async_loads() {
    static const bool on = [] {
        const char* e = std::getenv("TANGRAM_ASYNC_LOADS");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

inline int pick_device(const std::string& gpu_id) {
    const char* env = std::getenv("TANGRAM_DEVICE");
    const std::string mode = env ? env : "auto";
    if (mode == "none") return TG_POOL_NO_DEVICE;
    int n = 0;
    tg_device_count(&n);
    if (mode != "auto") return std::atoi(mode.c_str());
    std::size_t i = gpu_id.size();
    while (i > 0 && gpu_id[i - 1] >= '0' && gpu_id[i - 1] <= '9') --i;
    if (i == gpu_id.size()) return TG_POOL_NO_DEVICE;
    const int d = std::atoi(gpu_id.c_str() + i);
    return d < n ? d : TG_POOL_NO_DEVICE;
}

// Data-plane totals of every pool, collected when the pool is released, so a
// driver can report what the bytes cost after the reference code is done.
inline std::vector<std::pair<std::string, tg_pool_info>>& finished_pools() {
    static std::vector<std::pair<std::string, tg_pool_info>> v;
    return v;
}

struct PoolDeleter {
    std::string gpu_id;
    bool record = true;  // snapshots (control-plane clones) are not reported
    void operator()(tg_pool* p) const {
        auto& live = tgs::live_pools();
        for (auto it = live.begin(); it != live.end(); ++it)
            if (it->second == p) {
                live.erase(it);
                break;
            }
        if (record) {
            tg_pool_sync(p, nullptr);  // an asynchronous load still in flight lands first
            tg_pool_info i{};
            tg_pool_info_get(p, &i);
            finished_pools().push_back({gpu_id, i});
        }
        tg_pool_destroy(p);
    }
};

// One pool shared by a store and its unmutated copies; `owner` is the store
// that keeps the pool when a sharer mutates (null: whoever mutates next).
struct Box {
    std::shared_ptr<tg_pool> pool;
    const void* owner = nullptr;
};

}  // namespace tgb

class ReuseStore {
public:
    ReuseStore() = default;

    explicit ReuseStore(GpuSpec spec) : gpu_(std::move(spec)) {
        tg_gpu_spec g{gpu_.gpu_id.c_str(), gpu_.pool_size, gpu_.pcie_bandwidth, gpu_.intra_copy_bandwidth,
                      gpu_.store_bandwidth};
        tg_pool* p = nullptr;
        if (int rc = tg_pool_create(&g, tgb::pick_device(gpu_.gpu_id), &p)) tgb::fail(rc, "tg_pool_create");
        box_ = std::make_shared<tgb::Box>(tgb::Box{std::shared_ptr<tg_pool>(p, tgb::PoolDeleter{gpu_.gpu_id}), this});
        tg_pool_info i{};
        tg_pool_info_get(p, &i);
        if (i.device >= 0 && tgs::peer_bandwidth() > 0) {  // every device pool peers with every other
            for (const auto& [gid, q] : tgs::live_pools()) {
                tg_pool_add_peer(p, q);
                tg_pool_add_peer(q, p);
            }
            tgs::live_pools()[gpu_.gpu_id] = p;
        }
    }

    ReuseStore(const ReuseStore& o) : gpu_(o.gpu_), box_(o.box_) {}
    ReuseStore(ReuseStore&& o) noexcept : gpu_(std::move(o.gpu_)), box_(std::move(o.box_)) {
        if (box_ && box_->owner == &o) box_->owner = this;
    }
    ~ReuseStore() {
        if (box_ && box_->owner == this) box_->owner = nullptr;  // a sharer may claim the device
    }
    ReuseStore& operator=(const ReuseStore& o) {
        if (this == &o || (box_ && box_ == o.box_)) return *this;
        if (!box_ || !o.box_) return *this = ReuseStore(o);
        adopt(o);
        return *this;
    }
    ReuseStore& operator=(ReuseStore&& o) noexcept(false) {
        if (this == &o || (box_ && box_ == o.box_)) return *this;
        if (!box_ || !o.box_) {  // nothing to keep: take the other store whole
            if (box_ && box_->owner == this) box_->owner = nullptr;
            gpu_ = std::move(o.gpu_);
            box_ = std::move(o.box_);
            if (box_ && box_->owner == &o) box_->owner = this;
            map_epoch_ = ~std::uint64_t{0};
            return *this;
        }
        adopt(o);
        return *this;
    }

    // The pool, for reads.
    tg_pool* handle() const { return box_ ? box_->pool.get() : nullptr; }
    // The pool, for a mutation: resolves sharing first (copy-on-write).
    tg_pool* mutable_handle() {
        if (!box_) return nullptr;
        if (box_->owner == nullptr) box_->owner = this;  // the owner is gone: this store keeps the device
        if (box_.use_count() > 1) {
            auto snap = std::make_shared<tgb::Box>(tgb::Box{clone_of(handle()), nullptr});
            if (box_->owner == this) {
                // the sharers keep the state they saw; this store keeps the device
                std::swap(box_->pool, snap->pool);
                box_.swap(snap);
                box_->owner = this;
                snap->owner = nullptr;
            } else {
                box_ = std::move(snap);  // detach to a snapshot of our own
                box_->owner = this;
            }
        }
        map_epoch_ = ~std::uint64_t{0};
        return box_->pool.get();
    }
    const GpuSpec& gpu() const { return gpu_; }
    Bytes pool_size() const { return gpu_.pool_size; }
    Bytes free_bytes() const { return info().free_bytes; }
    Bytes kv_bytes() const { return info().kv_bytes; }
    Bytes pinned_tensor_bytes() const { return info().pinned_tensor_bytes; }
    Bytes pinned_bytes() const { return info().pinned_bytes; }
    Bytes reusable_bytes() const { return info().reusable_bytes; }
    Bytes bytes_merged_total() const { return info().bytes_merged_total; }
    Bytes bytes_transferred_total() const { return info().bytes_transferred_total; }
    std::uint64_t evictions_total() const { return info().evictions_total; }

    // Rebuilt from the pool's tensor list only when its epoch changed.
    const std::unordered_map<TensorId, TensorEntry, TensorIdHash>& tensor_map() const {
        const tg_pool_info i = info();
        if (i.epoch == map_epoch_) return tensors_cache_;
        std::uint64_t n = 0;
        tg_pool_tensors(handle(), nullptr, 0, &n);
        std::vector<tg_tensor_entry> buf(n);
        if (int rc = tg_pool_tensors(handle(), buf.data(), n, &n)) tgb::fail(rc, "tg_pool_tensors");
        tensors_cache_.clear();
        for (const auto& e : buf)
            tensors_cache_[tgb::wid(e.id)] = TensorEntry{e.offset, e.size, e.model_id, e.last_access, e.pinned != 0};
        map_epoch_ = i.epoch;
        return tensors_cache_;
    }

    const RegionList& regions() const {
        std::uint64_t n = 0;
        tg_regions(handle(), nullptr, 0, &n);
        std::vector<tg_region> buf(n);
        tg_regions(handle(), buf.data(), n, &n);
        std::vector<Region> regs;
        regs.reserve(n);
        for (const auto& r : buf)
            regs.push_back(Region{r.offset, r.size, static_cast<RegionKind>(r.kind), tgb::wid(r.tensor), r.block_id});
        regions_cache_ = RegionList::from_snapshot(gpu_.pool_size, regs);
        return regions_cache_;
    }

    void set_model_alpha(const std::string& model_id, double alpha) {
        tg_set_model_alpha(mutable_handle(), model_id.c_str(), alpha);
    }

    std::pair<std::vector<TensorId>, std::vector<TensorSpec>> lookup(const ModelSpec& model) const {
        tgb::ModelView v(model);
        std::vector<std::uint8_t> mask(model.tensors.size() + 1, 0);
        tg_lookup(handle(), &v.spec, mask.data(), nullptr);
        std::pair<std::vector<TensorId>, std::vector<TensorSpec>> out;
        for (std::size_t i = 0; i < model.tensors.size(); ++i)
            if (mask[i]) out.first.push_back(model.tensors[i].id);
            else out.second.push_back(model.tensors[i]);
        return out;
    }

    Bytes reuse_size(const ModelSpec& model) const {
        tgb::ModelView v(model);
        std::uint64_t s = 0;
        tg_reuse_size(handle(), &v.spec, &s);
        return s;
    }

    std::vector<EvictionCandidate> eviction_candidates(const ModelStatsTable& stats,
                                                       const std::string& exclude_model) const {
        tgb::StatsHandle sh(stats);
        std::uint32_t n = 0;
        tg_eviction_candidates(handle(), sh.h, exclude_model.c_str(), nullptr, 0, &n);
        std::vector<tg_eviction> buf(n);
        tg_eviction_candidates(handle(), sh.h, exclude_model.c_str(), buf.data(), n, &n);
        std::vector<EvictionCandidate> out;
        for (const auto& e : buf) out.push_back({tgb::wid(e.tensor), e.size, e.cost, e.last_access, e.model_id});
        return out;
    }

    Result<LoadOutcome> load_model(const ModelSpec& model, const ModelStatsTable& stats, Seconds clock,
                                   const LoadPolicy& policy = {}) {
        tgb::ModelView v(model);
        tgb::StatsHandle sh(stats);
        tg_load_policy pol{};
        pol.merge = policy.merge == MergePolicy::GlobalMerge ? 1 : 0;
        pol.strictness = policy.strictness == PackingStrictness::LiteralGuard ? 1 : 0;
        pol.random_eviction = policy.random_eviction ? 1 : 0;
        if (policy.rng) {
            pol.uniform_below = [](void* c, std::uint64_t n) { return static_cast<Rng*>(c)->uniform_below(n); };
            pol.rng_ctx = policy.rng;
        }
        pol.flags = TG_LOAD_DEFAULT | (tgb::async_loads() ? TG_LOAD_ASYNC : 0u) |
                    (tgs::peer_bandwidth() > 0 ? TG_LOAD_PEER : 0u);
        LoadOutcome out;
        const int rc = tgb::domain(tg_load_model(mutable_handle(), &v.spec, sh.h, clock, &pol, &out.device), "tg_load_model");
        if (rc) return static_cast<Error>(rc - 1);
        const tg_load_outcome& o = out.device;
        std::vector<tg_tensor_id> ids(o.n_hits);
        tg_last_hits(handle(), ids.data(), o.n_hits);
        for (const auto& i : ids) out.hit_tensors.push_back(tgb::wid(i));
        std::unordered_map<TensorId, const TensorSpec*, TensorIdHash> by_id;
        for (const auto& t : model.tensors) by_id.emplace(t.id, &t);
        ids.assign(o.n_misses, {});
        tg_last_misses(handle(), ids.data(), o.n_misses);
        for (const auto& i : ids) out.missed_tensors.push_back(*by_id.at(tgb::wid(i)));
        out.bytes_transferred = o.bytes_transferred;
        out.bytes_merged = o.bytes_merged;
        out.eviction_cost_total = o.eviction_cost_total;
        std::vector<tg_eviction> ev(o.n_evictions);
        tg_last_evictions(handle(), ev.data(), o.n_evictions);
        for (const auto& e : ev) out.plan.evictions.push_back({tgb::wid(e.tensor), e.size, e.cost, e.last_access, e.model_id});
        std::vector<tg_relocation> rl(o.n_relocations);
        tg_last_relocations(handle(), rl.data(), o.n_relocations);
        for (const auto& r : rl) out.plan.relocations.push_back({tgb::wid(r.tensor), r.from, r.to, r.size});
        std::vector<tg_placement> pl(o.n_placements);
        tg_last_placements(handle(), pl.data(), o.n_placements);
        for (const auto& p : pl) out.plan.placements.push_back({*by_id.at(tgb::wid(p.tensor)), p.offset});
        out.plan.total_eviction_cost = o.total_eviction_cost;
        out.plan.total_merge_cost = o.total_merge_cost;
        out.plan.pgp_merge_cost = o.pgp_merge_cost;
        out.plan.initial_merge_cost = o.initial_merge_cost;
        out.plan.fallback_evictions = o.fallback_evictions;
        return out;
    }

    void end_instance(const std::string& model_id) { tg_end_instance(mutable_handle(), model_id.c_str()); }

    Status evict_tensor(const TensorId& id) { return status(tg_evict_tensor(mutable_handle(), tgb::cid(id)), "evict"); }

    void evict_model(const std::string& model_id) { tg_evict_model(mutable_handle(), model_id.c_str()); }

    Status move_tensor(const TensorId& id, Bytes new_offset) {
        return status(tg_move_tensor(mutable_handle(), tgb::cid(id), new_offset), "tg_move_tensor");
    }

    Result<Bytes> alloc_kv_region(Bytes size, std::uint64_t block_id) {
        std::uint64_t off = 0;
        const int rc = tgb::domain(tg_alloc_kv_region(mutable_handle(), size, block_id, &off), "tg_alloc_kv_region");
        if (rc) return static_cast<Error>(rc - 1);
        return off;
    }

    Status free_kv_region(Bytes offset) { return status(tg_free_kv_region(mutable_handle(), offset), "tg_free_kv_region"); }

    Status validate() const { return status(tg_validate(handle()), "tg_validate"); }

    nlohmann::json dump() const {
        std::uint64_t need = 0;
        tg_dump(handle(), nullptr, 0, &need);
        std::string s(need, '\0');
        if (int rc = tg_dump(handle(), s.data(), need, &need)) tgb::fail(rc, "tg_dump");
        s.resize(need ? need - 1 : 0);
        return nlohmann::json::parse(s);
    }

private:
    static Status status(int rc, const char* where) {
        rc = tgb::domain(rc, where);
        if (rc) return static_cast<Error>(rc - 1);
        return ok_status();
    }
    tg_pool_info info() const {
        tg_pool_info i{};
        tg_pool_info_get(handle(), &i);
        return i;
    }

    static std::shared_ptr<tg_pool> clone_of(tg_pool* p) {
        tg_pool* c = nullptr;
        if (int rc = tg_pool_clone(p, &c)) tgb::fail(rc, "tg_pool_clone");
        return std::shared_ptr<tg_pool>(c, tgb::PoolDeleter{"", false});
    }
    void adopt(const ReuseStore& o) {
        tg_pool* dst = mutable_handle();
        if (int rc = tg_pool_assign(dst, o.handle())) tgb::fail(rc, "tg_pool_assign");
        gpu_ = o.gpu_;
    }

    GpuSpec gpu_;
    std::shared_ptr<tgb::Box> box_;
    mutable std::unordered_map<TensorId, TensorEntry, TensorIdHash> tensors_cache_;
    mutable std::uint64_t map_epoch_ = ~std::uint64_t{0};
    mutable RegionList regions_cache_;
};

}  // namespace warmsim
