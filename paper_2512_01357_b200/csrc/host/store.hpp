// Control plane of one GPU's unified pool: the tensor index plus the
// load / evict / move / KV-region lifecycle.  Decisions are bit-identical to
// the reference ReuseStore (reuse_store.hpp:50-345); the byte movement each
// decision implies is executed by the device data plane (pool.cpp), which is
// why planning and applying are separate steps here.
#pragma once

#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "model.hpp"
#include "planner.hpp"
#include "regions.hpp"

namespace tg {

// Device-side failure (CUDA error, missing host source, ...).  Thrown by the
// data plane and converted to an error code at the C-ABI boundary.
struct DeviceError : std::runtime_error {
    int code;
    DeviceError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

// Uniform draws for random-eviction order (reuse_store.hpp:143-147).
class Uniform {
public:
    virtual ~Uniform() = default;
    virtual u64 uniform_below(u64 n) = 0;
};

// mt19937_64 stream + rejection-sampled uniform_below; the same stream the
// reference Rng produces (rng.hpp:18-73).
class Rng final : public Uniform {
public:
    explicit Rng(u64 seed) : gen_(seed) {}
    u64 next() { return gen_(); }
    u64 uniform_below(u64 n) override {
        const u64 limit = UINT64_MAX - UINT64_MAX % n;
        u64 x;
        do x = gen_();
        while (x >= limit);
        return x % n;
    }

private:
    std::mt19937_64 gen_;
};

// Caller-owned random stream (e.g. the simulator's own Rng behind the facade).
class UniformCallback final : public Uniform {
public:
    UniformCallback(void* ctx, u64 (*fn)(void*, u64)) : ctx_(ctx), fn_(fn) {}
    u64 uniform_below(u64 n) override { return fn_(ctx_, n); }

private:
    void* ctx_;
    u64 (*fn_)(void*, u64);
};

struct LoadOptions {
    MergeMode merge = MergeMode::PartitionedGain;
    Strictness strictness = Strictness::Functional;
    bool random_eviction = false;
    Uniform* rng = nullptr;
};

struct Digest {
    u64 hi = 0, lo = 0;
    bool operator==(const Digest& o) const { return hi == o.hi && lo == o.lo; }
};

struct Entry {
    u64 off = 0;
    u64 size = 0;
    std::string model;
    double last_access = 0;
    bool pinned = false;
    // `digest` is the tensor's content truth: the fingerprint of its source
    // bytes (measured when placed, or the manifest / peer digest they were
    // checked against).  Not a statement about the resident bytes.
    bool has_digest = false;
    Digest digest;
    // The resident bytes are not known to equal the content: a load wrote
    // them and has not verified (or failed to land / repair) them.  Suspect
    // tensors are never exported to peers or used as byte sources, and are
    // verified (re-sent when unverifiable) on their next reuse whatever the
    // load flags say.  Data-plane state only: not part of the dump.
    bool suspect = false;
};

struct LoadDecision {
    std::vector<u32> hits;    // indices into model.tensors, model order
    std::vector<u32> misses;  // indices into model.tensors, model order
    std::vector<Key> hit_keys;
    std::vector<TensorDesc> miss_desc;
    u64 bytes_transferred = 0;
    Plan plan;                // placements index into miss_desc
    PoolMap after;            // layout once the plan is applied
};

class Store {
public:
    Store() = default;
    explicit Store(GpuDesc gpu) : gpu_(std::move(gpu)), map_(gpu_.pool_size) {}

    const GpuDesc& gpu() const { return gpu_; }
    u64 pool_size() const { return gpu_.pool_size; }
    u64 free_bytes() const { return map_.free_total(); }
    u64 kv_bytes() const { return kv_bytes_; }
    u64 pinned_tensor_bytes() const { return pinned_tensor_bytes_; }
    u64 pinned_bytes() const { return pinned_tensor_bytes_ + kv_bytes_; }
    u64 reusable_bytes() const { return gpu_.pool_size - pinned_bytes(); }
    u64 merged_total() const { return merged_total_; }
    u64 transferred_total() const { return transferred_total_; }
    u64 evictions_total() const { return evictions_total_; }
    const PoolMap& map() const { return map_; }
    const std::unordered_map<Key, Entry, KeyHash>& tensors() const { return tensors_; }
    // Changes whenever the tensor map's offsets, sizes, pins or access times
    // change; values are unique process-wide, so copies and restores compare
    // unequal to any other state.  (Drives the device index republish.)
    u64 epoch() const { return epoch_; }
    Entry* entry(const Key& k) {
        auto it = tensors_.find(k);
        return it == tensors_.end() ? nullptr : &it->second;
    }
    void set_alpha(const std::string& model, double a) { alpha_[model] = a; }

    // lookup / reuse_size (reuse_store.hpp:81-97)
    void lookup(const ModelDesc& m, std::vector<u32>* hits, std::vector<u32>* misses) const;
    u64 reuse_size(const ModelDesc& m) const;
    // eviction_candidates (reuse_store.hpp:99-115)
    std::vector<Candidate> candidates(const StatsView& stats, const std::string& exclude) const;

    // load_model, split in two (reuse_store.hpp:120-174).  decide() performs
    // the alpha update, the capacity check, lookup and planning without
    // touching the layout; commit() applies the decision and pins.
    Res<LoadDecision> decide(const ModelDesc& m, const StatsView& stats, const LoadOptions& opt);
    void commit(const ModelDesc& m, LoadDecision& d, double clock);

    void end_instance(const std::string& model);
    St evict_tensor(const Key& k);
    void evict_model(const std::string& model);
    St move_tensor(const Key& k, u64 to);
    Res<u64> alloc_kv_region(u64 size, u64 block_id);
    St free_kv_region(u64 off);

    // KV block runs carved by the block allocator (kv.cpp).
    void carve_kv_run(u64 off, u64 nblocks, u64 block_len, u64 first_block);
    // Release every KV extent inside [off, off+bytes) (teardown of a run).
    void release_kv_range(u64 off, u64 bytes);

    St validate() const;
    std::string dump_json() const;

    // Engines armed for device-decided KV batches (K4D) hold a mirror of the
    // free runs: while any is armed, nothing may change the layout.  Engines
    // hold a weak handle on the count, so an engine destroyed while armed
    // releases its arm, and one outliving the store touches nothing; copies
    // of a store (snapshots) start with a count of their own at zero.
    class ArmCount {
    public:
        ArmCount() : c_(std::make_shared<int>(0)) {}
        ArmCount(const ArmCount&) : ArmCount() {}
        ArmCount& operator=(const ArmCount&) { return *this; }
        int value() const { return *c_; }
        std::weak_ptr<int> handle() const { return c_; }

    private:
        std::shared_ptr<int> c_;
    };
    u32 kv_armed() const { return static_cast<u32>(kv_armed_.value()); }
    std::weak_ptr<int> kv_arm_handle() const { return kv_armed_.handle(); }

private:
    ArmCount kv_armed_;
    void touch();
    u64 epoch_ = 0;
    double alpha_of(const std::string& m) const {
        auto it = alpha_.find(m);
        return it == alpha_.end() ? 1.0 : it->second;
    }

    GpuDesc gpu_;
    PoolMap map_;
    std::unordered_map<Key, Entry, KeyHash> tensors_;
    std::map<std::string, double> alpha_;
    u64 kv_bytes_ = 0;
    u64 pinned_tensor_bytes_ = 0;
    u64 merged_total_ = 0;
    u64 transferred_total_ = 0;
    u64 evictions_total_ = 0;
};

}  // namespace tg
