// extern "C" boundary (include/tangram.h).  Converts C structs to the host
// control-plane types, maps domain errors to codes (ordinal + 1) and every
// device/runtime exception to a TG_ERR_* code with a thread-local detail.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/tangram.h"
#include "../device/common.cuh"
#include "../device/kernels.hpp"
#include "kv.hpp"
#include "index.hpp"
#include "pool.hpp"
#include "sched.hpp"

using namespace tg;

struct tg_pool {
    std::unique_ptr<Pool> pool;
    LoadReport last;
    std::vector<std::string> strs;  // backing store for returned model ids
};
struct tg_stats {
    RequestShares own;
    std::unique_ptr<ExternalStats> ext;  // caller-owned statistics (tg_stats_create_external)
    const StatsView& s_view() const { return ext ? static_cast<const StatsView&>(*ext) : own; }
};
struct tg_rng {
    Rng r;
};
struct tg_kv {
    std::unique_ptr<KvAllocator> a;
    int device = -2;  // -2: not yet bound to a pool
};
struct tg_model {
    ModelDesc m;
    std::vector<tg_tensor_spec> view;
    void refresh() {
        view.clear();
        for (const auto& t : m.tensors)
            view.push_back(tg_tensor_spec{{t.id.hi, t.id.lo}, t.name.c_str(), t.size, t.model_id.c_str()});
    }
};
struct tg_snapshot {
    Pool::Snapshot* s = nullptr;
};

namespace {

thread_local std::string g_detail;

int code_of(const St& s) { return s.ok() ? 0 : 1 + static_cast<int>(s.error()); }
int code_of(Err e) { return 1 + static_cast<int>(e); }

template <class F>
int guard(F&& f) {
    try {
        return f();
    } catch (const DeviceError& e) {
        g_detail = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_detail = e.what();
        return TG_ERR_INTERNAL;
    }
}

Key key_of(tg_tensor_id id) { return Key{id.hi, id.lo}; }
tg_tensor_id id_of(const Key& k) { return tg_tensor_id{k.hi, k.lo}; }

ModelDesc model_of(const tg_model_spec* s) {
    ModelDesc m;
    m.model_id = s->model_id ? s->model_id : "";
    m.total_size = s->total_size;
    m.alpha = s->latency_sensitivity;
    m.location = s->location ? Location::ModelStore : Location::ModelCache;
    m.bytes_per_token = s->bytes_per_token;
    m.tensors.reserve(s->n_tensors);
    for (uint32_t i = 0; i < s->n_tensors; ++i) {
        const tg_tensor_spec& t = s->tensors[i];
        m.tensors.push_back(TensorDesc{key_of(t.id), t.model_id ? t.model_id : m.model_id, t.name ? t.name : "", t.size});
    }
    return m;
}

LoadOptions options_of(const tg_load_policy* p, std::unique_ptr<UniformCallback>* keep) {
    LoadOptions o;
    if (!p) return o;
    o.merge = p->merge ? MergeMode::GlobalMerge : MergeMode::PartitionedGain;
    o.strictness = p->strictness ? Strictness::LiteralGuard : Strictness::Functional;
    o.random_eviction = p->random_eviction != 0;
    if (p->rng) {
        o.rng = &p->rng->r;
    } else if (p->uniform_below) {
        *keep = std::make_unique<UniformCallback>(p->rng_ctx, p->uniform_below);
        o.rng = keep->get();
    }
    return o;
}

// Bind a KV engine to the pool's device on first use (KvEngine takes the
// store per call, kv_engine.hpp:75, so binding is lazy).
int bind_kv(tg_kv* kv, tg_pool* p) {
    if (p->pool->store().kv_armed() || kv->a->armed()) {
        g_detail = "a KV engine is armed on this pool: tg_kv_device_sync first";
        return TG_ERR_KV_ARMED;
    }
    const int dev = p->pool->device();
    if (kv->device == -2) {
        kv->device = dev;
        if (dev >= 0) kv->a->attach_device(p->pool->make_kv_device());
        return 0;
    }
    if (kv->device != dev) {
        g_detail = "KV engine used with pools on different devices";
        return TG_ERR_BAD_ARG;
    }
    return 0;
}

}  // namespace

extern "C" {

int tg_version(void) { return 1; }

const char* tg_error_string(int code) {
    if (code == 0) return "ok";
    if (code >= 1 && code <= 10) return err_name(static_cast<Err>(code - 1));
    switch (code) {
        case TG_ERR_CUDA: return "CUDA error";
        case TG_ERR_NO_DEVICE: return "no device";
        case TG_ERR_NO_SOURCE: return "no byte source for a missed tensor";
        case TG_ERR_BUFFER: return "buffer too small";
        case TG_ERR_BAD_ARG: return "bad argument";
        case TG_ERR_VERIFY: return "fingerprint verification failed";
        case TG_ERR_KV_ARMED: return "a KV engine is armed for device batches";
        case TG_ERR_KV_LOG: return "device KV batch log overflowed";
        default: return "internal error";
    }
}

const char* tg_last_error_detail(void) { return g_detail.c_str(); }

uint64_t tg_kernel_launches(void) { return g_kernel_launches.load(); }

int tg_device_count(int* n) {
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        cudaGetLastError();
    }
    return 0;
}

// ---- ids / catalog --------------------------------------------------------------
int tg_murmur3_x64_128(const void* data, uint64_t len, uint64_t seed, tg_digest* out) {
    const Key k = murmur3_x64_128(data, len, seed);
    *out = tg_digest{k.hi, k.lo};
    return 0;
}

int tg_tensor_key(const char* model_id, const char* name, const int64_t* shape, int32_t ndim, int32_t dtype,
                  tg_tensor_id* out) {
    if (!model_id || !name || dtype < 0 || dtype > 3) return TG_ERR_BAD_ARG;
    *out = id_of(tensor_key(model_id, name, shape, ndim, static_cast<Dtype>(dtype)));
    return 0;
}

int tg_model_make(const char* model_id, uint64_t total, int32_t layers, uint64_t bpt, int32_t location, double alpha,
                  tg_model** out) {
    if (!model_id || layers <= 0) return TG_ERR_BAD_ARG;
    auto* m = new tg_model{make_model(model_id, total, layers, bpt, location ? Location::ModelStore : Location::ModelCache, alpha), {}};
    m->refresh();
    *out = m;
    return 0;
}

uint32_t tg_model_catalog_size(void) { return static_cast<uint32_t>(default_catalog().size()); }

int tg_model_default_catalog(uint32_t index, tg_model** out) {
    auto cat = default_catalog();
    if (index >= cat.size()) return TG_ERR_BAD_ARG;
    auto* m = new tg_model{cat[index], {}};
    m->refresh();
    *out = m;
    return 0;
}

void tg_model_destroy(tg_model* m) { delete m; }

int tg_model_view(const tg_model* m, tg_model_spec* out) {
    if (!m) return TG_ERR_BAD_ARG;
    *out = tg_model_spec{m->m.model_id.c_str(), m->view.data(), static_cast<uint32_t>(m->view.size()), m->m.total_size,
                         m->m.alpha, m->m.location == Location::ModelStore ? 1 : 0, m->m.bytes_per_token};
    return 0;
}

// Tensor-parallel shard r of N: shard of a tensor of n bytes
// = bytes [r*ceil(n/N), min(n, (r+1)*ceil(n/N))).  Ids are keyed on the
// shard's own (model, name, shape) so shards never alias each other.
int tg_model_shard(const tg_model* m, uint32_t rank, uint32_t world, tg_model** out) {
    if (!m || world == 0 || rank >= world) return TG_ERR_BAD_ARG;
    auto* s = new tg_model{};
    const std::string suffix = "#tp" + std::to_string(world) + "." + std::to_string(rank);
    s->m.model_id = m->m.model_id + suffix;
    s->m.alpha = m->m.alpha;
    s->m.location = m->m.location;
    s->m.bytes_per_token = m->m.bytes_per_token / world;
    for (const auto& t : m->m.tensors) {
        const u64 chunk = (t.size + world - 1) / world;
        const u64 b = std::min<u64>(t.size, rank * chunk), e = std::min<u64>(t.size, (rank + 1) * chunk);
        if (e <= b) continue;
        TensorDesc d;
        d.model_id = s->m.model_id;
        d.name = t.name + suffix;
        d.size = e - b;
        const std::int64_t elems = static_cast<std::int64_t>(d.size / 2);
        d.id = tensor_key(d.model_id, d.name, &elems, 1, Dtype::F16);
        ShardLineage::get().put(d.id, ShardOf{t.id, b, d.size});
        s->m.tensors.push_back(d);
        s->m.total_size += d.size;
    }
    std::sort(s->m.tensors.begin(), s->m.tensors.end(),
              [](const TensorDesc& a, const TensorDesc& b) { return a.name < b.name; });
    s->refresh();
    *out = s;
    return 0;
}

int tg_lineage_register(tg_tensor_id child, tg_tensor_id parent, uint64_t begin, uint64_t size) {
    ShardLineage::get().put(key_of(child), ShardOf{key_of(parent), begin, size});
    return 0;
}
int tg_lineage_get(tg_tensor_id child, tg_tensor_id* parent, uint64_t* begin, uint64_t* size) {
    ShardOf s;
    if (!ShardLineage::get().find(key_of(child), &s)) return code_of(Err::NotFound);
    if (parent) *parent = id_of(s.parent);
    if (begin) *begin = s.begin;
    if (size) *size = s.size;
    return 0;
}

// ---- stats / rng ------------------------------------------------------------------
int tg_stats_create(double decay, tg_stats** out) {
    *out = new tg_stats{RequestShares(decay), nullptr};
    return 0;
}
int tg_stats_create_external(void* ctx, double (*miss_probability)(void*, const char*),
                             double (*load_bandwidth_or)(void*, const char*, double), tg_stats** out) {
    if (!miss_probability || !load_bandwidth_or || !out) return TG_ERR_BAD_ARG;
    *out = new tg_stats{RequestShares(), std::make_unique<ExternalStats>(ctx, miss_probability, load_bandwidth_or)};
    return 0;
}
void tg_stats_destroy(tg_stats* s) { delete s; }
int tg_stats_record_request(tg_stats* s, const char* m, double t) { return code_of(s->own.record_request(m, t)); }
int tg_stats_record_eviction(tg_stats* s, const char* m, double t) { return code_of(s->own.record_eviction(m, t)); }
int tg_stats_set_load_bandwidth(tg_stats* s, const char* m, double bw) {
    s->own.set_load_bandwidth(m, bw);
    return 0;
}
double tg_stats_miss_probability(const tg_stats* s, const char* m) { return s->own.miss_probability(m); }

int tg_rng_create(uint64_t seed, tg_rng** out) {
    *out = new tg_rng{Rng(seed)};
    return 0;
}
void tg_rng_destroy(tg_rng* r) { delete r; }
uint64_t tg_rng_uniform_below(tg_rng* r, uint64_t n) { return r->r.uniform_below(n); }

// ---- pool ---------------------------------------------------------------------------
// An asynchronous load (TG_LOAD_ASYNC) still in flight is finished before
// any operation that mutates the pool or reads digests / suspect state
// (a deferred failure is reported by tg_pool_sync).
static void settle(const tg_pool* p) {
    if (p && p->pool && p->pool->has_pending()) p->pool->complete_pending();
}

int tg_pool_create(const tg_gpu_spec* g, int32_t device, tg_pool** out) {
    return guard([&] {
        if (!g || !out) return TG_ERR_BAD_ARG;
        GpuDesc d{g->gpu_id ? g->gpu_id : "gpu0", g->pool_size, g->pcie_bandwidth, g->intra_copy_bandwidth,
                  g->store_bandwidth};
        if (device >= 0) {
            int n = 0;
            if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n) {
                cudaGetLastError();
                g_detail = "no CUDA device " + std::to_string(device);
                return TG_ERR_NO_DEVICE;
            }
        }
        auto p = std::make_unique<tg_pool>();
        p->pool = std::make_unique<Pool>(d, device < 0 ? -1 : device);
        *out = p.release();
        return 0;
    });
}

void tg_pool_destroy(tg_pool* p) { delete p; }

int tg_pool_clone(const tg_pool* p, tg_pool** out) {
    settle(p);
    return guard([&] {
        if (!p || !out) return TG_ERR_BAD_ARG;
        auto c = std::make_unique<tg_pool>();
        c->pool = std::make_unique<Pool>(p->pool->store().gpu(), -1);
        c->pool->adopt_store(p->pool->store());
        *out = c.release();
        return 0;
    });
}

int tg_pool_assign(tg_pool* dst, const tg_pool* src) {
    settle(dst);
    return guard([&] {
        if (!dst || !src) return TG_ERR_BAD_ARG;
        if (dst == src) return 0;
        if (dst->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        dst->pool->adopt_store(src->pool->store());
        dst->pool->publish_index();
        return 0;
    });
}

int tg_pool_tensors(const tg_pool* p, tg_tensor_entry* buf, uint64_t cap, uint64_t* n) {
    settle(p);
    if (!p || !n) return TG_ERR_BAD_ARG;
    const auto& t = p->pool->store().tensors();
    *n = t.size();
    if (!buf) return 0;
    uint64_t i = 0;
    for (const auto& [k, e] : t) {
        if (i == cap) return TG_ERR_BUFFER;
        buf[i++] = tg_tensor_entry{id_of(k), e.off, e.size, e.last_access, e.pinned ? 1 : 0, e.suspect ? 1 : 0,
                                   e.model.c_str()};
    }
    return 0;
}

int tg_pool_info_get(const tg_pool* p, tg_pool_info* o) {
    if (!p || !o) return TG_ERR_BAD_ARG;
    const Store& s = p->pool->store();
    *o = tg_pool_info{s.pool_size(),       s.free_bytes(),        s.kv_bytes(),
                      s.pinned_tensor_bytes(), s.pinned_bytes(),  s.reusable_bytes(),
                      s.merged_total(),    s.transferred_total(), s.evictions_total(),
                      s.map().region_count(), s.map().extent_count(), s.tensors().size(),
                      s.map().largest_free(), p->pool->device(),  p->pool->arena(),
                      0, 0.0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const Pool::Totals& t = p->pool->totals();
    o->loads = t.loads;
    o->data_plane_ms = t.data_plane_ms;
    o->pcie_bytes = t.pcie_bytes;
    o->peer_bytes = t.peer_bytes;
    o->device_src_bytes = t.device_src_bytes;
    o->fingerprint_bytes = t.fingerprint_bytes;
    o->relocated_bytes = t.relocated_bytes;
    o->epoch = s.epoch();
    o->verify_mismatches = t.verify_mismatches;
    o->repaired_bytes = t.repaired_bytes;
    o->failed_loads = t.failed_loads;
    return 0;
}

int tg_pool_stream(const tg_pool* p, void** s) {
    if (!p || !p->pool->has_device()) return TG_ERR_NO_DEVICE;
    *s = p->pool->stream();
    return 0;
}

int tg_set_model_alpha(tg_pool* p, const char* m, double a) {
    p->pool->store().set_alpha(m, a);
    return 0;
}

static void fill_outcome(const LoadReport& r, tg_load_outcome* out) {
    const Plan& pl = r.decision.plan;
    std::memset(out, 0, sizeof *out);
    out->n_hits = static_cast<uint32_t>(r.decision.hits.size());
    out->n_misses = static_cast<uint32_t>(r.decision.misses.size());
    out->n_evictions = static_cast<uint32_t>(pl.evictions.size());
    out->n_relocations = static_cast<uint32_t>(pl.relocations.size());
    out->n_placements = static_cast<uint32_t>(pl.placements.size());
    out->n_waves = r.waves;
    out->fallback_evictions = pl.fallback_evictions;
    out->bytes_transferred = r.decision.bytes_transferred;
    out->bytes_merged = r.decision.misses.empty() ? 0 : pl.total_merge_cost;
    out->eviction_cost_total = r.decision.misses.empty() ? 0.0 : pl.total_eviction_cost;
    out->total_merge_cost = pl.total_merge_cost;
    out->pgp_merge_cost = pl.pgp_merge_cost;
    out->initial_merge_cost = pl.initial_merge_cost;
    out->total_eviction_cost = pl.total_eviction_cost;
    out->pcie_bytes = r.pcie_bytes;
    out->peer_bytes = r.peer_bytes;
    out->device_src_bytes = r.device_src_bytes;
    out->fingerprint_bytes = r.fingerprint_bytes;
    out->repaired_bytes = r.repaired_bytes;
    out->verify_mismatches = r.verify_mismatches;
    out->expected_mismatches = r.expected_mismatches;
    out->plan_us = r.t.plan_us;
    out->total_ms = r.t.total_ms;
    out->relocate_ms = r.t.relocate_ms;
    out->h2d_ms = r.t.h2d_ms;
    out->peer_ms = r.t.peer_ms;
    out->fp_kernel_ms = r.t.fp_kernel_ms;
    out->fp_reuse_ms = r.t.fp_reuse_ms;
    out->fp_reuse_max_ms = r.t.fp_reuse_max_ms;
    out->host_issue_us = r.t.host_issue_us;
    out->host_wait_us = r.t.host_wait_us;
    out->host_total_us = r.t.host_total_us;
    out->suspect_tensors = r.suspect_after;
    out->kernel_end_ms = r.t.kernel_end_ms;
    out->gated_h2d_start_ms = r.t.gated_h2d_start_ms;
}

int tg_load_model(tg_pool* p, const tg_model_spec* ms, const tg_stats* s, double clock, const tg_load_policy* pol,
                  tg_load_outcome* out) {
    return guard([&] {
        if (!p || !ms || !s) return TG_ERR_BAD_ARG;
        if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        const ModelDesc m = model_of(ms);
        u32 flags = static_cast<u32>(TG_LOAD_DEFAULT);
        if (pol && (pol->flags & TG_LOAD_EXPLICIT)) flags = pol->flags & ~static_cast<u32>(TG_LOAD_EXPLICIT);
        else if (pol && pol->flags) flags = pol->flags;
        LoadReport& r = p->last;
        std::unique_ptr<UniformCallback> cb;
        int rc = 0;
        try {
            St st = p->pool->load_model(m, s->s_view(), clock, options_of(pol, &cb), flags, &r);
            if (!st) return code_of(st);
        } catch (const DeviceError& e) {
            // After the commit the outcome still describes the decision taken
            // (and how many tensors it left suspect); before it, nothing changed.
            if (!r.committed) throw;
            g_detail = e.what();
            rc = e.code;
        }
        if (out) fill_outcome(r, out);
        if (p->pool->has_device()) p->pool->publish_index();
        return rc;
    });
}

int tg_pool_sync(tg_pool* p, tg_load_outcome* out) {
    return guard([&] {
        if (!p) return TG_ERR_BAD_ARG;
        const bool had = p->pool->has_pending();
        const int rc = p->pool->complete_pending();
        if (rc) g_detail = p->pool->last_completed_error();
        if (had) p->last = p->pool->last_completed();  // tg_last_* now describe the completed load
        if (out) {
            if (had) fill_outcome(p->last, out);
            else std::memset(out, 0, sizeof *out);
        }
        return rc;
    });
}

int tg_failpoint(const char* name, int64_t nth) {
    if (!name) return TG_ERR_BAD_ARG;
    Failpoints::arm(name, nth);
    return 0;
}

uint32_t tg_last_hits(const tg_pool* p, tg_tensor_id* buf, uint32_t cap) {
    const auto& d = p->last.decision;
    uint32_t n = 0;
    for (u32 i = 0; i < d.hits.size(); ++i, ++n)
        if (buf && n < cap) buf[n] = id_of(d.hit_keys[i]);
    return n;
}

uint32_t tg_last_misses(const tg_pool* p, tg_tensor_id* buf, uint32_t cap) {
    const auto& d = p->last.decision;
    uint32_t n = 0;
    for (const auto& t : d.miss_desc) {
        if (buf && n < cap) buf[n] = id_of(t.id);
        ++n;
    }
    return n;
}

uint32_t tg_last_evictions(const tg_pool* p, tg_eviction* buf, uint32_t cap) {
    const auto& ev = p->last.decision.plan.evictions;
    const uint32_t n = static_cast<uint32_t>(ev.size());
    for (uint32_t i = 0; buf && i < n && i < cap; ++i)
        buf[i] = tg_eviction{id_of(ev[i].tensor), ev[i].size, ev[i].cost, ev[i].last_access, ev[i].model_id.c_str()};
    return n;
}

uint32_t tg_last_relocations(const tg_pool* p, tg_relocation* buf, uint32_t cap) {
    const auto& rl = p->last.decision.plan.relocations;
    const uint32_t n = static_cast<uint32_t>(rl.size());
    for (uint32_t i = 0; buf && i < n && i < cap; ++i)
        buf[i] = tg_relocation{id_of(rl[i].tensor), rl[i].from, rl[i].to, rl[i].size,
                               i < p->last.reloc_wave.size() ? p->last.reloc_wave[i] : 0};
    return n;
}

uint32_t tg_last_placements(const tg_pool* p, tg_placement* buf, uint32_t cap) {
    const auto& d = p->last.decision;
    const auto& pl = d.plan.placements;
    const uint32_t n = static_cast<uint32_t>(pl.size());
    for (uint32_t i = 0; buf && i < n && i < cap; ++i) {
        const TensorDesc& t = d.miss_desc[pl[i].tensor];
        buf[i] = tg_placement{id_of(t.id), pl[i].off, t.size,
                              i < p->last.placement_src.size() ? p->last.placement_src[i] : 0u};
    }
    return n;
}

uint32_t tg_last_digests(const tg_pool* p, tg_digest* buf, uint32_t cap) {
    const auto& g = p->last.digests;
    const uint32_t n = static_cast<uint32_t>(g.size());
    for (uint32_t i = 0; buf && i < n && i < cap; ++i) buf[i] = tg_digest{g[i].hi, g[i].lo};
    return n;
}

int tg_end_instance(tg_pool* p, const char* m) {
    settle(p);
    return guard([&] {
        p->pool->store().end_instance(m);
        p->pool->publish_index();
        return 0;
    });
}
int tg_evict_tensor(tg_pool* p, tg_tensor_id id) {
    settle(p);
    return guard([&] {
        if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        const int rc = code_of(p->pool->store().evict_tensor(key_of(id)));
        p->pool->publish_index();
        return rc;
    });
}
int tg_evict_model(tg_pool* p, const char* m) {
    settle(p);
    return guard([&] {
        if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        p->pool->store().evict_model(m);
        p->pool->publish_index();
        return 0;
    });
}
int tg_move_tensor(tg_pool* p, tg_tensor_id id, uint64_t to) {
    settle(p);
    return guard([&] {
        if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        const int rc = code_of(p->pool->move_tensor(key_of(id), to));
        p->pool->publish_index();
        return rc;
    });
}
int tg_alloc_kv_region(tg_pool* p, uint64_t size, uint64_t block_id, uint64_t* off) {
    settle(p);
    if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
    auto r = p->pool->store().alloc_kv_region(size, block_id);
    if (!r) return code_of(r.error());
    *off = r.value();
    return 0;
}
int tg_free_kv_region(tg_pool* p, uint64_t off) {
    settle(p);
    if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
    return code_of(p->pool->store().free_kv_region(off));
}

int tg_lookup(const tg_pool* p, const tg_model_spec* ms, uint8_t* mask, uint64_t* reuse) {
    const ModelDesc m = model_of(ms);
    std::vector<u32> hits, misses;
    p->pool->store().lookup(m, &hits, &misses);
    if (mask) {
        std::memset(mask, 0, m.tensors.size());
        for (u32 i : hits) mask[i] = 1;
    }
    if (reuse) *reuse = p->pool->store().reuse_size(m);
    return 0;
}
int tg_reuse_size(const tg_pool* p, const tg_model_spec* ms, uint64_t* out) {
    *out = p->pool->store().reuse_size(model_of(ms));
    return 0;
}
int tg_peer_reuse_size(const tg_pool* p, const tg_model_spec* ms, uint64_t* out) {
    *out = p->pool->peer_reuse_size(model_of(ms));
    return 0;
}

int tg_eviction_candidates(tg_pool* p, const tg_stats* s, const char* exclude, tg_eviction* buf, uint32_t cap,
                           uint32_t* n) {
    auto c = p->pool->store().candidates(s->s_view(), exclude ? exclude : "");
    *n = static_cast<uint32_t>(c.size());
    p->strs.clear();
    p->strs.reserve(c.size());
    for (uint32_t i = 0; i < c.size(); ++i) {
        p->strs.push_back(c[i].model_id);
        if (buf && i < cap) buf[i] = tg_eviction{id_of(c[i].tensor), c[i].size, c[i].cost, c[i].last_access, nullptr};
    }
    for (uint32_t i = 0; buf && i < c.size() && i < cap; ++i) buf[i].model_id = p->strs[i].c_str();
    return *n > cap && buf ? TG_ERR_BUFFER : 0;
}

int tg_validate(const tg_pool* p) {
    settle(p);
    return code_of(p->pool->store().validate());
}

int tg_dump(const tg_pool* p, char* buf, uint64_t cap, uint64_t* needed) {
    const std::string s = p->pool->store().dump_json();
    if (needed) *needed = s.size() + 1;
    if (!buf || cap < s.size() + 1) return TG_ERR_BUFFER;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

int tg_regions(const tg_pool* p, tg_region* buf, uint64_t cap, uint64_t* n) {
    const auto regs = p->pool->store().map().expanded();
    *n = regs.size();
    for (uint64_t i = 0; buf && i < regs.size() && i < cap; ++i)
        buf[i] = tg_region{regs[i].off, regs[i].len, static_cast<int32_t>(regs[i].kind), id_of(regs[i].tensor),
                           regs[i].block};
    return buf && cap < regs.size() ? TG_ERR_BUFFER : 0;
}

int tg_tensor_info_get(const tg_pool* p, tg_tensor_id id, tg_tensor_info* o) {
    settle(p);
    const auto& t = p->pool->store().tensors();
    auto it = t.find(key_of(id));
    if (it == t.end()) return code_of(Err::NotFound);
    const Entry& e = it->second;
    *o = tg_tensor_info{e.off, e.size, e.last_access, e.pinned, e.has_digest, {e.digest.hi, e.digest.lo},
                        p->pool->has_device() ? p->pool->arena() + e.off : nullptr, e.suspect, 0};
    return 0;
}

int tg_pool_index_image(const tg_pool* p, tg_index_slot* buf, uint64_t cap_slots, uint64_t* capacity) {
    return guard([&] {
        if (!p || !capacity) return TG_ERR_BAD_ARG;
        static_assert(sizeof(tg_index_slot) == sizeof(IndexSlot), "index slot layout");
        const std::vector<IndexSlot> img = build_index_image(p->pool->store());
        *capacity = img.size();
        if (buf) std::memcpy(buf, img.data(), std::min<uint64_t>(cap_slots, img.size()) * sizeof(IndexSlot));
        return 0;
    });
}
int tg_pool_device_index(tg_pool* p, const tg_index_slot** table, uint64_t* capacity) {
    settle(p);
    return guard([&] {
        if (!p || !table || !capacity) return TG_ERR_BAD_ARG;
        if (!p->pool->has_device()) return TG_ERR_NO_DEVICE;
        p->pool->publish_index();
        *table = static_cast<const tg_index_slot*>(p->pool->device_index(capacity));
        return 0;
    });
}
int tg_index_lookup(tg_pool* p, const tg_tensor_id* ids, uint32_t n, tg_index_hit* out) {
    settle(p);
    return guard([&] {
        if (!p || (n && (!ids || !out))) return TG_ERR_BAD_ARG;
        if (!p->pool->has_device()) return TG_ERR_NO_DEVICE;
        std::vector<Key> keys(n);
        for (uint32_t i = 0; i < n; ++i) keys[i] = key_of(ids[i]);
        std::vector<u64> r;
        p->pool->index_lookup(keys, &r);
        for (uint32_t i = 0; i < n; ++i)
            out[i] = tg_index_hit{r[3 * i], r[3 * i + 1], static_cast<uint32_t>(r[3 * i + 2] & 1),
                                  static_cast<uint32_t>(r[3 * i + 2] >> 32)};
        return 0;
    });
}

int tg_fingerprint_tensor(tg_pool* p, tg_tensor_id id, tg_digest* out) {
    settle(p);
    return guard([&] {
        if (!p->pool->store().tensors().count(key_of(id))) return code_of(Err::NotFound);
        const Digest d = p->pool->fingerprint_resident(key_of(id));
        *out = tg_digest{d.hi, d.lo};
        return 0;
    });
}

int tg_pool_add_peer(tg_pool* p, tg_pool* peer) {
    settle(p);
    return guard([&] {
        if (!p || !peer || p == peer) return TG_ERR_BAD_ARG;
        p->pool->add_peer(peer->pool.get());
        return 0;
    });
}

static std::vector<RemoteEntry> entries_of(const tg_index_entry* idx, uint64_t n) {
    std::vector<RemoteEntry> v;
    v.reserve(n);
    for (uint64_t i = 0; i < n; ++i)
        v.push_back(RemoteEntry{key_of(idx[i].id), idx[i].offset, idx[i].size, Digest{idx[i].digest.hi, idx[i].digest.lo}});
    return v;
}

int tg_pool_export_ipc(const tg_pool* p, void* handle) {
    settle(p);
    return guard([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == TG_IPC_HANDLE_BYTES, "IPC handle size");
        cudaIpcMemHandle_t h;
        p->pool->export_handle(&h);
        std::memcpy(handle, &h, sizeof h);
        return 0;
    });
}

int tg_pool_index(const tg_pool* p, tg_index_entry* buf, uint64_t cap, uint64_t* n) {
    settle(p);
    const auto idx = p->pool->index();
    *n = idx.size();
    for (uint64_t i = 0; buf && i < idx.size() && i < cap; ++i)
        buf[i] = tg_index_entry{id_of(idx[i].id), idx[i].off, idx[i].size, {idx[i].digest.hi, idx[i].digest.lo}};
    return buf && cap < idx.size() ? TG_ERR_BUFFER : 0;
}

int tg_pool_attach_remote(tg_pool* p, const void* handle, const tg_index_entry* idx, uint64_t n, int32_t* peer_id) {
    settle(p);
    return guard([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        const int id = p->pool->attach_remote(h, entries_of(idx, n));
        if (peer_id) *peer_id = id;
        return 0;
    });
}

int tg_pool_update_remote(tg_pool* p, int32_t peer_id, const tg_index_entry* idx, uint64_t n) {
    settle(p);
    return guard([&] {
        p->pool->update_remote(peer_id, entries_of(idx, n));
        return 0;
    });
}

int tg_pool_snapshot(tg_pool* p, tg_snapshot** out) {
    settle(p);
    return guard([&] {
        if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        *out = new tg_snapshot{p->pool->snapshot()};
        return 0;
    });
}
int tg_pool_restore(tg_pool* p, const tg_snapshot* s) {
    settle(p);
    return guard([&] {
        if (p->pool->store().kv_armed()) return TG_ERR_KV_ARMED;
        p->pool->restore(s->s);
        p->pool->publish_index();
        return 0;
    });
}
void tg_snapshot_destroy(tg_snapshot* s) {
    if (!s) return;
    Pool::drop(s->s);
    delete s;
}

// ---- host sources ------------------------------------------------------------------
int tg_host_register(tg_tensor_id id, const void* ptr, uint64_t size, const tg_digest* expected) {
    if (!ptr && size) return TG_ERR_BAD_ARG;
    HostSource s;
    s.ptr = ptr;
    s.size = size;
    s.has_expected = expected != nullptr;
    if (expected) s.expected = Digest{expected->hi, expected->lo};
    cudaPointerAttributes a{};
    if (ptr && cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type == cudaMemoryTypeDevice) {
        s.on_device = true;
        s.device = a.device;
    }
    cudaGetLastError();
    SourceRegistry::get().put(key_of(id), s);
    return 0;
}
int tg_file_register(tg_tensor_id id, const char* path, uint64_t file_offset, uint64_t size,
                     const tg_digest* expected) {
    if (!path || !*path) return TG_ERR_BAD_ARG;
    HostSource s;
    s.size = size;
    s.has_expected = expected != nullptr;
    if (expected) s.expected = Digest{expected->hi, expected->lo};
    s.path = path;
    s.file_off = file_offset;
    SourceRegistry::get().put(key_of(id), s);
    return 0;
}
int tg_host_unregister(tg_tensor_id id) {
    SourceRegistry::get().erase(key_of(id));
    return 0;
}
int tg_host_clear(void) {
    SourceRegistry::get().clear();
    return 0;
}
int tg_host_alloc(uint64_t size, void** out) {
    return guard([&] {
        if (cudaMallocHost(out, size) != cudaSuccess) {
            cudaGetLastError();
            g_detail = "cudaMallocHost failed";
            return TG_ERR_CUDA;
        }
        return 0;
    });
}
int tg_host_free(void* p) { return cudaFreeHost(p) == cudaSuccess ? 0 : TG_ERR_CUDA; }

// ---- raw device helpers --------------------------------------------------------------
int tg_fingerprint_device(const void* dptr, uint64_t n, int32_t device, tg_digest* out) {
    return guard([&] {
        Digest d;
        fingerprint_device(dptr, n, device, &d);
        *out = tg_digest{d.hi, d.lo};
        return 0;
    });
}
int tg_bench_fingerprint(const void* const* dptrs, const uint64_t* ns, uint32_t n_bufs, int32_t device, int32_t reps,
                         double* ms, tg_digest* out) {
    return guard([&] {
        std::vector<std::pair<const void*, u64>> b;
        for (uint32_t i = 0; i < n_bufs; ++i) b.push_back({dptrs[i], ns[i]});
        std::vector<Digest> d;
        *ms = bench_fingerprint(b, device, reps < 1 ? 1 : reps, &d);
        for (uint32_t i = 0; out && i < n_bufs; ++i) out[i] = tg_digest{d[i].hi, d[i].lo};
        return 0;
    });
}
int tg_copy_fingerprint(const uint64_t* triples, uint32_t n_moves, int32_t device, int32_t reps, double* ms,
                        tg_digest* out) {
    return guard([&] {
        std::vector<MoveDesc> mv;
        for (uint32_t i = 0; i < n_moves; ++i) mv.push_back(MoveDesc{triples[3 * i], triples[3 * i + 1], triples[3 * i + 2]});
        std::vector<Digest> d;
        const double t = bench_copy_fp(mv, device, reps < 0 ? 0 : reps, &d);
        if (ms) *ms = t;
        for (uint32_t i = 0; out && i < n_moves; ++i) out[i] = tg_digest{d[i].hi, d[i].lo};
        return 0;
    });
}
int tg_bench_relocate(const uint64_t* triples /*src,dst,len*/, uint32_t n_moves, int32_t device, int32_t reps,
                      double* ms) {
    return guard([&] {
        std::vector<MoveDesc> mv;
        for (uint32_t i = 0; i < n_moves; ++i) mv.push_back(MoveDesc{triples[3 * i], triples[3 * i + 1], triples[3 * i + 2]});
        *ms = bench_relocate(mv, device, reps < 1 ? 1 : reps);
        return 0;
    });
}
int tg_synth_fill_device(tg_tensor_id id, uint64_t begin, uint64_t len, void* dptr, int32_t device) {
    return guard([&] {
        synth_fill_device(key_of(id), begin, len, dptr, device);
        return 0;
    });
}
int tg_synth_fill_host(tg_tensor_id id, uint64_t begin, uint64_t len, void* dst, int32_t threads) {
    // host generator for small test inputs; large checkpoints use the device
    // generator + one D2H.
    const u64 seed = id.hi ^ ((id.lo << 17) | (id.lo >> 47));
    auto fill = [&](u64 b, u64 e) {
        auto* out = static_cast<std::uint8_t*>(dst);
        for (u64 pos = b; pos < e;) {
            const u64 w = pos >> 3;
            u64 z = seed ^ (w * 0x9E3779B97F4A7C15ULL);
            z += 0x9E3779B97F4A7C15ULL;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            z ^= z >> 31;
            const u64 b0 = pos & 7, nb = std::min<u64>(8 - b0, e - pos);
            std::memcpy(out + (pos - begin), reinterpret_cast<const std::uint8_t*>(&z) + b0, nb);
            pos += nb;
        }
    };
    if (threads <= 1 || len < (1u << 22)) {
        fill(begin, begin + len);
        return 0;
    }
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t) {
        u64 b = begin + len * t / threads, e = begin + len * (t + 1) / threads;
        ts.emplace_back(fill, b, e);
    }
    for (auto& t : ts) t.join();
    return 0;
}
int tg_device_alloc(int32_t device, uint64_t size, void** out) {
    return guard([&] {
        DeviceScope ds(device);
        TG_CUDA(cudaMalloc(out, size));
        return 0;
    });
}
int tg_device_free(int32_t device, void* p) {
    return guard([&] {
        DeviceScope ds(device);
        TG_CUDA(cudaFree(p));
        return 0;
    });
}
int tg_memcpy(void* dst, const void* src, uint64_t n) {
    return guard([&] {
        TG_CUDA(cudaMemcpy(dst, src, n, cudaMemcpyDefault));
        return 0;
    });
}

// ---- KV engine ---------------------------------------------------------------------------
int tg_kv_create(const char* model_id, uint64_t bs, uint64_t bpt, tg_kv** out) {
    if (!model_id || bs == 0) return TG_ERR_BAD_ARG;
    *out = new tg_kv{std::make_unique<KvAllocator>(model_id, bs, bpt), -2};
    return 0;
}
void tg_kv_destroy(tg_kv* kv) { delete kv; }
int tg_kv_clone(const tg_kv* kv, tg_kv** out) {
    if (kv->a->armed()) return TG_ERR_KV_ARMED;
    return guard([&] {
        *out = new tg_kv{std::make_unique<KvAllocator>(*kv->a), kv->device};
        return 0;
    });
}

int tg_kv_ensure_capacity(tg_kv* kv, tg_pool* p, const tg_stats* s, uint64_t rid, uint64_t tokens, uint64_t* granted,
                          uint64_t cap, uint64_t* n_granted) {
    settle(p);
    return guard([&] {
        if (int rc = bind_kv(kv, p)) return rc;
        std::vector<u64> g;
        u64 n = 0;
        const bool want = granted && p->pool->has_device();
        St st = kv->a->ensure_capacity(p->pool->store(), s->s_view(), rid, tokens, want ? &g : nullptr, &n);
        if (n_granted) *n_granted = n;
        if (want)
            for (u64 i = 0; i < g.size() && i < cap; ++i) granted[i] = g[i];
        p->pool->publish_index();  // a contended grant may have evicted tensors
        return code_of(st);
    });
}

int tg_kv_batch_allocate(tg_kv* kv, tg_pool* p, const tg_stats* s, const uint64_t* rids, const uint64_t* tokens,
                         uint64_t n, uint64_t* counts, uint64_t* pbns, uint64_t cap, uint64_t* total) {
    settle(p);
    return guard([&] {
        if (int rc = bind_kv(kv, p)) return rc;
        std::vector<std::pair<u64, u64>> reqs(n);
        for (uint64_t i = 0; i < n; ++i) reqs[i] = {rids[i], tokens[i]};
        std::vector<u64> c, g;
        const bool want = pbns && p->pool->has_device();
        St st = kv->a->batch_allocate(p->pool->store(), s->s_view(), reqs, &c, want ? &g : nullptr);
        u64 t = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (counts) counts[i] = c[i];
            t += c[i];
        }
        if (total) *total = t;
        if (want)
            for (u64 i = 0; i < g.size() && i < cap; ++i) pbns[i] = g[i];
        p->pool->publish_index();
        return code_of(st);
    });
}

int tg_kv_release_request(tg_kv* kv, uint64_t rid) {
    if (kv->a->armed()) return TG_ERR_KV_ARMED;
    return guard([&] { return code_of(kv->a->release_request(rid)); });
}
int tg_kv_teardown(tg_kv* kv, tg_pool* p) {
    settle(p);
    return guard([&] {
        if (int rc = bind_kv(kv, p)) return rc;
        kv->a->teardown(p->pool->store());
        return 0;
    });
}
int tg_kv_urgent_reclaim(tg_kv* kv, tg_pool* p, const tg_stats* s, uint64_t blocks) {
    settle(p);
    return guard([&] {
        if (int rc = bind_kv(kv, p)) return rc;
        const int rc = code_of(kv->a->urgent_reclaim(p->pool->store(), s->s_view(), blocks));
        p->pool->publish_index();
        return rc;
    });
}
int tg_kv_table(const tg_kv* kv, uint64_t rid, uint64_t* pbns, uint64_t cap, uint64_t* n, uint64_t* token_count) {
    if (kv->a->armed()) return TG_ERR_KV_ARMED;
    return guard([&] {
        if (!kv->a->has_request(rid)) return code_of(Err::NotFound);
        if (token_count) *token_count = kv->a->request_tokens(rid);
        if (n) *n = kv->a->request_blocks(rid);
        if (!pbns) return 0;
        std::vector<u64> t;
        u64 tok = 0;
        St st = kv->a->table(rid, &t, &tok);
        for (u64 i = 0; i < t.size() && i < cap; ++i) pbns[i] = t[i];
        return code_of(st);
    });
}
int tg_kv_address_table(const tg_kv* kv, uint64_t* triples, uint64_t cap, uint64_t* n) {
    u64 cnt = 0;
    std::vector<std::pair<u64, u64>> rows;  // (pbn, off)
    for (const KvRun& r : kv->a->runs())
        for (u64 i = 0; i < r.count; ++i) rows.push_back({r.first_pbn + i, r.off + i * kv->a->block_bytes()});
    std::sort(rows.begin(), rows.end());
    for (const auto& [pbn, off] : rows) {
        if (triples && cnt < cap) {
            triples[3 * cnt] = pbn;
            triples[3 * cnt + 1] = off;
            triples[3 * cnt + 2] = kv->a->block_bytes();
        }
        ++cnt;
    }
    *n = cnt;
    return triples && cnt > cap ? TG_ERR_BUFFER : 0;
}
int tg_kv_stats_get(const tg_kv* kv, tg_kv_stats* o) {
    const KvCounters& c = kv->a->counters();
    *o = tg_kv_stats{c.pool_invocations, c.alloc_batches,       c.blocks_from_free_list, c.blocks_from_pool,
                     c.reclaim_events,   kv->a->free_list_size(), kv->a->active_requests(), kv->a->next_pbn(),
                     kv->a->block_bytes()};
    return 0;
}
int tg_kv_device_tables(const tg_kv* kv, void** tables, uint64_t* stride, void** addr) {
    KvDevice* d = kv->a->device();
    if (!d) return TG_ERR_NO_DEVICE;
    *tables = d->table_ptr();
    *stride = d->table_stride();
    *addr = d->addr_ptr();
    return 0;
}

static int kv_tokens(tg_kv* kv, tg_pool* p, const uint64_t* slots, const uint64_t* pos, void* buf, uint32_t n,
                     void* stream, bool write) {
    return guard([&] {
        KvDevice* d = kv->a->device();
        if (!d || !p->pool->has_device()) return TG_ERR_NO_DEVICE;
        if (kv->device != p->pool->device()) {
            g_detail = "KV engine and pool on different devices";
            return TG_ERR_BAD_ARG;
        }
        const u64 bt = kv->a->block_tokens(), tb = kv->a->block_bytes() / bt;
        return d->tokens(p->pool->arena(), p->pool->store().pool_size(), bt, tb, slots, pos,
                         static_cast<std::uint8_t*>(buf), n, write, stream);
    });
}
int tg_kv_token_faults(tg_kv* kv, uint64_t* faults) {
    return guard([&] {
        KvDevice* d = kv ? kv->a->device() : nullptr;
        if (!d) return TG_ERR_NO_DEVICE;
        if (!faults) return TG_ERR_BAD_ARG;
        *faults = d->token_faults();
        return 0;
    });
}
int tg_kv_wait_tables(tg_kv* kv, void* stream) {
    return guard([&] {
        KvDevice* d = kv ? kv->a->device() : nullptr;
        if (!d) return TG_ERR_NO_DEVICE;
        d->order_after_updates(stream);
        return 0;
    });
}
int tg_kv_reserve(tg_kv* kv, tg_pool* p, uint32_t max_requests, uint64_t max_blocks_per_request,
                  uint64_t max_blocks) {
    settle(p);
    return guard([&] {
        if (!kv || !p) return TG_ERR_BAD_ARG;
        if (int rc = bind_kv(kv, p)) return rc;
        KvDevice* d = kv->a->device();
        if (!d) return TG_ERR_NO_DEVICE;
        return d->reserve(max_requests, max_blocks_per_request, max_blocks, max_blocks + 1);
    });
}
int tg_kv_write_tokens(tg_kv* kv, tg_pool* p, const uint64_t* slots, const uint64_t* pos, const void* buf, uint32_t n,
                       void* stream) {
    settle(p);
    return kv_tokens(kv, p, slots, pos, const_cast<void*>(buf), n, stream, true);
}
int tg_kv_read_tokens(tg_kv* kv, tg_pool* p, const uint64_t* slots, const uint64_t* pos, void* buf, uint32_t n,
                      void* stream) {
    settle(p);
    return kv_tokens(kv, p, slots, pos, buf, n, stream, false);
}

int tg_kv_request_slot(const tg_kv* kv, uint64_t rid, uint32_t* slot) {
    if (!slot) return TG_ERR_BAD_ARG;
    if (!kv->a->has_request(rid)) return code_of(Err::NotFound);
    *slot = kv->a->request_slot(rid);
    return 0;
}
int tg_kv_device_arm(tg_kv* kv, tg_pool* p, uint64_t max_blocks_per_request, uint32_t max_requests,
                     uint32_t max_batches) {
    settle(p);
    return guard([&] {
        if (max_requests > kKvDevMaxRequests) {
            g_detail = "max_requests above the per-batch limit";
            return TG_ERR_BAD_ARG;
        }
        if (int rc = bind_kv(kv, p)) return rc;
        return code_of(kv->a->arm(p->pool->store(), max_blocks_per_request, max_requests, max_batches));
    });
}
int tg_kv_batch_allocate_device(tg_kv* kv, const uint64_t* d_slots, const uint64_t* d_tokens, uint32_t n,
                                void* stream) {
    return guard([&] {
        if (!kv->a->armed()) {
            g_detail = "engine not armed (tg_kv_device_arm)";
            return TG_ERR_BAD_ARG;
        }
        return kv->a->enqueue_device(d_slots, d_tokens, n, stream);
    });
}
int tg_kv_device_sync(tg_kv* kv, tg_pool* p, const tg_stats* s, uint64_t* applied, uint64_t* replayed) {
    settle(p);
    return guard([&] {
        if (!kv->a->armed()) return TG_ERR_BAD_ARG;
        KvAllocator::SyncReport r;
        St st = kv->a->sync(p->pool->store(), s->s_view(), &r);
        if (applied) *applied = r.applied;
        if (replayed) *replayed = r.replayed;
        p->pool->publish_index();  // a replayed contended batch may have evicted tensors
        if (r.overflow) {
            g_detail = "device KV batch log overflowed: batches were dropped";
            return TG_ERR_KV_LOG;
        }
        return code_of(st);
    });
}

// ---- planner ------------------------------------------------------------------------------------
struct tg_plan {
    Plan plan;
    std::vector<TensorDesc> tensors;
};

int tg_plan_allocation(const tg_region* regions, uint64_t n_regions, const tg_tensor_spec* new_tensors,
                       uint32_t n_new, const tg_eviction* candidates, uint32_t n_cand, const tg_tensor_id* immovable,
                       uint32_t n_imm, int32_t strictness, int32_t merge, int32_t keep_order, tg_plan** out) {
    return guard([&] {
        if (!out || (n_regions && !regions)) return TG_ERR_BAD_ARG;
        std::vector<Region> regs;
        u64 pool = 0;
        for (uint64_t i = 0; i < n_regions; ++i) {
            const tg_region& r = regions[i];
            regs.push_back(Region{r.offset, r.size, static_cast<Kind>(r.kind), key_of(r.tensor), r.block_id});
            pool = std::max<u64>(pool, r.offset + r.size);
        }
        const PoolMap map = PoolMap::from_regions(pool, regs);
        auto p = std::make_unique<tg_plan>();
        for (uint32_t i = 0; i < n_new; ++i)
            p->tensors.push_back(TensorDesc{key_of(new_tensors[i].id),
                                            new_tensors[i].model_id ? new_tensors[i].model_id : "",
                                            new_tensors[i].name ? new_tensors[i].name : "", new_tensors[i].size});
        PlanInput in;
        in.pool = &map;
        in.tensors = &p->tensors;
        for (uint32_t i = 0; i < n_cand; ++i)
            in.candidates.push_back(Candidate{key_of(candidates[i].tensor), candidates[i].size, candidates[i].cost,
                                              candidates[i].last_access,
                                              candidates[i].model_id ? candidates[i].model_id : ""});
        for (uint32_t i = 0; i < n_imm; ++i) in.immovable.insert(key_of(immovable[i]));
        in.strictness = strictness ? Strictness::LiteralGuard : Strictness::Functional;
        in.merge = merge ? MergeMode::GlobalMerge : MergeMode::PartitionedGain;
        in.keep_candidate_order = keep_order != 0;
        PoolMap work;
        auto res = make_plan(in, &work);
        if (!res) return code_of(res.error());
        p->plan = std::move(res.value());
        *out = p.release();
        return 0;
    });
}

uint32_t tg_plan_evictions(const tg_plan* p, tg_eviction* buf, uint32_t cap) {
    const auto& ev = p->plan.evictions;
    for (uint32_t i = 0; buf && i < ev.size() && i < cap; ++i)
        buf[i] = tg_eviction{id_of(ev[i].tensor), ev[i].size, ev[i].cost, ev[i].last_access, ev[i].model_id.c_str()};
    return static_cast<uint32_t>(ev.size());
}

uint32_t tg_plan_relocations(const tg_plan* p, tg_relocation* buf, uint32_t cap) {
    const auto& rl = p->plan.relocations;
    for (uint32_t i = 0; buf && i < rl.size() && i < cap; ++i)
        buf[i] = tg_relocation{id_of(rl[i].tensor), rl[i].from, rl[i].to, rl[i].size, 0};
    return static_cast<uint32_t>(rl.size());
}

uint32_t tg_plan_placements(const tg_plan* p, tg_placement* buf, uint32_t cap) {
    const auto& pl = p->plan.placements;
    for (uint32_t i = 0; buf && i < pl.size() && i < cap; ++i) {
        const TensorDesc& t = p->tensors[pl[i].tensor];
        buf[i] = tg_placement{id_of(t.id), pl[i].off, t.size, 0};
    }
    return static_cast<uint32_t>(pl.size());
}

int tg_plan_costs(const tg_plan* p, double* ec, uint64_t* tm, uint64_t* pgp, uint64_t* init, uint64_t* fb) {
    if (ec) *ec = p->plan.total_eviction_cost;
    if (tm) *tm = p->plan.total_merge_cost;
    if (pgp) *pgp = p->plan.pgp_merge_cost;
    if (init) *init = p->plan.initial_merge_cost;
    if (fb) *fb = p->plan.fallback_evictions;
    return 0;
}

void tg_plan_destroy(tg_plan* p) { delete p; }

// ---- scheduler ------------------------------------------------------------------------------
static GpuView view_of(const tg_gpu_snapshot& g) {
    return GpuView{g.gpu_id ? g.gpu_id : "", g.available != 0, g.pool_size, g.free_bytes, g.pcie_bandwidth,
                   g.store_bandwidth, g.nvlink_bandwidth};
}

int tg_schedule(const uint32_t* req, uint32_t n_req, const tg_gpu_snapshot* gpus, uint32_t n_gpus,
                const tg_model_spec* models, uint32_t n_models, const uint64_t* reuse, const uint64_t* peer_reuse,
                uint32_t batch_size, uint64_t block_tokens, int32_t* assignment, double* estimates) {
    return guard([&] {
        std::vector<u32> r(req, req + n_req);
        std::vector<GpuView> g;
        for (uint32_t i = 0; i < n_gpus; ++i) g.push_back(view_of(gpus[i]));
        std::vector<ModelDesc> ms;
        for (uint32_t i = 0; i < n_models; ++i) ms.push_back(model_of(&models[i]));
        std::vector<std::vector<u64>> ru(n_gpus, std::vector<u64>(n_models)), pr;
        for (uint32_t a = 0; a < n_gpus; ++a)
            for (uint32_t b = 0; b < n_models; ++b) ru[a][b] = reuse[a * n_models + b];
        if (peer_reuse) {
            pr.assign(n_gpus, std::vector<u64>(n_models));
            for (uint32_t a = 0; a < n_gpus; ++a)
                for (uint32_t b = 0; b < n_models; ++b) pr[a][b] = peer_reuse[a * n_models + b];
        }
        std::vector<std::vector<double>> est;
        auto out = schedule(r, g, ms, ru, pr, batch_size, block_tokens, estimates ? &est : nullptr);
        for (uint32_t i = 0; i < n_req; ++i) {
            assignment[i] = out[i];
            if (estimates)
                for (uint32_t k = 0; k < n_gpus; ++k) estimates[i * n_gpus + k] = est[i][k];
        }
        return 0;
    });
}

double tg_estimate_load_time(const tg_model_spec* m, uint64_t reuse, const tg_gpu_snapshot* g, uint64_t peer) {
    return estimate_load_time(model_of(m), reuse, view_of(*g), peer);
}

}  // extern "C"
