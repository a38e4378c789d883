// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// JSON-in / JSON-out C-ABI over the *unmodified* reference headers
// (/root/reference/proj/include/warmsim/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libwarmsim_ref.so.  Used by tests/ (differential parity against
// the product library), by tests/golden/make_golden.py (fixture generation) and
// by bench.py's cpu_baseline / --impl reference leg (timing the reference's own
// CPU control plane).  Nothing here is a restatement: every call forwards to the
// reference implementation:
//   ReuseStore           reuse_store.hpp:50-345
//   KvEngine             kv_engine.hpp:43-239
//   plan_allocation      packing.hpp:311-483
//   brute_force_oracle   packing_oracle.hpp:78-181
//   schedule             scheduler.hpp:79-120
//   ModelStatsTable      model.hpp:70-133
//   make_model/catalog   catalog.hpp:37-90
//   Simulator            simulator.hpp:202-856
//   generate_trace       workload.hpp:194-253
//   murmur3/fingerprint  types.hpp:77-146
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "json.hpp"
#include "warmsim/catalog.hpp"
#include "warmsim/kv_engine.hpp"
#include "warmsim/model.hpp"
#include "warmsim/packing.hpp"
#include "warmsim/packing_oracle.hpp"
#include "warmsim/region_pool.hpp"
#include "warmsim/reuse_store.hpp"
#include "warmsim/rng.hpp"
#include "warmsim/scheduler.hpp"
#include "warmsim/simulator.hpp"
#include "warmsim/types.hpp"
#include "warmsim/workload.hpp"

using nlohmann::json;
using namespace warmsim;

namespace {

thread_local std::string g_out;

const char* emit(const json& j) {
    g_out = j.dump();
    return g_out.c_str();
}

TensorId id_from_hex(const std::string& h) {
    TensorId id;
    id.hi = std::stoull(h.substr(0, 16), nullptr, 16);
    id.lo = std::stoull(h.substr(16, 16), nullptr, 16);
    return id;
}

json model_to_json(const ModelSpec& m) {
    json j;
    j["model_id"] = m.model_id;
    j["total_size"] = m.total_size;
    j["latency_sensitivity"] = m.latency_sensitivity;
    j["location"] = to_string(m.location);
    j["bytes_per_token"] = m.bytes_per_token;
    auto ts = json::array();
    for (const auto& t : m.tensors)
        ts.push_back({{"id", t.id.hex()}, {"name", t.name}, {"size", t.size}, {"model_id", t.model_id}});
    j["tensors"] = ts;
    return j;
}

ModelSpec model_from_json(const json& j) {
    ModelSpec m;
    m.model_id = j.at("model_id").get<std::string>();
    m.total_size = j.at("total_size").get<Bytes>();
    m.latency_sensitivity = j.value("latency_sensitivity", 1.0);
    m.location = j.value("location", std::string("model_cache")) == "model_store"
                     ? ModelLocation::ModelStore
                     : ModelLocation::ModelCache;
    m.bytes_per_token = j.value("bytes_per_token", Bytes{0});
    for (const auto& t : j.at("tensors")) {
        TensorSpec s;
        s.id = id_from_hex(t.at("id").get<std::string>());
        s.name = t.at("name").get<std::string>();
        s.size = t.at("size").get<Bytes>();
        s.model_id = t.value("model_id", m.model_id);
        m.tensors.push_back(s);
    }
    return m;
}

json plan_to_json(const AllocationPlan& p) {
    json j;
    auto ev = json::array();
    for (const auto& e : p.evictions)
        ev.push_back({{"tensor", e.tensor.hex()}, {"size", e.size}, {"cost", e.cost},
                      {"last_access", e.last_access}, {"model", e.model_id}});
    auto rl = json::array();
    for (const auto& r : p.relocations)
        rl.push_back({{"tensor", r.tensor.hex()}, {"from", r.from}, {"to", r.to}, {"size", r.size}});
    auto pl = json::array();
    for (const auto& x : p.placements)
        pl.push_back({{"tensor", x.tensor.id.hex()}, {"offset", x.offset}, {"size", x.tensor.size}});
    j["evictions"] = ev;
    j["relocations"] = rl;
    j["placements"] = pl;
    j["total_eviction_cost"] = p.total_eviction_cost;
    j["total_merge_cost"] = p.total_merge_cost;
    j["pgp_merge_cost"] = p.pgp_merge_cost;
    j["initial_merge_cost"] = p.initial_merge_cost;
    j["fallback_evictions"] = p.fallback_evictions;
    return j;
}

Region region_from_json(const json& r) {
    Region out;
    out.offset = r.at("offset").get<Bytes>();
    out.size = r.at("size").get<Bytes>();
    const auto st = r.at("state").get<std::string>();
    out.kind = st == "free" ? RegionKind::Free : st == "tensor" ? RegionKind::Tensor : RegionKind::KvBlock;
    if (out.kind == RegionKind::Tensor) out.tensor = id_from_hex(r.at("tensor").get<std::string>());
    if (out.kind == RegionKind::KvBlock) out.block_id = r.value("block", std::uint64_t{0});
    return out;
}

json err(Error e) { return json{{"ok", false}, {"error", static_cast<int>(e)}}; }

struct Registry {
    std::map<int, std::unique_ptr<ReuseStore>> stores;
    std::map<int, std::unique_ptr<ModelStatsTable>> stats;
    std::map<int, std::unique_ptr<KvEngine>> kvs;
    std::map<int, std::unique_ptr<Rng>> rngs;
    int next = 1;
};
Registry& reg() {
    static Registry r;
    return r;
}

LoadPolicy policy_from_json(const json& j) {
    LoadPolicy p;
    p.merge = j.value("merge", 0) ? MergePolicy::GlobalMerge : MergePolicy::PartitionedGain;
    p.strictness = j.value("strictness", 0) ? PackingStrictness::LiteralGuard : PackingStrictness::Functional;
    p.random_eviction = j.value("random_eviction", false);
    const int rng = j.value("rng", 0);
    p.rng = rng ? reg().rngs.at(rng).get() : nullptr;
    return p;
}

json outcome_to_json(const LoadOutcome& o) {
    json j;
    j["ok"] = true;
    auto h = json::array();
    for (const auto& id : o.hit_tensors) h.push_back(id.hex());
    auto m = json::array();
    for (const auto& t : o.missed_tensors) m.push_back(t.id.hex());
    j["hits"] = h;
    j["misses"] = m;
    j["bytes_transferred"] = o.bytes_transferred;
    j["bytes_merged"] = o.bytes_merged;
    j["eviction_cost_total"] = o.eviction_cost_total;
    j["plan"] = plan_to_json(o.plan);
    return j;
}

json kv_state(const KvEngine& kv) {
    json j;
    // Tables are only reachable per request id; the caller passes the ids it
    // cares about through ref_kv_table.  Here: address table + counters.
    auto at = json::array();
    for (const auto& [pbn, ext] : kv.address_table()) at.push_back({pbn, ext.first, ext.second});
    j["address_table"] = at;
    j["free_list_size"] = kv.free_list_size();
    j["active_requests"] = kv.active_requests();
    const auto& s = kv.stats();
    j["stats"] = {{"pool_invocations", s.pool_invocations}, {"alloc_batches", s.alloc_batches},
                  {"blocks_from_free_list", s.blocks_from_free_list},
                  {"blocks_from_pool", s.blocks_from_pool}, {"reclaim_events", s.reclaim_events}};
    return j;
}

}  // namespace

extern "C" {

// ---- ids / hashing --------------------------------------------------------
void ref_murmur3(const void* data, std::uint64_t len, std::uint64_t seed, std::uint64_t out[2]) {
    const TensorId id = detail::murmur3_x64_128(data, len, seed);
    out[0] = id.hi;
    out[1] = id.lo;
}

const char* ref_fingerprint(const char* model_id, const char* name, const std::int64_t* shape, int ndim,
                            int etype) {
    std::vector<std::int64_t> s(shape, shape + ndim);
    return emit(fingerprint(model_id, name, s, static_cast<ElementType>(etype)).hex());
}

// ---- catalog --------------------------------------------------------------
const char* ref_default_catalog() {
    auto arr = json::array();
    for (const auto& m : default_catalog()) arr.push_back(model_to_json(m));
    return emit(arr);
}

const char* ref_make_model(const char* model_id, std::uint64_t total, int layers, std::uint64_t bpt) {
    return emit(model_to_json(make_model(model_id, total, layers, bpt)));
}

// ---- stats ----------------------------------------------------------------
int ref_stats_create(double decay) {
    auto& r = reg();
    r.stats[r.next] = std::make_unique<ModelStatsTable>(decay);
    return r.next++;
}
int ref_stats_record_request(int h, const char* model_id, double t) {
    auto st = reg().stats.at(h)->record_request(model_id, t);
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
int ref_stats_record_eviction(int h, const char* model_id, double t) {
    auto st = reg().stats.at(h)->record_eviction(model_id, t);
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
void ref_stats_set_load_bandwidth(int h, const char* model_id, double b) {
    reg().stats.at(h)->set_load_bandwidth(model_id, b);
}
double ref_stats_miss_probability(int h, const char* model_id) {
    return reg().stats.at(h)->miss_probability(model_id);
}

int ref_rng_create(std::uint64_t seed) {
    auto& r = reg();
    r.rngs[r.next] = std::make_unique<Rng>(seed);
    return r.next++;
}

// ---- store ----------------------------------------------------------------
int ref_store_create(const char* gpu_id, std::uint64_t pool, double pcie, double intra, double store_bw) {
    auto& r = reg();
    GpuSpec g{gpu_id, pool, pcie, intra, store_bw};
    r.stores[r.next] = std::make_unique<ReuseStore>(g);
    return r.next++;
}
int ref_store_clone(int h) {
    auto& r = reg();
    r.stores[r.next] = std::make_unique<ReuseStore>(*r.stores.at(h));
    return r.next++;
}
void ref_destroy(int h) {
    auto& r = reg();
    r.stores.erase(h);
    r.stats.erase(h);
    r.kvs.erase(h);
    r.rngs.erase(h);
}

const char* ref_load_model(int store, const char* model_json, int stats, double clock, const char* policy_json) {
    auto& r = reg();
    const ModelSpec m = model_from_json(json::parse(model_json));
    const LoadPolicy p = policy_from_json(json::parse(policy_json));
    auto res = r.stores.at(store)->load_model(m, *r.stats.at(stats), clock, p);
    if (!res.ok()) return emit(err(res.error()));
    return emit(outcome_to_json(res.value()));
}

// Same as ref_load_model but also reports the wall time of load_model itself
// (the reference's CPU control plane) in ns; used by the CPU baseline.
const char* ref_load_model_timed(int store, const char* model_json, int stats, double clock,
                                 const char* policy_json) {
    auto& r = reg();
    const ModelSpec m = model_from_json(json::parse(model_json));
    const LoadPolicy p = policy_from_json(json::parse(policy_json));
    const auto t0 = std::chrono::steady_clock::now();
    auto res = r.stores.at(store)->load_model(m, *r.stats.at(stats), clock, p);
    const auto t1 = std::chrono::steady_clock::now();
    json j = res.ok() ? outcome_to_json(res.value()) : err(res.error());
    j["ns"] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    return emit(j);
}

void ref_end_instance(int store, const char* model_id) { reg().stores.at(store)->end_instance(model_id); }

int ref_evict_tensor(int store, const char* hex) {
    auto st = reg().stores.at(store)->evict_tensor(id_from_hex(hex));
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
void ref_evict_model(int store, const char* model_id) { reg().stores.at(store)->evict_model(model_id); }
int ref_move_tensor(int store, const char* hex, std::uint64_t to) {
    auto st = reg().stores.at(store)->move_tensor(id_from_hex(hex), to);
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
int ref_alloc_kv_region(int store, std::uint64_t size, std::uint64_t block_id, std::uint64_t* off) {
    auto res = reg().stores.at(store)->alloc_kv_region(size, block_id);
    if (!res.ok()) return 1 + static_cast<int>(res.error());
    *off = res.value();
    return 0;
}
int ref_free_kv_region(int store, std::uint64_t off) {
    auto st = reg().stores.at(store)->free_kv_region(off);
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
int ref_validate(int store) {
    auto st = reg().stores.at(store)->validate();
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
const char* ref_dump(int store) { return emit(reg().stores.at(store)->dump()); }

const char* ref_store_info(int store) {
    const auto& s = *reg().stores.at(store);
    return emit(json{{"pool_size", s.pool_size()}, {"free_bytes", s.free_bytes()},
                     {"kv_bytes", s.kv_bytes()}, {"pinned_tensor_bytes", s.pinned_tensor_bytes()},
                     {"pinned_bytes", s.pinned_bytes()}, {"reusable_bytes", s.reusable_bytes()},
                     {"bytes_merged_total", s.bytes_merged_total()},
                     {"bytes_transferred_total", s.bytes_transferred_total()},
                     {"evictions_total", s.evictions_total()}, {"region_count", s.regions().region_count()},
                     {"largest_free", s.regions().largest_free()}});
}

const char* ref_lookup(int store, const char* model_json) {
    const ModelSpec m = model_from_json(json::parse(model_json));
    auto [hits, misses] = reg().stores.at(store)->lookup(m);
    json j;
    j["hits"] = json::array();
    for (const auto& h : hits) j["hits"].push_back(h.hex());
    j["misses"] = json::array();
    for (const auto& t : misses) j["misses"].push_back(t.id.hex());
    j["reuse_size"] = reg().stores.at(store)->reuse_size(m);
    return emit(j);
}

const char* ref_eviction_candidates(int store, int stats, const char* exclude) {
    auto c = reg().stores.at(store)->eviction_candidates(*reg().stats.at(stats), exclude);
    auto arr = json::array();
    for (const auto& e : c)
        arr.push_back({{"tensor", e.tensor.hex()}, {"size", e.size}, {"cost", e.cost},
                       {"last_access", e.last_access}, {"model", e.model_id}});
    return emit(arr);
}

// ---- KV engine ------------------------------------------------------------
int ref_kv_create(const char* model_id, std::uint64_t bs, std::uint64_t bpt) {
    auto& r = reg();
    r.kvs[r.next] = std::make_unique<KvEngine>(model_id, bs, bpt);
    return r.next++;
}
const char* ref_kv_batch_allocate(int kv, int store, int stats, const std::uint64_t* rids,
                                  const std::uint64_t* tokens, std::uint64_t n) {
    auto& r = reg();
    std::vector<std::pair<std::uint64_t, std::uint64_t>> req;
    for (std::uint64_t i = 0; i < n; ++i) req.push_back({rids[i], tokens[i]});
    const auto t0 = std::chrono::steady_clock::now();
    auto res = r.kvs.at(kv)->batch_allocate(*r.stores.at(store), *r.stats.at(stats), req);
    const auto t1 = std::chrono::steady_clock::now();
    json j;
    j["ns"] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    if (!res.ok()) {
        j["ok"] = false;
        j["error"] = static_cast<int>(res.error());
        return emit(j);
    }
    j["ok"] = true;
    j["granted"] = res.value();
    return emit(j);
}
const char* ref_kv_ensure_capacity(int kv, int store, int stats, std::uint64_t rid, std::uint64_t tokens) {
    auto& r = reg();
    auto res = r.kvs.at(kv)->ensure_capacity(*r.stores.at(store), *r.stats.at(stats), rid, tokens);
    if (!res.ok()) return emit(err(res.error()));
    return emit(json{{"ok", true}, {"granted", res.value()}});
}
int ref_kv_release_request(int kv, std::uint64_t rid) {
    auto st = reg().kvs.at(kv)->release_request(rid);
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
void ref_kv_teardown(int kv, int store) { reg().kvs.at(kv)->instance_teardown(*reg().stores.at(store)); }
int ref_kv_urgent_reclaim(int kv, int store, int stats, std::uint64_t blocks) {
    auto& r = reg();
    auto st = r.kvs.at(kv)->urgent_reclaim(*r.stores.at(store), *r.stats.at(stats), blocks);
    return st.ok() ? 0 : 1 + static_cast<int>(st.error());
}
const char* ref_kv_table(int kv, std::uint64_t rid) {
    const auto* t = reg().kvs.at(kv)->table(rid);
    if (!t) return emit(json(nullptr));
    auto arr = json::array();
    for (const auto& [lbn, pbn] : t->lbn_to_pbn) arr.push_back({lbn, pbn});
    return emit(json{{"request_id", t->request_id}, {"token_count", t->token_count}, {"lbn_to_pbn", arr}});
}
const char* ref_kv_state(int kv) { return emit(kv_state(*reg().kvs.at(kv))); }

// ---- planner-level ----------------------------------------------------------
// request: {"regions":[...dump regions...], "new_tensors":[{id,size,model_id,name}],
//           "candidates":[{tensor,size,cost,last_access,model}], "immovable":[hex],
//           "strictness":0|1, "merge_policy":0|1, "randomize_eviction":bool}
const char* ref_plan_allocation(const char* request_json) {
    const json j = json::parse(request_json);
    PlanRequest req;
    for (const auto& r : j.at("regions")) req.regions.push_back(region_from_json(r));
    for (const auto& t : j.at("new_tensors")) {
        TensorSpec s;
        s.id = id_from_hex(t.at("id").get<std::string>());
        s.size = t.at("size").get<Bytes>();
        s.model_id = t.value("model_id", std::string(""));
        s.name = t.value("name", std::string(""));
        req.new_tensors.push_back(s);
    }
    for (const auto& c : j.at("candidates")) {
        EvictionCandidate e;
        e.tensor = id_from_hex(c.at("tensor").get<std::string>());
        e.size = c.at("size").get<Bytes>();
        e.cost = c.at("cost").get<double>();
        e.last_access = c.at("last_access").get<double>();
        e.model_id = c.value("model", std::string(""));
        req.candidates.push_back(e);
    }
    for (const auto& h : j.value("immovable", json::array())) req.immovable.insert(id_from_hex(h.get<std::string>()));
    req.strictness = j.value("strictness", 0) ? PackingStrictness::LiteralGuard : PackingStrictness::Functional;
    req.merge_policy = j.value("merge_policy", 0) ? MergePolicy::GlobalMerge : MergePolicy::PartitionedGain;
    req.randomize_eviction = j.value("randomize_eviction", false);
    auto res = plan_allocation(req);
    if (!res.ok()) return emit(err(res.error()));
    json out = plan_to_json(res.value());
    out["ok"] = true;
    return emit(out);
}

const char* ref_try_packing(const std::uint64_t* sizes, std::uint64_t n, std::uint64_t c1, std::uint64_t c2,
                            int strictness) {
    std::vector<TensorSpec> ts;
    for (std::uint64_t i = 0; i < n; ++i) {
        TensorSpec t;
        t.id = TensorId{0, i};
        t.size = sizes[i];
        ts.push_back(t);
    }
    auto r = try_packing(ts, c1, c2, strictness ? PackingStrictness::LiteralGuard : PackingStrictness::Functional);
    json j{{"success", r.success}};
    j["first"] = json::array();
    j["second"] = json::array();
    for (const auto& t : r.first) j["first"].push_back(t.size);
    for (const auto& t : r.second) j["second"].push_back(t.size);
    return emit(j);
}

const char* ref_brute_force_oracle(const char* instance_json) {
    const json j = json::parse(instance_json);
    OracleInstance inst;
    for (const auto& r : j.at("regions")) inst.regions.push_back(region_from_json(r));
    for (const auto& t : j.at("new_tensors")) {
        TensorSpec s;
        s.id = id_from_hex(t.at("id").get<std::string>());
        s.size = t.at("size").get<Bytes>();
        inst.new_tensors.push_back(s);
    }
    for (const auto& c : j.at("candidates")) {
        EvictionCandidate e;
        e.tensor = id_from_hex(c.at("tensor").get<std::string>());
        e.size = c.at("size").get<Bytes>();
        e.cost = c.at("cost").get<double>();
        inst.candidates.push_back(e);
    }
    for (const auto& h : j.value("immovable", json::array())) inst.immovable.insert(id_from_hex(h.get<std::string>()));
    inst.intra_copy_bandwidth = j.value("intra_copy_bandwidth", 1.0);
    auto res = brute_force_oracle(inst);
    if (!res.ok()) return emit(err(res.error()));
    const auto& o = res.value();
    return emit(json{{"ok", true}, {"feasible", o.feasible}, {"best_cost", o.feasible ? o.best_cost : -1.0},
                     {"eviction_cost", o.eviction_cost}, {"merge_bytes", o.merge_bytes}});
}

// ---- scheduler --------------------------------------------------------------
// in: {"requests":[model ids], "snapshots":[{gpu_id,available,pool_size,free_bytes,
//      reuse:{model:bytes}, pcie, store}], "models":[model json], "batch_size", "block_size_tokens"}
static const char* ref_schedule_impl(const char* in_json);
const char* ref_schedule(const char* in_json) {
    try {
        return ref_schedule_impl(in_json);
    } catch (const std::exception& e) {
        return emit(json{{"exception", e.what()}});
    }
}
static const char* ref_schedule_impl(const char* in_json) {
    const json j = json::parse(in_json);
    std::vector<std::string> reqs = j.at("requests").get<std::vector<std::string>>();
    std::vector<GpuSnapshot> snaps;
    for (const auto& s : j.at("snapshots")) {
        GpuSnapshot g;
        g.gpu_id = s.at("gpu_id").get<std::string>();
        g.available = s.value("available", true);
        g.pool_size = s.at("pool_size").get<Bytes>();
        g.free_bytes = s.value("free_bytes", Bytes{0});
        const json reuse = s.value("reuse", json::object());
        for (const auto& [k, v] : reuse.items()) g.reuse_size_by_model[k] = v.get<Bytes>();
        g.pcie_bandwidth = s.at("pcie").get<double>();
        g.store_bandwidth = s.at("store").get<double>();
        snaps.push_back(g);
    }
    std::map<std::string, ModelSpec> registry;
    for (const auto& m : j.at("models")) {
        auto spec = model_from_json(m);
        registry.emplace(spec.model_id, spec);
    }
    SchedulerConfig cfg{j.value("batch_size", 1u), j.value("block_size_tokens", std::uint64_t{16})};
    auto d = schedule(reqs, snaps, registry, cfg);
    json out;
    out["assignments"] = json::array();
    for (const auto& [m, g] : d.assignments) out["assignments"].push_back({m, g});
    out["deferred"] = d.deferred;
    out["entries"] = json::array();
    for (const auto& e : d.entries) {
        json je{{"model_id", e.model_id}};
        je["candidates"] = json::array();
        for (const auto& [g, est] : e.candidates) je["candidates"].push_back({g, est});
        je["chosen"] = e.chosen ? json(*e.chosen) : json(nullptr);
        out["entries"].push_back(je);
    }
    return emit(out);
}

// ---- workload / simulator -----------------------------------------------------
const char* ref_sample_lengths(std::uint64_t seed, const char* dataset, std::uint64_t n) {
    Rng rng(seed);
    auto prof = default_length_profiles();
    auto arr = json::array();
    for (std::uint64_t i = 0; i < n; ++i) {
        auto [p, o] = sample_lengths(prof, dataset, rng);
        arr.push_back({p, o});
    }
    return emit(arr);
}

// in: {"trace": {seed,num_requests,locality,mean_interarrival,zipf_s,repeat_probability},
//      "sim": {n_gpus,pool_size,pcie,intra,store,mode,batch_size,keep_alive,merge,eviction,strictness}}
const char* ref_simulate(const char* in_json) {
    const json j = json::parse(in_json);
    const auto catalog = default_catalog();
    const json& tj = j.at("trace");
    TraceSpec ts;
    ts.seed = tj.value("seed", std::uint64_t{42});
    ts.num_requests = tj.at("num_requests").get<std::uint64_t>();
    ts.locality = locality_from_string(tj.value("locality", std::string("L3")));
    ts.mean_interarrival = tj.value("mean_interarrival", 1.0);
    ts.zipf_s = tj.value("zipf_s", 1.1);
    ts.repeat_probability = tj.value("repeat_probability", 0.6);
    for (const auto& m : catalog) ts.model_ids.push_back(m.model_id);
    const Trace trace = generate_trace(ts);
    const json& sj = j.at("sim");
    SimConfig cfg;
    const int n = sj.at("n_gpus").get<int>();
    for (int g = 0; g < n; ++g)
        cfg.gpus.push_back(GpuSpec{"gpu" + std::to_string(g), sj.at("pool_size").get<Bytes>(),
                                   sj.value("pcie", 55e9), sj.value("intra", 3000e9), sj.value("store", 12e9)});
    cfg.mode = sim_mode_from_string(sj.value("mode", std::string("reuse_odkv")));
    cfg.batch_size = sj.value("batch_size", 1u);
    cfg.keep_alive = sj.value("keep_alive", 240.0);
    cfg.merge = sj.value("merge", 0) ? MergePolicy::GlobalMerge : MergePolicy::PartitionedGain;
    cfg.eviction = sj.value("eviction", 0) ? EvictionSelection::Random : EvictionSelection::MinCost;
    cfg.strictness = sj.value("strictness", 0) ? PackingStrictness::LiteralGuard : PackingStrictness::Functional;
    Simulator sim(cfg, catalog);
    const auto t0 = std::chrono::steady_clock::now();
    RunMetrics m = sim.run(trace);
    const auto t1 = std::chrono::steady_clock::now();
    json out;
    out["ns"] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    out["total_bytes_transferred"] = m.aggregates.total_bytes_transferred;
    out["total_bytes_merged"] = m.aggregates.total_bytes_merged;
    out["cold_starts"] = m.aggregates.cold_starts;
    out["warm_joins"] = m.aggregates.warm_joins;
    out["evictions"] = m.evictions;
    out["mean_ttft"] = m.aggregates.mean_ttft;
    out["p99_ttft"] = m.aggregates.p99_ttft;
    out["makespan"] = m.makespan;
    out["deferral_events"] = m.deferral_events;
    out["early_terminations"] = m.early_terminations;
    out["kv"] = {m.kv.pool_invocations, m.kv.alloc_batches, m.kv.blocks_from_free_list, m.kv.blocks_from_pool,
                 m.kv.reclaim_events};
    auto recs = json::array();
    for (const auto& r : m.records)
        recs.push_back({r.request_id, r.gpu_id, r.cold_start, r.bytes_transferred, r.bytes_merged, r.ttft});
    out["records"] = recs;
    return emit(out);
}

}  // extern "C"
