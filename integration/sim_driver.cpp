// Drop-in check driver: runs the reference's own discrete-event Simulator
// (simulator.hpp, unmodified) on a generated trace and prints RunMetrics as
// JSON.  Built twice by integration/Makefile: once against the pure reference
// headers, once with integration/ first on the include path so that
// "warmsim/reuse_store.hpp" and "warmsim/kv_engine.hpp" resolve to the B200
// bindings.  tests/test_dropin.py requires byte-identical output.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>

#include "json.hpp"
#include "warmsim/catalog.hpp"
#include "warmsim/simulator.hpp"
#include "warmsim/workload.hpp"

int main(int argc, char** argv) {
    using namespace warmsim;
    if (argc < 11) {
        std::fprintf(stderr,
                     "usage: %s mode n_gpus pool_gib batch keep_alive n_requests seed eviction merge locality "
                     "[model,model,...]\n",
                     argv[0]);
        return 2;
    }
    const std::string mode = argv[1];
    const int n = std::atoi(argv[2]);
    const double pool_gib = std::atof(argv[3]);
    // optional 11th argument: the catalog models the trace draws from
    // (default: all of default_catalog())
    auto catalog = default_catalog();
    if (argc > 11) {
        std::vector<ModelSpec> keep;
        std::stringstream ss(argv[11]);
        for (std::string id; std::getline(ss, id, ',');)
            for (const auto& m : catalog)
                if (m.model_id == id) keep.push_back(m);
        catalog = keep;
    }
    TraceSpec ts;
    ts.seed = std::strtoull(argv[7], nullptr, 10);
    ts.num_requests = std::strtoull(argv[6], nullptr, 10);
    ts.locality = locality_from_string(argv[10]);
    ts.mean_interarrival = 0.5;
    for (const auto& m : catalog) ts.model_ids.push_back(m.model_id);
    const Trace trace = generate_trace(ts);
    SimConfig cfg;
    for (int g = 0; g < n; ++g)
        cfg.gpus.push_back(GpuSpec{"gpu" + std::to_string(g), static_cast<Bytes>(pool_gib * (1ull << 30)), 55e9,
                                   3000e9, 12e9});
    cfg.mode = sim_mode_from_string(mode);
    cfg.batch_size = static_cast<std::uint32_t>(std::atoi(argv[4]));
    cfg.keep_alive = std::atof(argv[5]);
    cfg.eviction = std::atoi(argv[8]) ? EvictionSelection::Random : EvictionSelection::MinCost;
    cfg.merge = std::atoi(argv[9]) ? MergePolicy::GlobalMerge : MergePolicy::PartitionedGain;
    cfg.emit_alloc_log = true;
    cfg.emit_sched_log = true;
    cfg.emit_timeseries = true;
#ifdef TANGRAM_BINDING
    // Byte sources for every catalog tensor (TANGRAM_SYNTH_SOURCES): "1" or
    // "device" synthesises them in HBM on device 0 (an HBM model cache: pools
    // place them with the load kernel); "host" in pinned host memory (pools
    // load them over their PCIe link).  Pools that own a device then move
    // real bytes.
    std::vector<void*> sources, host_sources;
    if (const char* mode = std::getenv("TANGRAM_SYNTH_SOURCES")) {
        const bool host = std::string(mode) == "host";
        void* scratch = nullptr;
        Bytes biggest = 0;
        for (const auto& model : catalog)
            for (const auto& t : model.tensors) biggest = std::max(biggest, t.size);
        if (host && tg_device_alloc(0, biggest, &scratch)) return 3;
        for (const auto& model : catalog)
            for (const auto& t : model.tensors) {
                void* d = nullptr;
                const tg_tensor_id id{t.id.hi, t.id.lo};
                int rc = 0;
                if (host) {
                    rc = tg_host_alloc(t.size, &d);
                    if (!rc) rc = tg_synth_fill_device(id, 0, t.size, scratch, 0);
                    if (!rc) rc = tg_memcpy(d, scratch, t.size);
                    if (!rc) host_sources.push_back(d);
                } else {
                    rc = tg_device_alloc(0, t.size, &d);
                    if (!rc) rc = tg_synth_fill_device(id, 0, t.size, d, 0);
                    if (!rc) sources.push_back(d);
                }
                if (rc || tg_host_register(id, d, t.size, nullptr)) {
                    std::fprintf(stderr, "source setup failed: %s\n", tg_last_error_detail());
                    return 3;
                }
            }
        if (scratch) tg_device_free(0, scratch);
    }
#endif
    RunMetrics m;
    double replay_s = 0, setup_s = 0, run_s = 0;
    try {
        using sclk = std::chrono::steady_clock;
        auto secs = [](sclk::time_point a, sclk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
        const auto t0 = sclk::now();
        auto t1 = t0;
        {
            Simulator sim(cfg, catalog);  // creates the pools (arena allocation)
            t1 = sclk::now();
            m = sim.run(trace);
        }  // the stores' destructors land any load still in flight
        const auto t3 = sclk::now();
        replay_s = secs(t0, t3);
        setup_s = secs(t0, t1);
        run_s = secs(t1, t3);  // the run plus landing every load still in flight
    } catch (const std::exception& e) {  // ConfigError / RuntimeInfeasible: compare those too
        std::cout << nlohmann::json{{"exception", e.what()}}.dump() << "\n";
        return 0;
    }
#ifndef TANGRAM_BINDING
    (void)replay_s;
    (void)setup_s;
    (void)run_s;
#endif
#ifdef TANGRAM_BINDING
    // data-plane totals per pool (stderr, so stdout stays comparable)
    auto pools = nlohmann::json::array();
    for (const auto& [gid, i] : tgb::finished_pools())
        pools.push_back({{"gpu_id", gid}, {"device", i.device}, {"loads", i.loads}, {"data_plane_ms", i.data_plane_ms},
                         {"pcie_bytes", i.pcie_bytes}, {"peer_bytes", i.peer_bytes},
                         {"device_src_bytes", i.device_src_bytes}, {"fingerprint_bytes", i.fingerprint_bytes},
                         {"relocated_bytes", i.relocated_bytes}, {"verify_mismatches", i.verify_mismatches},
                         {"repaired_bytes", i.repaired_bytes}, {"failed_loads", i.failed_loads}});
    // replay_s: wall time of the simulator's construction, run and
    // destruction (every pool's data plane has finished inside it)
    std::cerr << nlohmann::json{{"pools", pools}, {"replay_s", replay_s}, {"setup_s", setup_s}, {"run_s", run_s}}.dump()
              << "\n";
    for (void* d : sources) tg_device_free(0, d);
    for (void* d : host_sources) tg_host_free(d);
#endif
    nlohmann::json j;
    auto recs = nlohmann::json::array();
    for (const auto& r : m.records)
        recs.push_back({r.request_id, r.model_id, r.gpu_id, r.t_arrival, r.t_scheduled, r.queued_time, r.t_init,
                        r.t_load, r.t_profile, r.t_prefill, r.ttft, r.t_complete, r.bytes_transferred,
                        r.bytes_merged, r.cold_start});
    j["records"] = recs;
    const auto& a = m.aggregates;
    j["aggregates"] = {a.mean_ttft, a.p99_ttft, a.mean_load, a.total_bytes_transferred, a.total_bytes_merged,
                       a.mean_pool_utilization, a.cold_starts, a.warm_joins};
    j["counters"] = {m.makespan, m.deferral_events, m.evictions, m.early_terminations, m.odkv_overhead_total,
                     m.load_compute_total, m.load_merge_total, m.load_transfer_total};
    j["kv"] = {m.kv.pool_invocations, m.kv.alloc_batches, m.kv.blocks_from_free_list, m.kv.blocks_from_pool,
               m.kv.reclaim_events};
    auto ts_arr = nlohmann::json::array();
    for (const auto& s : m.timeseries) ts_arr.push_back({s.t, s.reusable, s.free_bytes, s.kv_bytes, s.utilization});
    j["timeseries"] = ts_arr;
    auto al = nlohmann::json::array();
    for (const auto& r : m.alloc_log) al.push_back({r.t, r.request_id, r.blocks, r.source});
    j["alloc_log"] = al;
    j["sched_log"] = m.sched_log;
    std::cout << j.dump() << "\n";
    return 0;
}
