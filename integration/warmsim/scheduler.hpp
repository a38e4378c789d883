// Drop-in binding: warmsim's affinity scheduler (scheduler.hpp:23-120) over
// the B200 library's schedule (tg_schedule, csrc/host/sched.cpp), with an
// opt-in peer term.
//
// Same declarations as the reference header, so the unmodified simulator
// compiles against it (-I<repo>/integration first).  By default the decision
// and every estimate are the reference's: (S - S') / B with B = pcie, or
// min(store, pcie) for Model Store models (scheduler.hpp:41-48); greedy queue
// order, ties to the smaller gpu_id, a chosen GPU leaves the pass
// (scheduler.hpp:79-120) — RunMetrics stay byte-identical.
//
// TANGRAM_PEER_SCHEDULE=<GB/s> turns the peer term on: bytes
// of the model that are missing on a GPU but resident and verified in another
// live device pool of this process move over NVLink at that bandwidth,
//     t = (S - S'_local - S'_peer) / B + S'_peer / B_nvlink,
// and the bindings link every device pool to every other one as an NVLink
// peer and load with TG_LOAD_PEER, so those misses really come from the peer
// pool instead of over PCIe.  Decisions then differ from the reference's by
// design (the reference has no peer term).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <limits>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "tangram.h"
#include "warmsim/model.hpp"
#include "warmsim/types.hpp"

namespace warmsim {

struct GpuSnapshot {
    std::string gpu_id;
    bool available = true;
    Bytes pool_size = 0;
    Bytes free_bytes = 0;
    std::map<std::string, Bytes> reuse_size_by_model;  // S' per model
    BytesPerSecond pcie_bandwidth = 0;
    BytesPerSecond store_bandwidth = 0;

    Bytes reuse_size_of(const std::string& model_id) const {
        auto it = reuse_size_by_model.find(model_id);
        return it == reuse_size_by_model.end() ? 0 : it->second;
    }
};

namespace tgs {

// NVLink bandwidth of the peer term (bytes/s); 0 = off (reference behaviour).
inline double peer_bandwidth() {
    static const double bw = [] {
        const char* e = std::getenv("TANGRAM_PEER_SCHEDULE");
        return e ? std::atof(e) * 1e9 : 0.0;
    }();
    return bw;
}

// Live device pools of this process by gpu_id (registered by the
// ReuseStore bindings): where the peer term looks for resident bytes.
inline std::map<std::string, tg_pool*>& live_pools() {
    static std::map<std::string, tg_pool*> m;
    return m;
}

inline tg_model_spec spec_of(const ModelSpec& m, std::vector<tg_tensor_spec>* t) {
    t->clear();
    for (const auto& x : m.tensors)
        t->push_back(tg_tensor_spec{tg_tensor_id{x.id.hi, x.id.lo}, x.name.c_str(), x.size, x.model_id.c_str()});
    return tg_model_spec{m.model_id.c_str(), t->data(), static_cast<uint32_t>(t->size()), m.total_size,
                         m.latency_sensitivity, m.location == ModelLocation::ModelStore ? 1 : 0, m.bytes_per_token};
}

inline tg_gpu_snapshot view_of(const GpuSnapshot& g) {
    return tg_gpu_snapshot{g.gpu_id.c_str(), g.available ? 1 : 0, g.pool_size, g.free_bytes, g.pcie_bandwidth,
                           g.store_bandwidth, peer_bandwidth()};
}

}  // namespace tgs

/// Expected loading time (S - S') / B (scheduler.hpp:41-48; peer term off).
inline Seconds estimate_load_time(const ModelSpec& model, Bytes reuse_size, const GpuSnapshot& gpu) {
    std::vector<tg_tensor_spec> t;
    const tg_model_spec m = tgs::spec_of(model, &t);
    tg_gpu_snapshot g = tgs::view_of(gpu);
    g.nvlink_bandwidth = 0;
    return tg_estimate_load_time(&m, reuse_size, &g, 0);
}

/// Feasibility (scheduler.hpp:52-54).
inline bool can_run(const ModelSpec& model, const GpuSnapshot& snapshot, Bytes kv_headroom) {
    return snapshot.available && model.total_size + kv_headroom <= snapshot.pool_size;
}

struct SchedulerConfig {
    std::uint32_t batch_size = 1;
    std::uint64_t block_size_tokens = 16;

    Bytes kv_headroom(const ModelSpec& model) const {
        return static_cast<Bytes>(batch_size) * block_size_tokens * model.bytes_per_token;
    }
};

struct ScheduleEntry {
    std::string model_id;
    std::vector<std::pair<std::string, Seconds>> candidates;  // (gpu_id, estimate)
    std::optional<std::string> chosen;
};

struct ScheduleDecision {
    std::vector<std::pair<std::string, std::string>> assignments;  // (model_id, gpu_id)
    std::vector<std::string> deferred;
    std::vector<ScheduleEntry> entries;
};

/// Greedy order-sensitive pass over the queue (scheduler.hpp:79-120) through
/// tg_schedule; the peer term when TANGRAM_PEER_SCHEDULE is set.
inline ScheduleDecision schedule(const std::vector<std::string>& requests, std::vector<GpuSnapshot> snapshots,
                                 const std::map<std::string, ModelSpec>& registry, const SchedulerConfig& config) {
    // the distinct models of the queue, in first-seen order
    std::vector<std::string> ids;
    std::vector<std::uint32_t> req;
    std::vector<bool> known;
    for (const auto& id : requests) {
        auto it = std::find(ids.begin(), ids.end(), id);
        if (it == ids.end()) {
            ids.push_back(id);
            it = ids.end() - 1;
        }
        req.push_back(static_cast<std::uint32_t>(it - ids.begin()));
        known.push_back(registry.count(id) > 0);
    }
    std::vector<std::vector<tg_tensor_spec>> tbuf(ids.size());
    std::vector<tg_model_spec> specs;
    static const ModelSpec none{};
    for (std::size_t i = 0; i < ids.size(); ++i) {
        auto r = registry.find(ids[i]);
        specs.push_back(tgs::spec_of(r == registry.end() ? none : r->second, &tbuf[i]));
    }
    // unknown models are deferred without being offered to tg_schedule
    std::vector<std::uint32_t> req_known;
    for (std::size_t i = 0; i < req.size(); ++i)
        if (known[i]) req_known.push_back(req[i]);
    const std::size_t ng = snapshots.size(), nm = ids.size();
    std::vector<tg_gpu_snapshot> gv;
    for (const auto& s : snapshots) gv.push_back(tgs::view_of(s));
    std::vector<uint64_t> reuse(ng * nm, 0), peer(ng * nm, 0);
    const bool with_peer = tgs::peer_bandwidth() > 0;
    for (std::size_t g = 0; g < ng; ++g)
        for (std::size_t m = 0; m < nm; ++m) {
            reuse[g * nm + m] = snapshots[g].reuse_size_of(ids[m]);
            if (with_peer && registry.count(ids[m])) {
                auto p = tgs::live_pools().find(snapshots[g].gpu_id);
                if (p != tgs::live_pools().end()) tg_peer_reuse_size(p->second, &specs[m], &peer[g * nm + m]);
            }
        }
    std::vector<int32_t> assign(req_known.size(), -1);
    std::vector<double> est(req_known.size() * ng, -1.0);
    if (!req_known.empty())
        tg_schedule(req_known.data(), static_cast<uint32_t>(req_known.size()), gv.data(), static_cast<uint32_t>(ng),
                    specs.data(), static_cast<uint32_t>(nm), reuse.data(), with_peer ? peer.data() : nullptr,
                    config.batch_size, config.block_size_tokens, assign.data(), est.data());
    ScheduleDecision out;
    std::size_t k = 0;
    for (std::size_t i = 0; i < requests.size(); ++i) {
        ScheduleEntry entry;
        entry.model_id = requests[i];
        if (!known[i]) {
            out.deferred.push_back(requests[i]);
            out.entries.push_back(std::move(entry));
            continue;
        }
        for (std::size_t g = 0; g < ng; ++g)
            if (est[k * ng + g] >= 0) entry.candidates.emplace_back(snapshots[g].gpu_id, est[k * ng + g]);
        if (assign[k] < 0) {
            out.deferred.push_back(requests[i]);
        } else {
            entry.chosen = snapshots[assign[k]].gpu_id;
            out.assignments.emplace_back(requests[i], snapshots[assign[k]].gpu_id);
        }
        out.entries.push_back(std::move(entry));
        ++k;
    }
    return out;
}

}  // namespace warmsim
