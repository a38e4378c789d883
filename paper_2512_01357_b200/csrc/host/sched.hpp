// GPU-affinity placement (Alg. 2).  schedule() reproduces the reference's
// greedy pass (scheduler.hpp:79-120): requests in queue order, each to the
// feasible GPU with the lowest expected load time, ties to the smaller
// gpu_id, a chosen GPU leaves the pass.  The B200 extension adds a peer term
// to the estimate: bytes resident in a peer GPU's pool move
// over NVLink instead of PCIe,
//     t = (S − S'_local − S'_peer) / B + S'_peer / B_nvlink,
// and reduces to the reference's (S − S') / B when B_nvlink = 0.
#pragma once

#include <algorithm>
#include <limits>
#include <string>
#include <vector>

#include "model.hpp"

namespace tg {

struct GpuView {
    std::string gpu_id;
    bool available = true;
    u64 pool_size = 0;
    u64 free_bytes = 0;
    double pcie_bw = 0;
    double store_bw = 0;
    double nvlink_bw = 0;  // 0: no peer term
};

inline double estimate_load_time(const ModelDesc& m, u64 reuse, const GpuView& g, u64 peer_reuse = 0) {
    const double bw = m.location == Location::ModelCache ? g.pcie_bw : std::min(g.store_bw, g.pcie_bw);
    if (g.nvlink_bw <= 0.0 || peer_reuse == 0) return static_cast<double>(m.total_size - reuse) / bw;
    return static_cast<double>(m.total_size - reuse - peer_reuse) / bw + static_cast<double>(peer_reuse) / g.nvlink_bw;
}

inline bool can_run(const ModelDesc& m, const GpuView& g, u64 kv_headroom) {
    return g.available && m.total_size + kv_headroom <= g.pool_size;
}

// reuse[g][m], peer_reuse[g][m] (may be empty); returns per-request GPU index or -1.
std::vector<int> schedule(const std::vector<u32>& requests, std::vector<GpuView> gpus,
                          const std::vector<ModelDesc>& models, const std::vector<std::vector<u64>>& reuse,
                          const std::vector<std::vector<u64>>& peer_reuse, u32 batch_size, u64 block_tokens,
                          std::vector<std::vector<double>>* estimates);

}  // namespace tg
