#include "sched.hpp"

namespace tg {

std::vector<int> schedule(const std::vector<u32>& requests, std::vector<GpuView> gpus,
                          const std::vector<ModelDesc>& models, const std::vector<std::vector<u64>>& reuse,
                          const std::vector<std::vector<u64>>& peer_reuse, u32 batch_size, u64 block_tokens,
                          std::vector<std::vector<double>>* estimates) {
    std::vector<int> out(requests.size(), -1);
    if (estimates) estimates->assign(requests.size(), std::vector<double>(gpus.size(), -1.0));
    for (std::size_t r = 0; r < requests.size(); ++r) {
        const u32 mi = requests[r];
        if (mi >= models.size()) continue;  // unknown model: deferred
        const ModelDesc& m = models[mi];
        const u64 headroom = static_cast<u64>(batch_size) * block_tokens * m.bytes_per_token;
        int best = -1;
        double best_t = std::numeric_limits<double>::infinity();
        for (std::size_t g = 0; g < gpus.size(); ++g) {
            if (!can_run(m, gpus[g], headroom)) continue;
            const u64 peer = peer_reuse.empty() ? 0 : peer_reuse[g][mi];
            const double t = estimate_load_time(m, reuse[g][mi], gpus[g], peer);
            if (estimates) (*estimates)[r][g] = t;
            if (t < best_t || (t == best_t && best >= 0 && gpus[g].gpu_id < gpus[best].gpu_id)) {
                best = static_cast<int>(g);
                best_t = t;
            }
        }
        if (best >= 0) {
            out[r] = best;
            gpus[best].available = false;
        }
    }
    return out;
}

}  // namespace tg
