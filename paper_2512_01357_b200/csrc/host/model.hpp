// Model / GPU descriptions and the request-share statistics that feed the
// eviction cost.  Field meanings follow model.hpp of the reference
// (TensorSpec 17-22, ModelSpec 30-37, GpuSpec 39-45, ModelStatsTable 70-133,
// eviction_cost 136-140).
#pragma once

#include <algorithm>
#include <cstdint>
#include <deque>
#include <map>
#include <string>
#include <vector>

#include "core.hpp"

namespace tg {

struct TensorDesc {
    Key id;
    std::string model_id;
    std::string name;
    u64 size = 0;
};

enum class Location : std::uint8_t { ModelCache = 0, ModelStore = 1 };

struct ModelDesc {
    std::string model_id;
    std::vector<TensorDesc> tensors;  // name order
    u64 total_size = 0;
    double alpha = 1.0;  // latency sensitivity
    Location location = Location::ModelCache;
    u64 bytes_per_token = 0;
};

struct GpuDesc {
    std::string gpu_id;
    u64 pool_size = 0;
    double pcie_bw = 0;
    double intra_bw = 0;
    double store_bw = 0;
};

// What the eviction cost needs from the request statistics
// (reuse_store.hpp:104-105): p_m and b_m per model.
class StatsView {
public:
    virtual ~StatsView() = default;
    virtual double miss_probability(const std::string& model) const = 0;
    virtual double load_bandwidth_or(const std::string& model, double fallback) const = 0;
};

// Statistics owned by the caller (e.g. the reference's own ModelStatsTable
// behind the C++ facade), read through callbacks.
class ExternalStats final : public StatsView {
public:
    using PFn = double (*)(void*, const char*);
    using BFn = double (*)(void*, const char*, double);
    ExternalStats(void* ctx, PFn p, BFn b) : ctx_(ctx), p_(p), b_(b) {}
    double miss_probability(const std::string& m) const override { return p_(ctx_, m.c_str()); }
    double load_bandwidth_or(const std::string& m, double f) const override { return b_(ctx_, m.c_str(), f); }

private:
    void* ctx_;
    PFn p_;
    BFn b_;
};

// Exponentially-decayed request counters; miss probability = share of the
// total.  Arithmetic order is kept statement-for-statement with
// model.hpp:87-105 so every double is bit-identical.
class RequestShares final : public StatsView {
public:
    explicit RequestShares(double decay = 0.95) : decay_(decay) {}

    St record_request(const std::string& model, double t) {
        if (t < last_t_) return Err::OrderingError;
        last_t_ = t;
        row(model);
        double total = 0.0;
        for (auto& [id, r] : rows_) {
            r.counter *= decay_;
            if (id == model) {
                r.counter += 1.0;
                r.history.push_back(t);
                if (r.history.size() > 16) r.history.pop_front();
            }
            total += r.counter;
        }
        for (auto& [id, r] : rows_) r.p_miss = total > 0.0 ? std::clamp(r.counter / total, 0.0, 1.0) : 0.0;
        return ok();
    }

    St record_eviction(const std::string& model, double t) {
        if (t < last_t_) return Err::OrderingError;
        last_t_ = t;
        row(model);
        return ok();
    }

    void set_load_bandwidth(const std::string& model, double bw) { row(model).load_bw = bw; }

    double miss_probability(const std::string& model) const override {
        auto it = rows_.find(model);
        return it == rows_.end() ? 0.0 : it->second.p_miss;
    }

    double load_bandwidth_or(const std::string& model, double fallback) const override {
        auto it = rows_.find(model);
        return (it != rows_.end() && it->second.load_bw > 0.0) ? it->second.load_bw : fallback;
    }

private:
    struct Row {
        std::deque<double> history;
        double p_miss = 0.0;
        double load_bw = 0.0;
        double counter = 0.0;
    };
    Row& row(const std::string& m) { return rows_[m]; }

    double decay_;
    double last_t_ = 0.0;
    std::map<std::string, Row> rows_;  // ordered: the fold order is part of the numerics
};

// c = p * (s / b) * alpha, same association as model.hpp:136-140.
inline double eviction_cost(u64 size, double p, double bw, double alpha) {
    return p * (static_cast<double>(size) / bw) * alpha;
}

// Synthetic catalog (catalog.hpp:37-90): embed ≈ 5 %, attn:mlp = 1:2 per layer.
ModelDesc make_model(const std::string& model_id, u64 total_size, int layers, u64 bytes_per_token,
                     Location loc = Location::ModelCache, double alpha = 1.0);
std::vector<ModelDesc> default_catalog();

}  // namespace tg
