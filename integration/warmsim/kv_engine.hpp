// Drop-in binding: warmsim::KvEngine backed by the B200 KV allocator
// (device-resident block tables, libtangram.so).  Declarations mirror
// kv_engine.hpp:26-239 of the reference; see reuse_store.hpp in this
// directory for how the binding is put on the include path.
//
// Granted PBN values live in HBM.  On a control-plane-only pool (no device)
// the engine still takes every decision (counts, carve runs, address table,
// stats) but block-number values are not materialised: returned vectors have
// the right lengths and hold kNoPbn.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "tangram.h"
#include "warmsim/model.hpp"
#include "warmsim/packing.hpp"
#include "warmsim/reuse_store.hpp"
#include "warmsim/types.hpp"

namespace warmsim {

struct KvBlockTable {
    std::uint64_t request_id = 0;
    std::uint64_t block_size_tokens = 16;
    std::map<std::uint64_t, std::uint64_t> lbn_to_pbn;
    std::uint64_t token_count = 0;
};

struct KvAllocStats {
    std::uint64_t pool_invocations = 0;
    std::uint64_t alloc_batches = 0;
    std::uint64_t blocks_from_free_list = 0;
    std::uint64_t blocks_from_pool = 0;
    std::uint64_t reclaim_events = 0;
};

class KvEngine {
public:
    static constexpr std::uint64_t kNoPbn = ~std::uint64_t{0};

    KvEngine() = default;
    KvEngine(std::string model_id, std::uint64_t block_size_tokens, Bytes bytes_per_token)
        : model_id_(std::move(model_id)), block_size_tokens_(block_size_tokens) {
        tg_kv* k = nullptr;
        if (int rc = tg_kv_create(model_id_.c_str(), block_size_tokens, bytes_per_token, &k))
            tgb::fail(rc, "tg_kv_create");
        kv_.reset(k);
    }
    KvEngine(const KvEngine& o) : model_id_(o.model_id_), block_size_tokens_(o.block_size_tokens_) {
        if (o.kv_) {
            tg_kv* k = nullptr;
            if (int rc = tg_kv_clone(o.kv_.get(), &k)) tgb::fail(rc, "tg_kv_clone");
            kv_.reset(k);
        }
    }
    KvEngine& operator=(const KvEngine& o) {
        if (this != &o) *this = KvEngine(o);
        return *this;
    }
    KvEngine(KvEngine&&) noexcept = default;
    KvEngine& operator=(KvEngine&&) noexcept = default;

    const std::string& model_id() const { return model_id_; }
    std::uint64_t block_size_tokens() const { return block_size_tokens_; }
    Bytes block_bytes() const { return kvstats().block_bytes; }
    const KvAllocStats& stats() const {
        const tg_kv_stats s = kvstats();
        stats_cache_ = KvAllocStats{s.pool_invocations, s.alloc_batches, s.blocks_from_free_list, s.blocks_from_pool,
                                    s.reclaim_events};
        return stats_cache_;
    }
    std::size_t free_list_size() const { return kvstats().free_list_size; }
    std::size_t active_requests() const { return kvstats().active_requests; }

    const KvBlockTable* table(std::uint64_t request_id) const {
        std::uint64_t n = 0, tok = 0;
        if (tg_kv_table(kv_.get(), request_id, nullptr, 0, &n, &tok) != 0) return nullptr;
        std::vector<std::uint64_t> pbns(n, kNoPbn);
        if (n) tg_kv_table(kv_.get(), request_id, pbns.data(), n, &n, &tok);  // NO_DEVICE leaves kNoPbn
        KvBlockTable& t = tables_cache_[request_id];
        t = KvBlockTable{request_id, block_size_tokens_, {}, tok};
        for (std::uint64_t i = 0; i < n; ++i) t.lbn_to_pbn[i] = pbns[i];
        return &t;
    }

    const std::map<std::uint64_t, std::pair<Bytes, Bytes>>& address_table() const {
        std::uint64_t n = 0;
        tg_kv_address_table(kv_.get(), nullptr, 0, &n);
        std::vector<std::uint64_t> tri(3 * n);
        tg_kv_address_table(kv_.get(), tri.data(), n, &n);
        addr_cache_.clear();
        for (std::uint64_t i = 0; i < n; ++i) addr_cache_[tri[3 * i]] = {tri[3 * i + 1], tri[3 * i + 2]};
        return addr_cache_;
    }

    static std::uint64_t blocks_for(std::uint64_t tokens, std::uint64_t block_size) {
        return (tokens + block_size - 1) / block_size;
    }

    Result<std::vector<std::uint64_t>> ensure_capacity(ReuseStore& store, const ModelStatsTable& stats,
                                                       std::uint64_t request_id, std::uint64_t new_token_count) {
        tgb::StatsHandle sh(stats);
        std::uint64_t have = 0;
        tg_kv_table(kv_.get(), request_id, nullptr, 0, &have, nullptr);
        const std::uint64_t want = blocks_for(new_token_count, block_size_tokens_);
        std::vector<std::uint64_t> g(want > have ? want - have : 0, kNoPbn);
        std::uint64_t n = 0;
        const int rc = tgb::domain(tg_kv_ensure_capacity(kv_.get(), store.mutable_handle(), sh.h, request_id, new_token_count,
                                                         g.data(), g.size(), &n),
                                   "tg_kv_ensure_capacity");
        if (rc) return static_cast<Error>(rc - 1);
        g.resize(n);
        return g;
    }

    Result<std::vector<std::vector<std::uint64_t>>> batch_allocate(
        ReuseStore& store, const ModelStatsTable& stats,
        const std::vector<std::pair<std::uint64_t, std::uint64_t>>& requests) {
        tgb::StatsHandle sh(stats);
        std::vector<std::uint64_t> rids, toks, counts(requests.size(), 0);
        std::uint64_t cap = 0;
        for (const auto& [r, t] : requests) {
            rids.push_back(r);
            toks.push_back(t);
            cap += blocks_for(t, block_size_tokens_);
        }
        std::vector<std::uint64_t> pbns(cap, kNoPbn);
        std::uint64_t total = 0;
        const int rc = tgb::domain(tg_kv_batch_allocate(kv_.get(), store.mutable_handle(), sh.h, rids.data(), toks.data(),
                                                        rids.size(), counts.data(), pbns.data(), cap, &total),
                                   "tg_kv_batch_allocate");
        if (rc) return static_cast<Error>(rc - 1);
        std::vector<std::vector<std::uint64_t>> out(requests.size());
        std::uint64_t k = 0;
        for (std::size_t i = 0; i < requests.size(); ++i) {
            out[i].assign(pbns.begin() + static_cast<long>(k), pbns.begin() + static_cast<long>(k + counts[i]));
            k += counts[i];
        }
        return out;
    }

    Status release_request(std::uint64_t request_id) {
        const int rc = tgb::domain(tg_kv_release_request(kv_.get(), request_id), "tg_kv_release_request");
        if (rc) return static_cast<Error>(rc - 1);
        return ok_status();
    }

    void instance_teardown(ReuseStore& store) {
        if (int rc = tg_kv_teardown(kv_.get(), store.mutable_handle())) tgb::fail(rc, "tg_kv_teardown");
    }

    Status urgent_reclaim(ReuseStore& store, const ModelStatsTable& stats, std::uint64_t needed_blocks) {
        tgb::StatsHandle sh(stats);
        const int rc = tgb::domain(tg_kv_urgent_reclaim(kv_.get(), store.mutable_handle(), sh.h, needed_blocks),
                                   "tg_kv_urgent_reclaim");
        if (rc) return static_cast<Error>(rc - 1);
        return ok_status();
    }

private:
    struct KvDeleter {
        void operator()(tg_kv* k) const { tg_kv_destroy(k); }
    };
    tg_kv_stats kvstats() const {
        tg_kv_stats s{};
        if (kv_) tg_kv_stats_get(kv_.get(), &s);
        return s;
    }

    std::string model_id_;
    std::uint64_t block_size_tokens_ = 16;
    std::unique_ptr<tg_kv, KvDeleter> kv_;
    mutable KvAllocStats stats_cache_;
    mutable std::map<std::uint64_t, KvBlockTable> tables_cache_;
    mutable std::map<std::uint64_t, std::pair<Bytes, Bytes>> addr_cache_;
};

}  // namespace warmsim
