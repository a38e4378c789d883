#include "kv.hpp"

#include "../device/common.cuh"

#include <algorithm>

namespace tg {

KvAllocator::KvAllocator(const KvAllocator& o)
    : model_(o.model_),
      block_tokens_(o.block_tokens_),
      block_bytes_(o.block_bytes_),
      next_pbn_(o.next_pbn_),
      free_count_(o.free_count_),
      reqs_(o.reqs_),
      free_slots_(o.free_slots_),
      rid_of_slot_(o.rid_of_slot_),
      slots_used_(o.slots_used_),
      runs_(o.runs_),
      ctr_(o.ctr_),
      dev_(o.dev_ ? o.dev_->clone() : nullptr) {}

KvAllocator::~KvAllocator() {
    if (armed_)
        if (auto c = armed_on_.lock()) --*c;
}

KvAllocator& KvAllocator::operator=(const KvAllocator& o) {
    if (this == &o) return *this;
    KvAllocator tmp(o);
    std::swap(*this, tmp);
    return *this;
}

u64 KvAllocator::request_blocks(u64 rid) const {
    auto it = reqs_.find(rid);
    return it == reqs_.end() ? 0 : it->second.blocks;
}
u64 KvAllocator::request_tokens(u64 rid) const {
    auto it = reqs_.find(rid);
    return it == reqs_.end() ? 0 : it->second.tokens;
}
u32 KvAllocator::request_slot(u64 rid) const {
    auto it = reqs_.find(rid);
    return it == reqs_.end() ? 0 : it->second.slot;
}

KvAllocator::Req& KvAllocator::req(u64 rid) {
    auto it = reqs_.find(rid);
    if (it != reqs_.end()) return it->second;
    Req r;
    if (!free_slots_.empty()) {
        r.slot = free_slots_.back();
        free_slots_.pop_back();
    } else {
        r.slot = slots_used_++;
        rid_of_slot_.resize(slots_used_);
    }
    rid_of_slot_[r.slot] = rid;
    return reqs_.emplace(rid, r).first->second;
}

// Σ ⌊run / block⌋ over free runs (kv_engine.hpp:197-201); runs shorter than
// one block contribute nothing, so start the size-ordered walk at one block.
u64 KvAllocator::fittable(const Store& s) const {
    u64 n = 0;
    s.map().for_each_free_by_size(block_bytes_, [&](u64, u64 len) { n += len / block_bytes_; });
    return n;
}

u64 KvAllocator::acquire(Store& s, const StatsView& st, u32 slot, u64 lbn0, u64 need, bool* touched,
                         KvBatchWork* w, bool* exhausted) {
    u64 got = 0;
    // LIFO free list first (kv_engine.hpp:205-210).
    if (free_count_ > 0) {
        const u64 k = std::min(free_count_, need);
        free_count_ -= k;
        w->pops += k;
        ctr_.blocks_from_free_list += k;
        got += k;
    }
    // Then best-fit carving: k blocks from the smallest adequate run equal k
    // sequential allocate_best_fit calls (the carved run's remainder stays
    // the unique smallest adequate run until it drops below one block).
    while (got < need) {
        *touched = true;
        u64 off, len;
        if (!s.map().best_fit(block_bytes_, &off, &len)) {
            if (!urgent_reclaim(s, st, 1).ok()) {
                *exhausted = true;
                break;
            }
            continue;
        }
        const u64 k = std::min(len / block_bytes_, need - got);
        s.carve_kv_run(off, k, block_bytes_, next_pbn_);
        const KvRun run{off, k, next_pbn_};
        runs_.push_back(run);
        w->carved.push_back(run);
        next_pbn_ += k;
        ctr_.blocks_from_pool += k;
        got += k;
    }
    if (got > 0) {
        w->grants.push_back(KvGrant{slot, lbn0, got});
        w->total += got;
    }
    return got;
}

St KvAllocator::ensure_one(Store& s, const StatsView& st, u64 rid, u64 tokens, KvBatchWork* w, u64* granted) {
    *granted = 0;
    Req& r = req(rid);
    if (tokens < r.tokens) return Err::InvalidArgument;
    const u64 want = blocks_for(tokens, block_tokens_);
    bool touched = false, exhausted = false;
    if (want > r.blocks) {
        const u64 got = acquire(s, st, r.slot, r.blocks, want - r.blocks, &touched, w, &exhausted);
        // `r` may have been invalidated by nothing (map nodes are stable).
        r.blocks += got;
        *granted = got;
        if (exhausted) return Err::PoolExhausted;
    }
    r.tokens = tokens;
    if (*granted > 0) {
        ++ctr_.alloc_batches;
        if (touched) ++ctr_.pool_invocations;
    }
    return ok();
}

int KvAllocator::flush(KvBatchWork& w, std::vector<u64>* pbns) {
    if (pbns) pbns->assign(w.total, 0);
    if (w.total == 0) return 0;
    if (!dev_) return 0;
    return dev_->apply_batch(w, block_bytes_, pbns ? pbns->data() : nullptr);
}

St KvAllocator::ensure_capacity(Store& s, const StatsView& st, u64 rid, u64 tokens, std::vector<u64>* granted,
                                u64* n_granted) {
    KvBatchWork w;
    w.free_before = free_count_;
    u64 g = 0;
    St res = ensure_one(s, st, rid, tokens, &w, &g);
    if (n_granted) *n_granted = g;
    const int rc = flush(w, granted);  // blocks granted before a failure stay granted
    if (rc) throw DeviceError(rc, "kv: device batch failed");
    return res;
}

St KvAllocator::batch_allocate(Store& s, const StatsView& st, const std::vector<std::pair<u64, u64>>& reqs,
                               std::vector<u64>* counts, std::vector<u64>* pbns) {
    NvtxRange nvtx("tg.kv_batch_allocate");
    counts->assign(reqs.size(), 0);
    u64 needed = 0;
    for (const auto& [rid, tokens] : reqs) {
        const u64 have = request_blocks(rid);
        const u64 want = blocks_for(tokens, block_tokens_);
        if (want > have) needed += want - have;
    }
    KvBatchWork w;
    w.free_before = free_count_;

    if (needed == 0) {  // token counts only; no pool dispatch
        for (std::size_t i = 0; i < reqs.size(); ++i) {
            u64 g = 0;
            if (St r = ensure_one(s, st, reqs[i].first, reqs[i].second, &w, &g); !r) return r;
        }
        if (pbns) pbns->clear();
        return ok();
    }

    const bool certainly_fits = free_count_ >= needed || free_count_ + fittable(s) >= needed;
    if (certainly_fits) {
        const KvCounters before = ctr_;
        for (std::size_t i = 0; i < reqs.size(); ++i) {
            St r = ensure_one(s, st, reqs[i].first, reqs[i].second, &w, &(*counts)[i]);
            if (!r) {  // partial effects persist, as in the reference (kv_engine.hpp:136)
                if (int rc = flush(w, pbns)) throw DeviceError(rc, "kv: device batch failed");
                return r;
            }
        }
        ctr_.alloc_batches = before.alloc_batches + 1;
        ctr_.pool_invocations = before.pool_invocations + (ctr_.pool_invocations > before.pool_invocations ? 1 : 0);
        if (int rc = flush(w, pbns)) throw DeviceError(rc, "kv: device batch failed");
        return ok();
    }

    // Contended path: run on copies of the host state so that a failure
    // leaves no trace (kv_engine.hpp:145-160).  Device state is untouched
    // until the batch commits.
    Store s_copy = s;
    std::unique_ptr<KvDevice> dev = std::move(dev_);
    KvAllocator a_copy = *this;
    dev_ = std::move(dev);
    const KvCounters before = ctr_;
    for (std::size_t i = 0; i < reqs.size(); ++i) {
        St r = a_copy.ensure_one(s_copy, st, reqs[i].first, reqs[i].second, &w, &(*counts)[i]);
        if (!r) {
            counts->assign(reqs.size(), 0);
            return r;
        }
    }
    a_copy.ctr_.alloc_batches = before.alloc_batches + 1;
    a_copy.ctr_.pool_invocations =
        before.pool_invocations + (a_copy.ctr_.pool_invocations > before.pool_invocations ? 1 : 0);
    s = std::move(s_copy);
    a_copy.dev_ = std::move(dev_);
    *this = std::move(a_copy);
    if (int rc = flush(w, pbns)) throw DeviceError(rc, "kv: device batch failed");
    return ok();
}

St KvAllocator::release_request(u64 rid) {
    auto it = reqs_.find(rid);
    if (it == reqs_.end()) return Err::NotFound;
    const Req r = it->second;
    if (dev_ && r.blocks > 0) {
        if (int rc = dev_->release(r.slot, r.blocks, free_count_)) throw DeviceError(rc, "kv: release failed");
    }
    free_count_ += r.blocks;
    free_slots_.push_back(r.slot);
    reqs_.erase(it);
    return ok();
}

void KvAllocator::teardown(Store& s) {
    for (const KvRun& r : runs_) s.release_kv_range(r.off, r.count * block_bytes_);
    runs_.clear();
    reqs_.clear();
    free_slots_.clear();
    rid_of_slot_.clear();
    slots_used_ = 0;
    free_count_ = 0;
    if (dev_) dev_->reset();
}

St KvAllocator::urgent_reclaim(Store& s, const StatsView& st, u64 blocks) {
    auto cands = s.candidates(st, model_);
    std::sort(cands.begin(), cands.end(), candidate_before);
    std::size_t next = 0;
    while (fittable(s) < blocks) {
        if (next >= cands.size()) return Err::PoolExhausted;
        s.evict_tensor(cands[next++].tensor);
    }
    ++ctr_.reclaim_events;
    return ok();
}

// ---- K4D -----------------------------------------------------------------------------
St KvAllocator::arm(Store& s, u64 max_blocks_per_request, u32 max_requests, u32 max_batches) {
    if (!dev_) throw DeviceError(101, "kv: device-decided batches need a device pool");
    if (armed_ || max_requests == 0 || max_batches == 0) return Err::InvalidArgument;
    KvArmSpec a;
    s.map().for_each_free_by_size(block_bytes_, [&](u64 off, u64 len) {
        a.run_off.push_back(off);
        a.run_blocks.push_back(len / block_bytes_);
    });
    a.slot_blocks.assign(slots_used_, 0);
    a.slot_tokens.assign(slots_used_, 0);
    u64 longest = 0;
    for (const auto& [rid, r] : reqs_) {
        a.slot_blocks[r.slot] = r.blocks;
        a.slot_tokens[r.slot] = r.tokens;
        longest = std::max(longest, r.blocks);
    }
    a.free_top = free_count_;
    a.next_pbn = next_pbn_;
    a.max_blocks_per_request = std::max(max_blocks_per_request, longest);
    a.max_requests = max_requests;
    a.max_batches = max_batches;
    a.block_tokens = block_tokens_;
    if (int rc = dev_->arm(a, block_bytes_)) throw DeviceError(rc, "kv: arm failed");
    armed_ = true;
    arm_max_requests_ = max_requests;
    armed_on_ = s.kv_arm_handle();
    if (auto c = armed_on_.lock()) ++*c;
    return ok();
}

int KvAllocator::enqueue_device(const u64* d_slots, const u64* d_tokens, u32 n, void* stream) {
    if (!armed_ || n > arm_max_requests_) return 104;  // TG_ERR_BAD_ARG
    return dev_->enqueue(d_slots, d_tokens, n, stream);
}

St KvAllocator::sync(Store& s, const StatsView& st, SyncReport* rep) {
    NvtxRange nvtx("tg.kv_device_sync");
    if (!armed_) return Err::InvalidArgument;
    // the decisions were taken against the free runs of the store armed on:
    // folding them into any other store would corrupt it
    if (armed_on_.expired()) {  // the armed store is gone: drain and disarm, fold nothing
        KvLog drained;
        dev_->read_log(&drained);
        armed_ = false;
        return Err::InvalidArgument;
    }
    if (armed_on_.lock() != s.kv_arm_handle().lock())
        throw DeviceError(104, "kv: sync against a pool the engine was not armed on");
    KvLog log;
    if (int rc = dev_->read_log(&log)) throw DeviceError(rc, "kv: device log read failed");
    armed_ = false;
    if (auto c = armed_on_.lock()) --*c;
    armed_on_.reset();
    rep->overflow = log.stalled == 2;
    St first = ok();
    for (const KvLogBatch& b : log.batches) {
        if (b.status == 0) {
            // the device's decisions, folded in exactly as batch_allocate's
            // certainly-fits path books them (kv_engine.hpp:127-141)
            u64 total = 0;
            for (const auto& [slot, tok] : b.reqs) {
                Req& r = reqs_.at(rid_of_slot_.at(slot));
                const u64 want = blocks_for(tok, block_tokens_);
                const u64 need = want > r.blocks ? want - r.blocks : 0;
                r.blocks += need;
                r.tokens = tok;
                total += need;
            }
            if (total != b.total) throw DeviceError(106, "kv: device batch disagrees with the host replay");
            if (total == 0) continue;
            free_count_ -= b.pops;
            ctr_.blocks_from_free_list += b.pops;
            u64 carved = 0;
            for (const KvRun& p : b.pieces) {
                if (p.first_pbn != next_pbn_) throw DeviceError(106, "kv: device PBNs out of sequence");
                s.carve_kv_run(p.off, p.count, block_bytes_, p.first_pbn);
                runs_.push_back(p);
                next_pbn_ += p.count;
                carved += p.count;
            }
            ctr_.blocks_from_pool += carved;
            ++ctr_.alloc_batches;
            if (carved) ++ctr_.pool_invocations;
            ++rep->applied;
        } else {
            std::vector<std::pair<u64, u64>> reqs;
            bool known = true;
            for (const auto& [slot, tok] : b.reqs) {
                if (slot >= rid_of_slot_.size() || !reqs_.count(rid_of_slot_[slot])) known = false;
                else reqs.push_back({rid_of_slot_[slot], tok});
            }
            ++rep->replayed;
            std::vector<u64> counts;
            St r = known ? batch_allocate(s, st, reqs, &counts, nullptr) : St(Err::InvalidArgument);
            if (!r && first) first = r;
        }
    }
    return first;
}

St KvAllocator::table(u64 rid, std::vector<u64>* lbn_to_pbn, u64* tokens) const {
    auto it = reqs_.find(rid);
    if (it == reqs_.end()) return Err::NotFound;
    *tokens = it->second.tokens;
    lbn_to_pbn->assign(it->second.blocks, 0);
    if (!dev_) throw DeviceError(101, "kv: block tables live on the device; pool has no device");
    if (it->second.blocks)
        if (int rc = dev_->read_table(it->second.slot, it->second.blocks, lbn_to_pbn->data()))
            throw DeviceError(rc, "kv: table read failed");
    return ok();
}

}  // namespace tg
