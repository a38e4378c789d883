// On-demand KV block allocator, control half.
//
// Semantics: the reference KvEngine (kv_engine.hpp:43-239) — per-request
// LBN→PBN tables, a LIFO free list absorbing released requests, PBNs from 1,
// best-fit carving of new blocks from the shared pool, urgent tensor reclaim
// under pressure, atomic batches.
//
// Split of work on B200: the host decides *how many* blocks each request gets,
// how many come off the free list, and which pool runs are carved (a carve of
// k blocks from the smallest adequate free run is one extent, see
// SURVEY §7 hard part 5 for why sequential best-fit equals this prefix
// carve).  The per-block expansion — which PBN lands in which table slot,
// free-list pops, PBN→offset address entries — is done by the device kernel
// in device/kv.cu, and the tables live in HBM where a paged-attention
// engine reads them.  The host keeps O(requests + runs) state only.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "store.hpp"

namespace tg {

struct KvCounters {
    u64 pool_invocations = 0;
    u64 alloc_batches = 0;
    u64 blocks_from_free_list = 0;
    u64 blocks_from_pool = 0;
    u64 reclaim_events = 0;
};

// A run of blocks carved in one piece: PBNs first..first+count-1 at
// consecutive offsets off, off+B, ...
struct KvRun {
    u64 off = 0;
    u64 count = 0;
    u64 first_pbn = 0;
};

// One table update of a batch: `count` new LBNs starting at `lbn0` for the
// request in table slot `slot`.
struct KvGrant {
    u32 slot = 0;
    u64 lbn0 = 0;
    u64 count = 0;
};

// Everything the device needs to materialise one batch.
struct KvBatchWork {
    std::vector<KvGrant> grants;
    u64 total = 0;      // blocks in the batch
    u64 pops = 0;       // first `pops` blocks come off the free list top
    u64 free_before = 0;  // free-list length before the batch
    std::vector<KvRun> carved;  // the rest, in order
};

// K4D: what arming an engine uploads (KvAllocator::arm).
struct KvArmSpec {
    std::vector<u64> run_off, run_blocks;       // free runs >= 1 block, ascending (size, offset)
    std::vector<u64> slot_blocks, slot_tokens;  // per table slot
    u64 free_top = 0, next_pbn = 1;
    u64 max_blocks_per_request = 0;
    u32 max_requests = 0, max_batches = 0;
    u64 block_tokens = 0;
};
// One batch of the device log, as read back at sync.
struct KvLogBatch {
    u64 status = 0;  // 0 decided and applied on the device, 1 left to the host
    u64 total = 0, pops = 0;
    std::vector<std::pair<u64, u64>> reqs;  // (slot, tokens)
    std::vector<KvRun> pieces;              // carved, in order
};
struct KvLog {
    std::vector<KvLogBatch> batches;
    u64 stalled = 0;  // 2: the log overflowed and batches were dropped
};

// Device half (device/kv.cu); null for control-plane-only pools.
class KvDevice {
public:
    // K4D: arm (synchronous), enqueue one batch (asynchronous, graph-capturable;
    // `stream` null = the engine's stream), read the log back (waits for the
    // enqueued batches).
    virtual int arm(const KvArmSpec& a, u64 block_bytes) = 0;
    virtual int enqueue(const u64* d_slots, const u64* d_tokens, u32 n, void* stream) = 0;
    virtual int read_log(KvLog* out) = 0;
    virtual ~KvDevice() = default;
    virtual int apply_batch(const KvBatchWork& w, u64 block_bytes, u64* out_pbns /*nullable, w.total*/) = 0;
    // append the request's table (LBN order) to the free list
    virtual int release(u32 slot, u64 blocks, u64 free_before) = 0;
    virtual int read_table(u32 slot, u64 blocks, u64* pbns) = 0;
    virtual int read_free_list(u64 n, u64* pbns) = 0;
    virtual int reserve(u32 slots, u64 blocks_per_slot, u64 free_cap, u64 pbn_cap) = 0;
    virtual std::unique_ptr<KvDevice> clone() const = 0;
    virtual void reset() = 0;
    virtual void* table_ptr() const = 0;
    virtual void* stream() const = 0;  // the stream table updates are ordered on
    virtual u64 table_stride() const = 0;
    virtual void* addr_ptr() const = 0;
    // make `stream` wait for every table update enqueued so far
    virtual void order_after_updates(void* stream) = 0;
    // block-table consumer (kv_tokens_launch), ordered after the table updates
    virtual int tokens(std::uint8_t* arena, u64 arena_bytes, u64 block_tokens, u64 token_bytes, const u64* slots,
                       const u64* pos, std::uint8_t* buf, u32 n, bool write, void* stream) = 0;
    virtual u64 token_faults() = 0;  // waits for the consumers launched so far
};

class KvAllocator {
public:
    KvAllocator(std::string model, u64 block_tokens, u64 bytes_per_token)
        : model_(std::move(model)), block_tokens_(block_tokens), block_bytes_(block_tokens * bytes_per_token) {}
    ~KvAllocator();
    KvAllocator(const KvAllocator& o);  // deep copy, device tables included (never armed)
    KvAllocator& operator=(const KvAllocator& o);
    KvAllocator(KvAllocator&&) noexcept = default;
    KvAllocator& operator=(KvAllocator&&) noexcept = default;

    const std::string& model() const { return model_; }
    u64 block_tokens() const { return block_tokens_; }
    u64 block_bytes() const { return block_bytes_; }
    const KvCounters& counters() const { return ctr_; }
    u64 free_list_size() const { return free_count_; }
    std::size_t active_requests() const { return reqs_.size(); }
    u64 next_pbn() const { return next_pbn_; }
    const std::vector<KvRun>& runs() const { return runs_; }
    bool has_request(u64 rid) const { return reqs_.count(rid) != 0; }
    u64 request_blocks(u64 rid) const;
    u64 request_tokens(u64 rid) const;
    u32 request_slot(u64 rid) const;

    void attach_device(std::unique_ptr<KvDevice> dev) { dev_ = std::move(dev); }
    KvDevice* device() const { return dev_.get(); }

    static u64 blocks_for(u64 tokens, u64 bs) { return (tokens + bs - 1) / bs; }

    // ensure_capacity (kv_engine.hpp:75-102).  `granted` (nullable) receives
    // the new PBNs; *n_granted their count.
    St ensure_capacity(Store& s, const StatsView& st, u64 rid, u64 tokens, std::vector<u64>* granted,
                       u64* n_granted);
    // batch_allocate (kv_engine.hpp:107-161).  counts[i] = blocks granted to
    // request i; `pbns` (nullable) receives all new PBNs in order.
    St batch_allocate(Store& s, const StatsView& st, const std::vector<std::pair<u64, u64>>& reqs,
                      std::vector<u64>* counts, std::vector<u64>* pbns);
    St release_request(u64 rid);
    void teardown(Store& s);
    St urgent_reclaim(Store& s, const StatsView& st, u64 blocks);

    // ---- K4D: device-decided batches ------------------------------------------
    // arm: upload the allocator state and a mirror of the pool's free runs;
    // until sync, batches of the engine's known requests (by table slot) are
    // decided and applied by kv_device_batch_kernel with no host round trip,
    // and the pool must not change (Store::kv_armed).  sync: fold the device's
    // decisions into the host state (pool regions, tables, counters — equal to
    // running the same batches through batch_allocate) and replay on the host
    // path every batch the device left to it; disarms.
    St arm(Store& s, u64 max_blocks_per_request, u32 max_requests, u32 max_batches);
    int enqueue_device(const u64* d_slots, const u64* d_tokens, u32 n, void* stream);
    struct SyncReport {
        u64 applied = 0, replayed = 0;
        bool overflow = false;
    };
    St sync(Store& s, const StatsView& st, SyncReport* rep);
    bool armed() const { return armed_; }
    u32 max_device_requests() const { return arm_max_requests_; }

    // table(rid) / address_table() readers.
    St table(u64 rid, std::vector<u64>* lbn_to_pbn, u64* tokens) const;
    void address_table(std::vector<KvRun>* runs) const { *runs = runs_; }

private:
    struct Req {
        u64 blocks = 0;
        u64 tokens = 0;
        u32 slot = 0;
    };
    u64 fittable(const Store& s) const;
    Req& req(u64 rid);
    // Acquire `need` blocks for `slot` in order; appends to *w.  Returns the
    // number granted (== need unless the pool is exhausted).
    u64 acquire(Store& s, const StatsView& st, u32 slot, u64 lbn0, u64 need, bool* touched, KvBatchWork* w,
                bool* exhausted);
    St ensure_one(Store& s, const StatsView& st, u64 rid, u64 tokens, KvBatchWork* w, u64* granted);
    int flush(KvBatchWork& w, std::vector<u64>* pbns);

    std::string model_;
    u64 block_tokens_ = 16;
    u64 block_bytes_ = 0;
    u64 next_pbn_ = 1;
    u64 free_count_ = 0;
    std::map<u64, Req> reqs_;
    std::vector<u32> free_slots_;
    std::vector<u64> rid_of_slot_;
    u32 slots_used_ = 0;
    bool armed_ = false;
    std::weak_ptr<int> armed_on_;  // the store's arm count (Store::kv_arm_handle)
    u32 arm_max_requests_ = 0;
    std::vector<KvRun> runs_;
    KvCounters ctr_;
    std::unique_ptr<KvDevice> dev_;
};

}  // namespace tg
