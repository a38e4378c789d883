// K4 — on-demand KV block allocation, device half (sm_100a).
//
// The host decides per batch how many blocks each request receives, how
// many come off the LIFO free list and which pool runs are carved (kv.cpp).
// This kernel materialises the batch in HBM with one thread per granted
// block: block k of the batch (request order, then LBN order — the order of
// the reference's sequential acquire_block calls, kv_engine.hpp:84-89 and
// 203-229) takes free_list[top-1-k] while k < pops, otherwise the next PBN
// of its carve run; it writes the request's LBN→PBN table entry and, for
// carved blocks, the PBN→offset address-table entry.
//
// K4D (kv_device_batch_kernel) takes the decision itself as well, for
// batches enqueued between KvAllocator::arm and ::sync: no host round trip
// per batch, so a decode loop can allocate its blocks inside a CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "../host/kv.hpp"
#include "common.cuh"
#include "kernels.hpp"

namespace tg {
namespace {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

__global__ void kv_batch_kernel(const KvBatchArgs a) {
    const u64 k = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= a.total) return;
    u32 lo = 0, hi = a.n_grants - 1;
    while (lo < hi) {
        const u32 mid = (lo + hi + 1) >> 1;
        if (a.grants[mid].start <= k) lo = mid;
        else hi = mid - 1;
    }
    const KvGrantDev g = a.grants[lo];
    const u64 lbn = g.lbn0 + (k - g.start);
    u64 pbn;
    if (k < a.pops) {
        pbn = a.free_list[a.free_before - 1 - k];
    } else {
        const u64 j = k - a.pops;
        u32 rl = 0, rh = a.n_runs - 1;
        while (rl < rh) {
            const u32 mid = (rl + rh + 1) >> 1;
            if (a.runs[mid].start <= j) rl = mid;
            else rh = mid - 1;
        }
        const KvRunDev r = a.runs[rl];
        pbn = r.first_pbn + (j - r.start);
        a.addr[pbn] = r.off + (j - r.start) * a.block_bytes;
    }
    a.tables[static_cast<u64>(g.slot) * a.stride + lbn] = pbn;
    if (a.out) a.out[k] = pbn;
}

// K4D: one batch decided and applied on the device (one CTA).  The decision
// is the reference's certainly-fits path (kv_engine.hpp:127-141): for each
// request in order, blocks ceil(tokens / B) - have, the LIFO free list first
// (kv_engine.hpp:205-210), then best-fit carving — which for equal blocks is
// a walk over the free runs in ascending (size, offset) order, each run
// carved from its start until it holds less than one block (SURVEY §7 hard
// part 5; the control block keeps the cursor of that walk).  A batch that
// would need the contended path (not certainly fitting: urgent reclaim), or
// that the device cannot decide alone (unknown slot, shrinking token count,
// a request twice, a table row too short, too many pieces) is left untouched
// and flagged; the host replays it, and every later batch of the session, on
// the reference path at sync time.
constexpr int kKvThreads = 1024;

__device__ __forceinline__ u32 block_excl_scan(u32 v, u32* s_warp, u32* total) {
    const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<u32>(o)) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        u32 t = lane < kKvThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= static_cast<u32>(o)) t += y;
        }
        s_warp[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const u32 before = (w ? s_warp[w - 1] : 0) + x - v;
    *total = s_warp[kKvThreads / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(kKvThreads) kv_device_batch_kernel(KvDevCtl* __restrict__ c,
                                                                     const u64* __restrict__ slots,
                                                                     const u64* __restrict__ tokens, u32 n) {
    __shared__ u32 s_pref[kKvDevMaxRequests + 1];
    __shared__ KvPiece s_piece[kKvDevMaxPieces];
    __shared__ u64 s_pstart[kKvDevMaxPieces + 1];
    __shared__ u32 s_warp[32];
    __shared__ u64 s_b, s_pops, s_npieces;
    __shared__ int s_fallback;
    const u32 tid = threadIdx.x;
    if (tid == 0) s_b = c->batches++;
    __syncthreads();
    const u64 b = s_b;
    if (b >= c->max_batches) {  // log full: the batch is lost, reported at sync
        if (tid == 0) c->stalled = 2;
        return;
    }
    std::uint8_t* entry = c->log + b * c->log_entry_bytes;
    auto* hdr = reinterpret_cast<KvLogHeader*>(entry);
    u64* req = reinterpret_cast<u64*>(entry + sizeof(KvLogHeader));
    auto* pcs = reinterpret_cast<KvPiece*>(entry + sizeof(KvLogHeader) + 16 * c->max_requests);
    for (u32 i = tid; i < n && i < c->max_requests; i += kKvThreads) {
        req[2 * i] = slots[i];
        req[2 * i + 1] = tokens[i];
    }
    const bool stalled = c->stalled != 0;
    if (stalled) {
        if (tid == 0) {
            hdr->n = n;
            hdr->status = 1;
            hdr->total = hdr->pops = hdr->n_pieces = 0;
        }
        return;
    }
    // need per request, and whether the device can decide the batch alone
    const u64 bs = c->block_tokens;
    int bad = n > c->max_requests;
    const u32 per = (n + kKvThreads - 1) / kKvThreads;  // contiguous chunk per thread
    u32 local = 0;
    for (u32 q = 0; q < per; ++q) {
        const u32 i = tid * per + q;
        if (i >= n) break;
        const u64 slot = slots[i], tok = tokens[i];
        u32 need = 0;
        if (slot >= c->n_slots) {
            bad = 1;
        } else {
            if (atomicExch(reinterpret_cast<unsigned long long*>(c->slot_mark + slot), b + 1) == b + 1) bad = 1;
            if (tok < c->slot_tokens[slot]) bad = 1;
            const u64 want = (tok + bs - 1) / bs, have = c->slot_blocks[slot];
            if (want > c->stride) bad = 1;
            else if (want > have) need = static_cast<u32>(want - have);
        }
        s_pref[i] = need;
        local += need;
    }
    bad = __syncthreads_or(bad);
    u32 total = 0;
    u32 run = block_excl_scan(local, s_warp, &total);
    for (u32 q = 0; q < per; ++q) {
        const u32 i = tid * per + q;
        if (i >= n) break;
        const u32 v = s_pref[i];
        s_pref[i] = run;
        run += v;
    }
    if (tid == 0) {
        s_pref[n] = total;
        int fb = bad || total > c->free_top + c->blocks_left;
        u64 pops = total < c->free_top ? total : c->free_top;
        u64 rem = total - pops, cur = c->run_cursor, used = c->run_used, np = 0, carved = 0;
        while (!fb && rem > 0) {
            if (np == kKvDevMaxPieces || cur >= c->n_runs) {
                fb = 1;
                break;
            }
            const u64 k = min(c->run_blocks[cur] - used, rem);
            s_piece[np] = KvPiece{c->run_off[cur] + used * c->block_bytes, k, c->next_pbn + carved};
            s_pstart[np] = carved;
            ++np;
            carved += k;
            rem -= k;
            used += k;
            if (used == c->run_blocks[cur]) {
                ++cur;
                used = 0;
            }
        }
        s_pstart[np] = carved;
        s_fallback = fb;
        s_pops = pops;
        s_npieces = np;
        if (fb) {
            hdr->n = n;
            hdr->status = 1;
            hdr->total = hdr->pops = hdr->n_pieces = 0;
            c->stalled = 1;
        } else {
            hdr->n = n;
            hdr->status = 0;
            hdr->total = total;
            hdr->pops = pops;
            hdr->n_pieces = np;
            for (u64 p = 0; p < np; ++p) pcs[p] = s_piece[p];
            c->run_cursor = cur;
            c->run_used = used;
        }
    }
    __syncthreads();
    if (s_fallback) return;
    const u64 pops = s_pops, np = s_npieces, top = c->free_top;
    // expand: block k of the batch -> (request, LBN) and its PBN
    for (u32 k = tid; k < total; k += kKvThreads) {
        u32 lo = 0, hi = n - 1;
        while (lo < hi) {
            const u32 mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        const u64 slot = slots[lo];
        const u64 lbn = c->slot_blocks[slot] + (k - s_pref[lo]);
        u64 pbn;
        if (k < pops) {
            pbn = c->free_list[top - 1 - k];
        } else {
            const u64 j = k - pops;
            u32 p = 0;
            while (p + 1 < np && s_pstart[p + 1] <= j) ++p;
            pbn = s_piece[p].first_pbn + (j - s_pstart[p]);
            c->addr[pbn] = s_piece[p].off + (j - s_pstart[p]) * c->block_bytes;
        }
        c->tables[slot * c->stride + lbn] = pbn;
    }
    __syncthreads();
    for (u32 i = tid; i < n; i += kKvThreads) {
        const u64 slot = slots[i];
        c->slot_blocks[slot] += s_pref[i + 1] - s_pref[i];
        c->slot_tokens[slot] = tokens[i];
    }
    if (tid == 0) {
        const u64 carved = total - pops;
        c->free_top = top - pops;
        c->next_pbn += carved;
        c->blocks_left -= carved;
    }
}

// One warp per token; 16-byte words when both ends allow it, bytes otherwise.
__global__ void kv_tokens_kernel(const KvTokensArgs a) {
    const u32 lane = threadIdx.x & 31;
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const u64 block_bytes = a.block_tokens * a.token_bytes;
    for (u64 i = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < a.n; i += warps) {
        const u64 p = a.pos[i], slot = a.slots[i], lbn = p / a.block_tokens;
        const u64 pbn = slot < a.n_slots && lbn < a.stride ? a.tables[slot * a.stride + lbn] : 0;
        const u64 off = pbn != 0 && pbn < a.n_pbns ? a.addr[pbn] : ~u64{0};
        if (off == ~u64{0} || off + block_bytes > a.arena_bytes) {
            if (lane == 0) atomicAdd(a.faults, 1ull);
            continue;
        }
        std::uint8_t* at = a.arena + off + (p % a.block_tokens) * a.token_bytes;
        std::uint8_t* b = a.buf + i * a.token_bytes;
        std::uint8_t* dst = a.write ? at : b;
        const std::uint8_t* src = a.write ? b : at;
        if (((reinterpret_cast<std::uintptr_t>(dst) | reinterpret_cast<std::uintptr_t>(src) | a.token_bytes) & 15) == 0) {
            for (u64 w = lane; w < a.token_bytes / 16; w += 32)
                reinterpret_cast<uint4*>(dst)[w] = reinterpret_cast<const uint4*>(src)[w];
        } else {
            for (u64 k = lane; k < a.token_bytes; k += 32) dst[k] = src[k];
        }
    }
}

__global__ void kv_copy_kernel(const u64* __restrict__ src, u64 n, u64* __restrict__ dst) {
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

// Device-resident tables of one KV engine.
class KvDeviceImpl final : public KvDevice {
public:
    // The engine owns its stream: block tables are independent of the arena
    // bytes (KV allocation moves no bytes), and an engine may outlive the
    // pool it was first used with.
    explicit KvDeviceImpl(int device) : dev_(device) {
        DeviceScope ds(dev_);
        TG_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    }
    ~KvDeviceImpl() override {
        release_all();
        if (s_) cudaStreamDestroy(s_);
    }

    int apply_batch(const KvBatchWork& w, u64 block_bytes, u64* out_pbns) override {
        DeviceScope ds(dev_);
        // capacity: slots / LBNs / free list / PBNs
        u32 max_slot = 0;
        u64 max_lbn = 0;
        for (const auto& g : w.grants) {
            max_slot = std::max(max_slot, g.slot + 1);
            max_lbn = std::max(max_lbn, g.lbn0 + g.count);
        }
        u64 max_pbn = 0;
        for (const auto& r : w.carved) max_pbn = std::max(max_pbn, r.first_pbn + r.count);
        grow(max_slot, max_lbn, 0, max_pbn + 1);

        // pack descriptors into pinned staging, one H2D
        const std::size_t ng = w.grants.size(), nr = w.carved.size();
        const std::size_t bytes = ng * sizeof(KvGrantDev) + nr * sizeof(KvRunDev);
        ensure_staging(bytes);
        auto* hg = reinterpret_cast<KvGrantDev*>(h_stage_);
        auto* hr = reinterpret_cast<KvRunDev*>(h_stage_ + ng * sizeof(KvGrantDev));
        u64 start = 0;
        for (std::size_t i = 0; i < ng; ++i) {
            hg[i] = KvGrantDev{start, w.grants[i].lbn0, w.grants[i].slot, 0};
            start += w.grants[i].count;
        }
        u64 cstart = 0;
        for (std::size_t i = 0; i < nr; ++i) {
            hr[i] = KvRunDev{cstart, w.carved[i].off, w.carved[i].first_pbn};
            cstart += w.carved[i].count;
        }
        TG_CUDA(cudaMemcpyAsync(d_stage_, h_stage_, bytes, cudaMemcpyHostToDevice, s_));
        if (out_pbns) ensure_out(w.total);
        KvBatchArgs a{};
        a.grants = reinterpret_cast<const KvGrantDev*>(d_stage_);
        a.n_grants = static_cast<u32>(ng);
        a.runs = reinterpret_cast<const KvRunDev*>(d_stage_ + ng * sizeof(KvGrantDev));
        a.n_runs = static_cast<u32>(nr);
        a.total = w.total;
        a.pops = w.pops;
        a.free_before = w.free_before;
        a.block_bytes = block_bytes;
        a.tables = tables_;
        a.stride = stride_;
        a.free_list = free_;
        a.addr = addr_;
        a.out = out_pbns ? d_out_ : nullptr;
        kv_batch_launch(a, s_);
        TG_CUDA(cudaGetLastError());
        if (out_pbns) {
            TG_CUDA(cudaMemcpyAsync(out_pbns, d_out_, w.total * sizeof(u64), cudaMemcpyDeviceToHost, s_));
            TG_CUDA(cudaStreamSynchronize(s_));
        } else {
            // the staging buffer is reused by the next batch: order the host
            // rewrite after this copy
            TG_CUDA(cudaEventRecord(stage_done_, s_));
        }
        return 0;
    }

    int release(u32 slot, u64 blocks, u64 free_before) override {
        DeviceScope ds(dev_);
        grow(0, 0, free_before + blocks, 0);
        kv_release_launch(tables_ + static_cast<u64>(slot) * stride_, blocks, free_ + free_before, s_);
        TG_CUDA(cudaGetLastError());
        return 0;
    }

    int read_table(u32 slot, u64 blocks, u64* pbns) override {
        DeviceScope ds(dev_);
        TG_CUDA(cudaMemcpyAsync(pbns, tables_ + static_cast<u64>(slot) * stride_, blocks * sizeof(u64),
                                cudaMemcpyDeviceToHost, s_));
        TG_CUDA(cudaStreamSynchronize(s_));
        return 0;
    }

    int read_free_list(u64 n, u64* pbns) override {
        DeviceScope ds(dev_);
        if (n == 0) return 0;
        TG_CUDA(cudaMemcpyAsync(pbns, free_, n * sizeof(u64), cudaMemcpyDeviceToHost, s_));
        TG_CUDA(cudaStreamSynchronize(s_));
        return 0;
    }

    int reserve(u32 slots, u64 blocks_per_slot, u64 free_cap, u64 pbn_cap) override {
        DeviceScope ds(dev_);
        grow(slots, blocks_per_slot, free_cap, pbn_cap);
        return 0;
    }

    std::unique_ptr<KvDevice> clone() const override {
        DeviceScope ds(dev_);
        auto c = std::make_unique<KvDeviceImpl>(dev_);
        c->grow(static_cast<u32>(slots_), stride_, free_cap_, pbn_cap_);
        TG_CUDA(cudaStreamSynchronize(s_));  // source tables complete
        cudaStream_t cs = c->s_;
        if (slots_ && stride_)
            TG_CUDA(cudaMemcpyAsync(c->tables_, tables_, slots_ * stride_ * sizeof(u64), cudaMemcpyDeviceToDevice, cs));
        if (free_cap_) TG_CUDA(cudaMemcpyAsync(c->free_, free_, free_cap_ * sizeof(u64), cudaMemcpyDeviceToDevice, cs));
        if (pbn_cap_) TG_CUDA(cudaMemcpyAsync(c->addr_, addr_, pbn_cap_ * sizeof(u64), cudaMemcpyDeviceToDevice, cs));
        TG_CUDA(cudaStreamSynchronize(cs));
        return c;
    }

    int arm(const KvArmSpec& a, u64 block_bytes) override {
        DeviceScope ds(dev_);
        u64 carvable = 0;
        for (u64 b : a.run_blocks) carvable += b;
        const u64 slots = a.slot_blocks.size();
        grow(static_cast<u32>(slots), a.max_blocks_per_request, a.free_top, a.next_pbn + carvable + 1);
        const u64 nr = a.run_off.size();
        const u64 entry = kv_log_entry_bytes(a.max_requests);
        // buffers are kept across arms when large enough (captured graphs
        // read every pointer from the control block, so a reallocation only
        // costs a re-upload)
        reserve_buf(&d_runs_, &runs_cap_, 2 * std::max<u64>(nr, 1));
        reserve_buf(&d_slots_, &slots_cap_, 3 * std::max<u64>(slots, 1));
        reserve_bytes(&d_log_, &log_cap_, entry * a.max_batches);
        // whole entries are read back at sync (unused request / piece space too)
        TG_CUDA(cudaMemsetAsync(d_log_, 0, entry * a.max_batches, s_));
        if (!d_ctl_) TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_ctl_), sizeof(KvDevCtl), s_));
        std::vector<u64> h(2 * nr + 2 * slots);
        std::copy(a.run_off.begin(), a.run_off.end(), h.begin());
        std::copy(a.run_blocks.begin(), a.run_blocks.end(), h.begin() + nr);
        std::copy(a.slot_blocks.begin(), a.slot_blocks.end(), h.begin() + 2 * nr);
        std::copy(a.slot_tokens.begin(), a.slot_tokens.end(), h.begin() + 2 * nr + slots);
        if (nr) TG_CUDA(cudaMemcpyAsync(d_runs_, h.data(), 2 * nr * sizeof(u64), cudaMemcpyHostToDevice, s_));
        if (slots) {
            TG_CUDA(cudaMemcpyAsync(d_slots_, h.data() + 2 * nr, 2 * slots * sizeof(u64), cudaMemcpyHostToDevice, s_));
            TG_CUDA(cudaMemsetAsync(d_slots_ + 2 * slots, 0, slots * sizeof(u64), s_));
        }
        KvDevCtl c{};
        c.tables = tables_;
        c.stride = stride_;
        c.free_list = free_;
        c.addr = addr_;
        c.run_off = d_runs_;
        c.run_blocks = d_runs_ + nr;
        c.n_runs = nr;
        c.slot_blocks = d_slots_;
        c.slot_tokens = d_slots_ + slots;
        c.slot_mark = d_slots_ + 2 * slots;
        c.n_slots = slots;
        c.log = d_log_;
        c.log_entry_bytes = entry;
        c.max_batches = a.max_batches;
        c.max_requests = a.max_requests;
        c.block_bytes = block_bytes;
        c.block_tokens = a.block_tokens;
        c.free_top = a.free_top;
        c.next_pbn = a.next_pbn;
        c.blocks_left = carvable;
        h_ctl_ = c;
        TG_CUDA(cudaMemcpyAsync(d_ctl_, &h_ctl_, sizeof(KvDevCtl), cudaMemcpyHostToDevice, s_));
        TG_CUDA(cudaStreamSynchronize(s_));
        max_requests_ = a.max_requests;
        max_batches_ = a.max_batches;
        log_entry_ = entry;
        captured_ = false;
        pending_ = false;
        return 0;
    }

    int enqueue(const u64* d_slots, const u64* d_tokens, u32 n, void* stream) override {
        DeviceScope ds(dev_);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s_;
        foreign_ = foreign_ || st != s_;
        kv_device_batch_launch(d_ctl_, d_slots, d_tokens, n, st);
        TG_CUDA(cudaGetLastError());
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        TG_CUDA(cudaStreamIsCapturing(st, &cs));
        if (cs != cudaStreamCaptureStatusNone) {
            captured_ = true;  // replays run outside our view: sync waits for the device
        } else {
            if (!done_) TG_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
            TG_CUDA(cudaEventRecord(done_, st));
            pending_ = true;
        }
        return 0;
    }

    int read_log(KvLog* out) override {
        DeviceScope ds(dev_);
        if (captured_) TG_CUDA(cudaDeviceSynchronize());
        else if (pending_) TG_CUDA(cudaEventSynchronize(done_));
        KvDevCtl c{};
        TG_CUDA(cudaMemcpyAsync(&c, d_ctl_, sizeof(KvDevCtl), cudaMemcpyDeviceToHost, s_));
        TG_CUDA(cudaStreamSynchronize(s_));
        const u64 nb = std::min(c.batches, max_batches_);
        std::vector<std::uint8_t> log(nb * log_entry_);
        if (nb) {
            TG_CUDA(cudaMemcpyAsync(log.data(), d_log_, log.size(), cudaMemcpyDeviceToHost, s_));
            TG_CUDA(cudaStreamSynchronize(s_));
        }
        out->stalled = c.stalled;
        out->batches.clear();
        for (u64 b = 0; b < nb; ++b) {
            const std::uint8_t* e = log.data() + b * log_entry_;
            KvLogHeader hd;
            std::memcpy(&hd, e, sizeof hd);
            KvLogBatch lb;
            lb.status = hd.status;
            lb.total = hd.total;
            lb.pops = hd.pops;
            const u64* rq = reinterpret_cast<const u64*>(e + sizeof(KvLogHeader));
            for (u64 i = 0; i < hd.n; ++i) lb.reqs.push_back({rq[2 * i], rq[2 * i + 1]});
            const auto* pc = reinterpret_cast<const KvPiece*>(e + sizeof(KvLogHeader) + 16 * max_requests_);
            for (u64 p = 0; p < hd.n_pieces; ++p) lb.pieces.push_back(KvRun{pc[p].off, pc[p].count, pc[p].first_pbn});
            out->batches.push_back(std::move(lb));
        }
        captured_ = pending_ = false;
        return 0;
    }

    void order_after_updates(void* stream) override {
        DeviceScope ds(dev_);
        auto st = static_cast<cudaStream_t>(stream);
        if (!st || st == s_) return;
        if (!updated_) TG_CUDA(cudaEventCreateWithFlags(&updated_, cudaEventDisableTiming));
        TG_CUDA(cudaEventRecord(updated_, s_));
        TG_CUDA(cudaStreamWaitEvent(st, updated_));
    }

    int tokens(std::uint8_t* arena, u64 arena_bytes, u64 block_tokens, u64 token_bytes, const u64* slots,
               const u64* pos, std::uint8_t* buf, u32 n, bool write, void* stream) override {
        DeviceScope ds(dev_);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s_;
        if (!d_faults_) {
            TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_faults_), sizeof(unsigned long long), s_));
            TG_CUDA(cudaMemsetAsync(d_faults_, 0, sizeof(unsigned long long), s_));
        }
        order_after_updates(st);  // the tables this batch reads are the ones granted so far
        foreign_ = foreign_ || st != s_;
        KvTokensArgs a{tables_, slots_, stride_, addr_, pbn_cap_, arena, arena_bytes, block_tokens, token_bytes,
                       slots, pos, buf, n, write, d_faults_};
        kv_tokens_launch(a, st);
        TG_CUDA(cudaGetLastError());
        return 0;
    }

    u64 token_faults() override {
        DeviceScope ds(dev_);
        if (!d_faults_) return 0;
        if (foreign_) TG_CUDA(cudaDeviceSynchronize());
        unsigned long long f = 0;
        TG_CUDA(cudaMemcpyAsync(&f, d_faults_, sizeof f, cudaMemcpyDeviceToHost, s_));
        TG_CUDA(cudaStreamSynchronize(s_));
        return f;
    }

    void reset() override {}
    void* table_ptr() const override { return tables_; }
    void* stream() const override { return s_; }
    u64 table_stride() const override { return stride_; }
    void* addr_ptr() const override { return addr_; }

private:
    static u64 grow_to(u64 have, u64 need) {
        if (need <= have) return have;
        u64 n = have ? have : 16;
        while (n < need) n *= 2;
        return n;
    }

    // Grow any of the four arrays, preserving contents (stream-ordered).  The
    // old arrays are retired, not freed: pointers handed out earlier
    // (tg_kv_device_tables, kernels on other streams or in graphs) stay valid
    // memory until the engine is destroyed — stale after the growth, never
    // dangling.  Growth doubles, so the retired arrays total less than the
    // live ones.
    void grow(u32 slots, u64 lbns, u64 free_need, u64 pbns) {
        const u64 ns = grow_to(slots_, slots), nl = grow_to(stride_, lbns);
        if (ns != slots_ || nl != stride_) {
            u64* t = nullptr;
            TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t), ns * nl * sizeof(u64), s_));
            TG_CUDA(cudaMemsetAsync(t, 0, ns * nl * sizeof(u64), s_));
            if (tables_ && slots_ && stride_)
                TG_CUDA(cudaMemcpy2DAsync(t, nl * sizeof(u64), tables_, stride_ * sizeof(u64), stride_ * sizeof(u64),
                                          slots_, cudaMemcpyDeviceToDevice, s_));
            if (tables_) retired_.push_back(tables_);
            tables_ = t;
            slots_ = ns;
            stride_ = nl;
        }
        grow_linear(&free_, &free_cap_, free_need);
        grow_linear(&addr_, &pbn_cap_, pbns);
    }

    void grow_linear(u64** p, u64* cap, u64 need) {
        const u64 n = grow_to(*cap, need);
        if (n == *cap) return;
        u64* q = nullptr;
        TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&q), n * sizeof(u64), s_));
        TG_CUDA(cudaMemsetAsync(q, 0, n * sizeof(u64), s_));
        if (*p && *cap) TG_CUDA(cudaMemcpyAsync(q, *p, *cap * sizeof(u64), cudaMemcpyDeviceToDevice, s_));
        if (*p) retired_.push_back(*p);
        *p = q;
        *cap = n;
    }

    void ensure_staging(std::size_t bytes) {
        if (stage_done_) TG_CUDA(cudaEventSynchronize(stage_done_));
        else TG_CUDA(cudaEventCreateWithFlags(&stage_done_, cudaEventDisableTiming));
        if (bytes <= stage_cap_) return;
        std::size_t n = stage_cap_ ? stage_cap_ : 4096;
        while (n < bytes) n *= 2;
        if (h_stage_) cudaFreeHost(h_stage_);
        if (d_stage_) TG_CUDA(cudaFreeAsync(d_stage_, s_));
        TG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_stage_), n));
        TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_stage_), n, s_));
        stage_cap_ = n;
    }

    void reserve_buf(u64** p, u64* cap, u64 n) {
        if (n <= *cap) return;
        if (*p) TG_CUDA(cudaFreeAsync(*p, s_));
        *cap = grow_to(*cap, n);
        TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), *cap * sizeof(u64), s_));
    }
    void reserve_bytes(std::uint8_t** p, u64* cap, u64 n) {
        if (n <= *cap) return;
        if (*p) TG_CUDA(cudaFreeAsync(*p, s_));
        *cap = n;
        TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), n, s_));
    }

    void ensure_out(u64 n) {
        if (n <= out_cap_) return;
        if (d_out_) TG_CUDA(cudaFreeAsync(d_out_, s_));
        out_cap_ = grow_to(out_cap_, n);
        TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_out_), out_cap_ * sizeof(u64), s_));
    }

    void release_all() {
        DeviceScope ds(dev_);
        cudaStreamSynchronize(s_);
        // batches enqueued on a caller's stream (or captured in a graph) may
        // still read the control block and tables
        if (foreign_) cudaDeviceSynchronize();
        for (u64* p : {tables_, free_, addr_, d_out_, d_runs_, d_slots_})
            if (p) cudaFree(p);
        for (u64* p : retired_) cudaFree(p);
        if (d_faults_) cudaFree(d_faults_);
        if (updated_) cudaEventDestroy(updated_);
        if (d_log_) cudaFree(d_log_);
        if (d_ctl_) cudaFree(d_ctl_);
        if (done_) cudaEventDestroy(done_);
        if (d_stage_) cudaFree(d_stage_);
        if (h_stage_) cudaFreeHost(h_stage_);
        if (stage_done_) cudaEventDestroy(stage_done_);
    }

    int dev_;
    cudaStream_t s_;
    u64* tables_ = nullptr;
    u64 slots_ = 0, stride_ = 0;
    u64* free_ = nullptr;
    u64 free_cap_ = 0;
    u64* addr_ = nullptr;
    u64 pbn_cap_ = 0;
    u64* d_out_ = nullptr;
    u64 out_cap_ = 0;
    std::uint8_t* h_stage_ = nullptr;
    std::uint8_t* d_stage_ = nullptr;
    std::size_t stage_cap_ = 0;
    cudaEvent_t stage_done_ = nullptr;
    // K4D
    KvDevCtl* d_ctl_ = nullptr;
    KvDevCtl h_ctl_{};
    u64* d_runs_ = nullptr;
    u64 runs_cap_ = 0;
    u64* d_slots_ = nullptr;
    u64 slots_cap_ = 0;
    std::uint8_t* d_log_ = nullptr;
    u64 log_cap_ = 0, log_entry_ = 0, max_requests_ = 0, max_batches_ = 0;
    cudaEvent_t done_ = nullptr;
    bool captured_ = false, pending_ = false, foreign_ = false;
    std::vector<u64*> retired_;            // grown-out arrays (see grow)
    unsigned long long* d_faults_ = nullptr;  // block-table consumer faults (kv_tokens_kernel)
    cudaEvent_t updated_ = nullptr;           // engine stream, for consumers on other streams
};

}  // namespace

void kv_batch_launch(const KvBatchArgs& a, cudaStream_t s) {
    if (a.total == 0) return;
    const unsigned blocks = static_cast<unsigned>((a.total + 255) / 256);
    kv_batch_kernel<<<blocks, 256, 0, s>>>(a);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void kv_device_batch_launch(KvDevCtl* d_ctl, const u64* d_slots, const u64* d_tokens, u32 n, cudaStream_t s) {
    kv_device_batch_kernel<<<1, kKvThreads, 0, s>>>(d_ctl, d_slots, d_tokens, n);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void kv_tokens_launch(const KvTokensArgs& a, cudaStream_t s) {
    if (a.n == 0 || a.token_bytes == 0) return;
    const u64 want = (static_cast<u64>(a.n) * 32 + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < 4096 ? want : 4096);
    kv_tokens_kernel<<<blocks, 256, 0, s>>>(a);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void kv_release_launch(const u64* table_row, u64 blocks, u64* free_list_dst, cudaStream_t s) {
    if (blocks == 0) return;
    const unsigned grid = static_cast<unsigned>((blocks + 255) / 256 < 1024 ? (blocks + 255) / 256 : 1024);
    kv_copy_kernel<<<grid, 256, 0, s>>>(table_row, blocks, free_list_dst);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

std::unique_ptr<KvDevice> make_kv_device(int device, cudaStream_t /*pool stream: not shared*/) {
    return std::make_unique<KvDeviceImpl>(device);
}

}  // namespace tg
