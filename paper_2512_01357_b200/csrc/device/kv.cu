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
#include <cuda_runtime.h>

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

    void reset() override {}
    void* table_ptr() const override { return tables_; }
    u64 table_stride() const override { return stride_; }
    void* addr_ptr() const override { return addr_; }

private:
    static u64 grow_to(u64 have, u64 need) {
        if (need <= have) return have;
        u64 n = have ? have : 16;
        while (n < need) n *= 2;
        return n;
    }

    // Grow any of the four arrays, preserving contents (stream-ordered).
    void grow(u32 slots, u64 lbns, u64 free_need, u64 pbns) {
        const u64 ns = grow_to(slots_, slots), nl = grow_to(stride_, lbns);
        if (ns != slots_ || nl != stride_) {
            u64* t = nullptr;
            TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t), ns * nl * sizeof(u64), s_));
            TG_CUDA(cudaMemsetAsync(t, 0, ns * nl * sizeof(u64), s_));
            if (tables_ && slots_ && stride_)
                TG_CUDA(cudaMemcpy2DAsync(t, nl * sizeof(u64), tables_, stride_ * sizeof(u64), stride_ * sizeof(u64),
                                          slots_, cudaMemcpyDeviceToDevice, s_));
            if (tables_) TG_CUDA(cudaFreeAsync(tables_, s_));
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
        if (*p) TG_CUDA(cudaFreeAsync(*p, s_));
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

    void ensure_out(u64 n) {
        if (n <= out_cap_) return;
        if (d_out_) TG_CUDA(cudaFreeAsync(d_out_, s_));
        out_cap_ = grow_to(out_cap_, n);
        TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_out_), out_cap_ * sizeof(u64), s_));
    }

    void release_all() {
        DeviceScope ds(dev_);
        cudaStreamSynchronize(s_);
        for (u64* p : {tables_, free_, addr_, d_out_})
            if (p) cudaFree(p);
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
};

}  // namespace

void kv_batch_launch(const KvBatchArgs& a, cudaStream_t s) {
    if (a.total == 0) return;
    const unsigned blocks = static_cast<unsigned>((a.total + 255) / 256);
    kv_batch_kernel<<<blocks, 256, 0, s>>>(a);
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
