// K3 — relocation / compaction kernel, sm_100a.
//
// Executes one hazard-free wave of the planner's relocations
// (packing.hpp:412-456 → reuse_store.hpp:323-327) as a batched memcpy with
// arbitrary byte alignment at both ends.  Every warp owns 32 KiB chunks of a
// move's 16-byte-aligned destination body: lanes load consecutive aligned
// source words (coalesced 512 B per warp instruction), borrow the next word
// from the neighbouring lane with a shuffle and funnel-shift into the
// destination alignment, then issue coalesced 16-byte streaming stores.
// Head and tail bytes (< 16 each) are copied bytewise by the chunk-0 warp.
// The same kernel performs peer pulls when `src` is a peer arena address.
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace tg {
namespace {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

constexpr u64 kChunkWords = 2048;  // 32 KiB of destination per warp task
constexpr int kUnroll = 4;

struct RelocArgs {
    MoveDesc mv[kMaxMovesPerLaunch];
    u32 prefix[kMaxMovesPerLaunch + 1];  // task prefix over moves
    u32 n;
};

__device__ __forceinline__ uint4 shfl_down4(uint4 v) {
    uint4 r;
    r.x = __shfl_down_sync(0xffffffffu, v.x, 1);
    r.y = __shfl_down_sync(0xffffffffu, v.y, 1);
    r.z = __shfl_down_sync(0xffffffffu, v.z, 1);
    r.w = __shfl_down_sync(0xffffffffu, v.w, 1);
    return r;
}

template <int Q>
__device__ __forceinline__ uint4 realign(uint4 w0, uint4 w1, u32 r8) {
    const u32 u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    uint4 o;
    o.x = __funnelshift_r(u[Q + 0], u[Q + 1], r8);
    o.y = __funnelshift_r(u[Q + 1], u[Q + 2], r8);
    o.z = __funnelshift_r(u[Q + 2], u[Q + 3], r8);
    o.w = __funnelshift_r(u[Q + 3], u[Q + 4], r8);
    return o;
}

// The aligned source word after the body: only its first `valid` bytes lie
// inside the source range (the move's tail bytes included), so it is read
// byte by byte when the rest would run past the end of the source —
// registered device sources (an HBM model cache) have no slack after them.
__device__ __forceinline__ uint4 load_last_word(const uint4* p, u32 valid) {
    if (valid >= 16) return __ldcs(p);
    u64 lo = 0, hi = 0;
    const std::uint8_t* b = reinterpret_cast<const std::uint8_t*>(p);
    for (u32 i = 0; i < valid; ++i) {
        const u64 v = b[i];
        if (i < 8) lo |= v << (8 * i);
        else hi |= v << (8 * (i - 8));
    }
    return make_uint4(static_cast<u32>(lo), static_cast<u32>(lo >> 32), static_cast<u32>(hi),
                      static_cast<u32>(hi >> 32));
}

// Copy destination words [w_begin, w_end) of one move.  `sa` is the aligned
// source word holding the byte that lands on destination word 0, `o` the
// byte offset inside it.  Q = o >> 2 selects the unrolled realignment; Q < 0
// means co-aligned (o == 0).  `last_valid`: bytes of word sa[w_total] inside
// the source range.
template <int Q>
__device__ __forceinline__ void copy_words(const uint4* __restrict__ sa, uint4* __restrict__ da, u64 w_begin,
                                           u64 w_end, u64 w_total, u32 last_valid, u32 r8, u32 lane) {
    for (u64 g = w_begin; g < w_end; g += 32 * kUnroll) {
        uint4 cur[kUnroll], nxt[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const u64 wi = g + u * 32 + lane;
            cur[u] = wi < w_end ? __ldcs(sa + wi) : make_uint4(0, 0, 0, 0);
        }
        if constexpr (Q >= 0) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const u64 wi = g + u * 32 + lane;
                nxt[u] = shfl_down4(cur[u]);
                if (wi < w_end && (lane == 31 || wi + 1 == w_end))
                    nxt[u] = wi + 1 == w_total ? load_last_word(sa + wi + 1, last_valid) : __ldcs(sa + wi + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const u64 wi = g + u * 32 + lane;
            if (wi >= w_end) continue;
            if constexpr (Q >= 0) __stcs(da + wi, realign<Q>(cur[u], nxt[u], r8));
            else __stcs(da + wi, cur[u]);
        }
    }
}

__global__ void __launch_bounds__(256) relocate_kernel(const __grid_constant__ RelocArgs a) {
    const u32 lane = threadIdx.x & 31;
    const u32 warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u32 nwarps = (gridDim.x * blockDim.x) >> 5;
    const u32 total = a.prefix[a.n];
    for (u32 t = warp; t < total; t += nwarps) {
        u32 m = 0;
        while (a.prefix[m + 1] <= t) ++m;
        const u64 c = t - a.prefix[m];
        const u64 src = a.mv[m].src, dst = a.mv[m].dst, len = a.mv[m].len;
        const u64 d0 = (dst + 15) & ~u64{15};
        const u64 d1 = (dst + len) & ~u64{15};
        if (d0 >= d1) {  // tiny move: no aligned body
            if (c == 0)
                for (u64 i = lane; i < len; i += 32)
                    reinterpret_cast<std::uint8_t*>(dst)[i] = reinterpret_cast<const std::uint8_t*>(src)[i];
            continue;
        }
        const u64 head = d0 - dst, tail = dst + len - d1;
        if (c == 0) {
            if (lane < head)
                reinterpret_cast<std::uint8_t*>(dst)[lane] = reinterpret_cast<const std::uint8_t*>(src)[lane];
            if (lane >= 16 && lane - 16 < tail)
                reinterpret_cast<std::uint8_t*>(d1)[lane - 16] =
                    reinterpret_cast<const std::uint8_t*>(src + (d1 - dst))[lane - 16];
        }
        const u64 nw = (d1 - d0) >> 4;
        const u64 wb = c * kChunkWords;
        const u64 we = wb + kChunkWords < nw ? wb + kChunkWords : nw;
        const u64 s0 = src + head;
        const u32 o = static_cast<u32>(s0 & 15);
        const uint4* sa = reinterpret_cast<const uint4*>(s0 - o);
        uint4* da = reinterpret_cast<uint4*>(d0);
        const u32 r8 = (o & 3) * 8;
        const u32 lv = o + static_cast<u32>(tail);  // source bytes in word sa[nw]
        if (o == 0) copy_words<-1>(sa, da, wb, we, nw, lv, 0, lane);
        else if (o < 4) copy_words<0>(sa, da, wb, we, nw, lv, r8, lane);
        else if (o < 8) copy_words<1>(sa, da, wb, we, nw, lv, r8, lane);
        else if (o < 12) copy_words<2>(sa, da, wb, we, nw, lv, r8, lane);
        else copy_words<3>(sa, da, wb, we, nw, lv, r8, lane);
    }
}

}  // namespace

void relocate_launch(const MoveDesc* moves, int n_moves, int sm_count, cudaStream_t s) {
    for (int base = 0; base < n_moves; base += kMaxMovesPerLaunch) {
        RelocArgs a{};
        a.n = static_cast<u32>(n_moves - base < kMaxMovesPerLaunch ? n_moves - base : kMaxMovesPerLaunch);
        a.prefix[0] = 0;
        for (u32 i = 0; i < a.n; ++i) {
            a.mv[i] = moves[base + i];
            const u64 d0 = (a.mv[i].dst + 15) & ~u64{15};
            const u64 d1 = (a.mv[i].dst + a.mv[i].len) & ~u64{15};
            const u64 nw = d1 > d0 ? (d1 - d0) >> 4 : 0;
            const u64 chunks = nw ? (nw + kChunkWords - 1) / kChunkWords : 1;
            a.prefix[i + 1] = a.prefix[i] + static_cast<u32>(chunks);
        }
        const u32 total = a.prefix[a.n];
        const u32 want = (total + 7) / 8;
        const u32 cap = static_cast<u32>(sm_count) * 4;
        relocate_kernel<<<want < cap ? want : cap, 256, 0, s>>>(a);
        g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    }
}

}  // namespace tg
