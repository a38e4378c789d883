// K3 — relocation / compaction kernel, sm_100a.
//
// Executes one hazard-free wave of the planner's relocations
// (packing.hpp:412-456 → reuse_store.hpp:323-327) as a batched memcpy with
// arbitrary byte alignment at both ends.  The same kernel performs peer pulls
// (src in a peer arena), re-shard pieces and move_tensor.
//
// Data path (TMA bulk copies, no register staging of aligned bytes):
//  * every warp owns a private ring of four 4 KiB(+16 B) shared-memory stages
//    with one mbarrier each; lane 0 streams the warp's chunks into the ring
//    with cp.async.bulk (global -> shared, complete_tx on the stage's
//    mbarrier), three chunks ahead;
//  * a chunk is 256 destination words (16 B) of a move's 16-byte-aligned
//    destination body; its source is the aligned word run that holds those
//    bytes (one word more when the source is shifted against the destination);
//  * co-aligned chunks ((src - dst) mod 16 == 0) go straight back out of the
//    landed stage with cp.async.bulk (shared -> global, bulk_group): no thread
//    touches the bytes;
//  * shifted chunks are realigned by the warp (two LDS.128, four funnel
//    shifts, one STS.128 per destination word) into one of two out-stages,
//    which the bulk store then drains;
//  * a stage is refilled only after the bulk store that read it has finished
//    reading (cp.async.bulk.wait_group.read), an out-stage is rewritten two
//    chunks later under the same wait.
// Head and tail bytes (< 16 each, outside the aligned body) and moves too
// small to have a body are copied bytewise by one warp per move before it
// joins the pipeline (moves of one launch never overlap).
//
// The register-staged predecessor (LDG/shuffle/funnel-shift/STG, 32 KiB per
// warp task) stays selectable for A/B runs with TANGRAM_K3=ldst.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "kernels.hpp"

namespace tg {
namespace {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

struct RelocArgs {
    MoveDesc mv[kMaxMovesPerLaunch];
    u32 prefix[kMaxMovesPerLaunch + 1];  // task prefix over moves
    u32 n;
};

// ---- shared helpers -----------------------------------------------------------------
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

// Geometry of one move's aligned destination body.
struct Body {
    u64 dst, src, len;
    u64 d0, nw;       // first aligned destination word address, body words
    u64 sa;           // aligned source word holding the byte that lands on d0
    u32 o;            // (src byte of d0) mod 16
    u32 last_valid;   // bytes of source word sa[nw] inside the source range
};

__device__ __forceinline__ Body body_of(const MoveDesc& m) {
    Body b;
    b.dst = m.dst;
    b.src = m.src;
    b.len = m.len;
    b.d0 = (m.dst + 15) & ~u64{15};
    const u64 d1 = (m.dst + m.len) & ~u64{15};
    b.nw = d1 > b.d0 ? (d1 - b.d0) >> 4 : 0;
    const u64 head = b.d0 - m.dst;
    const u64 s0 = m.src + head;
    b.o = static_cast<u32>(s0 & 15);
    b.sa = s0 - b.o;
    const u64 tail = b.nw ? m.dst + m.len - d1 : 0;
    b.last_valid = b.o + static_cast<u32>(tail);
    return b;
}

// Head / tail bytes of a move (and the whole of a move without an aligned
// body), bytewise by one warp.
__device__ __forceinline__ void copy_edges(const MoveDesc& m, u32 lane) {
    auto* d = reinterpret_cast<std::uint8_t*>(m.dst);
    const auto* s = reinterpret_cast<const std::uint8_t*>(m.src);
    const u64 d0 = (m.dst + 15) & ~u64{15};
    const u64 d1 = (m.dst + m.len) & ~u64{15};
    if (d0 >= d1) {
        for (u64 i = lane; i < m.len; i += 32) d[i] = s[i];
        return;
    }
    const u64 head = d0 - m.dst, tail = m.dst + m.len - d1;
    if (lane < head) d[lane] = s[lane];
    if (lane >= 16 && lane - 16 < tail) d[(d1 - m.dst) + (lane - 16)] = s[(d1 - m.dst) + (lane - 16)];
}

// ---- K3 (TMA bulk) ------------------------------------------------------------------
constexpr u32 kChunkWords = 256;            // 4 KiB of destination per chunk
constexpr u32 kTaskChunks = 8;              // 32 KiB of contiguous destination per warp task
constexpr u64 kTaskWords = u64{kChunkWords} * kTaskChunks;
constexpr int kRing = 4;                    // in-stages per warp (3 chunks ahead)
constexpr int kWarps = 8;                   // one CTA per SM
constexpr u32 kInBytes = kChunkWords * 16 + 16;
constexpr u32 kOutBytes = kChunkWords * 16;
constexpr u32 kWarpSmem = kRing * kInBytes + 2 * kOutBytes;
constexpr u32 kSmemBytes = kWarps * kWarpSmem + kWarps * kRing * 8;

__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    u32 done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_load(u32 smem, const void* gmem, u32 bytes, u32 bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem),
                 "l"(gmem), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* gmem, u32 smem, u32 bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem), "r"(smem), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// One chunk of the warp's stream: destination words [wb, we) of move m.
struct Chunk {
    int m = -1;
    u64 wb = 0, we = 0;
};

// The warp's k-th chunk: task = warp + (k / kTaskChunks) * nwarps, chunk
// k mod kTaskChunks of it (tasks without that many chunks are skipped —
// only a move's last task is short).
struct ChunkStream {
    const RelocArgs* a;
    u32 warp, nwarps, total_tasks;
    u32 task = 0, sub = 0;  // position of the next chunk
    int m = 0;

    __device__ void start(const RelocArgs* args, u32 w, u32 nw) {
        a = args;
        warp = w;
        nwarps = nw;
        total_tasks = a->prefix[a->n];
        task = w;
        sub = 0;
        m = 0;
    }
    __device__ Chunk next() {
        Chunk c;
        while (task < total_tasks) {
            while (a->prefix[m + 1] <= task) ++m;  // tasks increase: the move index only moves forward
            const Body b = body_of(a->mv[m]);
            const u64 wb = static_cast<u64>(task - a->prefix[m]) * kTaskWords + static_cast<u64>(sub) * kChunkWords;
            if (wb < b.nw) {
                c.m = m;
                c.wb = wb;
                c.we = wb + kChunkWords < b.nw ? wb + kChunkWords : b.nw;
                if (++sub == kTaskChunks) {
                    sub = 0;
                    task += nwarps;
                }
                return c;
            }
            sub = 0;
            task += nwarps;
        }
        return c;
    }
};

// Source words a chunk loads by TMA (the partial last word, if any, is
// fetched bytewise).
__device__ __forceinline__ u32 chunk_load_words(const Body& b, const Chunk& c, bool* partial_last) {
    u64 n = c.we - c.wb;
    *partial_last = false;
    if (b.o) {
        if (c.we == b.nw && b.last_valid < 16) *partial_last = true;
        else n += 1;
    }
    return static_cast<u32>(n);
}

template <int Q>
__device__ __forceinline__ void shift_chunk(const uint4* in, uint4* out, u32 words, u32 r8, u32 lane) {
#pragma unroll 4
    for (u32 w = lane; w < words; w += 32) out[w] = realign<Q>(in[w], in[w + 1], r8);
}

__global__ void __launch_bounds__(kWarps * 32, 1) relocate_bulk_kernel(const __grid_constant__ RelocArgs a) {
    extern __shared__ __align__(128) std::uint8_t smem[];
    const u32 lane = threadIdx.x & 31;
    const u32 wid = threadIdx.x >> 5;
    const u32 warp = blockIdx.x * kWarps + wid;
    const u32 nwarps = gridDim.x * kWarps;

    // edges of moves m = warp (mod nwarps): before this warp's chunks, no
    // other warp touches those bytes
    for (u32 m = warp; m < a.n; m += nwarps) copy_edges(a.mv[m], lane);

    std::uint8_t* wbase = smem + wid * kWarpSmem;
    const u32 in0 = smem_u32(wbase);
    const u32 out0 = in0 + kRing * kInBytes;
    const u32 bar0 = smem_u32(smem + kWarps * kWarpSmem + wid * kRing * 8);
    if (lane == 0) {
        for (int s = 0; s < kRing; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();

    ChunkStream cs;
    cs.start(&a, warp, nwarps);
    Chunk ring[kRing];  // chunk held by each stage (uniform across the warp)
    auto issue = [&](int slot, const Chunk& c) {
        ring[slot] = c;
        if (c.m < 0 || lane != 0) return;
        const Body b = body_of(a.mv[c.m]);
        bool partial;
        const u32 nwords = chunk_load_words(b, c, &partial);
        const u32 bar = bar0 + 8 * slot;
        mbar_expect_tx(bar, nwords * 16);
        bulk_load(in0 + slot * kInBytes, reinterpret_cast<const void*>(b.sa + 16 * c.wb), nwords * 16, bar);
    };
    for (int s = 0; s < kRing - 1; ++s) issue(s, cs.next());
    ring[kRing - 1] = Chunk{};

    for (u32 k = 0;; ++k) {
        const int slot = static_cast<int>(k % kRing);
        const Chunk c = ring[slot];
        if (c.m < 0) break;
        __syncwarp();
        mbar_wait(bar0 + 8 * slot, (k / kRing) & 1);
        const Body b = body_of(a.mv[c.m]);
        bool partial;
        const u32 nwords = chunk_load_words(b, c, &partial);
        const u32 words = static_cast<u32>(c.we - c.wb);
        auto* in = reinterpret_cast<uint4*>(wbase + slot * kInBytes);
        u32 store_from = in0 + slot * kInBytes;
        if (b.o) {
            if (partial && lane == 0) in[nwords] = load_last_word(reinterpret_cast<const uint4*>(b.sa) + b.nw, b.last_valid);
            __syncwarp();
            auto* out = reinterpret_cast<uint4*>(wbase + kRing * kInBytes + (k & 1) * kOutBytes);
            const u32 r8 = (b.o & 3) * 8;
            switch (b.o >> 2) {
                case 0: shift_chunk<0>(in, out, words, r8, lane); break;
                case 1: shift_chunk<1>(in, out, words, r8, lane); break;
                case 2: shift_chunk<2>(in, out, words, r8, lane); break;
                default: shift_chunk<3>(in, out, words, r8, lane); break;
            }
            fence_proxy_async();  // the shifted words (generic proxy) before the bulk store reads them
            store_from = out0 + (k & 1) * kOutBytes;
        }
        __syncwarp();
        if (lane == 0) {
            bulk_store(reinterpret_cast<void*>(b.d0 + 16 * c.wb), store_from, words * 16);
            // every store but this one has finished reading shared memory:
            // the stage of chunk k - 1 and the out-stage of chunk k - 1's
            // predecessor are free
            bulk_wait_read<1>();
        }
        // refill the stage of chunk k - 1 with chunk k + kRing - 1
        issue(static_cast<int>((k + kRing - 1) % kRing), cs.next());
    }
    if (lane == 0) bulk_wait_all();
}

// ---- K3 (register staged, A/B) ----------------------------------------------------
constexpr u64 kLdstChunkWords = 2048;  // 32 KiB of destination per warp task
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 shfl_down4(uint4 v) {
    uint4 r;
    r.x = __shfl_down_sync(0xffffffffu, v.x, 1);
    r.y = __shfl_down_sync(0xffffffffu, v.y, 1);
    r.z = __shfl_down_sync(0xffffffffu, v.z, 1);
    r.w = __shfl_down_sync(0xffffffffu, v.w, 1);
    return r;
}

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

__global__ void __launch_bounds__(256) relocate_ldst_kernel(const __grid_constant__ RelocArgs a) {
    const u32 lane = threadIdx.x & 31;
    const u32 warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u32 nwarps = (gridDim.x * blockDim.x) >> 5;
    const u32 total = a.prefix[a.n];
    for (u32 m = warp; m < a.n; m += nwarps) copy_edges(a.mv[m], lane);
    for (u32 t = warp; t < total; t += nwarps) {
        u32 m = 0;
        while (a.prefix[m + 1] <= t) ++m;
        const Body b = body_of(a.mv[m]);
        if (b.nw == 0) continue;
        const u64 wb = (t - a.prefix[m]) * kLdstChunkWords;
        const u64 we = wb + kLdstChunkWords < b.nw ? wb + kLdstChunkWords : b.nw;
        const auto* sa = reinterpret_cast<const uint4*>(b.sa);
        auto* da = reinterpret_cast<uint4*>(b.d0);
        const u32 r8 = (b.o & 3) * 8;
        if (b.o == 0) copy_words<-1>(sa, da, wb, we, b.nw, b.last_valid, 0, lane);
        else if (b.o < 4) copy_words<0>(sa, da, wb, we, b.nw, b.last_valid, r8, lane);
        else if (b.o < 8) copy_words<1>(sa, da, wb, we, b.nw, b.last_valid, r8, lane);
        else if (b.o < 12) copy_words<2>(sa, da, wb, we, b.nw, b.last_valid, r8, lane);
        else copy_words<3>(sa, da, wb, we, b.nw, b.last_valid, r8, lane);
    }
}

bool use_ldst() {
    static const bool on = [] {
        const char* e = std::getenv("TANGRAM_K3");
        return e && std::strcmp(e, "ldst") == 0;
    }();
    return on;
}

}  // namespace

void relocate_launch(const MoveDesc* moves, int n_moves, int sm_count, cudaStream_t s) {
    const bool ldst = use_ldst();
    const u64 task_words = ldst ? kLdstChunkWords : kTaskWords;
    static const bool attr = [] {
        return cudaFuncSetAttribute(relocate_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) ==
               cudaSuccess;
    }();
    (void)attr;
    for (int base = 0; base < n_moves; base += kMaxMovesPerLaunch) {
        RelocArgs a{};
        a.n = static_cast<u32>(n_moves - base < kMaxMovesPerLaunch ? n_moves - base : kMaxMovesPerLaunch);
        a.prefix[0] = 0;
        for (u32 i = 0; i < a.n; ++i) {
            a.mv[i] = moves[base + i];
            const u64 d0 = (a.mv[i].dst + 15) & ~u64{15};
            const u64 d1 = (a.mv[i].dst + a.mv[i].len) & ~u64{15};
            const u64 nw = d1 > d0 ? (d1 - d0) >> 4 : 0;
            a.prefix[i + 1] = a.prefix[i] + static_cast<u32>((nw + task_words - 1) / task_words);
        }
        const u32 total = a.prefix[a.n];
        if (ldst) {
            const u32 want = (total + 7) / 8 > 0 ? (total + 7) / 8 : 1;
            const u32 cap = static_cast<u32>(sm_count) * 4;
            relocate_ldst_kernel<<<want < cap ? want : cap, 256, 0, s>>>(a);
        } else {
            // one CTA per SM; fewer when the wave has fewer tasks (edges are
            // spread over the warps too, so at least one CTA runs)
            const u32 want = (total + kWarps - 1) / kWarps > 0 ? (total + kWarps - 1) / kWarps : 1;
            const u32 cap = static_cast<u32>(sm_count);
            relocate_bulk_kernel<<<want < cap ? want : cap, kWarps * 32, kSmemBytes, s>>>(a);
        }
        g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    }
}

}  // namespace tg
