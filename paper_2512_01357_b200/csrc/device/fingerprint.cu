// K1 content fingerprint (tgfp1) and the load kernel, sm_100a.
//
// One lane hashes one 4 KiB leaf with MurmurHash3 x64-128 (seed = leaf
// index, the reference's leaf function types.hpp:77-124); a warp owns a tile
// of 32 consecutive leaves of one tensor.  Leaf digests are folded with
// wrap-around 64-bit sums (order-free, so leaves may be hashed in any order
// and by any number of warps) and flushed with one 64-bit atomic per warp
// per tensor change; a finalize kernel turns (ΣH, ΣL, n) into the root.
//
// Tensors sit at arbitrary byte offsets in the arena (catalog sizes are odd
// byte counts), so every lane reads aligned 16-byte words and realigns them
// in registers with funnel shifts; the shift is uniform per tensor, hence
// per warp, and selects one of four unrolled bodies.  The same kernel moves
// bytes (relocations, device-source placements) and fingerprints them from
// the move's own read: the load kernel below.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "../host/murmur_mix.hpp"
#include "kernels.hpp"

namespace tg {
namespace {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

// leaf_digest over a generic (shared-memory) pointer: plain loads, 4-byte
// words funnel-shifted into blocks.
__device__ void leaf_digest_generic(const std::uint8_t* p, u32 len, u64 seed, u64& d1, u64& d2) {
    mm::W32 h1 = mm::w_of(seed), h2 = h1;
    const u32 nblk = len >> 4;
    const u32 o = static_cast<u32>(reinterpret_cast<std::uintptr_t>(p) & 3);
    const u32* wp = reinterpret_cast<const u32*>(p - o);
    const u32 r8 = o * 8;
    for (u32 j = 0; j < nblk; ++j) {
        u32 u[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) u[q] = (q < 4 || o) ? wp[4 * j + q] : 0u;
        const u32 a = __funnelshift_r(u[0], u[1], r8), b = __funnelshift_r(u[1], u[2], r8);
        const u32 c = __funnelshift_r(u[2], u[3], r8), d = __funnelshift_r(u[3], u[4], r8);
        mm::body_dev(h1, h2, mm::W32{a, b}, mm::W32{c, d});
    }
    const u32 rem = len & 15;
    u64 t1 = 0, t2 = 0;
    const std::uint8_t* tp = p + (static_cast<u64>(nblk) << 4);
    for (u32 b = 0; b < rem; ++b) {
        const u64 v = tp[b];
        if (b < 8) t1 |= v << (8 * b);
        else t2 |= v << (8 * (b - 8));
    }
    u64 f1 = mm::u_of(h1), f2 = mm::u_of(h2);
    mm::finish(f1, f2, t1, t2, rem, len);
    d1 = f1;
    d2 = f2;
}

__device__ __forceinline__ u64 warp_sum(u64 v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    return v;
}

// ---- staging ---------------------------------------------------------------------
// A stage is 8 blocks (128 B) of each of a warp's 32 leaves, copied into
// shared memory with coalesced 16-byte cp.async (LDGSTS); every lane then
// reads its own leaf's words with conflict-free LDS.128.  (Design history:
// per-lane direct loads were L1-wavefront bound, per-lane TMA bulk copies
// serialised on uniform operands.)
constexpr int kStageBlocks = 8;
constexpr int kSlotWords = kStageBlocks + 1;
constexpr int kStagesPerLeaf = static_cast<int>(kLeafBytes / 16) / kStageBlocks;  // 32

// The 9th (realignment) word of a stage is the first word of the next 128
// bytes — at a leaf's last stage, of the next leaf, read long before: no
// 256-byte prefetch for it (that re-fetched 256 B per leaf from DRAM).
__device__ __forceinline__ void cp_async16_noprefetch(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// First `valid` (< 16) bytes only, the rest of the 16-byte slot zero-filled:
// a source word that runs past the end of the tensor is never read beyond it
// (registered device sources have no slack after them).
__device__ __forceinline__ void cp_async16_partial(void* smem, const void* gmem, u32 valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    // L2::256B: the L2 fetches the whole 256-byte pair of lines, so a leaf's
    // next stage (the next line) is an L2 hit and DRAM sees 256-byte requests
    // (16 GiB aligned: verify 6.11 -> 6.49 TB/s, copy 5.63 -> 6.01 r+w;
    // unaligned cases unchanged — tools/phase_sweep.py).
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// One LDS.128 for a 16-byte staged word.  Plain uint4 loads whose components
// are only partly used get split into LDS.64 pairs, and a half-warp LDS.64
// phase sees leaves l and l+8 on the same swizzled bank pair (2-way conflict).
__device__ __forceinline__ uint4 lds128(const uint4* p) {
    uint4 v;
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(s));
    return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Stage layout: 32 slots of 8 words (128 B) with the word index
// XOR-swizzled by (leaf & 7), plus a 32-word column holding each leaf's 9th
// (realignment) word.  Tiles that only fingerprint fill that column at a
// leaf's last stage alone and otherwise read word 0 of the next stage.  Copy i of a lane is leaf 4i + lane/8, word lane%8: one
// base register plus the immediate 16 KiB·i per LDGSTS, no predicates on full
// tiles, and both the LDGSTS writes and the per-lane LDS.128 reads are bank
// conflict free.
constexpr int kV3StageWords = 32 * kStageBlocks + 32;  // slots + extra column

template <int Q>
__device__ __forceinline__ void v3_hash_stage(const uint4* stage_buf, const uint4* xw, u32 lane, u32 r8, mm::W32& h1,
                                              mm::W32& h2) {
    const uint4* slot = stage_buf + lane * 8;
    const u32 key = lane & 7;
    uint4 w[kSlotWords];
#pragma unroll
    for (int q = 0; q < kStageBlocks; ++q) w[q] = lds128(slot + (q ^ key));
    w[kStageBlocks] = lds128(xw);
#pragma unroll
    for (int b = 0; b < kStageBlocks; ++b) {
        const u32 u[8] = {w[b].x, w[b].y, w[b].z, w[b].w, w[b + 1].x, w[b + 1].y, w[b + 1].z, w[b + 1].w};
        const u32 a = __funnelshift_r(u[Q + 0], u[Q + 1], r8);
        const u32 c = __funnelshift_r(u[Q + 1], u[Q + 2], r8);
        const u32 d = __funnelshift_r(u[Q + 2], u[Q + 3], r8);
        const u32 e = __funnelshift_r(u[Q + 3], u[Q + 4], r8);
        mm::body_dev(h1, h2, mm::W32{a, c}, mm::W32{d, e});
    }
}

// 16-byte-aligned leaves: the blocks are the staged words themselves.
__device__ __forceinline__ void v3_hash_stage_aligned(const uint4* stage_buf, u32 lane, mm::W32& h1, mm::W32& h2) {
    const uint4* slot = stage_buf + lane * 8;
    const u32 key = lane & 7;
#pragma unroll
    for (int b = 0; b < kStageBlocks; ++b) {
        const uint4 w = lds128(slot + (b ^ key));
        mm::body_dev(h1, h2, mm::W32{w.x, w.y}, mm::W32{w.z, w.w});
    }
}

// A warp's view of one tile: the tensor, the tile's first leaf, the number of
// full leaves in it, and the source alignment o (uniform per tensor).
struct TileRef {
    const std::uint8_t* a0;  // aligned base of leaf 0 of the tile
    const std::uint8_t* base;  // tensor base
    u64 n;                   // tensor bytes
    u64 leaf0;
    u64 seed0;               // the task's leaf_base: seed of leaf l is seed0 + l
    u32 nfull;
    u32 o;
    int task;
};

// xw: the leaf's 9th word — the extra column, or word 0 of the leaf's next
// stage when that stage has landed in the ring.
__device__ __forceinline__ void v4_hash(const uint4* stage_buf, const uint4* xw, const TileRef& tr, u32 lane,
                                        mm::W32& h1, mm::W32& h2) {
    if (tr.o == 0) {
        v3_hash_stage_aligned(stage_buf, lane, h1, h2);
        return;
    }
    const u32 r8 = (tr.o & 3) * 8;
    switch (tr.o >> 2) {
        case 0: v3_hash_stage<0>(stage_buf, xw, lane, r8, h1, h2); break;
        case 1: v3_hash_stage<1>(stage_buf, xw, lane, r8, h1, h2); break;
        case 2: v3_hash_stage<2>(stage_buf, xw, lane, r8, h1, h2); break;
        default: v3_hash_stage<3>(stage_buf, xw, lane, r8, h1, h2); break;
    }
}

__global__ void fp_finalize_kernel(const FpTask* __restrict__ tasks, u32 n_tasks, const u64* __restrict__ sums,
                                   u64* __restrict__ digests) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tasks) return;
    u64 h1 = 0, h2 = 0;
    mm::body(h1, h2, sums[2 * i], sums[2 * i + 1]);
    mm::finish(h1, h2, tasks[i].n, 0, 8, 24);
    digests[2 * i] = h1;
    digests[2 * i + 1] = h2;
}

// ---- K3F: copy + fingerprint in one pass ------------------------------------------
// Moves a tensor (relocation wave member, HBM-cache or peer placement) and
// computes its tgfp1 digest from the same staged bytes, so the bytes cross
// HBM once in each direction instead of copy (r+w) + fingerprint (r).
// Staging and hashing are v4's.  The destination is written from the staged
// slots: with o = src & 15, od = dst & 15 and delta = (o - od) mod 16, the
// 16-byte destination word of leaf l, stage s, index q holds tensor bytes
// [x, x+16), x = 4096 l + 128 s - o + delta + 16 q — slot bytes delta+16q..,
// i.e. slot words q, q+1 funnel-shifted by delta.  These words tile the
// tensor without gaps or overlaps; the ones that would reach outside
// [0, 4096 F) (F = full leaves) are left to an edge pass that copies the
// head (< 16 B) and the tail (< 4 KiB + 16 B) bytewise.
//
// Those words are stored one 128-byte destination line per leaf and stage:
// with k = ((dst + delta - o) mod 128) / 16, line lane q takes word
// (q - k) mod 8 of stage s when q >= k, else of stage s - 1 (still in the
// ring), and each leaf stores the k words of its stage 31 that spill into
// the next line after its last stage.  An unaligned 128-byte run would
// touch two lines and five sectors per leaf-stage and leave half sectors
// for L2 to merge (measured: 3.4 vs 5.0 TB/s for delta = 8, dst % 32 = 8).
struct CopyTileRef {
    TileRef t;
    std::uint8_t* dst;  // destination of tensor byte 0 (nullptr: fingerprint only)
    u32 delta;
    u32 k;               // destination line phase of the word grid, in words
    u64 x_first, x_end;  // full-word writes cover tensor bytes [x_first, x_end)
    int gate, wave;
};

// K1 runs through the load kernel too: an FpTask is a fingerprint-only task.
__device__ __forceinline__ CopyFpTask as_copy_task(const CopyFpTask& t) { return t; }
__device__ __forceinline__ CopyFpTask as_copy_task(const FpTask& t) {
    return CopyFpTask{t.base, nullptr, t.n, t.tile0, -1, -1, 0};
}

// Task of tile t: the last task with tile0 <= t.  A warp takes its tiles in
// increasing order, so the search starts at the task of its previous tile
// (`hint`, tile0 <= t) and scans 32 tasks per round with one load per lane —
// one dependent L2 round trip per tile instead of log2(n_tasks).
template <class Task>
__device__ __forceinline__ u32 find_task(const Task* __restrict__ tasks, u32 n_tasks, u64 t, u32 hint, u32 lane) {
    for (u32 base = hint;; base += 31) {
        const u32 i = base + lane;
        const unsigned m = __ballot_sync(0xffffffffu, i < n_tasks && tasks[i].tile0 <= t);
        if (m != 0xffffffffu || base + 32 >= n_tasks) return base + 31 - __clz(m);  // lane 0 always set
    }
}

// A/B knob (TANGRAM_TILE_ORDER=forward): dispense a task's tiles first-first.
__constant__ bool tile_order_reversed = true;

template <class Task>
__device__ __forceinline__ CopyTileRef copy_tile_ref(const Task* __restrict__ tasks, u32 n_tasks, u64 t,
                                                     u64 total_tiles, u32 hint, u32 lane) {
    CopyTileRef r{};
    r.t.task = -1;
    if (t >= total_tiles) return r;
    const u32 lo = find_task(tasks, n_tasks, t, hint, lane);
    const CopyFpTask tk = as_copy_task(tasks[lo]);
    r.t.task = static_cast<int>(lo);
    r.t.base = tk.src;
    r.t.n = tk.n;
    r.t.seed0 = tk.leaf_base & ~kRawSums;
    // A task's tiles are dispensed last-first: the tile holding the partial
    // leaf and the tail bytes (one lane hashes that leaf serially) comes
    // early, so the launch's final tiles are plain full tiles and the tail
    // of the launch is shorter.
    const u64 task_tiles = ((tk.n + kLeafBytes - 1) / kLeafBytes + kLeavesPerTile - 1) / kLeavesPerTile;
    r.t.leaf0 = (tile_order_reversed ? task_tiles - 1 - (t - tk.tile0) : t - tk.tile0) * kLeavesPerTile;
    const u64 full = tk.n / kLeafBytes;
    r.t.nfull = full > r.t.leaf0 ? static_cast<u32>(min(full - r.t.leaf0, u64{32})) : 0u;
    const std::uint8_t* p0 = tk.src + r.t.leaf0 * kLeafBytes;
    r.t.o = static_cast<u32>(reinterpret_cast<std::uintptr_t>(p0) & 15);
    r.t.a0 = p0 - r.t.o;
    r.dst = tk.dst;
    r.gate = tk.gate;
    r.wave = tk.wave;
    if (!tk.dst) return r;  // delta = k = 0: no realignment, no writes
    const u32 od = static_cast<u32>(reinterpret_cast<std::uintptr_t>(tk.dst) & 15);
    r.delta = (r.t.o - od) & 15;
    // first x >= 0 on the grid x ≡ delta - o (mod 16); last with x + 16 <= 4096 F
    const long long x0 = static_cast<long long>(r.delta) - static_cast<long long>(r.t.o);
    r.k = static_cast<u32>(((reinterpret_cast<std::uintptr_t>(tk.dst) + static_cast<std::uintptr_t>(x0)) & 127) >> 4);
    r.x_first = static_cast<u64>(x0 < 0 ? x0 + 16 : x0);
    const u64 lim = full * kLeafBytes;
    r.x_end = lim >= r.x_first + 16 ? r.x_first + ((lim - r.x_first) / 16) * 16 : r.x_first;
    return r;
}

template <int QD>
__device__ __forceinline__ uint4 realign_words(uint4 w0, uint4 w1, u32 r8) {
    const u32 u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    return make_uint4(__funnelshift_r(u[QD + 0], u[QD + 1], r8), __funnelshift_r(u[QD + 1], u[QD + 2], r8),
                      __funnelshift_r(u[QD + 2], u[QD + 3], r8), __funnelshift_r(u[QD + 3], u[QD + 4], r8));
}

// Store one destination line per leaf of the tile: lane -> leaf 4i + lane/8,
// line word q = lane%8, which is word j = (q - k) mod 8 of stage `so` (s for
// q >= k, s - 1 for q < k; see CopyTileRef).  The lane's tensor offset and
// swizzled smem positions are computed once; copy i adds 16 KiB (4 leaves),
// interior tiles skip the edge test.  SHIFT = false is the delta = 0 case:
// the staged word is the destination word.
template <int QD, bool SHIFT>
__device__ __forceinline__ void write_lines(const uint4* cur_buf, const uint4* prev_buf, const CopyTileRef& c, int s,
                                            bool use_cur, bool use_prev, bool check, u32 r8, u32 lane) {
    const u32 g = lane >> 3, q = lane & 7;
    const bool from_cur = q >= c.k;
    if (!(from_cur ? use_cur : use_prev)) return;
    const u32 j = (q - c.k) & 7;
    const int so = from_cur ? s : s - 1;
    const uint4* sbuf = from_cur ? cur_buf : prev_buf;
    const uint4* base = sbuf + g * 8;
    const uint4* extra = sbuf + 32 * kStageBlocks + g;
    const u32 pa0 = j ^ g, pb0 = j ^ (4u ^ g);
    const u32 pa1 = ((j + 1) & 7) ^ g, pb1 = ((j + 1) & 7) ^ (4u ^ g);
    const long long x_lane = static_cast<long long>((c.t.leaf0 + g) * kLeafBytes) + 16LL * j +
                             static_cast<long long>(c.delta) - static_cast<long long>(c.t.o) + 128LL * so;
    std::uint8_t* dst_lane = c.dst + x_lane;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const u32 l = 4 * i + g;
        if (l >= c.t.nfull) continue;
        const long long x = x_lane + 16384LL * i;
        if (check && (x < static_cast<long long>(c.x_first) || x + 16 > static_cast<long long>(c.x_end))) continue;
        const uint4 w0 = lds128(base + 32 * i + ((i & 1) ? pb0 : pa0));
        uint4 v = w0;
        if constexpr (SHIFT) {
            const uint4 w1 = lds128(j == 7 ? extra + 4 * i : base + 32 * i + ((i & 1) ? pb1 : pa1));
            v = realign_words<QD>(w0, w1, r8);
        }
        __stcs(reinterpret_cast<uint4*>(dst_lane + 16384LL * i), v);
    }
}

// Up to three line stores of one iteration (paired mode: line s - 1, line s,
// and after a leaf's last stage the spill line) through ONE instance of the
// unrolled store body: job t takes (cur, prev, stage, use_cur, use_prev) from
// the arguments by index, in a loop that is not unrolled — the load kernel's
// instruction footprint matters (warps of one SM run different alignment
// variants; ncu shows no_instructions stalls).
template <int QD, bool SHIFT>
__device__ __forceinline__ void write_line_jobs(const uint4* b0, const uint4* b1, const uint4* b2, int s, int nj,
                                                bool first_prev, const CopyTileRef& c, bool check, u32 r8, u32 lane) {
#pragma unroll 1
    for (int t = 0; t < nj; ++t) {
        // t = 0: line s - 1 (cur b1, prev b0); t = 1: line s (cur b2, prev b1);
        // t = 2: spill line s + 1 (no cur, prev b2)
        const uint4* cur = t == 0 ? b1 : b2;
        const uint4* prev = t == 0 ? b0 : (t == 1 ? b1 : b2);
        write_lines<QD, SHIFT>(cur, prev, c, s - 1 + t, t < 2, t == 0 ? first_prev : true, check, r8, lane);
    }
}

__device__ __forceinline__ void write_pair_dispatch(const uint4* b0, const uint4* b1, const uint4* b2, int s, int nj,
                                                    bool first_prev, const CopyTileRef& c, u32 lane) {
    const long long tile_lo = static_cast<long long>(c.t.leaf0 * kLeafBytes) - 16;
    const long long tile_hi = static_cast<long long>((c.t.leaf0 + c.t.nfull) * kLeafBytes) + 16;
    const bool check = tile_lo < static_cast<long long>(c.x_first) || tile_hi > static_cast<long long>(c.x_end);
    if (c.delta == 0) {
        write_line_jobs<0, false>(b0, b1, b2, s, nj, first_prev, c, check, 0, lane);
        return;
    }
    const u32 r8 = (c.delta & 3) * 8;
    switch (c.delta >> 2) {
        case 0: write_line_jobs<0, true>(b0, b1, b2, s, nj, first_prev, c, check, r8, lane); break;
        case 1: write_line_jobs<1, true>(b0, b1, b2, s, nj, first_prev, c, check, r8, lane); break;
        case 2: write_line_jobs<2, true>(b0, b1, b2, s, nj, first_prev, c, check, r8, lane); break;
        default: write_line_jobs<3, true>(b0, b1, b2, s, nj, first_prev, c, check, r8, lane); break;
    }
}

__device__ __forceinline__ void write_lines_dispatch(const uint4* cur_buf, const uint4* prev_buf, const CopyTileRef& c,
                                                     int s, bool use_cur, bool use_prev, u32 lane) {
    // the whole tile is inside [x_first, x_end) unless it holds the tensor's
    // first or last full leaf (its words are within 16 bytes of its leaves)
    const long long tile_lo = static_cast<long long>(c.t.leaf0 * kLeafBytes) - 16;
    const long long tile_hi = static_cast<long long>((c.t.leaf0 + c.t.nfull) * kLeafBytes) + 16;
    const bool check = tile_lo < static_cast<long long>(c.x_first) || tile_hi > static_cast<long long>(c.x_end);
    if (c.delta == 0) {
        write_lines<0, false>(cur_buf, prev_buf, c, s, use_cur, use_prev, check, 0, lane);
        return;
    }
    const u32 r8 = (c.delta & 3) * 8;
    switch (c.delta >> 2) {
        case 0: write_lines<0, true>(cur_buf, prev_buf, c, s, use_cur, use_prev, check, r8, lane); break;
        case 1: write_lines<1, true>(cur_buf, prev_buf, c, s, use_cur, use_prev, check, r8, lane); break;
        case 2: write_lines<2, true>(cur_buf, prev_buf, c, s, use_cur, use_prev, check, r8, lane); break;
        default: write_lines<3, true>(cur_buf, prev_buf, c, s, use_cur, use_prev, check, r8, lane); break;
    }
}

// The extra (9th) word of every leaf-stage is needed by the writes whenever
// delta > 0, by the hash whenever o > 0; load it when it holds a tensor byte.
__device__ __forceinline__ void copy_issue(uint4* stage_buf, const CopyTileRef& c, int s, u32 lane, bool next_words) {
    const TileRef& tr = c.t;
    if (tr.task < 0 || tr.nfull == 0) {
        cp_async_commit();
        return;
    }
    const std::uint8_t* src_lane =
        tr.a0 + static_cast<u64>(lane >> 3) * kLeafBytes + (lane & 7) * 16 + static_cast<u64>(s) * 128;
    const u64 extra_word = (tr.leaf0 + lane) * kLeafBytes + static_cast<u64>(s) * 128 + 128;  // tensor offset + o
    const bool extra = (tr.o != 0 || c.delta != 0) && (!next_words || s == kStagesPerLeaf - 1) && extra_word - tr.o < tr.n;
    const std::uint8_t* src_extra = tr.a0 + static_cast<u64>(lane) * kLeafBytes + static_cast<u64>(s) * 128 + 128;
    const u32 leaf_in_group = lane >> 3, q = lane & 7;
    if (tr.nfull == 32) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const u32 key = ((4 * i) & 7) ^ leaf_in_group;
            cp_async16(stage_buf + (4 * i + leaf_in_group) * 8 + (q ^ key), src_lane + static_cast<u64>(i) * 16384);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const u32 l = 4 * i + leaf_in_group;
            if (l < tr.nfull) cp_async16(stage_buf + l * 8 + (q ^ (l & 7)), src_lane + static_cast<u64>(i) * 16384);
        }
    }
    if (extra && lane < tr.nfull) {
        const u64 left = tr.n - (extra_word - tr.o);  // tensor bytes from the word's start (> 0)
        if (left >= 16) cp_async16_noprefetch(stage_buf + 32 * kStageBlocks + lane, src_extra);
        else cp_async16_partial(stage_buf + 32 * kStageBlocks + lane, src_extra, static_cast<u32>(left));
    }
    cp_async_commit();
}

// Release-ordered add: the warp's reads and stores before it (ordered by the
// preceding __syncwarp) are visible to whoever acquires the counter.
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ u64 ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Tiles are handed out in task order by one counter, so every tile of the
// wave a gated tile waits for was taken earlier by a running warp: the wait
// always ends, whatever the residency.  Reads never wait: a wave never writes
// into a later wave's (or an in-place task's) source bytes.
__device__ __forceinline__ u64 next_tile(unsigned long long* counter, u32 lane) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(counter, 1ull);
    return __shfl_sync(0xffffffffu, t, 0);
}

// Stage ring of the load kernel: four slots per warp, six warps per CTA, two
// CTAs (2 x 108 KiB) per SM.
//  * Tasks that write (kPair): the stores of stages s - 1 and s go out
//    together at odd s, so each leaf receives 256 contiguous bytes at a time.
//    With single 128-byte lines 4 KiB apart DRAM write efficiency drops
//    (B200, plain register copies: 4.94 TB/s r+w for 128-byte pieces, 5.87
//    for 256-byte pieces, 6.0 contiguous — tools/store_pattern.cu).  A line
//    of stage s reads stage s and the last words of stage s - 1, so a pair at
//    odd s reads s - 2 .. s; after it both s - 2 and s - 1 are refilled, so
//    two or three stages are in flight.
//  * Fingerprint-only launches (K1), or TANGRAM_LOAD_RING=single: one line per
//    stage; a line reads s - 1 and s, and two stages are in flight.
template <int STAGES, int WARPS, bool PAIR, bool NEXT = false>
struct CopyCfg {
    static constexpr bool kNext = NEXT;
    static constexpr int kStages = STAGES;
    static constexpr int kWarps = WARPS;
    static constexpr bool kPair = PAIR;
    static constexpr int kAhead = STAGES - 1;  // single-line ring: stages in flight + 1
    static constexpr int kWarpWords = STAGES * kV3StageWords;
    static constexpr int kSmemBytes = WARPS * kWarpWords * 16;
};
using CfgSingle = CopyCfg<4, 6, false>;
using CfgPair = CopyCfg<4, 6, true>;
// K1 (fingerprint-only launches): three slots and eight warps per CTA — the
// shared memory of four slots x six warps, 16 instead of 12 resident warps
// per SM (A/B on one box: K1 8 GiB misaligned +1.7 %, warm reloads of
// opt1.3B / qwen3B / opt13B 1.5-2 % faster).  TANGRAM_K1_RING=4x6 selects
// the four-slot ring for A/B runs.
using CfgFpNext = CopyCfg<3, 8, false, true>;
using CfgFpNext46 = CopyCfg<4, 6, false, true>;

template <class Task, class Cfg>
__device__ __forceinline__ void load_tiles(const Task* __restrict__ tasks, u32 n_tasks, u64 total_tiles,
                                           u64* __restrict__ sums, unsigned long long* __restrict__ sync,
                                           const u64* __restrict__ need, bool verify_next) {
    constexpr int kStagesRing = Cfg::kStages;
    constexpr int kAhead = Cfg::kAhead;
    extern __shared__ uint4 smem[];
    const u32 lane = threadIdx.x & 31;
    const u32 wid = threadIdx.x >> 5;
    uint4* wbuf = smem + wid * Cfg::kWarpWords;
    CopyTileRef cur = copy_tile_ref(tasks, n_tasks, next_tile(sync, lane), total_tiles, 0u, lane);
    if (cur.t.task < 0) return;
    CopyTileRef nxt = copy_tile_ref(tasks, n_tasks, next_tile(sync, lane), total_tiles, static_cast<u32>(cur.t.task),
                                    lane);
    int cur_task = -1;
    u64 acc_h = 0, acc_l = 0;
    u32 buf = 0;
    // Fingerprint-only single ring: a stage's 9th words are word 0 of the
    // next stage (waited for before hashing), so only the leaf's last stage
    // loads the extra column — one uncoalesced 32-line request per leaf
    // instead of one per stage.
    constexpr bool kFpNext = std::is_same<Task, FpTask>::value && Cfg::kNext && !Cfg::kPair;
    constexpr int kPrologue = Cfg::kPair ? 3 : kAhead;  // stages 0 .. kPrologue - 1 before the loop
#pragma unroll
    for (int s = 0; s < kPrologue; ++s)
        copy_issue(wbuf + s * kV3StageWords, cur, s, lane, kFpNext || (Cfg::kPair && verify_next && cur.dst == nullptr));
    while (cur.t.task >= 0) {
        if (cur.t.task != cur_task) {
            if (cur_task >= 0) {
                const u64 sh = warp_sum(acc_h), sl = warp_sum(acc_l);
                if (lane == 0) {
                    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur_task), sh);
                    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur_task + 1), sl);
                }
            }
            cur_task = cur.t.task;
            acc_h = acc_l = 0;
        }
        const bool writes = cur.dst != nullptr;
        if (writes && cur.gate >= 0) {
            if (lane == 0) {
                const u64 want = need[cur.gate];
                while (ld_acquire(sync + 1 + cur.gate) < want) __nanosleep(256);
            }
            __syncwarp();
        }
        const u64 my_leaf = cur.t.seed0 + cur.t.leaf0 + lane;
        mm::W32 h1 = mm::w_of(my_leaf), h2 = h1;
        // The line stores of stage s also read stage s - 1 (pairs: s - 2 .. s),
        // so the ring slot refilled with stage s + kAhead is the one no store
        // reads any more: that of s - 1 (single lines) or s - 2 (pairs).
        auto issue = [&](int stage, int slot) {
            uint4* dst = wbuf + slot * kV3StageWords;
            // verify tiles of paired launches take the next-stage words too
            if (stage < kStagesPerLeaf)
                copy_issue(dst, cur, stage, lane, kFpNext || (Cfg::kPair && verify_next && cur.dst == nullptr));
            else
                copy_issue(dst, nxt, stage - kStagesPerLeaf, lane, kFpNext || (Cfg::kPair && verify_next && nxt.dst == nullptr));
        };
        for (int s = 0; s < kStagesPerLeaf; ++s) {
            const uint4* sb = wbuf + buf * kV3StageWords;
            const u32 b1 = (buf + kStagesRing - 1) % kStagesRing, b2 = (buf + kStagesRing - 2) % kStagesRing;
            const uint4* sp = wbuf + b1 * kV3StageWords;
            if constexpr (Cfg::kPair) {
                // Ring schedule: at odd s the pair (s - 1, s) is stored and
                // both of its older slots (s - 2, s - 1) are refilled at once
                // with s + 2 and s + 3; at even s nothing is refilled.  Stages
                // up to s + 2 (even s) or s + 1 (odd s) have been issued.
                // Verify tiles (no stores) run the fingerprint-only schedule:
                // refill the slot of s - 1 with s + 3, wait for s and s + 1,
                // realign from the next stage's word 0.  Both schedules leave
                // the next tile's stages 0..2 issued in slots (stage mod 4), so
                // tiles of either kind follow each other.
                if (writes || !verify_next) {
                    if (s & 1) cp_async_wait<1>();
                    else cp_async_wait<2>();
                    __syncwarp();
                    if (s & 1) {
                        if (writes && cur.t.nfull) {
                            const uint4* spp = wbuf + b2 * kV3StageWords;
                            const int nj = (s == kStagesPerLeaf - 1 && cur.k) ? 3 : 2;
                            write_pair_dispatch(spp, sp, sb, s, nj, s > 1, cur, lane);
                        }
                        __syncwarp();
                        issue(s + 2, static_cast<int>(b2));
                        issue(s + 3, static_cast<int>(b1));
                    }
                } else {
                    __syncwarp();
                    issue(s + 3, static_cast<int>(b1));
                    cp_async_wait<2>();
                    __syncwarp();
                }
                const uint4* xw = (!writes && verify_next && s < kStagesPerLeaf - 1)
                                      ? wbuf + ((buf + 1) % kStagesRing) * kV3StageWords + lane * 8 + (lane & 7)
                                      : sb + 32 * kStageBlocks + lane;
                if (lane < cur.t.nfull) v4_hash(sb, xw, cur.t, lane, h1, h2);
            } else if constexpr (kFpNext) {
                // slot of s - 1 is free (no line stores): refill first, then
                // wait for s and s + 1
                issue(s + kAhead, static_cast<int>((buf + kAhead) % kStagesRing));
                cp_async_wait<kAhead - 1>();
                __syncwarp();
                const uint4* nb = wbuf + ((buf + 1) % kStagesRing) * kV3StageWords;
                const uint4* xw = s < kStagesPerLeaf - 1 ? nb + lane * 8 + (lane & 7) : sb + 32 * kStageBlocks + lane;
                if (lane < cur.t.nfull) v4_hash(sb, xw, cur.t, lane, h1, h2);
                __syncwarp();
            } else {
                cp_async_wait<kAhead - 1>();
                __syncwarp();
                if (writes && cur.t.nfull) write_lines_dispatch(sb, sp, cur, s, true, s > 0, lane);
                if (s == kStagesPerLeaf - 1 && writes && cur.t.nfull && cur.k)
                    write_lines_dispatch(nullptr, sb, cur, kStagesPerLeaf, false, true, lane);
                if (lane < cur.t.nfull) v4_hash(sb, sb + 32 * kStageBlocks + lane, cur.t, lane, h1, h2);
                __syncwarp();
                issue(s + kAhead, static_cast<int>((buf + kAhead) % kStagesRing));
            }
            buf = (buf + 1) % kStagesRing;
        }
        if (lane < cur.t.nfull) {
            u64 f1 = mm::u_of(h1), f2 = mm::u_of(h2);
            mm::finish(f1, f2, 0, 0, 0, kLeafBytes);
            acc_h += f1;
            acc_l += f2;
        }
        // The tensor's last tile: the partial leaf (< 4 KiB) and, for moves,
        // the bytes no full word covers (head < 16 B; tail = [x_end, n)).
        // The warp stages [from, n) in the ring slot stage 31 just released
        // (one round of coalesced loads), then hashes the partial leaf and
        // copies the tail from shared memory — a per-byte global loop here
        // costs tens of microseconds of DRAM latency at the end of a launch.
        if (cur.t.leaf0 + 32 >= (cur.t.n + kLeafBytes - 1) / kLeafBytes) {
            const u64 pl = (cur.t.n / kLeafBytes) * kLeafBytes;  // partial leaf start
            const u64 from = writes ? min(cur.x_end, pl) : pl;
            if (from < cur.t.n) {
                __syncwarp();
                uint4* tb = wbuf + ((buf + kStagesRing - 1) % kStagesRing) * kV3StageWords;
                const std::uint8_t* g0 = cur.t.base + from;
                const u32 ga = static_cast<u32>(reinterpret_cast<std::uintptr_t>(g0) & 15);
                const uint4* gw = reinterpret_cast<const uint4*>(g0 - ga);
                const u32 nw = static_cast<u32>((ga + (cur.t.n - from) + 15) / 16);
                const std::uint8_t* gend = cur.t.base + cur.t.n;
                for (u32 w = lane; w < nw; w += 32) {
                    const std::uint8_t* wa = reinterpret_cast<const std::uint8_t*>(gw + w);
                    if (wa + 16 <= gend) {
                        tb[w] = __ldg(gw + w);
                    } else {  // the last word: only the bytes before the end of the tensor
                        u64 lo = 0, hi = 0;
                        for (u32 i = 0; wa + i < gend; ++i) {
                            const u64 v = wa[i];
                            if (i < 8) lo |= v << (8 * i);
                            else hi |= v << (8 * (i - 8));
                        }
                        tb[w] = make_uint4(static_cast<u32>(lo), static_cast<u32>(lo >> 32), static_cast<u32>(hi),
                                           static_cast<u32>(hi >> 32));
                    }
                }
                __syncwarp();
                const std::uint8_t* sbytes = reinterpret_cast<const std::uint8_t*>(tb) + ga;
                if (lane == cur.t.nfull && pl < cur.t.n) {
                    u64 d1, d2;
                    leaf_digest_generic(sbytes + (pl - from), static_cast<u32>(cur.t.n - pl),
                                        cur.t.seed0 + pl / kLeafBytes, d1, d2);
                    acc_h += d1;
                    acc_l += d2;
                }
                if (writes)
                    for (u64 b = lane; b < cur.t.n - from; b += 32) cur.dst[from + b] = sbytes[b];
                __syncwarp();
            }
            if (writes)
                for (u64 b = lane; b < cur.x_first && b < cur.t.n; b += 32) cur.dst[b] = cur.t.base[b];
        }
        if (cur.wave >= 0) {  // this tile's source bytes are all read
            __syncwarp();
            if (lane == 0) red_release_add(sync + 1 + cur.wave, 1ull);
        }
        const u32 hint = static_cast<u32>(nxt.t.task >= 0 ? nxt.t.task : cur.t.task);
        cur = nxt;
        nxt = copy_tile_ref(tasks, n_tasks, next_tile(sync, lane), total_tiles, hint, lane);
    }
    cp_async_wait<0>();
    if (cur_task >= 0) {
        const u64 sh = warp_sum(acc_h), sl = warp_sum(acc_l);
        if (lane == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur_task), sh);
            atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur_task + 1), sl);
        }
    }
}

// tgfp1 root of one task from its leaf sums (types.hpp:77-124 over
// le64 H || le64 L || le64 n).
__device__ __forceinline__ void digest_of(u64 sum_h, u64 sum_l, u64 n, u64* out) {
    u64 h1 = 0, h2 = 0;
    mm::body(h1, h2, sum_h, sum_l);
    mm::finish(h1, h2, n, 0, 8, 24);
    out[0] = h1;
    out[1] = h2;
}

// The last warp of the launch to finish writes every task's digest, so a load
// needs no second kernel (threadFenceReduction pattern at warp granularity:
// each warp's sums are device-visible before its ticket, the last ticket
// sees them all).  No shared memory and no CTA barrier: a static __shared__
// flag here shifts the dynamic stage ring and cost K1 8-12 % (A/B on one
// box, 8 GiB: 5.6-5.9 vs 6.4-6.8 TB/s).
__device__ __forceinline__ u64 globaltimer_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ bool raw_sums(const FpTask&) { return false; }
__device__ __forceinline__ bool raw_sums(const CopyFpTask& t) { return (t.leaf_base & kRawSums) != 0; }

// The last warp's work, kept out of line: it runs once per launch and stays
// out of the tile loop's code (A/B on one box against the inlined form and
// against the kernel without stamps / clean-up: K1, move + fingerprint and
// verify rates within 1.5 %).
template <class Task>
__device__ __noinline__ void finalize_tail(const Task* __restrict__ tasks, u32 n_tasks, const u64* sums,
                                           u64* __restrict__ digests, unsigned long long* done, u64* stamps,
                                           bool clean, unsigned long long* sync) {
    const u32 lane = threadIdx.x & 31;
    for (u32 i = lane; i < n_tasks; i += 32) {
        const u64 sh = __ldcg(sums + 2 * i), sl = __ldcg(sums + 2 * i + 1);
        if (raw_sums(tasks[i])) {  // a piece of a tensor: the host adds the pieces
            digests[2 * i] = sh;
            digests[2 * i + 1] = sl;
        } else {
            digest_of(sh, sl, tasks[i].n, digests + 2 * i);
        }
    }
    if (clean) {       // every other warp is done with them: leave the stage zeroed for the next launch
        __syncwarp();  // (every lane has read its tasks' sums)
        u64* s = const_cast<u64*>(sums);
        for (u32 i = lane; i < 2 * n_tasks; i += 32) s[i] = 0;
        for (u32 i = lane; sync + i <= done; i += 32) sync[i] = 0;
    }
    if (stamps) {  // the launch's end, after the digests (the host may poll it)
        __threadfence_system();
        if (lane == 0) *reinterpret_cast<volatile u64*>(stamps + 1) = globaltimer_ns();
    }
}

template <class Task>
__device__ __forceinline__ void finalize_if_last(const Task* __restrict__ tasks, u32 n_tasks,
                                                 const u64* __restrict__ sums, u64* __restrict__ digests,
                                                 unsigned long long* __restrict__ done, u64* stamps, bool clean,
                                                 unsigned long long* sync) {
    const u32 lane = threadIdx.x & 31;
    __threadfence();
    __syncwarp();
    unsigned long long ticket = 0;
    if (lane == 0) ticket = atomicAdd(done, 1ull);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket != static_cast<unsigned long long>(gridDim.x) * (blockDim.x >> 5) - 1) return;
    __threadfence();
    finalize_tail(tasks, n_tasks, sums, digests, done, stamps, clean, sync);
}

template <class Task, class Cfg>
__global__ void __launch_bounds__(Cfg::kWarps * 32, 2)
    copy_fp_kernel(const Task* __restrict__ tasks, u32 n_tasks, u64 total_tiles, u64* __restrict__ sums,
                   unsigned long long* __restrict__ sync, const u64* __restrict__ need, bool verify_next,
                   u64* __restrict__ digests, unsigned long long* __restrict__ done, u64* __restrict__ stamps,
                   bool clean) {
    // stamps (nullable, host-mapped): globaltimer at the first CTA's start and
    // at the finalizer's end — the kernel's span without an event query
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0) stamps[0] = globaltimer_ns();
    load_tiles<Task, Cfg>(tasks, n_tasks, total_tiles, sums, sync, need, verify_next);
    finalize_if_last(tasks, n_tasks, sums, digests, done, stamps, clean, sync);
}

__global__ void copy_fp_finalize_kernel(const CopyFpTask* __restrict__ tasks, u32 n_tasks,
                                        const u64* __restrict__ sums, u64* __restrict__ digests) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tasks) return;
    if (raw_sums(tasks[i])) {
        digests[2 * i] = sums[2 * i];
        digests[2 * i + 1] = sums[2 * i + 1];
        return;
    }
    u64 h1 = 0, h2 = 0;
    mm::body(h1, h2, sums[2 * i], sums[2 * i + 1]);
    mm::finish(h1, h2, tasks[i].n, 0, 8, 24);
    digests[2 * i] = h1;
    digests[2 * i + 1] = h2;
}

}  // namespace

// Load-kernel configuration of launches with writing tasks (TANGRAM_LOAD_RING
// = "single" selects the four-slot single-line ring for A/B runs).
// Writing launches use the paired-store ring unless TANGRAM_LOAD_RING=single
// (A/B runs).
static bool pair_ring() {
    static const bool pair = [] {
        const char* e = std::getenv("TANGRAM_LOAD_RING");
        return !(e && std::strcmp(e, "single") == 0);
    }();
    return pair;
}

// Verify tiles of writing launches realign from the next stage (A/B:
// TANGRAM_VERIFY_NEXT=0 keeps the extra column at every stage).
static bool verify_next() {
    static const bool on = [] {
        const char* e = std::getenv("TANGRAM_VERIFY_NEXT");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

std::uint64_t copy_fp_resident_warps(int sm_count) { return static_cast<u64>(sm_count) * 2 * CfgPair::kWarps; }

namespace {
void set_tile_order_once() {
    static const bool done = [] {
        const char* e = std::getenv("TANGRAM_TILE_ORDER");
        if (e && std::strcmp(e, "forward") == 0) {
            const bool f = false;
            cudaMemcpyToSymbol(tile_order_reversed, &f, sizeof(f));
        }
        return true;
    }();
    (void)done;
}

template <class Task, class Cfg>
void load_kernel_launch_cfg(const Task* d_tasks, u32 n_tasks, u64 total_tiles, u64* d_sums, u64* d_digests,
                            u64* d_sync, const u64* d_need, u32 n_waves, int sm_count, cudaStream_t s,
                            bool sync_zeroed, u64* stamps, bool clean) {
    static const bool attr = [] {
        return cudaFuncSetAttribute(copy_fp_kernel<Task, Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Cfg::kSmemBytes) == cudaSuccess;
    }();
    (void)attr;
    set_tile_order_once();
    if (!sync_zeroed) cudaMemsetAsync(d_sync, 0, (2 + n_waves) * sizeof(u64), s);
    const u64 want = (total_tiles + Cfg::kWarps - 1) / Cfg::kWarps;
    const u64 cap = static_cast<u64>(sm_count) * 2;
    const unsigned blocks = static_cast<unsigned>(want < cap ? want : cap);
    auto* sync = reinterpret_cast<unsigned long long*>(d_sync);
    copy_fp_kernel<Task, Cfg><<<blocks, Cfg::kWarps * 32, Cfg::kSmemBytes, s>>>(
        d_tasks, n_tasks, total_tiles, d_sums, sync, d_need, verify_next(), d_digests, sync + 1 + n_waves, stamps, clean);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

template <class Task>
void load_kernel_launch(const Task* d_tasks, u32 n_tasks, u64 total_tiles, u64* d_sums, u64* d_digests, u64* d_sync,
                        const u64* d_need, u32 n_waves, int sm_count, cudaStream_t s, bool sync_zeroed,
                        bool writes, u64* stamps = nullptr, bool clean = false) {
    static const bool ring46 = [] {
        const char* e = std::getenv("TANGRAM_K1_RING");
        return e && std::strcmp(e, "4x6") == 0;
    }();
    if (!writes && ring46)
        load_kernel_launch_cfg<Task, CfgFpNext46>(d_tasks, n_tasks, total_tiles, d_sums, d_digests, d_sync, d_need, n_waves,
                                                  sm_count, s, sync_zeroed, stamps, clean);
    else if (!writes && !(std::getenv("TANGRAM_FP_NEXT") && std::strcmp(std::getenv("TANGRAM_FP_NEXT"), "0") == 0))
        load_kernel_launch_cfg<Task, CfgFpNext>(d_tasks, n_tasks, total_tiles, d_sums, d_digests, d_sync, d_need, n_waves,
                                                sm_count, s, sync_zeroed, stamps, clean);
    else if (writes && pair_ring())
        load_kernel_launch_cfg<Task, CfgPair>(d_tasks, n_tasks, total_tiles, d_sums, d_digests, d_sync, d_need, n_waves,
                                              sm_count, s, sync_zeroed, stamps, clean);
    else
        load_kernel_launch_cfg<Task, CfgSingle>(d_tasks, n_tasks, total_tiles, d_sums, d_digests, d_sync, d_need, n_waves,
                                                sm_count, s, sync_zeroed, stamps, clean);
}
}  // namespace

void copy_fp_launch(const CopyFpTask* d_tasks, u32 n_tasks, u64 total_tiles, u64* d_sums, u64* d_digests, u64* d_sync,
                    const u64* d_need, u32 n_waves, int sm_count, cudaStream_t s, bool sync_zeroed, u64* stamps,
                    bool clean) {
    if (n_tasks == 0) return;
    if (total_tiles > 0) {
        load_kernel_launch(d_tasks, n_tasks, total_tiles, d_sums, d_digests, d_sync, d_need, n_waves, sm_count, s,
                           sync_zeroed, /*writes=*/true, stamps, clean);
        return;
    }
    copy_fp_finalize_kernel<<<(n_tasks + 127) / 128, 128, 0, s>>>(d_tasks, n_tasks, d_sums, d_digests);  // empty tensors only
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void fp_launch(const FpTask* d_tasks, u32 n_tasks, u64 total_tiles, u64* d_sums, u64* d_digests, u64* d_sync,
               int sm_count, cudaStream_t s, bool sync_zeroed, u64* stamps, bool clean) {
    if (n_tasks == 0) return;
    // K1 is the load kernel with fingerprint-only tasks
    if (total_tiles > 0) {
        load_kernel_launch(d_tasks, n_tasks, total_tiles, d_sums, d_digests, d_sync, nullptr, 0, sm_count, s,
                           sync_zeroed, /*writes=*/false, stamps, clean);
        return;
    }
    fp_finalize_kernel<<<(n_tasks + 127) / 128, 128, 0, s>>>(d_tasks, n_tasks, d_sums, d_digests);  // empty tensors only
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace tg
