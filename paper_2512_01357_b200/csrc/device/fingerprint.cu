// K1 — content fingerprint kernel (tgfp1), sm_100a.
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
// per warp, and selects one of four unrolled bodies.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "../host/murmur_mix.hpp"
#include "kernels.hpp"

namespace tg {
namespace {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

__device__ __forceinline__ u64 pack64(u32 lo, u32 hi) { return (static_cast<u64>(hi) << 32) | lo; }

// Hash `nblk` 16-byte blocks starting `4*Q + r8/8` bytes past the aligned
// word pointer `wp`.
template <int Q>
__device__ __forceinline__ void hash_blocks(const uint4* __restrict__ wp, u32 nblk, u32 r8, mm::W32& h1, mm::W32& h2) {
    uint4 w0 = __ldg(wp);
#pragma unroll 4
    for (u32 j = 0; j < nblk; ++j) {
        const uint4 w1 = __ldg(wp + j + 1);
        const u32 u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        const u32 a = __funnelshift_r(u[Q + 0], u[Q + 1], r8);
        const u32 b = __funnelshift_r(u[Q + 1], u[Q + 2], r8);
        const u32 c = __funnelshift_r(u[Q + 2], u[Q + 3], r8);
        const u32 d = __funnelshift_r(u[Q + 3], u[Q + 4], r8);
        mm::body_dev(h1, h2, mm::W32{a, b}, mm::W32{c, d});
        w0 = w1;
    }
}

__device__ __forceinline__ void hash_blocks_aligned(const uint4* __restrict__ wp, u32 nblk, mm::W32& h1, mm::W32& h2) {
#pragma unroll 4
    for (u32 j = 0; j < nblk; ++j) {
        const uint4 w = __ldg(wp + j);
        mm::body_dev(h1, h2, mm::W32{w.x, w.y}, mm::W32{w.z, w.w});
    }
}

// murmur3_x64_128(p[0..len), seed) for len <= 4096.
__device__ void leaf_digest(const std::uint8_t* p, u32 len, u64 seed, u64& d1, u64& d2) {
    mm::W32 h1 = mm::w_of(seed), h2 = h1;
    const u32 nblk = len >> 4;
    const u32 o = static_cast<u32>(reinterpret_cast<std::uintptr_t>(p) & 15);
    const uint4* wp = reinterpret_cast<const uint4*>(p - o);
    if (nblk) {
        const u32 r8 = (o & 3) * 8;
        switch (o >> 2) {
            case 0:
                if (o == 0) hash_blocks_aligned(wp, nblk, h1, h2);
                else hash_blocks<0>(wp, nblk, r8, h1, h2);
                break;
            case 1: hash_blocks<1>(wp, nblk, r8, h1, h2); break;
            case 2: hash_blocks<2>(wp, nblk, r8, h1, h2); break;
            default: hash_blocks<3>(wp, nblk, r8, h1, h2); break;
        }
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

__global__ void __launch_bounds__(256) fp_leaves_kernel(const FpTask* __restrict__ tasks, u32 n_tasks,
                                                        u64 total_tiles, u64* __restrict__ sums) {
    const u32 lane = threadIdx.x & 31;
    const u64 warp = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    int cur = -1;
    u64 acc_h = 0, acc_l = 0;
    for (u64 t = warp; t < total_tiles; t += nwarps) {
        // task owning tile t: last i with tasks[i].tile0 <= t
        u32 lo = 0, hi = n_tasks - 1;
        while (lo < hi) {
            const u32 mid = (lo + hi + 1) >> 1;
            if (tasks[mid].tile0 <= t) lo = mid;
            else hi = mid - 1;
        }
        const int ti = static_cast<int>(lo);
        if (ti != cur) {
            if (cur >= 0) {
                const u64 sh = warp_sum(acc_h), sl = warp_sum(acc_l);
                if (lane == 0) {
                    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur), sh);
                    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur + 1), sl);
                }
            }
            cur = ti;
            acc_h = acc_l = 0;
        }
        const FpTask tk = tasks[ti];
        const u64 leaf = (t - tk.tile0) * kLeavesPerTile + lane;
        const u64 off = leaf * kLeafBytes;
        if (off < tk.n) {
            const u64 rest = tk.n - off;
            const u32 len = rest < kLeafBytes ? static_cast<u32>(rest) : static_cast<u32>(kLeafBytes);
            u64 d1, d2;
            leaf_digest(tk.base + off, len, leaf, d1, d2);
            acc_h += d1;
            acc_l += d2;
        }
    }
    if (cur >= 0) {
        const u64 sh = warp_sum(acc_h), sl = warp_sum(acc_l);
        if (lane == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur), sh);
            atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur + 1), sl);
        }
    }
}

// ---- v1: shared-memory staged leaves ------------------------------------------
// The v0 kernel above issues one 16-byte load per lane from 32 different 4 KiB
// leaves, so every LDG touches 32 L1 lines and the L1 wavefront rate caps it
// near 16 B/clk/SM.  v1 stages each warp's 32 leaves through shared memory
// with cp.async: a stage is 8 blocks (128 B) + 1 realignment word per leaf,
// copied with coalesced 16-byte LDGSTS (lanes walk the 9-word slots of
// consecutive leaves), then every lane reads its own slot with conflict-free
// LDS.128 (slot stride 9 words → 8 consecutive lanes hit 8 distinct bank
// quads).  Three stages in flight per warp, 8 warps per CTA, 2 CTAs per SM.
constexpr int kStageBlocks = 8;
constexpr int kSlotWords = kStageBlocks + 1;
constexpr int kStages = 3;
constexpr int kStagesPerLeaf = static_cast<int>(kLeafBytes / 16) / kStageBlocks;  // 32
constexpr int kWarpsPerCta = 8;
constexpr int kWarpSmemWords = kStages * 32 * kSlotWords;
constexpr int kSmemBytes = kWarpsPerCta * kWarpSmemWords * 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Stage `s` of the tile's full leaves: words [8s, 8s+9) of every leaf's
// aligned window (the 9th only when the data is misaligned, so it always
// holds at least one byte of the leaf).
__device__ __forceinline__ void issue_stage(uint4* buf, const std::uint8_t* a0, u32 nfull, bool extra, int s,
                                            u32 lane) {
#pragma unroll
    for (int i = 0; i < kSlotWords; ++i) {
        const u32 f = i * 32 + lane;
        const u32 l = f / kSlotWords, q = f % kSlotWords;
        if (l < nfull && (q < kStageBlocks || extra))
            cp_async16(buf + l * kSlotWords + q, a0 + static_cast<u64>(l) * kLeafBytes + s * 128 + q * 16);
    }
    cp_async_commit();
}

template <int Q>
__device__ __forceinline__ void hash_stage(const uint4* slot, u32 r8, mm::W32& h1, mm::W32& h2) {
    uint4 w[kSlotWords];
#pragma unroll
    for (int q = 0; q < kSlotWords; ++q) w[q] = slot[q];
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

template <int Q>
__device__ __forceinline__ void hash_full_leaves(uint4* wbuf, const std::uint8_t* a0, u32 nfull, bool extra, u32 r8,
                                                 u32 lane, mm::W32& h1, mm::W32& h2) {
    constexpr int kStride = 32 * kSlotWords;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) issue_stage(wbuf + s * kStride, a0, nfull, extra, s, lane);
    for (int s = 0; s < kStagesPerLeaf; ++s) {
        const int nxt = s + kStages - 1;
        if (nxt < kStagesPerLeaf) issue_stage(wbuf + (nxt % kStages) * kStride, a0, nfull, extra, nxt, lane);
        else cp_async_commit();
        cp_async_wait<kStages - 1>();
        __syncwarp();
        if (lane < nfull) hash_stage<Q>(wbuf + (s % kStages) * kStride + lane * kSlotWords, r8, h1, h2);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kWarpsPerCta * 32, 2)
    fp_smem_kernel(const FpTask* __restrict__ tasks, u32 n_tasks, u64 total_tiles, u64* __restrict__ sums) {
    extern __shared__ uint4 smem[];
    const u32 lane = threadIdx.x & 31;
    const u32 wid = threadIdx.x >> 5;
    uint4* wbuf = smem + wid * kWarpSmemWords;
    const u64 nwarps = static_cast<u64>(gridDim.x) * kWarpsPerCta;
    int cur = -1;
    u64 acc_h = 0, acc_l = 0;
    for (u64 t = static_cast<u64>(blockIdx.x) * kWarpsPerCta + wid; t < total_tiles; t += nwarps) {
        u32 lo = 0, hi = n_tasks - 1;
        while (lo < hi) {
            const u32 mid = (lo + hi + 1) >> 1;
            if (tasks[mid].tile0 <= t) lo = mid;
            else hi = mid - 1;
        }
        const int ti = static_cast<int>(lo);
        if (ti != cur) {
            if (cur >= 0) {
                const u64 sh = warp_sum(acc_h), sl = warp_sum(acc_l);
                if (lane == 0) {
                    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur), sh);
                    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur + 1), sl);
                }
            }
            cur = ti;
            acc_h = acc_l = 0;
        }
        const FpTask tk = tasks[ti];
        const u64 leaf0 = (t - tk.tile0) * kLeavesPerTile;
        const u64 full_leaves = tk.n / kLeafBytes;
        const u32 nfull = full_leaves > leaf0 ? static_cast<u32>(min(full_leaves - leaf0, u64{32})) : 0u;
        const std::uint8_t* p0 = tk.base + leaf0 * kLeafBytes;
        const u32 o = static_cast<u32>(reinterpret_cast<std::uintptr_t>(p0) & 15);
        const std::uint8_t* a0 = p0 - o;
        const u64 my_leaf = leaf0 + lane;
        mm::W32 h1 = mm::w_of(my_leaf), h2 = h1;
        if (nfull) {
            const u32 r8 = (o & 3) * 8;
            const bool extra = o != 0;
            switch (o >> 2) {
                case 0: hash_full_leaves<0>(wbuf, a0, nfull, extra, r8, lane, h1, h2); break;
                case 1: hash_full_leaves<1>(wbuf, a0, nfull, extra, r8, lane, h1, h2); break;
                case 2: hash_full_leaves<2>(wbuf, a0, nfull, extra, r8, lane, h1, h2); break;
                default: hash_full_leaves<3>(wbuf, a0, nfull, extra, r8, lane, h1, h2); break;
            }
        }
        if (lane < nfull) {
            u64 f1 = mm::u_of(h1), f2 = mm::u_of(h2);
            mm::finish(f1, f2, 0, 0, 0, kLeafBytes);
            acc_h += f1;
            acc_l += f2;
        } else if (lane == nfull && my_leaf * kLeafBytes < tk.n) {
            // the tensor's trailing partial leaf, hashed straight from global
            const u32 len = static_cast<u32>(tk.n - my_leaf * kLeafBytes);
            u64 d1, d2;
            leaf_digest(tk.base + my_leaf * kLeafBytes, len, my_leaf, d1, d2);
            acc_h += d1;
            acc_l += d2;
        }
    }
    if (cur >= 0) {
        const u64 sh = warp_sum(acc_h), sl = warp_sum(acc_l);
        if (lane == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur), sh);
            atomicAdd(reinterpret_cast<unsigned long long*>(sums + 2 * cur + 1), sl);
        }
    }
}

// root = murmur3(le64 H ‖ le64 L ‖ le64 n, seed 0): one body block + an
// 8-byte tail.
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

}  // namespace

void fp_launch(const FpTask* d_tasks, u32 n_tasks, u64 total_tiles, u64* d_sums, u64* d_digests, int sm_count,
               cudaStream_t s) {
    if (n_tasks == 0) return;
    static const bool v0 = [] {
        const char* e = std::getenv("TANGRAM_FP_KERNEL");
        return e && std::strcmp(e, "v0") == 0;
    }();
    if (total_tiles > 0 && v0) {
        const u64 want = (total_tiles + 7) / 8;  // 8 warps per block
        const u64 cap = static_cast<u64>(sm_count) * 4;
        const unsigned blocks = static_cast<unsigned>(want < cap ? want : cap);
        fp_leaves_kernel<<<blocks, 256, 0, s>>>(d_tasks, n_tasks, total_tiles, d_sums);
        g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    } else if (total_tiles > 0) {
        static const bool attr = [] {
            return cudaFuncSetAttribute(fp_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) ==
                   cudaSuccess;
        }();
        (void)attr;
        const u64 want = (total_tiles + kWarpsPerCta - 1) / kWarpsPerCta;
        const u64 cap = static_cast<u64>(sm_count) * 2;
        const unsigned blocks = static_cast<unsigned>(want < cap ? want : cap);
        fp_smem_kernel<<<blocks, kWarpsPerCta * 32, kSmemBytes, s>>>(d_tasks, n_tasks, total_tiles, d_sums);
        g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    }
    fp_finalize_kernel<<<(n_tasks + 127) / 128, 128, 0, s>>>(d_tasks, n_tasks, d_sums, d_digests);
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace tg
