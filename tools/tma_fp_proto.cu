// Prototype (tools, not product): K1 tgfp1 leaf hashing with the staging done
// by TMA tensor copies instead of per-lane cp.async + funnel shifts.
//
// A tensor at byte phase o is viewed as a 2-D uint8 tensor map: dim 0 = byte
// in leaf (extent 4096 + 16, so a box may run up to 15 bytes into the next
// row), dim 1 = leaf (stride 4096 B).  One box {128 B, 32 leaves} at
// (o + 128 s, 32 t) is stage s of tile t: ONE instruction per warp stage,
// issued by lane 0, lands leaf-aligned in shared memory with the 128-byte
// swizzle (chunk q of row r at q ^ (r & 7), the same conflict-free layout
// the load kernel builds by hand), so every phase hashes on the aligned body:
// 8 LDS.128 per 128 B, no funnel shifts, no 9th word.  Completion through one
// mbarrier per ring slot (expect_tx 4096 B).
//
// Prints one JSON line per (config, phase): GB/s over an 8 GiB tensor
// (inputs >> L2), and whether (ΣH, ΣL) equals a one-thread-per-leaf
// reference kernel on the first 256 MiB.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2512_01357_b200/csrc/host
//        tools/tma_fp_proto.cu -o tma_fp_proto -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "murmur_mix.hpp"

using u64 = std::uint64_t;
using u32 = std::uint32_t;
using namespace tg;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("{\"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(u64* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_expect(u64* b, u32 tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* b, u32 parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int x, int y, u64* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint4 lds128(u32 a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

template <int STAGES, int WARPS, bool SWZ = true>
__global__ void __launch_bounds__(WARPS * 32, 2)
    fp_tma(const __grid_constant__ CUtensorMap tm, u32 o, u64 n_leaves, u64 n_tiles, u64* sums) {
    extern __shared__ std::uint8_t smem_raw[];
    __shared__ u64 bars[WARPS][STAGES];
    std::uint8_t* smem = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    std::uint8_t* wbuf = smem + wid * STAGES * 4096;
    u64* bar = bars[wid];
    if (lane == 0) {
        for (int i = 0; i < STAGES; ++i) mbar_init(bar + i);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const u64 gw = static_cast<u64>(blockIdx.x) * WARPS + wid, nw = static_cast<u64>(gridDim.x) * WARPS;
    const u64 my_tiles = gw < n_tiles ? (n_tiles - gw + nw - 1) / nw : 0;
    const u64 total = my_tiles * 32;
    auto issue = [&](u64 g) {
        if (g >= total || lane != 0) return;
        const u64 t = gw + (g >> 5) * nw;
        const int slot = static_cast<int>(g % STAGES);
        mbar_expect(bar + slot, 4096);
        tma_2d(wbuf + slot * 4096, &tm, static_cast<int>(o + 128 * (g & 31)), static_cast<int>(32 * t), bar + slot);
    };
    for (int g = 0; g < STAGES - 1; ++g) issue(g);
    u64 acc_h = 0, acc_l = 0;
    mm::W32 h1{}, h2{};
    const u32 key = lane & 7;
    for (u64 g = 0; g < total; ++g) {
        issue(g + STAGES - 1);
        const int slot = static_cast<int>(g % STAGES);
        mbar_wait(bar + slot, static_cast<u32>((g / STAGES) & 1));
        const u64 t = gw + (g >> 5) * nw;
        const u64 leaf = 32 * t + lane;
        const u32 s = static_cast<u32>(g & 31);
        if (s == 0) h1 = h2 = mm::w_of(leaf);
        if (leaf < n_leaves) {
            const u32 row = smem_u32(wbuf + slot * 4096 + lane * 128);
#pragma unroll
            for (u32 q = 0; q < 8; ++q) {
                const uint4 w = lds128(row + ((SWZ ? (q ^ key) : q) << 4));
                mm::body_dev(h1, h2, mm::W32{w.x, w.y}, mm::W32{w.z, w.w});
            }
            if (s == 31) {
                u64 f1 = mm::u_of(h1), f2 = mm::u_of(h2);
                mm::finish(f1, f2, 0, 0, 0, 4096);
                acc_h += f1;
                acc_l += f2;
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) {
        acc_h += __shfl_xor_sync(0xffffffffu, acc_h, k);
        acc_l += __shfl_xor_sync(0xffffffffu, acc_l, k);
    }
    if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(sums), acc_h);
        atomicAdd(reinterpret_cast<unsigned long long*>(sums + 1), acc_l);
    }
}

// Reference: one thread per leaf, byte loads.
__global__ void fp_ref(const std::uint8_t* base, u64 n_leaves, u64* sums) {
    const u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    if (i >= n_leaves) return;
    const std::uint8_t* p = base + 4096 * i;
    mm::W32 h1 = mm::w_of(i), h2 = h1;
    for (int b = 0; b < 256; ++b) {
        u32 w[4];
        for (int k = 0; k < 4; ++k)
            w[k] = p[16 * b + 4 * k] | (p[16 * b + 4 * k + 1] << 8) | (p[16 * b + 4 * k + 2] << 16) |
                   (static_cast<u32>(p[16 * b + 4 * k + 3]) << 24);
        mm::body_dev(h1, h2, mm::W32{w[0], w[1]}, mm::W32{w[2], w[3]});
    }
    u64 f1 = mm::u_of(h1), f2 = mm::u_of(h2);
    mm::finish(f1, f2, 0, 0, 0, 4096);
    atomicAdd(reinterpret_cast<unsigned long long*>(sums), f1);
    atomicAdd(reinterpret_cast<unsigned long long*>(sums + 1), f2);
}

__global__ void fill(u64* p, u64 n) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n; i += static_cast<u64>(gridDim.x) * blockDim.x) {
        u64 z = (i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        p[i] = z ^ (z >> 31);
    }
}

static bool g_aligned_only = false;
static CUtensorMapSwizzle g_swz = CU_TENSOR_MAP_SWIZZLE_128B;
static CUresult make_map(CUtensorMap* tm, const void* base, u64 n_leaves) {
    cuuint64_t gdim[2] = {4096 + 16, n_leaves};
    cuuint64_t gstride[1] = {4096};
    cuuint32_t box[2] = {128, 32};
    cuuint32_t estr[2] = {1, 1};
    return cuTensorMapEncodeTiled(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, g_swz,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <int STAGES, int WARPS, bool SWZ = true>
static void run(const std::uint8_t* buf, u64 gib, u64* d_sums, int sms) {
    constexpr int smem = STAGES * WARPS * 4096 + 1024;
    g_swz = SWZ ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    CK(cudaFuncSetAttribute(fp_tma<STAGES, WARPS, SWZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (u32 o : {0u, 3u, 8u, 13u}) {
        if (g_aligned_only && o % 16) continue;
        // parity on 256 MiB
        const u64 cl = (256ull << 20) / 4096;
        CUtensorMap tm;
        CUresult r = make_map(&tm, buf, cl);
        if (r != CUDA_SUCCESS) {
            std::printf("{\"stages\": %d, \"warps\": %d, \"phase\": %u, \"encode_error\": %d}\n", STAGES, WARPS, o, (int)r);
            return;
        }
        u64 h[4];
        CK(cudaMemset(d_sums, 0, 32));
        const u64 ct = (cl + 31) / 32;
        const unsigned cb = static_cast<unsigned>(std::min<u64>((ct + WARPS - 1) / WARPS, 2ull * sms));
        fp_tma<STAGES, WARPS, SWZ><<<cb, WARPS * 32, smem>>>(tm, o, cl, ct, d_sums);
        fp_ref<<<(cl + 255) / 256, 256>>>(buf + o, cl, d_sums + 2);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, d_sums, 32, cudaMemcpyDeviceToHost));
        const bool ok = h[0] == h[2] && h[1] == h[3];
        // rate on gib GiB
        const u64 nl = (gib << 30) / 4096;
        r = make_map(&tm, buf, nl);
        const u64 nt = nl / 32;
        const unsigned blocks = static_cast<unsigned>(std::min<u64>((nt + WARPS - 1) / WARPS, 2ull * sms));
        fp_tma<STAGES, WARPS, SWZ><<<blocks, WARPS * 32, smem>>>(tm, o, nl, nt, d_sums);
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        const int reps = 5;
        CK(cudaEventRecord(a));
        for (int i = 0; i < reps; ++i) fp_tma<STAGES, WARPS, SWZ><<<blocks, WARPS * 32, smem>>>(tm, o, nl, nt, d_sums);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        ms /= reps;
        std::printf("{\"swizzle\": %d, \"stages\": %d, \"warps\": %d, \"ctas\": %u, \"phase\": %u, \"ms\": %.4f, \"GBps\": %.1f, \"parity\": %s}\n",
                    (int)SWZ, STAGES, WARPS, blocks, o, ms, nl * 4096.0 / ms / 1e6, ok ? "true" : "false");
        std::fflush(stdout);
    }
}

int main(int argc, char** argv) {
    const u64 gib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 8;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::uint8_t* buf = nullptr;
    const u64 bytes = (gib << 30) + (1 << 20);
    CK(cudaMalloc(&buf, bytes));
    fill<<<4 * sms, 256>>>(reinterpret_cast<u64*>(buf), bytes / 8);
    u64* d_sums = nullptr;
    CK(cudaMalloc(&d_sums, 64));
    const int mode = argc > 2 ? std::atoi(argv[2]) : 0;
    g_aligned_only = mode == 2;
    if (mode == 1) {
        run<4, 6, false>(buf, gib, d_sums, sms);
        run<3, 10, false>(buf, gib, d_sums, sms);
        return 0;
    }
    run<4, 6>(buf, gib, d_sums, sms);
    run<3, 8>(buf, gib, d_sums, sms);
    run<6, 4>(buf, gib, d_sums, sms);
    run<8, 3>(buf, gib, d_sums, sms);
    run<2, 8>(buf, gib, d_sums, sms);
    run<2, 12>(buf, gib, d_sums, sms);
    run<3, 10>(buf, gib, d_sums, sms);
    return 0;
}
