// Microbenchmark (tools, not product): DRAM efficiency of copy access
// patterns on B200, the evidence behind the load kernel's paired stores.
//  kernel 0: contiguous, each warp copies 512 B per instruction (K3-like)
//  kernel 1: leaf-strided, each instruction covers 4 lines 4 KiB apart; a
//            warp walks 32 leaves x 128 B per stage (single-line stores)
//  kernel 2: like 1 with 256 B per leaf per stage (paired stores)
//  kernel 3: like 1 with 8 warps per CTA, 4 CTAs
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/store_pattern.cu -o store_pattern
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void copy_contig(const uint4* __restrict__ s, uint4* __restrict__ d, u64 n16) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n16; i += (u64)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(s + i); __stcs(d + i, v);
    }
}
template <int LINES_PER_LEAF>
__global__ void copy_leaf(const uint8_t* __restrict__ s, uint8_t* __restrict__ d, u64 tiles) {
    const unsigned lane = threadIdx.x & 31, wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    const unsigned g = lane >> 3, q = lane & 7;
    for (u64 t = wid; t < tiles; t += nw) {
        const u64 base = t * 131072ull;
        for (int st = 0; st < 32 / LINES_PER_LEAF; ++st) {
            uint4 v[8 * LINES_PER_LEAF];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int l = 0; l < LINES_PER_LEAF; ++l)
                    v[i * LINES_PER_LEAF + l] = __ldcs(reinterpret_cast<const uint4*>(
                        s + base + (u64)(4 * i + g) * 4096 + (st * LINES_PER_LEAF + l) * 128 + q * 16));
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int l = 0; l < LINES_PER_LEAF; ++l)
                    __stcs(reinterpret_cast<uint4*>(d + base + (u64)(4 * i + g) * 4096 + (st * LINES_PER_LEAF + l) * 128 + q * 16),
                           v[i * LINES_PER_LEAF + l]);
        }
    }
}
int main() {
    const u64 n = 8ull << 30;
    uint8_t *a, *b;
    cudaMalloc(&a, n); cudaMalloc(&b, n);
    cudaMemset(a, 1, n); cudaMemset(b, 2, n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int k = 0; k < 4; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            const int reps = 5;
            for (int r = 0; r < reps; ++r) {
                if (k == 0) copy_contig<<<148 * 8, 256>>>((const uint4*)a, (uint4*)b, n / 16);
                if (k == 1) copy_leaf<1><<<148 * 2, 192>>>(a, b, n / 131072);
                if (k == 2) copy_leaf<2><<<148 * 2, 192>>>(a, b, n / 131072);
                if (k == 3) copy_leaf<1><<<148 * 4, 256>>>(a, b, n / 131072);
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("{\"kernel\": %d, \"GBps_rw\": %.0f}\n", k, 2.0 * n * reps / (ms / 1e3) / 1e9);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
