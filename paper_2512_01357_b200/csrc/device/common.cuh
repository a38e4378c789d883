// Shared helpers for the sm_100a data plane.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <string>

#include "../host/store.hpp"

namespace tg {

constexpr int kErrCuda = 100;

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(kErrCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
#define TG_CUDA(x) ::tg::cuda_check((x), #x)

// NVTX range for the phases of a load / KV batch (visible in Nsight Systems;
// header-only NVTX3, a no-op without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// RAII device guard.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) TG_CUDA(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace tg
