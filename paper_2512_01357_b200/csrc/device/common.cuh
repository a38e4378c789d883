// Shared helpers for the sm_100a data plane.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../host/store.hpp"

namespace tg {

constexpr int kErrCuda = 100;

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(kErrCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
#define TG_CUDA(x) ::tg::cuda_check((x), #x)

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
