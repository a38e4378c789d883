// Latency of one tg_load_model call as a C/C++ host sees it: CUDA events on
// the pool stream recorded immediately before and after the C-ABI call (so
// host planning, launches, the data plane, the digest readback and the
// host's bookkeeping after the sync are all inside), plus the host wall clock
// of the call.  Test/bench tooling only: bench.py's warm-reload rows call
// through this so that Python's ctypes overhead is not charged to the load.
#include <chrono>

#include <cuda_runtime.h>

#include "tangram.h"

extern "C" int tgt_time_load(tg_pool* p, const tg_model_spec* spec, tg_stats* st, double clock,
                             const tg_load_policy* pol, tg_load_outcome* out, double* event_ms, double* wall_us) {
    void* sp = nullptr;
    if (int rc = tg_pool_stream(p, &sp)) return rc;
    auto s = static_cast<cudaStream_t>(sp);
    static cudaEvent_t a = nullptr, b = nullptr;
    if (!a) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
    }
    cudaStreamSynchronize(s);
    const auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(a, s);
    const int rc = tg_load_model(p, spec, st, clock, pol, out);
    cudaEventRecord(b, s);
    const auto t1 = std::chrono::steady_clock::now();
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    *event_ms = ms;
    *wall_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
    return rc;
}
