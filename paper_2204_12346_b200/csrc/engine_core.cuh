// engine_core.cuh — the engine's host-side core shared by its CUDA
// translation units (engine.cu, gswarm.cu): context and window objects, the
// per-context lock, error texts, counted copies, stream-ordered allocation.
#pragma once

#include "sirdgpu.h"

#include "engine_internal.h"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

using namespace sirdgpu;

// Independent swarm partitions run as separate launch sequences on their own
// streams so one partition's per-iteration tail overlaps the next
// partition's iteration (swarms never synchronise with each other).
#ifndef SG_LANES
#define SG_LANES 32
#endif
constexpr int kMaxLanes = SG_LANES;

struct sg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // Every entry point that touches the context's stream, scratch buffers,
    // lanes or plans holds this lock, so threads may share one context (the
    // reference's objectives are reentrant); the C++ layer nests calls, hence
    // recursive.  Error texts are kept per calling thread (last_errors()).
    std::recursive_mutex mu;
    std::atomic<uint64_t> launches{0};
    // host <-> device bytes copied by the context's calls (telemetry: the
    // e2e byte counts of bench.py)
    std::atomic<uint64_t> h2d_bytes{0}, d2h_bytes{0};
    int sm_count = 0;
    // reusable scratch for sg_eval_costs (host-buffer path)
    double* d_pos = nullptr;
    double* d_cost = nullptr;
    size_t scratch_n = 0;
    // side streams for concurrent swarm partitions (see step_group)
    cudaStream_t side[kMaxLanes] = {};
    cudaEvent_t fork = nullptr;
    cudaEvent_t join[kMaxLanes] = {};
    // the C5 band pipeline: ensemble evaluation and band selection streams
    static constexpr int kBandSlots = 2;  // windows in flight (one evaluation stream each; 3 measured no faster)
    cudaStream_t band_eval[kBandSlots] = {}, band_sel = nullptr;
    // band-selection telemetry (device): days resolved from the ensemble's
    // fused histogram, days that took the histogram pass
    unsigned long long* band_stats = nullptr;
};

struct sg_window {
    sg_ctx* ctx = nullptr;
    DevWindow host{};          // device pointers inside
    DevWindow* d_desc = nullptr;
    ObsDay* d_obs = nullptr;
    ObsDay* d_robs = nullptr;
    unsigned char* d_flag = nullptr;
    unsigned char* d_block = nullptr;  // the one allocation holding desc/obs/robs/flags
    size_t smem = 0;
};

// sg_last_error text per (calling thread, context): a failing call and the
// caller's sg_last_error() see the same message even when other threads use
// the context concurrently.
inline std::unordered_map<const sg_ctx*, std::string>& last_errors() {
    static thread_local std::unordered_map<const sg_ctx*, std::string> m;
    return m;
}

inline int fail(sg_ctx* ctx, int code, const std::string& msg) {
    if (ctx) last_errors()[ctx] = msg;
    return code;
}

using CtxLock = std::lock_guard<std::recursive_mutex>;

// Every host <-> device copy of the engine goes through here (counted per
// context, sg_ctx_copy_bytes).
inline cudaError_t copy_async(sg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
    if (kind == cudaMemcpyHostToDevice) ctx->h2d_bytes += bytes;
    else if (kind == cudaMemcpyDeviceToHost) ctx->d2h_bytes += bytes;
    return cudaMemcpyAsync(dst, src, bytes, kind, st);
}

// NVTX range around an entry point (visible in nsys/ncu timelines; a no-op
// without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define SG_ENTRY(ctx, name)       \
    CtxLock sg_lock_((ctx)->mu);  \
    NvtxRange sg_nvtx_(name)

inline int cuda_fail(sg_ctx* ctx, cudaError_t e, const char* what) {
    const int code = e == cudaErrorMemoryAllocation ? SG_ERR_OUT_OF_MEMORY : SG_ERR_CUDA;
    return fail(ctx, code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define SG_CUDA(ctx, call)                                  \
    do {                                                    \
        const cudaError_t e_ = (call);                      \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// on the context stream; the pool keeps freed blocks, see sg_ctx_create), so
// repeated calls of the calibration API do not pay cudaMalloc/cudaFree.
template <class T>
cudaError_t dalloc(T** p, size_t count, cudaStream_t st) {
    return cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T), st);
}


// RAII bundle of device allocations for one call / plan (stream-ordered).
struct DevBufs {
    cudaStream_t st = nullptr;
    std::vector<void*> ptrs;
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        const cudaError_t e = dalloc(p, count, st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~DevBufs() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

