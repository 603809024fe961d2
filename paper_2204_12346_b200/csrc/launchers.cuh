// launchers.cuh — host-side launchers of the templated kernels, one struct
// per kernel family with run() for every (objective family, metric,
// substeps: 24 / -1 = any count with the t_k table / 0 = generic) specialisation.  engine.cu dispatches to them; family.cu
// instantiates them, once per objective family, so the heavy kernel
// templates compile in parallel translation units (build.py).
#pragma once

#include "kernels.cuh"

#include <cuda_runtime.h>

namespace sirdgpu {

// Opt in to the dynamic shared memory a launch needs beyond the default
// 48 KB, which covers static + dynamic together: every kernel here has less
// than 8 KB of static shared memory (the cluster kernel's partials 1 KB,
// its warp minima and window descriptor ~3.6 KB), so dynamic segments past
// 40 KB opt in.
template <class KernelPtr>
cudaError_t prepare_smem(KernelPtr k, size_t smem) {
    if (smem > 40 * 1024)
        return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    return cudaSuccess;
}

template <int F, int M, int S>
struct EvalLaunch {
    static void run(const DevWindow* w, const double* pos, size_t n, double* costs, size_t smem, cudaStream_t st,
                    cudaError_t* err);
};

// out of class: not implicitly inline, so `extern template` keeps engine.cu from instantiating it
template <int F, int M, int S>
void EvalLaunch<F, M, S>::run(const DevWindow* w, const double* pos, size_t n, double* costs, size_t smem, cudaStream_t st,
                    cudaError_t* err) {
    auto k = eval_costs_kernel<F, M, S>;
    *err = prepare_smem(k, smem);
    if (*err != cudaSuccess) return;
    const unsigned grid = static_cast<unsigned>((n + kEvalThreads - 1) / kEvalThreads);
    k<<<grid, kEvalThreads, smem, st>>>(w, pos, n, costs);
    *err = cudaGetLastError();
}

template <int F, int M, int S>
struct StepLaunch {
    static void run(unsigned grid, uint32_t cta_offset, const CtaTask* tasks, const DevSwarm* sw, const PsoPlanes& P,
                    DevSwarmState* state, uint64_t it, size_t smem, cudaStream_t st, cudaError_t* err);
};

// out of class: not implicitly inline, so `extern template` keeps engine.cu from instantiating it
template <int F, int M, int S>
void StepLaunch<F, M, S>::run(unsigned grid, uint32_t cta_offset, const CtaTask* tasks, const DevSwarm* sw, const PsoPlanes& P,
                    DevSwarmState* state, uint64_t it, size_t smem, cudaStream_t st, cudaError_t* err) {
    auto k = pso_step_kernel<F, M, S>;
    if (it == 0) {
        *err = prepare_smem(k, smem);
        if (*err != cudaSuccess) return;
    }
    k<<<grid, kStepThreads, smem, st>>>(tasks, sw, P, state, it, cta_offset);
    *err = cudaGetLastError();
}

template <int F, int M, int S>
struct SwarmLaunch {
    // n_swarms clusters of `cluster` CTAs (thread-block clusters, one swarm each)
    static void run(unsigned n_swarms, unsigned cluster, unsigned threads, uint32_t swarm_offset, const DevSwarm* sw,
                    const DevWindow* wins, const PsoPlanes& P, DevSwarmState* state, size_t smem, cudaStream_t st,
                    cudaError_t* err);
};

// out of class: not implicitly inline, so `extern template` keeps engine.cu from instantiating it
template <int F, int M, int S>
void SwarmLaunch<F, M, S>::run(unsigned n_swarms, unsigned cluster, unsigned threads, uint32_t swarm_offset, const DevSwarm* sw,
                    const DevWindow* wins, const PsoPlanes& P, DevSwarmState* state, size_t smem, cudaStream_t st,
                    cudaError_t* err) {
    auto k = pso_swarm_kernel<F, M, S>;
    *err = prepare_smem(k, smem);
    if (*err != cudaSuccess) return;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_swarms * cluster);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cluster;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    *err = cudaLaunchKernelEx(&cfg, k, sw, wins, P, state, swarm_offset);
}

template <int F, int M, int S>
struct EnsembleLaunch {
    static void run(const DevWindow* w, const DevWindow& fwin, const double* lo, const double* hi, uint64_t seed,
                    size_t n, int horizon, double* costs, double* params, double* deaths, size_t sstride,
                    size_t dstride, const uint32_t* perm, const double* planes, int out_by_slot, SelDay* days,
                    unsigned int* hist, unsigned long long* ramp_count, EnsNext next, size_t smem,
                    cudaStream_t st, cudaError_t* err);
};

// out of class: not implicitly inline, so `extern template` keeps engine.cu from instantiating it
template <int F, int M, int S>
void EnsembleLaunch<F, M, S>::run(const DevWindow* w, const DevWindow& fwin, const double* lo, const double* hi, uint64_t seed,
                    size_t n, int horizon, double* costs, double* params, double* deaths, size_t sstride,
                    size_t dstride, const uint32_t* perm, const double* planes, int out_by_slot, SelDay* days,
                    unsigned int* hist, unsigned long long* ramp_count, EnsNext next, size_t smem,
                    cudaStream_t st, cudaError_t* err) {
    auto k = ensemble_kernel<F, M, S>;
    *err = prepare_smem(k, smem);
    if (*err != cudaSuccess) return;
    const unsigned grid = static_cast<unsigned>((n + kEvalThreads - 1) / kEvalThreads);
    k<<<grid, kEvalThreads, smem, st>>>(w, fwin, lo, hi, seed, n, horizon, costs, params, deaths, sstride,
                                        dstride, perm, planes, out_by_slot, days, hist, ramp_count, next);
    *err = cudaGetLastError();
}


// Explicit instantiation lists: INST = extern (declaration, engine.cu) or
// empty (definition, family.cu).
#define SG_LAUNCH_ONE(INST, F, M, S)          \
    INST template struct EvalLaunch<F, M, S>;  \
    INST template struct StepLaunch<F, M, S>;  \
    INST template struct SwarmLaunch<F, M, S>; \
    INST template struct EnsembleLaunch<F, M, S>;
#define SG_LAUNCH_FAMILY_SUB(INST, F, S) \
    SG_LAUNCH_ONE(INST, F, 0, S) SG_LAUNCH_ONE(INST, F, 1, S) SG_LAUNCH_ONE(INST, F, 2, S) SG_LAUNCH_ONE(INST, F, 3, S)
#define SG_LAUNCH_FAMILY(INST, F) \
    SG_LAUNCH_FAMILY_SUB(INST, F, 24) SG_LAUNCH_FAMILY_SUB(INST, F, -24) SG_LAUNCH_FAMILY_SUB(INST, F, -1) \
    SG_LAUNCH_FAMILY_SUB(INST, F, 0)

}  // namespace sirdgpu
