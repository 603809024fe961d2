// engine.cu — implementation of the C-ABI declared in include/sirdgpu.h.
//
// Host side of the B200 particle-window cost engine: contexts, window
// descriptors, launch planning for batched swarms, and the status/error
// plumbing that the C++ and Python layers turn back into the reference's
// exception types.  There is no CPU fallback anywhere: every numeric result
// is produced by the kernels in kernels.cuh.
#include "sirdgpu.h"

#include "engine_core.cuh"
#include "launchers.cuh"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

// The launchers of the templated kernels are instantiated in family.cu (one
// object per objective family, compiled in parallel by build.py).
namespace sirdgpu {
SG_LAUNCH_FAMILY(extern, 0)
SG_LAUNCH_FAMILY(extern, 1)
}  // namespace sirdgpu

namespace {

// Divisor admissibility for the 3-op exact division (sird_device.cuh
// div_exact; proof in DESIGN.md §4): |b| in [2^-60, 2^60] and the odd part of
// b's 53-bit significand below 2^53/3.
bool divisor_admits_fast_path(double b) {
    if (!std::isfinite(b) || b == 0.0) return false;
    const double a = std::fabs(b);
    if (a < 0x1.0p-60 || a > 0x1.0p60) return false;
    uint64_t bits;
    std::memcpy(&bits, &a, sizeof bits);
    uint64_t m = (bits & ((1ULL << 52) - 1)) | (1ULL << 52);
    while ((m & 1ULL) == 0) m >>= 1;
    return m < (1ULL << 53) / 3;
}

// The ramp's 2-op division q = fma(a, y, RN(a*y_lo)) needs the
// divisor's odd part below 2^50 on top of the 3-op conditions.
bool divisor_admits_two_op(double b) {
    if (!divisor_admits_fast_path(b)) return false;
    const double a = std::fabs(b);
    uint64_t bits;
    std::memcpy(&bits, &a, sizeof bits);
    uint64_t m = (bits & ((1ULL << 52) - 1)) | (1ULL << 52);
    while ((m & 1ULL) == 0) m >>= 1;
    return m < (1ULL << 50);
}

// objectives.cpp:61-69 — scale of one compartment's residuals.
double compartment_scale(const double* obs, int n) {
    // the same std::minmax_element as the reference: with NaN among the
    // values the chosen elements depend on its comparison order
    const auto [lo, hi] = std::minmax_element(obs, obs + n);
    const double range = *hi - *lo;
    return range > 0.0 ? 1.0 / range : 1.0 / std::max(1.0, std::fabs(*lo));
}

// Kernel specialisation of a window: 24 = the reference default substep count
// with the t_k table in shared memory; 0 = generic runtime substeps.
// -1 = any other substep count whose t_k table fits shared memory.
int kernel_sub(int n_days, int substeps) {
    if (substeps == 24) return uses_fast_grid(n_days, substeps) ? 24 : kSub24NoTable;
    return uses_time_table(n_days, substeps) ? -1 : 0;
}

bool valid_spec(int family, int metric) {
    return (family == SG_FAMILY_D_ONLY || family == SG_FAMILY_IRD_JOINT) && metric >= SG_METRIC_MXSE &&
           metric <= SG_METRIC_MAPE;
}

// ---- template dispatch over (family, metric, substeps == 24) ------------------
template <template <int, int, int> class K, class... Args>
void dispatch(int family, int metric, int substeps, Args&&... args) {
    // substeps: the kernel_sub() of the window(s): 24, -1 (table, runtime count) or 0
#define SG_CASE(F, M)                                                           \
    if (family == F && metric == M) {                                           \
        if (substeps == 24) K<F, M, 24>::run(std::forward<Args>(args)...);      \
        else if (substeps == -24) K<F, M, -24>::run(std::forward<Args>(args)...); \
        else if (substeps == -1) K<F, M, -1>::run(std::forward<Args>(args)...); \
        else K<F, M, 0>::run(std::forward<Args>(args)...);                      \
        return;                                                                 \
    }
    SG_CASE(0, 0) SG_CASE(0, 1) SG_CASE(0, 2) SG_CASE(0, 3)
    SG_CASE(1, 0) SG_CASE(1, 1) SG_CASE(1, 2) SG_CASE(1, 3)
#undef SG_CASE
}

// Trajectory launcher shared by sg_integrate_batch and sg_forecast_batch.
int launch_integrate(sg_ctx* ctx, const DevWindow& w, const double* d_params, const double* d_init, int init_stride,
                     int hold, size_t n, double* d_states, unsigned char* d_fin) {
    const unsigned grid = static_cast<unsigned>((n + kEvalThreads - 1) / kEvalThreads);
    const size_t smem = static_cast<size_t>(w.substeps + tgrid_entries(w.n_days, w.substeps)) * sizeof(double);
    if (uses_fast_grid(w.n_days, w.substeps)) {
        SG_CUDA(ctx, prepare_smem(integrate_kernel<24>, smem));
        integrate_kernel<24><<<grid, kEvalThreads, smem, ctx->stream>>>(w, d_params, d_init, init_stride, hold, n,
                                                                        d_states, d_fin);
    } else if (uses_time_table(w.n_days, w.substeps)) {
        SG_CUDA(ctx, prepare_smem(integrate_kernel<-1>, smem));
        integrate_kernel<-1><<<grid, kEvalThreads, smem, ctx->stream>>>(w, d_params, d_init, init_stride, hold, n,
                                                                        d_states, d_fin);
    } else {
        SG_CUDA(ctx, prepare_smem(integrate_kernel<0>, smem));
        integrate_kernel<0><<<grid, kEvalThreads, smem, ctx->stream>>>(w, d_params, d_init, init_stride, hold, n,
                                                                       d_states, d_fin);
    }
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    return SG_OK;
}

DevWindow integration_window(int n_days, int substeps, double N) {
    DevWindow w{};
    w.n_days = n_days;
    w.substeps = substeps;
    w.N = N;
    w.h = 1.0 / static_cast<double>(substeps);  // model.cpp:90
    w.fast_N = divisor_admits_two_op(N) ? 1 : 0;
    w.rN = 1.0 / N;
    // 1/N = rN + e/N exactly with e = 1 - rN*N (exact by fma); rN_lo = RN(e/N)
    w.rN_lo = std::fma(-w.rN, N, 1.0) / N;
    w.init_finite = 1;
    return w;
}

}  // namespace

extern "C" {

int sg_abi_version(void) { return SG_ABI_VERSION; }

int sg_ctx_create(int device, sg_ctx** out) {
    if (!out) return SG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0) return SG_ERR_NO_DEVICE;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SG_ERR_NO_DEVICE;
    if (prop.major != 10) return SG_ERR_NO_DEVICE;  // built for sm_100a only
    sg_ctx* ctx = new (std::nothrow) sg_ctx;
    if (!ctx) return SG_ERR_OUT_OF_MEMORY;
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return SG_ERR_CUDA;
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;  // keep freed blocks for the next plan
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = ctx;
    return SG_OK;
}

void sg_ctx_destroy(sg_ctx* ctx) {
    if (!ctx) return;
    {
        // wait for any call still inside the context before tearing it down
        CtxLock wait_for_callers(ctx->mu);
    }
    last_errors().erase(ctx);
    cudaSetDevice(ctx->device);
    cudaFreeAsync(ctx->d_pos, ctx->stream);
    cudaFreeAsync(ctx->d_cost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    for (int l = 0; l < kMaxLanes; ++l) {
        if (ctx->side[l]) cudaStreamDestroy(ctx->side[l]);
        if (ctx->join[l]) cudaEventDestroy(ctx->join[l]);
    }
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    if (ctx->band_stats) cudaFree(ctx->band_stats);
    for (cudaStream_t e : ctx->band_eval)
        if (e) cudaStreamDestroy(e);
    if (ctx->band_sel) cudaStreamDestroy(ctx->band_sel);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* sg_last_error(const sg_ctx* ctx) {
    if (!ctx) return "null context";
    auto& m = last_errors();
    auto it = m.find(ctx);
    return it == m.end() ? "" : it->second.c_str();
}

}  // extern "C"

void sg_set_last_error(sg_ctx* ctx, const std::string& message) {
    if (ctx) last_errors()[ctx] = message;
}

extern "C" {

uint64_t sg_ctx_launch_count(const sg_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

void sg_ctx_copy_bytes(const sg_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = ctx ? ctx->h2d_bytes.load() : 0;
    if (d2h) *d2h = ctx ? ctx->d2h_bytes.load() : 0;
}

int sg_ctx_band_stats(sg_ctx* ctx, uint64_t* fused_days, uint64_t* pass_days, uint64_t* ramp_substeps) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    SG_ENTRY(ctx, "sg_ctx_band_stats");
    unsigned long long v[3] = {0, 0, 0};
    if (ctx->band_stats) {
        SG_CUDA(ctx, cudaSetDevice(ctx->device));
        SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        SG_CUDA(ctx, cudaMemcpy(v, ctx->band_stats, sizeof v, cudaMemcpyDeviceToHost));
    }
    if (fused_days) *fused_days = v[0];
    if (pass_days) *pass_days = v[1];
    if (ramp_substeps) *ramp_substeps = v[2];
    return SG_OK;
}

void* sg_ctx_stream(const sg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int sg_window_create(sg_ctx* ctx, const double* infectious, const double* recovered_cum, const double* deaths_cum,
                     int n_days, sg_state init, double population, int substeps, int family, int metric,
                     sg_window** out) {
    if (!ctx || !out) return SG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (!infectious || !recovered_cum || !deaths_cum)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "window series must not be null");
    if (!valid_spec(family, metric)) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "unknown objective spec");
    SG_ENTRY(ctx, "sg_window_create");
    // integrate_euler's guards (model.cpp:78-80)
    if (n_days < 1 || substeps < 1 || !(population > 0.0))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT,
                    "integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    sg_window* w = new (std::nothrow) sg_window;
    if (!w) return fail(ctx, SG_ERR_OUT_OF_MEMORY, "host allocation failed");
    w->ctx = ctx;
    DevWindow& d = w->host;
    d = integration_window(n_days, substeps, population);
    d.family = family;
    d.metric = metric;
    d.init[0] = init.S;
    d.init[1] = init.I;
    d.init[2] = init.R;
    d.init[3] = init.D;
    d.init_finite = std::isfinite(init.S + init.I + init.R + init.D) ? 1 : 0;  // model.cpp:83
    const double* series[3] = {infectious, recovered_cum, deaths_cum};
    std::vector<ObsDay> obs(n_days), robs(n_days);
    std::vector<unsigned char> flag(3 * static_cast<size_t>(n_days));
    for (int c = 0; c < 3; ++c) {
        d.scale[c] = 1.0;
        d.kept[c] = 0.0;
        if (family == SG_FAMILY_IRD_JOINT && metric != SG_METRIC_MAPE) d.scale[c] = compartment_scale(series[c], n_days);
        size_t kept = 0;
        for (int k = 0; k < n_days; ++k) {
            const double o = series[c][k];
            obs[k].v[c] = o;
            robs[k].v[c] = 1.0 / o;
            unsigned char f = kObsSlow;
            if (o == 0.0) f = kObsSkip;
            else if (divisor_admits_fast_path(o)) f = kObsFast;
            flag[3 * static_cast<size_t>(k) + c] = f;
            if (o != 0.0) ++kept;
        }
        d.kept[c] = static_cast<double>(kept);
    }
    // Day-0 contribution of objective_value (objectives.cpp:15-55 at k = 0):
    // the prediction on day 0 is the initial state for every particle
    // (model.cpp:85), so it is computed once here, with the device's
    // operation order (e = (obs - pred) * scale; MXSE max(0, e*e); MSE
    // 0 + e*e; MAE 0 + |e|; MAPE 0 + |(obs - pred) / obs| unless obs == 0).
    // MXSE by largest |obs - pred|: exact when every scale is
    // finite and positive (always for D-only, scale 1).
    d.mxse_abs = 1;
    if (family == SG_FAMILY_IRD_JOINT)
        for (int c = 0; c < 3; ++c)
            if (!(std::isfinite(d.scale[c]) && d.scale[c] > 0.0)) d.mxse_abs = 0;
    {
        const double pred[3] = {init.I, init.R, init.D};
        for (int c = 0; c < 3; ++c) {
            const double o = series[c][0];
            double a = 0.0;
            if (metric == SG_METRIC_MAPE) {
                if (o != 0.0) a = 0.0 + std::fabs((o - pred[c]) / o);
            } else {
                double e = o - pred[c];
                if (family == SG_FAMILY_IRD_JOINT) e = e * d.scale[c];
                const double e2 = e * e;
                // std::max(0.0, x) == (0.0 < x) ? x : 0.0 (objectives.cpp:22-26): a NaN residual
                // leaves the accumulator at 0, in both forms
                const double ad = std::fabs(o - pred[c]);
                if (metric == SG_METRIC_MXSE) a = d.mxse_abs ? ((0.0 < ad) ? ad : 0.0) : ((0.0 < e2) ? e2 : 0.0);
                else if (metric == SG_METRIC_MSE) a = 0.0 + e2;
                else a = 0.0 + std::fabs(e);
            }
            d.acc0[c] = a;
        }
    }
    // Substep times, staged by every CTA that evaluates this window:
    // subh[sub] = RN(sub*h) and t_k = RN(RN(day-1) + subh[sub]) (model.cpp:94),
    // the same IEEE operations as stage_times on the device.
    const int n_tgrid = tgrid_entries(n_days, substeps);
    std::vector<double> times(static_cast<size_t>(substeps) + n_tgrid);
    for (int i = 0; i < substeps; ++i) times[i] = static_cast<double>(i) * d.h;
    for (int k = 0; k < n_tgrid; ++k) {
        const int day = k / substeps;
        times[substeps + k] = static_cast<double>(day) + static_cast<double>(k - day * substeps) * d.h;
    }
    // One device block: descriptor | times | obs | robs | flags.
    // Every section starts 16-byte aligned and is padded to a 16-byte
    // multiple: the step kernel stages them with bulk copies (CtaTask).
    const size_t obs_b = sizeof(ObsDay) * static_cast<size_t>(n_days);
    const size_t obs_b16 = (obs_b + 15) & ~size_t(15);
    const size_t off_times = (sizeof(DevWindow) + 255) & ~size_t(255);
    const size_t times_b = (times.size() * sizeof(double) + 15) & ~size_t(15);
    const size_t off_obs = off_times + times_b;
    const size_t off_robs = off_obs + obs_b16;
    const size_t off_flag = off_robs + obs_b16;
    const size_t total = off_flag + ((flag.size() + 15) & ~size_t(15));
    unsigned char* block = nullptr;
    cudaError_t e = dalloc(&block, total, ctx->stream);
    if (e == cudaSuccess) {
        w->d_block = block;
        w->d_desc = reinterpret_cast<DevWindow*>(block);
        w->d_obs = reinterpret_cast<ObsDay*>(block + off_obs);
        w->d_robs = reinterpret_cast<ObsDay*>(block + off_robs);
        w->d_flag = block + off_flag;
        d.obs = w->d_obs;
        d.robs = w->d_robs;
        d.obs_flag = w->d_flag;
        d.times = reinterpret_cast<const double*>(block + off_times);
        std::vector<unsigned char> staging(total, 0);
        std::memcpy(staging.data(), &d, sizeof d);
        std::memcpy(staging.data() + off_times, times.data(), times.size() * sizeof(double));
        std::memcpy(staging.data() + off_obs, obs.data(), obs_b);
        std::memcpy(staging.data() + off_robs, robs.data(), obs_b);
        std::memcpy(staging.data() + off_flag, flag.data(), flag.size());
        e = copy_async(ctx, block, staging.data(), total, cudaMemcpyHostToDevice, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    }
    if (e != cudaSuccess) {
        sg_window_destroy(w);
        return cuda_fail(ctx, e, "sg_window_create");
    }
    w->smem = kernel_smem_bytes(n_days, substeps, metric, uses_fast_grid(n_days, substeps));
    if (w->smem > 200 * 1024) {
        sg_window_destroy(w);
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "window too long for shared-memory staging");
    }
    *out = w;
    return SG_OK;
}

void sg_window_destroy(sg_window* w) {
    if (!w) return;
    CtxLock lock(w->ctx->mu);
    if (w->d_block) cudaFreeAsync(w->d_block, w->ctx->stream);
    delete w;
}

int sg_eval_costs_device(sg_window* w, const double* d_positions, size_t n, double* d_costs, void* cuda_stream) {
    if (!w) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = w->ctx;
    if (n == 0) return SG_OK;
    if (!d_positions || !d_costs) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null device buffer");
    SG_ENTRY(ctx, "sg_eval_costs_device");
    cudaStream_t st = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->stream;
    cudaError_t err = cudaSuccess;
    dispatch<EvalLaunch>(w->host.family, w->host.metric, kernel_sub(w->host.n_days, w->host.substeps), w->d_desc, d_positions, n, d_costs,
                         w->smem, st, &err);
    ctx->launches += 1;
    if (err != cudaSuccess) return cuda_fail(ctx, err, "eval_costs_kernel");
    return SG_OK;
}

int sg_eval_costs(sg_window* w, const double* positions, size_t n, size_t dim, double* costs) {
    if (!w) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = w->ctx;
    // calibration.cpp:141-143
    if (dim != 6) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "window objective expects 6-dim positions");
    if (n == 0) return SG_OK;
    if (!positions || !costs) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_eval_costs");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    if (ctx->scratch_n < n) {
        cudaFreeAsync(ctx->d_pos, ctx->stream);
        cudaFreeAsync(ctx->d_cost, ctx->stream);
        ctx->d_pos = nullptr;
        ctx->d_cost = nullptr;
        ctx->scratch_n = 0;
        SG_CUDA(ctx, dalloc(&ctx->d_pos, 6 * n, ctx->stream));
        SG_CUDA(ctx, dalloc(&ctx->d_cost, n, ctx->stream));
        ctx->scratch_n = n;
    }
    SG_CUDA(ctx, copy_async(ctx, ctx->d_pos, positions, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
    const int rc = sg_eval_costs_device(w, ctx->d_pos, n, ctx->d_cost, ctx->stream);
    if (rc) return rc;
    SG_CUDA(ctx, copy_async(ctx, costs, ctx->d_cost, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_integrate_batch(sg_ctx* ctx, const double* params, size_t n, sg_state init, double population, int n_days,
                       int substeps, double* states, uint8_t* finite) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (n_days < 1 || substeps < 1 || !(population > 0.0))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT,
                    "integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
    if (n == 0) return SG_OK;
    if (!params || !states || !finite) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_integrate_batch");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double *d_p, *d_init, *d_states;
    unsigned char* d_fin;
    SG_CUDA(ctx, b.alloc(&d_p, 6 * n));
    SG_CUDA(ctx, b.alloc(&d_init, 4));
    SG_CUDA(ctx, b.alloc(&d_states, n * static_cast<size_t>(n_days) * 4));
    SG_CUDA(ctx, b.alloc(&d_fin, n));
    const double s0[4] = {init.S, init.I, init.R, init.D};
    SG_CUDA(ctx, copy_async(ctx, d_p, params, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_init, s0, sizeof s0, cudaMemcpyHostToDevice, ctx->stream));
    const DevWindow w = integration_window(n_days, substeps, population);
    const int rc = launch_integrate(ctx, w, d_p, d_init, 0, 0, n, d_states, d_fin);
    if (rc) return rc;
    SG_CUDA(ctx, copy_async(ctx, states, d_states, sizeof(double) * n * n_days * 4, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, finite, d_fin, n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_integrate_states(sg_ctx* ctx, const double* params, const sg_state* inits, size_t n, double population,
                        int n_days, int substeps, double* states, uint8_t* finite) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (n_days < 1 || substeps < 1 || !(population > 0.0))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT,
                    "integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
    if (n == 0) return SG_OK;
    if (!params || !inits || !states || !finite) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_integrate_states");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double *d_p, *d_init, *d_states;
    unsigned char* d_fin;
    SG_CUDA(ctx, b.alloc(&d_p, 6 * n));
    SG_CUDA(ctx, b.alloc(&d_init, 4 * n));
    SG_CUDA(ctx, b.alloc(&d_states, n * static_cast<size_t>(n_days) * 4));
    SG_CUDA(ctx, b.alloc(&d_fin, n));
    SG_CUDA(ctx, copy_async(ctx, d_p, params, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_init, inits, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, ctx->stream));
    const DevWindow w = integration_window(n_days, substeps, population);
    const int rc = launch_integrate(ctx, w, d_p, d_init, 4, 0, n, d_states, d_fin);
    if (rc) return rc;
    SG_CUDA(ctx, copy_async(ctx, states, d_states, sizeof(double) * n * n_days * 4, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, finite, d_fin, n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_integrate_states_r2(sg_ctx* ctx, const double* params, const sg_state* inits, const double* observed_d,
                           size_t n, double population, int n_days, int substeps, double* states, uint8_t* finite,
                           double* r2) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (n_days < 1 || substeps < 1 || !(population > 0.0))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT,
                    "integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
    if (n == 0) return SG_OK;
    if (!params || !inits || !observed_d || !states || !finite || !r2)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_integrate_states_r2");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double *d_p, *d_init, *d_states, *d_obs, *d_r2;
    unsigned char* d_fin;
    const size_t nd = n * static_cast<size_t>(n_days);
    SG_CUDA(ctx, b.alloc(&d_p, 6 * n));
    SG_CUDA(ctx, b.alloc(&d_init, 4 * n));
    SG_CUDA(ctx, b.alloc(&d_states, nd * 4));
    SG_CUDA(ctx, b.alloc(&d_fin, n));
    SG_CUDA(ctx, b.alloc(&d_obs, nd));
    SG_CUDA(ctx, b.alloc(&d_r2, n));
    SG_CUDA(ctx, copy_async(ctx, d_p, params, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_init, inits, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_obs, observed_d, sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream));
    const DevWindow w = integration_window(n_days, substeps, population);
    const int rc = launch_integrate(ctx, w, d_p, d_init, 4, 0, n, d_states, d_fin);
    if (rc) return rc;
    r2_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(d_states, d_obs, n, n_days, d_r2);
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    SG_CUDA(ctx, copy_async(ctx, states, d_states, sizeof(double) * nd * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, finite, d_fin, n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, r2, d_r2, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_forecast_batch(sg_ctx* ctx, const double* params, const sg_state* junction, size_t n, double population,
                      int horizon, int substeps, double* states, uint8_t* finite) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (horizon < 0 || substeps < 1 || !(population > 0.0))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "forecast needs horizon >= 0, substeps >= 1, population > 0");
    if (n == 0) return SG_OK;
    if (!params || !junction || !states || !finite) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_forecast_batch");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    const int n_days = horizon + 1;
    DevBufs b;
    b.st = ctx->stream;
    double *d_p, *d_init, *d_states;
    unsigned char* d_fin;
    SG_CUDA(ctx, b.alloc(&d_p, 6 * n));
    SG_CUDA(ctx, b.alloc(&d_init, 4 * n));
    SG_CUDA(ctx, b.alloc(&d_states, n * static_cast<size_t>(n_days) * 4));
    SG_CUDA(ctx, b.alloc(&d_fin, n));
    static_assert(sizeof(sg_state) == 4 * sizeof(double), "sg_state layout");
    SG_CUDA(ctx, copy_async(ctx, d_p, params, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_init, junction, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, ctx->stream));
    const DevWindow w = integration_window(n_days, substeps, population);
    const int rc = launch_integrate(ctx, w, d_p, d_init, 4, 1, n, d_states, d_fin);
    if (rc) return rc;
    SG_CUDA(ctx, copy_async(ctx, states, d_states, sizeof(double) * n * n_days * 4, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, finite, d_fin, n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

}  // extern "C"

// ---- swarms ---------------------------------------------------------------------

namespace {

bool swarm_config_valid(const sg_swarm_desc& d, std::string* why) {
    // PsoConfig::validate / SearchBounds::validate (pso.cpp:16-34)
    if (d.n_particles == 0 || d.max_iters == 0) {
        *why = "pso: n_particles and max_iters must be positive";
        return false;
    }
    if (!std::isfinite(d.inertia) || !std::isfinite(d.cognitive) || !std::isfinite(d.social)) {
        *why = "pso: coefficients must be finite";
        return false;
    }
    for (int k = 0; k < 6; ++k) {
        if (!std::isfinite(d.lower[k]) || !std::isfinite(d.upper[k]) || d.lower[k] > d.upper[k]) {
            *why = "pso: bound " + std::to_string(k) + " is invalid";
            return false;
        }
    }
    if (!d.window) {
        *why = "swarm has no window";
        return false;
    }
    return true;
}

// One launch group: swarms sharing (family, metric, substeps == 24).  The
// runtime-substep kernel (SUB == 0) reads the substep count from each
// swarm's staged window, so mixed counts may share a launch.
struct SwarmGroup {
    int family = 0, metric = 0, substeps = 24;
    std::vector<size_t> idx;          // positions in the caller's descriptor array
    std::vector<uint64_t> max_iters;  // per swarm
    struct Lane {
        uint32_t cta_begin, n_ctas, swarm_begin, n_swarms;
    };
    std::vector<Lane> lanes;  // swarm partitions launched on separate streams
    bool persistent = false;  // every swarm <= kPersistMax: one CTA per swarm, one launch
    unsigned threads = 0;     // persistent CTA size
    unsigned cluster = 1;     // persistent CTAs per swarm (thread-block cluster)
    size_t n_total = 0, n_ctas = 0, smem = 0;
    uint64_t iters = 0;               // max over swarms
    DevSwarm* d_sw = nullptr;
    uint32_t* d_cta = nullptr;
    CtaTask* d_task = nullptr;
    DevWindow* d_win = nullptr;
    DevSwarmState* d_state = nullptr;
    PsoPlanes P{};
    DevBufs bufs;
    // The flat step launches of a run (all lanes, all iterations) as one
    // CUDA graph, captured at the third run of the plan: instantiating a
    // 4000-node graph costs tens of ms, so plans run once or twice (every
    // calibration call, timing loops with one warm-up) never pay it.
    int runs = 0;
    cudaGraphExec_t steps_exec = nullptr;
    ~SwarmGroup() {
        if (steps_exec) cudaGraphExecDestroy(steps_exec);
    }
};

}  // namespace

struct sg_plan {
    sg_ctx* ctx = nullptr;
    std::vector<SwarmGroup*> groups;
    std::vector<int> status;          // per descriptor: SG_OK or validation failure
    size_t n_desc = 0;
    uint64_t evals = 0;
    bool ran = false;
    ~sg_plan() {
        for (SwarmGroup* g : groups) delete g;
    }
};

namespace {

int build_group(sg_ctx* ctx, const sg_swarm_desc* descs, SwarmGroup& g) {
    std::vector<const sg_window*> wins;
    std::vector<DevSwarm> sw(g.idx.size());
    std::vector<uint32_t> cta_swarm;
    uint64_t offset = 0;
    uint32_t n_groups_total = 0;
    for (size_t j = 0; j < g.idx.size(); ++j) {
        const sg_swarm_desc& d = descs[g.idx[j]];
        auto it = std::find(wins.begin(), wins.end(), d.window);
        const int wi = static_cast<int>(it - wins.begin());
        if (it == wins.end()) wins.push_back(d.window);
        g.smem = std::max(g.smem, d.window->smem);
        DevSwarm& s = sw[j];
        s.window = wi;
        s.repair = d.repair_time_order ? 1 : 0;
        s.n = d.n_particles;
        s.offset = offset;
        s.max_iters = d.max_iters;
        s.cta_begin = static_cast<uint32_t>(cta_swarm.size());
        s.n_ctas = static_cast<uint32_t>((d.n_particles + kStepThreads * kNP - 1) / (kStepThreads * kNP));
        s.n_groups = (s.n_ctas + kFoldGroupCtas - 1) / kFoldGroupCtas;
        s.group_begin = n_groups_total;
        n_groups_total += s.n_groups;
        for (int k = 0; k < 6; ++k) {
            s.lo[k] = d.lower[k];
            s.hi[k] = d.upper[k];
        }
        s.w = d.inertia;
        s.c1 = d.cognitive;
        s.c2 = d.social;
        s.seed = d.seed;
        for (uint32_t c = 0; c < s.n_ctas; ++c) cta_swarm.push_back(static_cast<uint32_t>(j));
        offset += d.n_particles;
        g.iters = std::max(g.iters, d.max_iters);
        g.max_iters.push_back(d.max_iters);
    }
    g.n_total = offset;
    g.n_ctas = cta_swarm.size();
    // Partition swarms into up to kPlanLanes lanes of about equal CTA count
    // (swarm boundaries only).  Lanes let one lane's per-iteration tail
    // overlap the others' iterations; that matters most when the plan is
    // about one wave (measured, rank 0's share of the sweep on 8 GPUs, 18
    // swarms / 576 CTAs: 74.3 ms with 2 lanes, 62.3 ms with 8; the full
    // sweep is the same with 4, 8 or 16, profiles/r02d_lanes.jsonl).  Plans
    // under one CTA per SM stay on one lane (host enqueue would dominate).
    {
        constexpr int kPlanLanes = 8;
        int want = g.n_ctas >= static_cast<size_t>(ctx->sm_count)
                       ? static_cast<int>(std::min<size_t>(std::min(kPlanLanes, kMaxLanes), sw.size()))
                       : 1;
        static const char* lanes_env = std::getenv("SG_PLAN_LANES");  // diagnostic override
        if (lanes_env) want = std::max(1, std::min(kMaxLanes, std::atoi(lanes_env)));
        const size_t target = (g.n_ctas + want - 1) / want;
        SwarmGroup::Lane cur{0, 0, 0, 0};
        for (const DevSwarm& s : sw) {
            if (cur.n_ctas > 0 && cur.n_ctas + s.n_ctas > target && static_cast<int>(g.lanes.size()) + 1 < want) {
                g.lanes.push_back(cur);
                cur = SwarmGroup::Lane{cur.cta_begin + cur.n_ctas, 0, cur.swarm_begin + cur.n_swarms, 0};
            }
            cur.n_ctas += s.n_ctas;
            cur.n_swarms += 1;
        }
        g.lanes.push_back(cur);
    }
    if (g.persistent) {
        uint64_t max_n = 0;
        for (const DevSwarm& s : sw) max_n = std::max(max_n, s.n);
        // At most one warp per SM sub-partition: spread the swarm over
        // ceil(n / 128) SMs (<= 8, a portable cluster).
        g.cluster = static_cast<unsigned>(
            std::min<uint64_t>(kSwarmClusterMax, std::max<uint64_t>(1, (max_n + kSwarmThreadsMax - 1) / kSwarmThreadsMax)));
        const uint64_t per_cta = (max_n + g.cluster - 1) / g.cluster;
        g.threads = static_cast<unsigned>(std::min<uint64_t>(kSwarmThreadsMax, (per_cta + 31) / 32 * 32));
    }
    std::vector<DevWindow> wtab(wins.size());
    for (size_t k = 0; k < wins.size(); ++k) wtab[k] = wins[k]->host;

    DevBufs& b = g.bufs;
    b.st = ctx->stream;
    PsoPlanes& P = g.P;
    SG_CUDA(ctx, b.alloc(&g.d_sw, sw.size()));
    SG_CUDA(ctx, b.alloc(&g.d_cta, g.n_ctas));
    SG_CUDA(ctx, b.alloc(&g.d_win, wtab.size()));
    SG_CUDA(ctx, b.alloc(&g.d_task, g.n_ctas));
    SG_CUDA(ctx, b.alloc(&g.d_state, sw.size()));
    SG_CUDA(ctx, b.alloc(&P.x, pblock_elems(g.n_total, 6)));
    SG_CUDA(ctx, b.alloc(&P.v, pblock_elems(g.n_total, 6)));
    SG_CUDA(ctx, b.alloc(&P.pb, pblock_elems(g.n_total, 6)));
    SG_CUDA(ctx, b.alloc(&P.pbc, g.n_total));
    SG_CUDA(ctx, b.alloc(&P.mt, pblock_elems(g.n_total, kMtN)));
    SG_CUDA(ctx, b.alloc(&P.part_cost, g.n_ctas * kStepWarps));
    SG_CUDA(ctx, b.alloc(&P.part_idx, g.n_ctas * kStepWarps));
    SG_CUDA(ctx, b.alloc(&P.gpart_cost, std::max<uint32_t>(n_groups_total, 1)));
    SG_CUDA(ctx, b.alloc(&P.gpart_idx, std::max<uint32_t>(n_groups_total, 1)));
    SG_CUDA(ctx, b.alloc(&P.group_arrived, std::max<uint32_t>(n_groups_total, 1)));
    SG_CUDA(ctx, cudaMemsetAsync(P.group_arrived, 0, sizeof(unsigned int) * std::max<uint32_t>(n_groups_total, 1),
                                 ctx->stream));
    SG_CUDA(ctx, b.alloc(&P.history, sw.size() * g.iters));
    P.stride = g.n_total;
    P.hist_stride = g.iters;
    cudaStream_t st = ctx->stream;
    SG_CUDA(ctx, copy_async(ctx, g.d_sw, sw.data(), sizeof(DevSwarm) * sw.size(), cudaMemcpyHostToDevice, st));
    SG_CUDA(ctx, copy_async(ctx, g.d_cta, cta_swarm.data(), sizeof(uint32_t) * g.n_ctas, cudaMemcpyHostToDevice, st));
    SG_CUDA(ctx, copy_async(ctx, g.d_win, wtab.data(), sizeof(DevWindow) * wtab.size(), cudaMemcpyHostToDevice, st));
    std::vector<CtaTask> tasks(g.n_ctas);
    for (size_t c = 0; c < g.n_ctas; ++c) {
        const DevSwarm& s = sw[cta_swarm[c]];
        const DevWindow& w = wtab[s.window];
        CtaTask& t = tasks[c];
        const uint64_t first = static_cast<uint64_t>(c - s.cta_begin) * kStepThreads * kNP;
        t.swarm = cta_swarm[c];
        t.n_valid = static_cast<uint32_t>(std::min<uint64_t>(kStepThreads * kNP, s.n - first));
        t.p0 = s.offset + first;
        t.i0 = first;
        t.max_iters = s.max_iters;
        t.win = g.d_win + s.window;
        t.times = w.times;
        t.obs = reinterpret_cast<const double*>(w.obs);
        const WindowLayout L = window_layout(w.n_days, w.substeps, w.metric);
        // field widths: the table is at most kMaxTgrid entries (+ subh), the
        // observations at most the 200 KB window limit of sg_window_create
        // (windows without a table stage cooperatively and ignore both sizes)
        const bool table = uses_time_table(w.n_days, w.substeps);
        if (L.times_bytes / 16 > 0xFFFF || (table && w.substeps > 0xFFFF) || L.obs_bytes > 0xFFFFFFFFu)
            return fail(ctx, SG_ERR_INVALID_ARGUMENT, "window too large for the step kernel's staging");
        // subh (+ the table when it is staged): the kSub24NoTable kernels
        // stage subh too, to compute their ramp times from it
        t.times_x16 = static_cast<uint16_t>(L.times_bytes / 16);
        t.obs_bytes = static_cast<uint32_t>(L.obs_bytes);
        t.substeps = static_cast<uint16_t>(table ? w.substeps : 0);
    }
    SG_CUDA(ctx, copy_async(ctx, g.d_task, tasks.data(), sizeof(CtaTask) * tasks.size(), cudaMemcpyHostToDevice, st));
    SG_CUDA(ctx, cudaStreamSynchronize(st));  // host vectors go out of scope
    return SG_OK;
}

int seed_group(sg_ctx* ctx, SwarmGroup& g) {
    if (g.persistent) return SG_OK;  // the persistent kernel seeds its own swarm
    pso_init_kernel<<<static_cast<unsigned>(g.n_ctas), kStepThreads, 0, ctx->stream>>>(g.d_sw, g.d_cta, g.P,
                                                                                      g.d_state);
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    return SG_OK;
}

int ensure_lanes(sg_ctx* ctx) {
    if (ctx->fork) return SG_OK;
    SG_CUDA(ctx, cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming));
    for (int l = 0; l < kMaxLanes; ++l) {
        SG_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->side[l], cudaStreamNonBlocking));
        SG_CUDA(ctx, cudaEventCreateWithFlags(&ctx->join[l], cudaEventDisableTiming));
    }
    return SG_OK;
}

int enqueue_steps(sg_ctx* ctx, SwarmGroup& g);

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SG_GRAPH");
        return !(e && e[0] == '0');
    }();
    return on;
}

int step_group(sg_ctx* ctx, SwarmGroup& g) {
    if (!g.persistent && graphs_enabled() && g.runs++ >= 2) {
        if (!g.steps_exec) {
            const int rc0 = g.lanes.size() > 1 ? ensure_lanes(ctx) : SG_OK;
            if (rc0) return rc0;
            SG_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            const uint64_t before = ctx->launches;
            const int rc = enqueue_steps(ctx, g);
            ctx->launches = before;  // counted when the graph runs
            cudaGraph_t graph = nullptr;
            const cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
            if (rc) {
                if (graph) cudaGraphDestroy(graph);
                return rc;
            }
            if (e != cudaSuccess) return cuda_fail(ctx, e, "plan graph capture");
            const cudaError_t ei = cudaGraphInstantiate(&g.steps_exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ei != cudaSuccess) {
                g.steps_exec = nullptr;
                return cuda_fail(ctx, ei, "plan graph instantiate");
            }
        }
        SG_CUDA(ctx, cudaGraphLaunch(g.steps_exec, ctx->stream));
        ctx->launches += g.iters * g.lanes.size();
        return SG_OK;
    }
    return enqueue_steps(ctx, g);
}

int enqueue_steps(sg_ctx* ctx, SwarmGroup& g) {
    if (g.persistent) {
        cudaError_t err = cudaSuccess;
        dispatch<SwarmLaunch>(g.family, g.metric, g.substeps, static_cast<unsigned>(g.idx.size()), g.cluster,
                              g.threads, 0u, g.d_sw, g.d_win, g.P, g.d_state, g.smem, ctx->stream, &err);
        ctx->launches += 1;
        if (err != cudaSuccess) return cuda_fail(ctx, err, "pso_swarm_kernel");
        return SG_OK;
    }
    const size_t n_lanes = g.lanes.size();
    if (n_lanes > 1) {
        const int rc = ensure_lanes(ctx);
        if (rc) return rc;
        SG_CUDA(ctx, cudaEventRecord(ctx->fork, ctx->stream));
        for (size_t l = 0; l < n_lanes; ++l) SG_CUDA(ctx, cudaStreamWaitEvent(ctx->side[l], ctx->fork, 0));
    }
    cudaError_t err = cudaSuccess;
    for (uint64_t it = 0; it < g.iters && err == cudaSuccess; ++it) {
        for (size_t l = 0; l < n_lanes && err == cudaSuccess; ++l) {
            const SwarmGroup::Lane& ln = g.lanes[l];
            cudaStream_t st = n_lanes > 1 ? ctx->side[l] : ctx->stream;
            dispatch<StepLaunch>(g.family, g.metric, g.substeps, ln.n_ctas, ln.cta_begin, g.d_task, g.d_sw, g.P,
                                 g.d_state, it, g.smem, st, &err);
            ctx->launches += 1;
        }
    }
    if (n_lanes > 1) {  // join the lanes even after a failed launch (capture and buffer order need it)
        for (size_t l = 0; l < n_lanes; ++l) {
            SG_CUDA(ctx, cudaEventRecord(ctx->join[l], ctx->side[l]));
            SG_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->join[l], 0));
        }
    }
    if (err != cudaSuccess) return cuda_fail(ctx, err, "pso_step_kernel");
    return SG_OK;
}

}  // namespace

extern "C" {

int sg_plan_create(sg_ctx* ctx, const sg_swarm_desc* swarms, size_t n_swarms, sg_plan** out) {
    if (!ctx || !out) return SG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (n_swarms > 0 && !swarms) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null swarm array");
    SG_ENTRY(ctx, "sg_plan_create");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    sg_plan* plan = new (std::nothrow) sg_plan;
    if (!plan) return fail(ctx, SG_ERR_OUT_OF_MEMORY, "host allocation failed");
    plan->ctx = ctx;
    plan->n_desc = n_swarms;
    plan->status.assign(n_swarms, SG_OK);
    std::string why;
    // Swarms of <= kPersistMax particles run as persistent clusters (one
    // launch, state in registers) when all of them fit in one wave of
    // cluster CTAs (2 per SM at the kernel's register use); a plan too large
    // for that fills the GPU better with the flat per-iteration kernels
    // (measured: 148 swarms x 256 particles 1.45x faster persistent, 296
    // even, C4's 4448 swarms flat).  SG_PERSIST_CTAS (diagnostic) overrides
    // the CTA budget.
    uint64_t n_small = 0, max_small = 0;
    for (size_t k = 0; k < n_swarms; ++k)
        if (swarms[k].n_particles <= static_cast<uint64_t>(kPersistMax)) {
            ++n_small;
            max_small = std::max<uint64_t>(max_small, swarms[k].n_particles);
        }
    static const char* persist_env = std::getenv("SG_PERSIST_CTAS");
    const uint64_t persist_budget = persist_env ? std::strtoull(persist_env, nullptr, 10)
                                                : 2 * static_cast<uint64_t>(ctx->sm_count);
    const bool small_plan = n_small * ((max_small + kSwarmThreadsMax - 1) / kSwarmThreadsMax) <= persist_budget;
    for (size_t k = 0; k < n_swarms; ++k) {
        if (!swarm_config_valid(swarms[k], &why)) {
            plan->status[k] = SG_ERR_INVALID_ARGUMENT;
            fail(ctx, SG_ERR_INVALID_ARGUMENT, why);
            continue;
        }
        if (swarms[k].window->ctx != ctx) {
            plan->status[k] = SG_ERR_INVALID_ARGUMENT;
            fail(ctx, SG_ERR_INVALID_ARGUMENT, "swarm window belongs to another context");
            continue;
        }
        const DevWindow& w = swarms[k].window->host;
        const int sub = kernel_sub(w.n_days, w.substeps);
        const bool pers = swarms[k].n_particles <= static_cast<uint64_t>(kPersistMax) && small_plan;
        SwarmGroup* g = nullptr;
        for (SwarmGroup* x : plan->groups)
            if (x->family == w.family && x->metric == w.metric && x->substeps == sub && x->persistent == pers) g = x;
        if (!g) {
            g = new (std::nothrow) SwarmGroup;
            if (!g) {
                delete plan;
                return fail(ctx, SG_ERR_OUT_OF_MEMORY, "host allocation failed");
            }
            g->family = w.family;
            g->metric = w.metric;
            g->substeps = sub;
            g->persistent = pers;
            plan->groups.push_back(g);
        }
        g->idx.push_back(k);
        plan->evals += swarms[k].n_particles * swarms[k].max_iters;
    }
    for (SwarmGroup* g : plan->groups) {
        const int rc = build_group(ctx, swarms, *g);
        if (rc) {
            delete plan;
            return rc;
        }
    }
    *out = plan;
    return SG_OK;
}

int sg_plan_run(sg_plan* plan) {
    if (!plan) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = plan->ctx;
    SG_ENTRY(ctx, "sg_plan_run");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    for (SwarmGroup* g : plan->groups) {
        int rc = seed_group(ctx, *g);
        if (!rc) rc = step_group(ctx, *g);
        if (rc) return rc;
    }
    plan->ran = true;
    return SG_OK;
}

int sg_plan_run_timed(sg_plan* plan, double* seed_ms, double* steps_ms) {
    if (!plan || !seed_ms || !steps_ms) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = plan->ctx;
    SG_ENTRY(ctx, "sg_plan_run_timed");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaEvent_t ev[3];
    for (cudaEvent_t& e : ev) SG_CUDA(ctx, cudaEventCreate(&e));
    *seed_ms = 0.0;
    *steps_ms = 0.0;
    int rc = SG_OK;
    for (SwarmGroup* g : plan->groups) {
        cudaEventRecord(ev[0], ctx->stream);
        rc = seed_group(ctx, *g);
        if (rc) break;
        cudaEventRecord(ev[1], ctx->stream);
        rc = step_group(ctx, *g);
        if (rc) break;
        cudaEventRecord(ev[2], ctx->stream);
        const cudaError_t e = cudaEventSynchronize(ev[2]);
        if (e != cudaSuccess) {
            rc = cuda_fail(ctx, e, "sg_plan_run_timed");
            break;
        }
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        *seed_ms += a;
        *steps_ms += b;
    }
    for (cudaEvent_t& e : ev) cudaEventDestroy(e);
    if (!rc) plan->ran = true;
    return rc;
}

uint64_t sg_plan_step_launches(const sg_plan* plan) {
    uint64_t n = 0;
    if (plan)
        for (const SwarmGroup* g : plan->groups) n += g->persistent ? 1 : g->iters * g->lanes.size();
    return n;
}

int sg_plan_results(sg_plan* plan, sg_swarm_result* results) {
    if (!plan || (!results && plan->n_desc)) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = plan->ctx;
    SG_ENTRY(ctx, "sg_plan_results");
    if (!plan->ran) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "plan has not been run");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    for (size_t k = 0; k < plan->n_desc; ++k) {
        results[k].status = plan->status[k];
        if (plan->status[k] != SG_OK) {
            results[k].best_cost = HUGE_VAL;
            for (double& v : results[k].best_position) v = 0.0;
        }
    }
    for (SwarmGroup* g : plan->groups) {
        std::vector<DevSwarmState> state(g->idx.size());
        std::vector<double> hist(g->idx.size() * g->iters);
        SG_CUDA(ctx, copy_async(ctx, state.data(), g->d_state, sizeof(DevSwarmState) * state.size(),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        SG_CUDA(ctx, copy_async(ctx, hist.data(), g->P.history, sizeof(double) * hist.size(), cudaMemcpyDeviceToHost,
                                     ctx->stream));
        SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        for (size_t j = 0; j < g->idx.size(); ++j) {
            sg_swarm_result& r = results[g->idx[j]];
            std::memcpy(r.best_position, state[j].best, sizeof r.best_position);
            r.best_cost = state[j].best_cost;
            if (r.cost_history)
                std::memcpy(r.cost_history, hist.data() + j * g->iters, sizeof(double) * g->max_iters[j]);
            // optimize() throws AllInfeasibleError when nothing finite was
            // found (pso.cpp:137-139).
            r.status = state[j].best_cost < HUGE_VAL ? SG_OK : SG_ERR_ALL_INFEASIBLE;
        }
    }
    return SG_OK;
}

uint64_t sg_plan_evals(const sg_plan* plan) { return plan ? plan->evals : 0; }

uint64_t sg_plan_ramp_substeps(sg_plan* plan) {
    if (!plan || !plan->ran) return 0;
    sg_ctx* ctx = plan->ctx;
    CtxLock lock(ctx->mu);
    uint64_t total = 0;
    for (SwarmGroup* g : plan->groups) {
        std::vector<DevSwarmState> state(g->idx.size());
        if (copy_async(ctx, state.data(), g->d_state, sizeof(DevSwarmState) * state.size(), cudaMemcpyDeviceToHost,
                            ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            return 0;
        for (const DevSwarmState& s : state) total += s.ramp_substeps;
    }
    return total;
}

void sg_plan_destroy(sg_plan* plan) {
    if (!plan) return;
    CtxLock lock(plan->ctx->mu);
    cudaSetDevice(plan->ctx->device);
    delete plan;
}

// Device bytes per particle of a plan (x, v, pb: 18; pbc: 1; 312
// engine words) — used to split oversized calls into sequential plans.
static constexpr size_t kBytesPerParticle = (18 + 1 + kMtN) * sizeof(double);

void sg_trace_phase(const char* what) {
    static const bool on = std::getenv("SG_TRACE") != nullptr;
    if (!on) return;
    static auto last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sg] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

int sg_fit_swarms(sg_ctx* ctx, const sg_swarm_desc* swarms, size_t n_swarms, sg_swarm_result* results) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (n_swarms == 0) return SG_OK;
    if (!swarms || !results) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null swarm arrays");
    SG_ENTRY(ctx, "sg_fit_swarms");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    // Split oversized calls into sequential plans that fit in 70% of the
    // free memory; the (slow, driver-locking) memory query only runs when
    // the call could come near the 180 GB of a B200.
    size_t want = 0;
    for (size_t k = 0; k < n_swarms; ++k) want += swarms[k].n_particles * kBytesPerParticle;
    size_t budget = want;
    if (want > (size_t(16) << 30)) {
        size_t free_b = 0, total_b = 0;
        SG_CUDA(ctx, cudaMemGetInfo(&free_b, &total_b));
        budget = std::max<size_t>(free_b / 10 * 7, size_t(1) << 28);
    }
    static const char* budget_env = std::getenv("SG_PLAN_BUDGET_BYTES");  // diagnostic: force the split
    if (budget_env) budget = std::min<size_t>(budget, std::strtoull(budget_env, nullptr, 10));
    size_t begin = 0;
    while (begin < n_swarms) {
        size_t end = begin, bytes = 0;
        while (end < n_swarms) {
            const size_t need = swarms[end].n_particles * kBytesPerParticle;
            if (end > begin && bytes + need > budget) break;
            bytes += need;
            ++end;
        }
        sg_plan* plan = nullptr;
        sg_trace_phase("fit_swarms: chunk");
        int rc = sg_plan_create(ctx, swarms + begin, end - begin, &plan);
        sg_trace_phase("plan_create");
        if (!rc) rc = sg_plan_run(plan);
        sg_trace_phase("plan_run");
        if (!rc) rc = sg_plan_results(plan, results + begin);
        sg_trace_phase("plan_results");
        sg_plan_destroy(plan);
        sg_trace_phase("plan_destroy");
        if (rc) return rc;
        begin = end;
    }
    return SG_OK;
}

// Days of t1/t2 per ordering-key step: 1 while the box's switch times stay
// below day 64, coarser beyond (the key has 64 steps per switch time).
static int order_step(const double upper[6]) {
    const double t = std::max(upper[2], upper[3]);
    return t < 63.0 ? 1 : static_cast<int>(std::min(4096.0, std::ceil((t + 1.0) / 64.0)));
}

// Ramp-coherent evaluation order of an ensemble: ens_sample_kernel draws
// every sample into SoA planes with its (day t1, day t2) key and counts the
// keys (ranking each sample within its key); a scan and an atomic-free
// scatter complete the counting sort into perm.
// key_count: 2 x kOrderKeys, the counts zero on entry (and again on exit).
// sample = false: the samples and key counts were drawn elsewhere (an
// earlier window's ensemble launch, EnsNext); only the scan and scatter run.
static int ensemble_order(sg_ctx* ctx, const double* d_lo, const double* d_hi, uint64_t seed, size_t n, int q,
                          double* planes, uint32_t* keys, unsigned int* key_count, uint32_t* perm, cudaStream_t st,
                          bool sample = true) {
    const unsigned grid = static_cast<unsigned>((n + kSampleThreads - 1) / kSampleThreads);
    if (sample) {
        ens_sample_kernel<<<grid, kSampleThreads, 0, st>>>(d_lo, d_hi, seed, n, q, planes, keys, key_count);
        ctx->launches += 1;
    }
    ens_scan_kernel<<<1, kBgThreads, 0, st>>>(key_count);
    ens_scatter_kernel<<<grid, kSampleThreads, 0, st>>>(keys, n, key_count + kOrderKeys, perm);
    ctx->launches += 2;
    SG_CUDA(ctx, cudaGetLastError());
    return SG_OK;
}

int sg_forecast_ensemble(sg_window* w, const double lower[6], const double upper[6], uint64_t seed, size_t n,
                         int horizon, double* costs, double* params_out, double* deaths_out) {
    if (!w) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = w->ctx;
    if (!lower || !upper || !deaths_out) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null buffer");
    if (horizon < 0) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "horizon must be >= 0");
    for (int k = 0; k < 6; ++k)
        if (!std::isfinite(lower[k]) || !std::isfinite(upper[k]) || lower[k] > upper[k])
            return fail(ctx, SG_ERR_INVALID_ARGUMENT, "pso: bound " + std::to_string(k) + " is invalid");
    if (n == 0) return SG_OK;
    SG_ENTRY(ctx, "sg_forecast_ensemble");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double *d_lo, *d_hi, *d_cost = nullptr, *d_par = nullptr, *d_D;
    SG_CUDA(ctx, b.alloc(&d_lo, 6));
    SG_CUDA(ctx, b.alloc(&d_hi, 6));
    if (costs) SG_CUDA(ctx, b.alloc(&d_cost, n));
    if (params_out) SG_CUDA(ctx, b.alloc(&d_par, 6 * n));
    SG_CUDA(ctx, b.alloc(&d_D, n * static_cast<size_t>(horizon + 1)));
    SG_CUDA(ctx, copy_async(ctx, d_lo, lower, 6 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_hi, upper, 6 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    DevWindow fwin = integration_window(horizon + 1, w->host.substeps, w->host.N);
    uint32_t* perm = nullptr;
    double* planes = nullptr;
    if (n <= static_cast<size_t>(INT32_MAX)) {
        uint32_t* keys;
        unsigned int* key_count;
        SG_CUDA(ctx, b.alloc(&planes, 6 * n));
        SG_CUDA(ctx, b.alloc(&keys, 2 * n));
        SG_CUDA(ctx, b.alloc(&perm, n));
        SG_CUDA(ctx, b.alloc(&key_count, 2 * kOrderKeys));
        SG_CUDA(ctx, cudaMemsetAsync(key_count, 0, sizeof(unsigned int) * kOrderKeys, ctx->stream));
        if (const int rc = ensemble_order(ctx, d_lo, d_hi, seed, n, order_step(upper), planes, keys, key_count, perm,
                                          ctx->stream))
            return rc;
    }
    cudaError_t err = cudaSuccess;
    dispatch<EnsembleLaunch>(w->host.family, w->host.metric, kernel_sub(w->host.n_days, w->host.substeps), w->d_desc,
                             fwin, d_lo, d_hi, seed, n, horizon, d_cost, d_par, d_D,
                             static_cast<size_t>(horizon + 1), size_t(1), perm, planes, 0, static_cast<SelDay*>(nullptr),
                             static_cast<unsigned int*>(nullptr), static_cast<unsigned long long*>(nullptr), EnsNext{},
                             w->smem, ctx->stream, &err);
    ctx->launches += 1;
    if (err != cudaSuccess) return cuda_fail(ctx, err, "ensemble_kernel");
    if (costs) SG_CUDA(ctx, copy_async(ctx, costs, d_cost, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (params_out)
        SG_CUDA(ctx, copy_async(ctx, params_out, d_par, 6 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, deaths_out, d_D, n * (horizon + 1) * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

// Order buffers of one window (samples, keys + ranks, permutation, key
// counts + cursors).
struct OrderBufs {
    double* planes = nullptr;
    uint32_t *keys = nullptr, *perm = nullptr;
    unsigned int* key_count = nullptr;
};

static int alloc_order_bufs(sg_ctx* ctx, DevBufs& b, OrderBufs& o, size_t n) {
    SG_CUDA(ctx, b.alloc(&o.planes, 6 * n));
    SG_CUDA(ctx, b.alloc(&o.keys, 2 * n));  // key, rank within the key
    SG_CUDA(ctx, b.alloc(&o.perm, n));
    SG_CUDA(ctx, b.alloc(&o.key_count, 2 * kOrderKeys));
    // zero once: ens_scan_kernel leaves the counts zero
    SG_CUDA(ctx, cudaMemsetAsync(o.key_count, 0, sizeof(unsigned int) * kOrderKeys, b.st));
    return SG_OK;
}

// Device buffers of one window in flight in the C5 pipeline (the order
// buffers bound per window from an OrderBufs).
struct BandSlot {
    double *planes = nullptr, *D = nullptr, *cand = nullptr, *scratch = nullptr, *vals = nullptr;
    uint32_t *keys = nullptr, *perm = nullptr;
    unsigned int *key_count = nullptr, *hist = nullptr;
    SelDay* days = nullptr;
    bool unordered = false;  // SG_BAND_ORDER=0 (diagnostic)
};

// The ensemble kernel reduces each day's key range and finite count as the
// forecast runs (lane d of a warp holds day d, so horizon < 32: REDUX per
// day, no barrier, no re-read of the plane — an earlier epilogue version that
// re-read the row and folded per CTA cost ~63 us per evaluation);
// SG_FUSED_RANGE=0 runs sel_range_kernel over the plane instead (A/B).
static bool fused_range(int horizon) {
    static const bool on = [] {
        const char* e = std::getenv("SG_FUSED_RANGE");
        return !(e && e[0] == '0');
    }();
    return on && horizon < 32;
}

// The ensemble kernel's fused histogram over predicted bins (SelDay);
// SG_FUSED_HIST=0 sends every day through the histogram pass (A/B).
static bool fused_hist() {
    static const bool on = [] {
        const char* e = std::getenv("SG_FUSED_HIST");
        return !(e && e[0] == '0');
    }();
    return on;
}

static void bind_order(BandSlot& s, const OrderBufs& o) {
    s.planes = o.planes;
    s.keys = o.keys;
    s.perm = o.perm;
    s.key_count = o.key_count;
}

static int alloc_band_slot(sg_ctx* ctx, DevBufs& b, BandSlot& s, size_t n, int n_days, bool with_order = true) {
    const size_t nd = n * static_cast<size_t>(n_days);
    if (with_order) {
        OrderBufs o;
        if (const int rc = alloc_order_bufs(ctx, b, o, n)) return rc;
        bind_order(s, o);
    }
    SG_CUDA(ctx, b.alloc(&s.D, nd));
    SG_CUDA(ctx, b.alloc(&s.cand, nd));
    SG_CUDA(ctx, b.alloc(&s.scratch, 2 * nd));  // only bins too full for one CTA's shared memory touch it
    SG_CUDA(ctx, b.alloc(&s.days, n_days));
    SG_CUDA(ctx, b.alloc(&s.hist, static_cast<size_t>(n_days) * kSelBins));
    SG_CUDA(ctx, b.alloc(&s.vals, static_cast<size_t>(n_days) * kBandRanks));
    // zero once: sel_locate_kernel leaves it zero
    SG_CUDA(ctx, cudaMemsetAsync(s.hist, 0, sizeof(unsigned int) * n_days * kSelBins, b.st));
    SG_CUDA(ctx, cudaMemsetAsync(s.days, 0, sizeof(SelDay) * n_days, b.st));  // no prediction for the first window
    return SG_OK;
}

// C5, stage 1 (integer work): the samples and their ramp-coherent order;
// the slot's day records reset for the selection.
static int enqueue_band_order(sg_ctx* ctx, BandSlot& s, cudaStream_t st, const double* d_lo, const double* d_hi,
                              uint64_t seed, size_t n, int q, int n_days, bool sample = true) {
    static const bool ordered = [] {  // SG_BAND_ORDER=0: samples drawn in the ensemble kernel, unordered (A/B)
        const char* e = std::getenv("SG_BAND_ORDER");
        return !(e && e[0] == '0');
    }();
    if (ordered) {
        if (const int rc =
                ensemble_order(ctx, d_lo, d_hi, seed, n, q, s.planes, s.keys, s.key_count, s.perm, st, sample))
            return rc;
    }
    s.unordered = !ordered;
    sel_init_kernel<<<static_cast<unsigned>((n_days + kBgThreads - 1) / kBgThreads), kBgThreads, 0, st>>>(
        s.days, n_days, fused_range(n_days - 1) && fused_hist() ? 1 : 0);
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    return SG_OK;
}

// Band telemetry (device): [0] days from the fused histogram, [1] days
// through the histogram pass, [2] ramp substeps of the evaluated windows.
static int ensure_band_stats(sg_ctx* ctx) {
    if (ctx->band_stats) return SG_OK;
    SG_CUDA(ctx, cudaMalloc(&ctx->band_stats, 3 * sizeof(unsigned long long)));
    SG_CUDA(ctx, cudaMemsetAsync(ctx->band_stats, 0, 3 * sizeof(unsigned long long), ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // once per context; zero before any stream adds to it
    return SG_OK;
}

// C5, stage 2 (FP64-bound): evaluation of the window and forecast into the
// slot's day-major deaths plane; with horizon < 32 the kernel also reduces
// each day's key range and finite count and fills the predicted-bin
// histogram as the forecast days arrive (BandDSink).
static int enqueue_band_eval(sg_ctx* ctx, sg_window* w, BandSlot& s, cudaStream_t st, const double* d_lo,
                             const double* d_hi, uint64_t seed, size_t n, int horizon, double* d_cost,
                             EnsNext next = EnsNext{}) {
    const int n_days = horizon + 1;
    const DevWindow fwin = integration_window(n_days, w->host.substeps, w->host.N);
    if (const int rc = ensure_band_stats(ctx)) return rc;
    cudaError_t err = cudaSuccess;
    // day-major columns in evaluation order: the bands only need each day's multiset
    dispatch<EnsembleLaunch>(w->host.family, w->host.metric, kernel_sub(w->host.n_days, w->host.substeps), w->d_desc,
                             fwin, d_lo, d_hi, seed, n, horizon, d_cost, static_cast<double*>(nullptr), s.D, size_t(1),
                             n, s.unordered ? nullptr : s.perm, s.unordered ? nullptr : s.planes, 1,
                             fused_range(horizon) ? s.days : nullptr, s.hist,
                             ctx->band_stats ? ctx->band_stats + 2 : nullptr, next, w->smem, st, &err);
    ctx->launches += 1;
    if (err != cudaSuccess) return cuda_fail(ctx, err, "ensemble_kernel");
    return SG_OK;
}

// C5, stage 3 (memory-bound): per forecast day the bins of the wanted
// ranks (calibration.cpp:17-25, 324-361) — located in the ensemble's fused
// histogram, or for the days whose prediction missed in a histogram pass
// over the plane — then a gather of those bins' values, one CTA per (bin,
// day) resolving the bin's wanted ranks in shared memory, and
// quantile_sorted turning them into the bands.
static int enqueue_band_select(sg_ctx* ctx, BandSlot& s, cudaStream_t st, size_t n, int n_days, double* d_bands,
                               unsigned long long* d_counts, bool standalone = false) {
    if (const int rc = ensure_band_stats(ctx)) return rc;
    const unsigned chunks = static_cast<unsigned>(std::min<size_t>(64, (n + 4095) / 4096));
    const dim3 grid(chunks, static_cast<unsigned>(n_days));
    if (!fused_range(n_days - 1) && !standalone) {  // standalone: the caller ran it
        sel_range_kernel<<<grid, kSampleThreads, 0, st>>>(s.D, n, s.days);
        ctx->launches += 1;
    }
    const dim3 hgrid(static_cast<unsigned>(std::min<size_t>(16, (n + 16383) / 16384)), static_cast<unsigned>(n_days));
    // the fused histogram, else (per day) the histogram pass over the plane
    sel_locate_kernel<<<static_cast<unsigned>(n_days), kBgThreads, 0, st>>>(s.hist, s.days, 0, ctx->band_stats);
    sel_hist_kernel<<<hgrid, kHistThreads, 0, st>>>(s.D, n, s.days, s.hist);
    sel_locate_kernel<<<static_cast<unsigned>(n_days), kBgThreads, 0, st>>>(s.hist, s.days, 1, nullptr);
    sel_gather_kernel<<<grid, kSampleThreads, 0, st>>>(s.D, n, s.days, s.cand);
    sel_finish_kernel<<<static_cast<unsigned>(kBandRanks * n_days), kSampleThreads, 0, st>>>(
        n_days, s.days, s.cand, s.scratch, n, s.vals);
    sel_bands_kernel<<<static_cast<unsigned>((n_days + kBgThreads - 1) / kBgThreads), kBgThreads, 0, st>>>(
        s.days, s.vals, d_bands, d_counts, n_days);
    ctx->launches += 6;
    SG_CUDA(ctx, cudaGetLastError());
    return SG_OK;
}

static int check_bands_args(sg_ctx* ctx, const double* lower, const double* upper, size_t n, int horizon) {
    if (horizon < 0) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "horizon must be >= 0");
    for (int k = 0; k < 6; ++k)
        if (!std::isfinite(lower[k]) || !std::isfinite(upper[k]) || lower[k] > upper[k])
            return fail(ctx, SG_ERR_INVALID_ARGUMENT, "pso: bound " + std::to_string(k) + " is invalid");
    if (n > static_cast<size_t>(INT32_MAX))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "ensemble too large for one device selection (n > 2^31)");
    return SG_OK;
}

int sg_forecast_ensemble_bands(sg_window* w, const double lower[6], const double upper[6], uint64_t seed, size_t n,
                               int horizon, double* bands, uint64_t* counts, double* costs) {
    if (!w) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = w->ctx;
    if (!lower || !upper || !bands || !counts) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null buffer");
    if (const int rc = check_bands_args(ctx, lower, upper, n, horizon)) return rc;
    const int n_days = horizon + 1;
    SG_ENTRY(ctx, "sg_forecast_ensemble_bands");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double *d_lo, *d_hi, *d_cost = nullptr, *d_bands;
    unsigned long long* d_counts;
    SG_CUDA(ctx, b.alloc(&d_lo, 6));
    SG_CUDA(ctx, b.alloc(&d_hi, 6));
    if (costs && n) SG_CUDA(ctx, b.alloc(&d_cost, n));
    SG_CUDA(ctx, b.alloc(&d_bands, 7 * static_cast<size_t>(n_days)));
    SG_CUDA(ctx, b.alloc(&d_counts, n_days));
    SG_CUDA(ctx, copy_async(ctx, d_lo, lower, 6 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_hi, upper, 6 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if (n == 0) {
        bands_kernel<<<n_days, 32, 0, ctx->stream>>>(nullptr, 0, d_bands, d_counts, n_days);  // k = 0: NaN bands
        ctx->launches += 1;
        SG_CUDA(ctx, cudaGetLastError());
    } else {
        BandSlot s;
        if (const int rc = alloc_band_slot(ctx, b, s, n, n_days)) return rc;
        if (const int rc = enqueue_band_order(ctx, s, ctx->stream, d_lo, d_hi, seed, n, order_step(upper), n_days))
            return rc;
        if (const int rc = enqueue_band_eval(ctx, w, s, ctx->stream, d_lo, d_hi, seed, n, horizon, d_cost)) return rc;
        if (const int rc = enqueue_band_select(ctx, s, ctx->stream, n, n_days, d_bands, d_counts)) return rc;
    }
    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "count width");
    SG_CUDA(ctx, copy_async(ctx, bands, d_bands, 7 * n_days * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, counts, d_counts, n_days * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    if (costs && n)
        SG_CUDA(ctx, copy_async(ctx, costs, d_cost, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_quantile_bands(sg_ctx* ctx, const double* values, size_t n, int n_days, double* bands, uint64_t* counts) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (n_days < 1 || (n && !values) || !bands || !counts) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null buffer");
    if (n > static_cast<size_t>(INT32_MAX)) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "too many values per day (> 2^31)");
    SG_ENTRY(ctx, "sg_quantile_bands");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double* d_bands;
    unsigned long long* d_counts;
    SG_CUDA(ctx, b.alloc(&d_bands, 7 * static_cast<size_t>(n_days)));
    SG_CUDA(ctx, b.alloc(&d_counts, n_days));
    if (n == 0) {
        bands_kernel<<<n_days, 32, 0, ctx->stream>>>(nullptr, 0, d_bands, d_counts, n_days);
        ctx->launches += 1;
    } else {
        BandSlot s;
        const size_t nd = n * static_cast<size_t>(n_days);
        SG_CUDA(ctx, b.alloc(&s.D, nd));
        SG_CUDA(ctx, b.alloc(&s.cand, nd));
        SG_CUDA(ctx, b.alloc(&s.scratch, 2 * nd));
        SG_CUDA(ctx, b.alloc(&s.days, n_days));
        SG_CUDA(ctx, b.alloc(&s.hist, static_cast<size_t>(n_days) * kSelBins));
        SG_CUDA(ctx, b.alloc(&s.vals, static_cast<size_t>(n_days) * kBandRanks));
        SG_CUDA(ctx, cudaMemsetAsync(s.hist, 0, sizeof(unsigned int) * n_days * kSelBins, ctx->stream));
        SG_CUDA(ctx, copy_async(ctx, s.D, values, sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream));
        sel_init_kernel<<<static_cast<unsigned>((n_days + 127) / 128), 128, 0, ctx->stream>>>(s.days, n_days, 0);
        const dim3 grid(static_cast<unsigned>(std::min<size_t>(64, (n + 4095) / 4096)), static_cast<unsigned>(n_days));
        sel_range_kernel<<<grid, kSampleThreads, 0, ctx->stream>>>(s.D, n, s.days);
        ctx->launches += 2;
        if (const int rc = enqueue_band_select(ctx, s, ctx->stream, n, n_days, d_bands, d_counts, true)) return rc;
    }
    SG_CUDA(ctx, cudaGetLastError());
    SG_CUDA(ctx, copy_async(ctx, bands, d_bands, 7 * n_days * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, counts, d_counts, n_days * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

// Many windows (C5): a two-slot pipeline on two streams.  The evaluation
// stream (low priority) runs window k's FP64-bound ensemble while the
// selection stream (high priority, so its memory-bound CTAs take SM slots
// as soon as ensemble CTAs retire) reduces window k-1 to bands.
static int ensure_band_streams(sg_ctx* ctx) {
    if (ctx->band_eval[0]) return SG_OK;
    int least = 0, greatest = 0;
    SG_CUDA(ctx, cudaDeviceGetStreamPriorityRange(&least, &greatest));
    // SG_BAND_PRIO (diagnostic A/B): priority of the selection stream
    // relative to the evaluation streams: high (default), equal or low.  At
    // low priority the selection's grids are dispatched only once an
    // evaluation grid has no CTAs left to place, so the evaluations stall on
    // the ordering (round 2: 217 ms vs 188 ms high; 213-268 ms with the
    // selection kernels cut to fit beside the ensemble's CTAs)
    static const char* prio = std::getenv("SG_BAND_PRIO");
    const std::string p = prio ? prio : "high";
    const int eval_prio = p == "low" ? greatest : least;
    const int sel_prio = p == "high" ? greatest : least;
    for (cudaStream_t& e : ctx->band_eval)
        SG_CUDA(ctx, cudaStreamCreateWithPriority(&e, cudaStreamNonBlocking, eval_prio));
    SG_CUDA(ctx, cudaStreamCreateWithPriority(&ctx->band_sel, cudaStreamNonBlocking, sel_prio));
    return SG_OK;
}

int sg_forecast_ensemble_bands_batch(sg_window* const* windows, size_t n_windows, const double lower[6],
                                     const double upper[6], const uint64_t* seeds, size_t n, int horizon,
                                     double* bands, uint64_t* counts) {
    if (!windows || n_windows == 0) return n_windows == 0 ? SG_OK : SG_ERR_INVALID_ARGUMENT;
    if (!windows[0]) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = windows[0]->ctx;
    if (!lower || !upper || !seeds || !bands || !counts) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null buffer");
    for (size_t k = 0; k < n_windows; ++k)
        if (!windows[k] || windows[k]->ctx != ctx)
            return fail(ctx, SG_ERR_INVALID_ARGUMENT, "windows must be non-null and share one context");
    if (const int rc = check_bands_args(ctx, lower, upper, n, horizon)) return rc;
    if (n == 0) {  // NaN bands for every window, like the single-window call
        for (size_t k = 0; k < n_windows; ++k) {
            const int rc = sg_forecast_ensemble_bands(windows[k], lower, upper, seeds[k], 0, horizon,
                                                      bands + 7 * static_cast<size_t>(horizon + 1) * k,
                                                      counts + static_cast<size_t>(horizon + 1) * k, nullptr);
            if (rc) return rc;
        }
        return SG_OK;
    }
    const int n_days = horizon + 1;
    const int q = order_step(upper);
    SG_ENTRY(ctx, "sg_forecast_ensemble_bands_batch");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    if (const int rc = ensure_lanes(ctx)) return rc;
    if (const int rc = ensure_band_streams(ctx)) return rc;
    if (const int rc = ensure_band_stats(ctx)) return rc;
    DevBufs b;
    b.st = ctx->stream;
    double *d_lo, *d_hi, *d_bands;
    unsigned long long* d_counts;
    SG_CUDA(ctx, b.alloc(&d_lo, 6));
    SG_CUDA(ctx, b.alloc(&d_hi, 6));
    SG_CUDA(ctx, b.alloc(&d_bands, 7 * static_cast<size_t>(n_days) * n_windows));
    SG_CUDA(ctx, b.alloc(&d_counts, static_cast<size_t>(n_days) * n_windows));
    constexpr int kSlots = sg_ctx::kBandSlots;  // band buffers (deaths plane, day records, histograms)
    constexpr int kOrd = 4;                      // order buffers: windows k..k+3 (samples drawn two ahead)
    BandSlot slot[kSlots];
    for (BandSlot& s : slot)
        if (const int rc = alloc_band_slot(ctx, b, s, n, n_days, false)) return rc;
    OrderBufs ord[kOrd];
    for (OrderBufs& o : ord)
        if (const int rc = alloc_order_bufs(ctx, b, o, n)) return rc;
    // SG_BAND_AHEAD=0 (A/B): every window's samples drawn on the selection
    // stream instead of by the ensemble launch two windows earlier
    static const bool ahead = [] {
        const char* e = std::getenv("SG_BAND_AHEAD");
        return !(e && e[0] == '0');
    }();
    SG_CUDA(ctx, copy_async(ctx, d_lo, lower, 6 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_hi, upper, 6 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    cudaEvent_t ordered[kOrd], evaluated[kOrd], selected[kSlots];
    for (int k = 0; k < kOrd; ++k) {
        SG_CUDA(ctx, cudaEventCreateWithFlags(&ordered[k], cudaEventDisableTiming));
        SG_CUDA(ctx, cudaEventCreateWithFlags(&evaluated[k], cudaEventDisableTiming));
    }
    for (int k = 0; k < kSlots; ++k) SG_CUDA(ctx, cudaEventCreateWithFlags(&selected[k], cudaEventDisableTiming));
    // Three stages per window: order (S) -> evaluate (E) -> select (S).  S
    // finishes window k+1's order while E evaluates window k, then runs
    // window k's selection.  Each band slot evaluates on its own stream:
    // nothing orders window k+1's evaluation after window k's, so its CTAs
    // fill the SMs window k's last wave leaves idle.  Window k's ensemble
    // launch also draws window k+2's samples and key counts (EnsNext: integer
    // work the FP64-bound launch absorbs), so S's order stage is the scan and
    // the scatter.  Order buffers rotate over 4 windows: launch k reads
    // ord[k%4] and writes ord[(k+2)%4], launch k+1 (concurrent) ord[(k+1)%4]
    // and ord[(k+3)%4]; ord[(k+2)%4] was last read by launch k-2, which
    // finished before window k-2's selection that launch k waits for.
    cudaStream_t S = ctx->band_sel;
    SG_CUDA(ctx, cudaEventRecord(ctx->fork, ctx->stream));  // buffers allocated, bounds uploaded
    for (cudaStream_t e : ctx->band_eval) SG_CUDA(ctx, cudaStreamWaitEvent(e, ctx->fork, 0));
    SG_CUDA(ctx, cudaStreamWaitEvent(S, ctx->fork, 0));
    auto step = [&](cudaError_t e) { return e == cudaSuccess ? SG_OK : cuda_fail(ctx, e, "band pipeline"); };
    bind_order(slot[0], ord[0]);
    int rc = enqueue_band_order(ctx, slot[0], S, d_lo, d_hi, seeds[0], n, q, n_days);
    if (!rc) rc = step(cudaEventRecord(ordered[0], S));
    for (size_t k = 0; k < n_windows && !rc; ++k) {
        const int j = static_cast<int>(k % kSlots), o = static_cast<int>(k % kOrd);
        cudaStream_t E = ctx->band_eval[j];
        // E: window k once ordered, into a band slot its previous window has
        // been reduced from
        rc = step(cudaStreamWaitEvent(E, ordered[o], 0));
        if (!rc && k >= kSlots) rc = step(cudaStreamWaitEvent(E, selected[j], 0));
        EnsNext next{};
        if (ahead && k + 2 < n_windows) {
            const OrderBufs& a2 = ord[(k + 2) % kOrd];
            next = EnsNext{seeds[k + 2], a2.planes, a2.keys, a2.key_count, q};
        }
        bind_order(slot[j], ord[o]);
        if (!rc) rc = enqueue_band_eval(ctx, windows[k], slot[j], E, d_lo, d_hi, seeds[k], n, horizon, nullptr, next);
        if (!rc) rc = step(cudaEventRecord(evaluated[o], E));
        // S: the next window's order, then window k's selection
        if (!rc && k + 1 < n_windows) {
            const int j1 = static_cast<int>((k + 1) % kSlots), o1 = static_cast<int>((k + 1) % kOrd);
            const bool drawn = ahead && k + 1 >= 2;  // by launch k-1
            // drawn: wait for launch k-1; else the order buffers' last reader, launch k-3
            if (drawn) rc = step(cudaStreamWaitEvent(S, evaluated[(k + kOrd - 1) % kOrd], 0));
            else if (k + 1 >= kOrd) rc = step(cudaStreamWaitEvent(S, evaluated[o1], 0));
            bind_order(slot[j1], ord[o1]);
            if (!rc) rc = enqueue_band_order(ctx, slot[j1], S, d_lo, d_hi, seeds[k + 1], n, q, n_days, !drawn);
            if (!rc) rc = step(cudaEventRecord(ordered[o1], S));
        }
        if (!rc) rc = step(cudaStreamWaitEvent(S, evaluated[o], 0));
        if (!rc)
            rc = enqueue_band_select(ctx, slot[j], S, n, n_days, d_bands + 7 * static_cast<size_t>(n_days) * k,
                                     d_counts + static_cast<size_t>(n_days) * k);
        if (!rc) rc = step(cudaEventRecord(selected[j], S));
    }
    // join the streams even after a failure: the buffers are released in ctx->stream order
    for (int e = 0; e < kSlots; ++e) {
        SG_CUDA(ctx, cudaEventRecord(ctx->join[e], ctx->band_eval[e]));
        SG_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->join[e], 0));
    }
    SG_CUDA(ctx, cudaEventRecord(ctx->join[kSlots], S));
    SG_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->join[kSlots], 0));
    for (int k = 0; k < kOrd; ++k) {
        cudaEventDestroy(ordered[k]);
        cudaEventDestroy(evaluated[k]);
    }
    for (int k = 0; k < kSlots; ++k) cudaEventDestroy(selected[k]);
    if (rc) return rc;
    SG_CUDA(ctx, copy_async(ctx, bands, d_bands, 7 * n_days * n_windows * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, counts, d_counts, n_days * n_windows * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                            ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

}  // extern "C"

// ---- diagnostics -------------------------------------------------------------------

#if SG_DAY_COUNTERS
extern "C" int sg_day_classes_u0(unsigned long long* out3);
extern "C" int sg_day_classes_u1(unsigned long long* out3);
extern "C" int sg_day_classes_u2(unsigned long long* out3);
extern "C" int sg_day_classes_u3(unsigned long long* out3);
extern "C" int sg_day_classes_u4(unsigned long long* out3);
extern "C" int sg_day_classes_u5(unsigned long long* out3);
extern "C" int sg_day_classes_u6(unsigned long long* out3);
extern "C" int sg_day_classes_u7(unsigned long long* out3);
#endif

extern "C" int sg_debug_day_classes(unsigned long long* out3) {
#if SG_DAY_COUNTERS
    int (*parts[8])(unsigned long long*) = {sg_day_classes_u0, sg_day_classes_u1, sg_day_classes_u2,
                                            sg_day_classes_u3, sg_day_classes_u4, sg_day_classes_u5,
                                            sg_day_classes_u6, sg_day_classes_u7};
    for (int k = 0; k < 3; ++k) out3[k] = 0;
    for (auto f : parts) {
        unsigned long long a[3];
        f(a);
        for (int k = 0; k < 3; ++k) out3[k] += a[k];
    }
    return SG_OK;
#else
    out3[0] = out3[1] = out3[2] = 0;
    return SG_ERR_INVALID_ARGUMENT;
#endif
}

namespace {

// 8 independent DADD/DMUL chains per thread, alternating, no FMA: the FP64
// pipe's issue rate for the operation mix of euler_substep.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = a + threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __dmul_rn(x[j], b);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __dadd_rn(x[j], a);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __dadd_rn(s, x[j]);
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

extern "C" int sg_probe_fp64_rate(sg_ctx* ctx, double* ops_per_s) {
    if (!ctx || !ops_per_s) return SG_ERR_INVALID_ARGUMENT;
    SG_ENTRY(ctx, "sg_probe_fp64_rate");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    double* d_out;
    SG_CUDA(ctx, b.alloc(&d_out, 1));
    const int iters = 4096;
    const unsigned grid = static_cast<unsigned>(ctx->sm_count * 8);  // 2048 threads / SM
    cudaEvent_t e0, e1;
    SG_CUDA(ctx, cudaEventCreate(&e0));
    SG_CUDA(ctx, cudaEventCreate(&e1));
    float best_ms = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        SG_CUDA(ctx, cudaEventRecord(e0, ctx->stream));
        fp64_probe_kernel<<<grid, 256, 0, ctx->stream>>>(d_out, iters, 1.0000001, 0.9999999);
        SG_CUDA(ctx, cudaEventRecord(e1, ctx->stream));
        SG_CUDA(ctx, cudaEventSynchronize(e1));
        float ms = 0.0f;
        SG_CUDA(ctx, cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0) best_ms = std::min(best_ms, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double ops = static_cast<double>(grid) * 256.0 * iters * 16.0;
    *ops_per_s = ops / (best_ms * 1e-3);
    return SG_OK;
}
