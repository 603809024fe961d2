// gswarm.cu — the rest of the reference's numeric API on the device:
//
//   sg_gswarm_*            Swarm / optimize (pso.hpp:41-93) for ANY dimension and
//                          ANY objective.  The swarm's state (positions,
//                          velocities, personal bests, one MT19937-64 engine per
//                          particle) lives in device memory and every PSO
//                          operation runs here; an objective the engine does not
//                          own (a host BatchObjective, e.g. the reference's
//                          acceptance sphere) receives the positions and returns
//                          the costs once per step, exactly where the reference
//                          calls it (pso.cpp:81).  A window objective evaluates
//                          in place on the device (eval_costs_kernel).
//   sg_objective_values    objective_value (objectives.cpp:95-120) of given
//   sg_metric_values       trajectories / metric_value (objectives.cpp:72-81)
//   sg_sird_rhs_batch      sird_rhs (model.cpp:66-74)
//
// The fused many-swarm kernels of engine.cu remain the fast path of
// optimize() for window objectives (sirdfit_b200::optimize dispatches there);
// this file serves the general API with the same arithmetic, bit for bit.
#define SG_FAMILY_TU 1  // the shared kernels of kernels.cuh live in engine.cu
#include "engine_core.cuh"

#include <cmath>
#include <new>

namespace sirdgpu {
namespace {

constexpr int kGThreads = 256;

__device__ __forceinline__ double pinf() { return __longlong_as_double(0x7FF0000000000000LL); }

// One value of the particle's engine at draw position `pos` (values drawn
// so far): the lazy in-place twist of word pos % 312 (sird_device.cuh).
__device__ __forceinline__ double gdraw(uint64_t* mt, uint64_t pos) {
    double u;
    mt_draw<1>(mt, static_cast<int>(pos % kMtN), &u);
    return u;
}

// Swarm::Swarm (pso.cpp:47-75): engine i = mt19937_64(mix_seed(seed, i)),
// x[d] = lo[d] + u * (hi[d] - lo[d]) for d in order, repair, v = 0, pbest = x,
// pbest cost = +inf.  Row-major n x dim planes (the BatchObjective layout).
__global__ void __launch_bounds__(kGThreads) gswarm_init_kernel(size_t n, int dim, const double* __restrict__ lo,
                                                                const double* __restrict__ hi, uint64_t seed,
                                                                int repair, uint64_t* __restrict__ mt,
                                                                double* __restrict__ x, double* __restrict__ v,
                                                                double* __restrict__ pb, double* __restrict__ pbc) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t* const e = mt + pblock_base(i, kMtN);
    uint64_t m = mix_seed(seed, i);
    e[0] = m;
    for (int j = 1; j < kMtN; ++j) {
        m = kMtF * (m ^ (m >> 62)) + static_cast<uint64_t>(j);
        e[32 * j] = m;
    }
    double* const xi = x + i * dim;
    for (int d = 0; d < dim; ++d) xi[d] = dadd(lo[d], dmul(gdraw(e, static_cast<uint64_t>(d)), dsub(hi[d], lo[d])));
    if (repair) repair_order(xi);  // repair_time_order (calibration.cpp:89-93), dim >= 4
    for (int d = 0; d < dim; ++d) {
        v[i * dim + d] = 0.0;
        pb[i * dim + d] = xi[d];
    }
    pbc[i] = pinf();
}

// Personal bests (pso.cpp:83-89) and the block's (cost, index) minimum of
// the personal-best costs.
__global__ void __launch_bounds__(kGThreads) gswarm_pbest_kernel(size_t n, int dim, const double* __restrict__ cost,
                                                                 const double* __restrict__ x, double* __restrict__ pb,
                                                                 double* __restrict__ pbc,
                                                                 double* __restrict__ part_cost,
                                                                 unsigned long long* __restrict__ part_idx) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double my_c = pinf();
    unsigned long long my_i = ~0ULL;
    if (i < n) {
        double p = pbc[i];
        const double c = cost[i];
        if (c < p) {
            p = c;
            pbc[i] = c;
            for (int d = 0; d < dim; ++d) pb[i * dim + d] = x[i * dim + d];
        }
        my_c = p;
        my_i = i;
    }
    __shared__ double sc[kGThreads / 32];
    __shared__ unsigned long long si[kGThreads / 32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double oc = __shfl_down_sync(0xFFFFFFFFu, my_c, off);
        const unsigned long long oi = __shfl_down_sync(0xFFFFFFFFu, my_i, off);
        if (better(oc, oi, my_c, my_i)) {
            my_c = oc;
            my_i = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sc[threadIdx.x >> 5] = my_c;
        si[threadIdx.x >> 5] = my_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kGThreads / 32; ++k)
            if (better(sc[k], si[k], my_c, my_i)) {
                my_c = sc[k];
                my_i = si[k];
            }
        part_cost[blockIdx.x] = my_c;
        part_idx[blockIdx.x] = my_i;
    }
}

// Global best (pso.cpp:90-96): the lowest (cost, index) over the block
// minima replaces the best only when strictly better.  One block.
__global__ void __launch_bounds__(kGThreads) gswarm_gbest_kernel(unsigned n_parts, int dim,
                                                                 const double* __restrict__ part_cost,
                                                                 const unsigned long long* __restrict__ part_idx,
                                                                 const double* __restrict__ pb,
                                                                 double* __restrict__ best,
                                                                 double* __restrict__ best_cost) {
    double my_c = pinf();
    unsigned long long my_i = ~0ULL;
    for (unsigned k = threadIdx.x; k < n_parts; k += blockDim.x)
        if (better(part_cost[k], part_idx[k], my_c, my_i)) {
            my_c = part_cost[k];
            my_i = part_idx[k];
        }
    __shared__ double sc[kGThreads];
    __shared__ unsigned long long si[kGThreads];
    sc[threadIdx.x] = my_c;
    si[threadIdx.x] = my_i;
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (unsigned k = 1; k < blockDim.x; ++k)
        if (better(sc[k], si[k], my_c, my_i)) {
            my_c = sc[k];
            my_i = si[k];
        }
    if (my_c < *best_cost) {
        *best_cost = my_c;
        for (int d = 0; d < dim; ++d) best[d] = pb[my_i * dim + d];
    }
}

// Swarm::move_particles (pso.cpp:103-127): per dimension r1 then r2 (always
// both), vel = w*v + (c1*r1)*(pbest - x) [+ (c2*r2)*(best - x)], clamp,
// repair.  `pos` = values drawn per engine before this move.
__global__ void __launch_bounds__(kGThreads) gswarm_move_kernel(size_t n, int dim, uint64_t pos, double w, double c1,
                                                                double c2, const double* __restrict__ lo,
                                                                const double* __restrict__ hi,
                                                                const double* __restrict__ best,
                                                                const double* __restrict__ best_cost, int repair,
                                                                uint64_t* __restrict__ mt, double* __restrict__ x,
                                                                double* __restrict__ v, const double* __restrict__ pb) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool have_best = *best_cost < pinf();
    uint64_t* const e = mt + pblock_base(i, kMtN);
    double* const xi = x + i * dim;
    for (int d = 0; d < dim; ++d) {
        const double r1 = gdraw(e, pos++);
        const double r2 = gdraw(e, pos++);
        const double xd = xi[d];
        double vel = dadd(dmul(w, v[i * dim + d]), dmul(dmul(c1, r1), dsub(pb[i * dim + d], xd)));
        if (have_best) vel = dadd(vel, dmul(dmul(c2, r2), dsub(best[d], xd)));
        v[i * dim + d] = vel;
        xi[d] = std_clamp(dadd(xd, vel), lo[d], hi[d]);
    }
    if (repair) repair_order(xi);
}

// objective_value (objectives.cpp:95-120) of stored trajectories, or
// metric_value (objectives.cpp:72-81) of given series: per item and
// compartment the reference's sequential accumulation over every day,
// IEEE operations in its order.  states: item k, day d, component c at
// states[(k * n_days + d) * 4 + c]; obs: n_days ObsDay (I, R, D), shared by
// all items (obs_stride 0) or one block per item.
__global__ void __launch_bounds__(128) score_kernel(int family, int metric, const ObsDay* __restrict__ obs,
                                                    size_t obs_stride, const double* __restrict__ scale3,
                                                    const double* __restrict__ states,
                                                    const unsigned char* __restrict__ finite, size_t n, int n_days,
                                                    double* __restrict__ out) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (finite && !finite[k]) {  // objectives.cpp:101-103
        out[k] = pinf();
        return;
    }
    const ObsDay* o = obs + k * obs_stride;
    const double* st = states + k * static_cast<size_t>(n_days) * 4;
    double worst = 0.0;
    for (int c = (family == kFamD ? 2 : 0); c < 3; ++c) {
        double acc = 0.0;
        double kept = 0.0;
        const double s = family == kFamD ? 1.0 : scale3[c];  // metric_value scales by 1.0
        for (int d = 0; d < n_days; ++d) {
            const double y = o[d].v[c];
            const double p = st[4 * d + 1 + c];
            if (metric == kMetMAPE) {
                if (y == 0.0) continue;
                acc = dadd(acc, fabs(ddiv(dsub(y, p), y)));
                kept = dadd(kept, 1.0);
                continue;
            }
            const double e = dmul(dsub(y, p), s);
            if (metric == kMetMXSE) acc = std_max(acc, dmul(e, e));
            else if (metric == kMetMSE) acc = dadd(acc, dmul(e, e));
            else acc = dadd(acc, fabs(e));
        }
        double v;
        if (metric == kMetMAPE) v = kept == 0.0 ? pinf() : ddiv(dmul(100.0, acc), kept);
        else if (metric == kMetMSE || metric == kMetMAE) v = ddiv(acc, static_cast<double>(n_days));
        else v = acc;
        worst = (family == kFamD || c == 0) ? v : std_max(worst, v);  // objectives.cpp:116-119
    }
    out[k] = worst;
}

// sird_rhs (model.cpp:66-74): inf = ((beta / N) * S) * I.
__global__ void rhs_kernel(const sg_state* __restrict__ s, const double* __restrict__ beta,
                           const double* __restrict__ gamma, const double* __restrict__ mu, double population,
                           size_t n, sg_state* __restrict__ out) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double inf = dmul(dmul(ddiv(beta[k], population), s[k].S), s[k].I);
    const double gI = dmul(gamma[k], s[k].I);
    const double mI = dmul(mu[k], s[k].I);
    out[k] = sg_state{-inf, dsub(dsub(inf, gI), mI), gI, mI};
}

}  // namespace
}  // namespace sirdgpu

struct sg_gswarm {
    sg_ctx* ctx = nullptr;
    size_t n = 0;
    int dim = 0;
    double w = 0, c1 = 0, c2 = 0;
    int repair = 0;
    uint64_t drawn = 0;  // values drawn per engine so far (uniform over the swarm)
    unsigned n_blocks = 0;
    double *x = nullptr, *v = nullptr, *pb = nullptr, *pbc = nullptr, *cost = nullptr;
    double *lo = nullptr, *hi = nullptr, *best = nullptr, *best_cost = nullptr, *part_cost = nullptr;
    unsigned long long* part_idx = nullptr;
    uint64_t* mt = nullptr;
    DevBufs bufs;
};

extern "C" {

int sg_gswarm_create(sg_ctx* ctx, int dim, const double* lower, const double* upper, uint64_t n_particles,
                     double inertia, double cognitive, double social, uint64_t seed, int repair_time_order,
                     sg_gswarm** out) {
    if (!ctx || !out) return SG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    // PsoConfig::validate / SearchBounds::validate (pso.cpp:16-34)
    if (n_particles == 0) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "pso: n_particles and max_iters must be positive");
    if (!std::isfinite(inertia) || !std::isfinite(cognitive) || !std::isfinite(social))
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "pso: coefficients must be finite");
    if (dim < 1 || !lower || !upper)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "pso: bounds must be non-empty and of equal dimension");
    for (int d = 0; d < dim; ++d)
        if (!std::isfinite(lower[d]) || !std::isfinite(upper[d]) || lower[d] > upper[d])
            return fail(ctx, SG_ERR_INVALID_ARGUMENT, "pso: bound " + std::to_string(d) + " is invalid");
    if (repair_time_order && dim < 4)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "repair_time_order needs positions of at least 4 dimensions");
    SG_ENTRY(ctx, "sg_gswarm_create");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    sg_gswarm* s = new (std::nothrow) sg_gswarm;
    if (!s) return fail(ctx, SG_ERR_OUT_OF_MEMORY, "host allocation failed");
    s->ctx = ctx;
    s->n = n_particles;
    s->dim = dim;
    s->w = inertia;
    s->c1 = cognitive;
    s->c2 = social;
    s->repair = repair_time_order ? 1 : 0;
    s->n_blocks = static_cast<unsigned>((n_particles + kGThreads - 1) / kGThreads);
    DevBufs& b = s->bufs;
    b.st = ctx->stream;
    const size_t nd = n_particles * static_cast<size_t>(dim);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = b.alloc(&s->x, nd);
    if (e == cudaSuccess) e = b.alloc(&s->v, nd);
    if (e == cudaSuccess) e = b.alloc(&s->pb, nd);
    if (e == cudaSuccess) e = b.alloc(&s->pbc, n_particles);
    if (e == cudaSuccess) e = b.alloc(&s->cost, n_particles);
    if (e == cudaSuccess) e = b.alloc(&s->lo, dim);
    if (e == cudaSuccess) e = b.alloc(&s->hi, dim);
    if (e == cudaSuccess) e = b.alloc(&s->best, dim);
    if (e == cudaSuccess) e = b.alloc(&s->best_cost, 1);
    if (e == cudaSuccess) e = b.alloc(&s->part_cost, s->n_blocks);
    if (e == cudaSuccess) e = b.alloc(&s->part_idx, s->n_blocks);
    if (e == cudaSuccess) e = b.alloc(&s->mt, pblock_elems(n_particles, kMtN));
    if (e == cudaSuccess) e = copy_async(ctx, s->lo, lower, sizeof(double) * dim, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = copy_async(ctx, s->hi, upper, sizeof(double) * dim, cudaMemcpyHostToDevice, ctx->stream);
    // best_position_ = 0, best_cost_ = +inf (pso.cpp:49, 63)
    if (e == cudaSuccess) e = cudaMemsetAsync(s->best, 0, sizeof(double) * dim, ctx->stream);
    const double inf = HUGE_VAL;
    if (e == cudaSuccess) e = copy_async(ctx, s->best_cost, &inf, sizeof inf, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        gswarm_init_kernel<<<s->n_blocks, kGThreads, 0, ctx->stream>>>(n_particles, dim, s->lo, s->hi, seed, s->repair,
                                                                       s->mt, s->x, s->v, s->pb, s->pbc);
        ctx->launches += 1;
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // the host `inf` goes out of scope
    if (e != cudaSuccess) {
        delete s;
        return cuda_fail(ctx, e, "sg_gswarm_create");
    }
    s->drawn = static_cast<uint64_t>(dim);
    *out = s;
    return SG_OK;
}

void sg_gswarm_destroy(sg_gswarm* s) {
    if (!s) return;
    CtxLock lock(s->ctx->mu);
    delete s;
}

const double* sg_gswarm_positions_device(const sg_gswarm* s) { return s ? s->x : nullptr; }
double* sg_gswarm_costs_device(sg_gswarm* s) { return s ? s->cost : nullptr; }

int sg_gswarm_get_positions(sg_gswarm* s, double* positions) {
    if (!s || !positions) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = s->ctx;
    SG_ENTRY(ctx, "sg_gswarm_get_positions");
    SG_CUDA(ctx, copy_async(ctx, positions, s->x, sizeof(double) * s->n * s->dim, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_gswarm_set_positions(sg_gswarm* s, const double* positions) {
    if (!s || !positions) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = s->ctx;
    SG_ENTRY(ctx, "sg_gswarm_set_positions");
    SG_CUDA(ctx, copy_async(ctx, s->x, positions, sizeof(double) * s->n * s->dim, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_gswarm_set_initial_positions(sg_gswarm* s, const double* positions) {
    // after a host repair hook at construction: pbest = the repaired positions (pso.cpp:70-74)
    const int rc = sg_gswarm_set_positions(s, positions);
    if (rc) return rc;
    sg_ctx* ctx = s->ctx;
    SG_ENTRY(ctx, "sg_gswarm_set_initial_positions");
    SG_CUDA(ctx, cudaMemcpyAsync(s->pb, s->x, sizeof(double) * s->n * s->dim, cudaMemcpyDeviceToDevice, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_gswarm_set_costs(sg_gswarm* s, const double* costs) {
    if (!s || !costs) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = s->ctx;
    SG_ENTRY(ctx, "sg_gswarm_set_costs");
    SG_CUDA(ctx, copy_async(ctx, s->cost, costs, sizeof(double) * s->n, cudaMemcpyHostToDevice, ctx->stream));
    return SG_OK;
}

int sg_gswarm_eval_window(sg_gswarm* s, sg_window* w) {
    if (!s || !w) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = s->ctx;
    if (s->dim != 6) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "window objective expects 6-dim positions");
    if (w->ctx != ctx) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "window belongs to another context");
    SG_ENTRY(ctx, "sg_gswarm_eval_window");
    return sg_eval_costs_device(w, s->x, s->n, s->cost, ctx->stream);
}

int sg_gswarm_step(sg_gswarm* s, double* best_cost) {
    if (!s) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = s->ctx;
    SG_ENTRY(ctx, "sg_gswarm_step");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    gswarm_pbest_kernel<<<s->n_blocks, kGThreads, 0, st>>>(s->n, s->dim, s->cost, s->x, s->pb, s->pbc, s->part_cost,
                                                           s->part_idx);
    gswarm_gbest_kernel<<<1, kGThreads, 0, st>>>(s->n_blocks, s->dim, s->part_cost, s->part_idx, s->pb, s->best,
                                                 s->best_cost);
    gswarm_move_kernel<<<s->n_blocks, kGThreads, 0, st>>>(s->n, s->dim, s->drawn, s->w, s->c1, s->c2, s->lo, s->hi,
                                                          s->best, s->best_cost, s->repair, s->mt, s->x, s->v, s->pb);
    ctx->launches += 3;
    SG_CUDA(ctx, cudaGetLastError());
    s->drawn += 2 * static_cast<uint64_t>(s->dim);
    if (best_cost) {
        SG_CUDA(ctx, copy_async(ctx, best_cost, s->best_cost, sizeof(double), cudaMemcpyDeviceToHost, st));
        SG_CUDA(ctx, cudaStreamSynchronize(st));
    }
    return SG_OK;
}

int sg_gswarm_best(sg_gswarm* s, double* best_position, double* best_cost) {
    if (!s || !best_position || !best_cost) return SG_ERR_INVALID_ARGUMENT;
    sg_ctx* ctx = s->ctx;
    SG_ENTRY(ctx, "sg_gswarm_best");
    SG_CUDA(ctx, copy_async(ctx, best_position, s->best, sizeof(double) * s->dim, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, best_cost, s->best_cost, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_objective_values(sg_ctx* ctx, int family, int metric, const double* infectious, const double* recovered_cum,
                        const double* deaths_cum, size_t n_days, const double* states, const uint8_t* finite, size_t n,
                        double* costs) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if ((family != SG_FAMILY_D_ONLY && family != SG_FAMILY_IRD_JOINT) || metric < SG_METRIC_MXSE ||
        metric > SG_METRIC_MAPE)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "unknown objective spec");
    if (n_days == 0) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "objective_value: observed and predicted must cover the same days");
    if (n == 0) return SG_OK;
    if (!infectious || !recovered_cum || !deaths_cum || !states || !costs)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_objective_values");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    const double* series[3] = {infectious, recovered_cum, deaths_cum};
    std::vector<ObsDay> obs(n_days);
    double scale[3] = {1.0, 1.0, 1.0};
    for (int c = 0; c < 3; ++c) {
        for (size_t d = 0; d < n_days; ++d) obs[d].v[c] = series[c][d];
        if (family == SG_FAMILY_IRD_JOINT && metric != SG_METRIC_MAPE) {
            // compartment_cost (objectives.cpp:61-69): the same std::minmax_element
            const auto [lo, hi] = std::minmax_element(series[c], series[c] + n_days);
            const double range = *hi - *lo;
            scale[c] = range > 0.0 ? 1.0 / range : 1.0 / std::max(1.0, std::fabs(*lo));
        }
    }
    DevBufs b;
    b.st = ctx->stream;
    ObsDay* d_obs;
    double *d_states, *d_costs, *d_scale;
    unsigned char* d_fin = nullptr;
    SG_CUDA(ctx, b.alloc(&d_obs, n_days));
    SG_CUDA(ctx, b.alloc(&d_states, n * n_days * 4));
    SG_CUDA(ctx, b.alloc(&d_costs, n));
    SG_CUDA(ctx, b.alloc(&d_scale, 3));
    SG_CUDA(ctx, copy_async(ctx, d_obs, obs.data(), sizeof(ObsDay) * n_days, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_states, states, sizeof(double) * n * n_days * 4, cudaMemcpyHostToDevice,
                            ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_scale, scale, sizeof scale, cudaMemcpyHostToDevice, ctx->stream));
    if (finite) {
        SG_CUDA(ctx, b.alloc(&d_fin, n));
        SG_CUDA(ctx, copy_async(ctx, d_fin, finite, n, cudaMemcpyHostToDevice, ctx->stream));
    }
    score_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(
        family, metric, d_obs, 0, d_scale, d_states, d_fin, n, static_cast<int>(n_days), d_costs);
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    SG_CUDA(ctx, copy_async(ctx, costs, d_costs, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host staging goes out of scope
    return SG_OK;
}

int sg_metric_values(sg_ctx* ctx, int metric, const double* observed, const double* predicted, size_t n_days,
                     size_t n, double* out) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (metric < SG_METRIC_MXSE || metric > SG_METRIC_MAPE)
        return fail(ctx, SG_ERR_INVALID_ARGUMENT, "unknown objective metric");
    if (n_days == 0) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "metric_value: series must be non-empty and of equal length");
    if (n == 0) return SG_OK;
    if (!observed || !predicted || !out) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_metric_values");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    // the series as the D column of observation days / trajectory states
    std::vector<ObsDay> obs(n * n_days);
    std::vector<double> st(n * n_days * 4, 0.0);
    for (size_t k = 0; k < n * n_days; ++k) {
        obs[k] = ObsDay{{0.0, 0.0, observed[k]}};
        st[4 * k + 3] = predicted[k];
    }
    DevBufs b;
    b.st = ctx->stream;
    ObsDay* d_obs;
    double *d_states, *d_out;
    SG_CUDA(ctx, b.alloc(&d_obs, obs.size()));
    SG_CUDA(ctx, b.alloc(&d_states, st.size()));
    SG_CUDA(ctx, b.alloc(&d_out, n));
    SG_CUDA(ctx, copy_async(ctx, d_obs, obs.data(), sizeof(ObsDay) * obs.size(), cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_states, st.data(), sizeof(double) * st.size(), cudaMemcpyHostToDevice, ctx->stream));
    score_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(
        kFamD, metric, d_obs, n_days, nullptr, d_states, nullptr, n, static_cast<int>(n_days), d_out);
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    SG_CUDA(ctx, copy_async(ctx, out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

int sg_sird_rhs_batch(sg_ctx* ctx, const sg_state* states, const double* beta, const double* gamma, const double* mu,
                      double population, size_t n, sg_state* out) {
    if (!ctx) return SG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SG_OK;
    if (!states || !beta || !gamma || !mu || !out) return fail(ctx, SG_ERR_INVALID_ARGUMENT, "null host buffer");
    SG_ENTRY(ctx, "sg_sird_rhs_batch");
    SG_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBufs b;
    b.st = ctx->stream;
    sg_state *d_s, *d_out;
    double *d_b, *d_g, *d_m;
    SG_CUDA(ctx, b.alloc(&d_s, n));
    SG_CUDA(ctx, b.alloc(&d_out, n));
    SG_CUDA(ctx, b.alloc(&d_b, n));
    SG_CUDA(ctx, b.alloc(&d_g, n));
    SG_CUDA(ctx, b.alloc(&d_m, n));
    SG_CUDA(ctx, copy_async(ctx, d_s, states, sizeof(sg_state) * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_b, beta, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_g, gamma, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    SG_CUDA(ctx, copy_async(ctx, d_m, mu, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    rhs_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(d_s, d_b, d_g, d_m, population, n,
                                                                                  d_out);
    ctx->launches += 1;
    SG_CUDA(ctx, cudaGetLastError());
    SG_CUDA(ctx, copy_async(ctx, out, d_out, sizeof(sg_state) * n, cudaMemcpyDeviceToHost, ctx->stream));
    SG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SG_OK;
}

}  // extern "C"
