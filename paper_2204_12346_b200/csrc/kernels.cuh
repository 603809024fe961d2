// kernels.cuh — sm_100a kernels of the particle-window cost engine.
//
//   eval_costs_kernel     boundary 1: BatchObjective body (calibration.cpp:140-154)
//   integrate_kernel      integrate_batch / forecast_extension trajectories
//   r2_kernel             fit_window's R^2(D) of the re-integrated fits
//   pso_init_kernel       Swarm::Swarm (pso.cpp:47-75) for many swarms
//   pso_step_kernel       Swarm::step (pso.cpp:77-101) fused: move -> evaluate ->
//                         personal best -> warp argmin -> last-warp global best
//                         (two-level for swarms over 32 CTAs)
//   pso_swarm_kernel      whole optimize() of small swarms, one thread-block
//                         cluster per swarm (partials pushed into every rank's
//                         shared memory with st.async + mbarrier)
//   ens_sample_kernel,    forecast-scenario ensemble (sample in ramp-coherent
//   ens_scan/scatter,     order, score when asked, forecast; on the band path
//   ensemble_kernel       also each day's key range, finite count and
//                         histogram over predicted bins)
//   sel_*_kernel          quantile bands by order-statistic selection
//
// Layout in HBM: particle state in particle blocks (32 particles x fields,
// so each warp's access to a field is one 256 B segment and a particle's
// fields sit at immediate offsets; the MT19937-64 engines the same with 312
// words).  Windows are staged in shared memory per CTA (bulk async copies in
// the step kernel) and read as broadcasts; trajectories stay in registers.
#pragma once

#include "sird_device.cuh"

#include <cooperative_groups.h>
#include <cstring>

namespace sirdgpu {

#ifndef SG_STEP_THREADS
#define SG_STEP_THREADS 128
#endif
#ifndef SG_STEP_MIN_BLOCKS
#define SG_STEP_MIN_BLOCKS 5
#endif

constexpr int kEvalThreads = 128;
constexpr int kStepThreads = SG_STEP_THREADS;
constexpr int kNP = 1;  // particles per thread in the flat step kernel (2, interleaved, measured slower)
// pso_step_kernel evaluates slot 0 only: raising kNP needs an evaluation loop
// over the slots first, or idle slots would enter finish_step with cost 0.
static_assert(kNP == 1, "pso_step_kernel evaluates one particle per thread");
constexpr int kStepWarps = kStepThreads / 32;

// Shared-memory staging of one window: the descriptor in static shared memory,
// the substep-time tables, obs (+ robs + flags for MAPE) in the dynamic
// segment (WindowLayout).
struct SmemWindow {
    const DevWindow* w;  // shared memory
    const ObsDay* obs;
    const ObsDay* robs;
    const unsigned char* flag;
    TimeGrid tg;
};

__host__ __device__ inline int tgrid_entries(int n_days, int substeps) {
    return uses_time_table(n_days, substeps) ? (n_days - 1) * substeps : 0;
}

// Shared-memory image of a window (dynamic segment, every section 16-byte
// aligned and padded): subh[substeps] + tgrid | obs | robs | flags (MAPE).
// The device block of a window (sg_window_create) uses the same section
// sizes from its times table on, so the step kernel stages it with one bulk
// copy per section.
struct WindowLayout {
    size_t times_bytes, obs_bytes, obs, robs, flag, total;
};

__host__ __device__ inline WindowLayout window_layout(int n_days, int substeps, int metric) {
    WindowLayout L;
    L.times_bytes = (static_cast<size_t>(substeps + tgrid_entries(n_days, substeps)) * sizeof(double) + 15) & ~size_t(15);
    L.obs_bytes = (static_cast<size_t>(n_days) * sizeof(ObsDay) + 15) & ~size_t(15);
    L.obs = L.times_bytes;
    L.robs = L.obs + L.obs_bytes;
    L.flag = L.robs + L.obs_bytes;
    L.total = metric == kMetMAPE ? L.flag + ((3 * static_cast<size_t>(n_days) + 15) & ~size_t(15)) : L.robs;
    return L;
}

__host__ __device__ inline size_t smem_window_bytes(int n_days, int substeps, int metric) {
    return window_layout(n_days, substeps, metric).total;
}

// Fill subh[sub] = RN(sub*h) and, when it fits, tgrid[k] = RN(RN(day-1) +
// subh[sub]) for k = (day-1)*S + sub — the t of model.cpp:94, bit for bit.
__device__ __forceinline__ TimeGrid stage_times(double* base, int n_days, int ns, double h) {
    double* subh = base;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) subh[i] = dmul(static_cast<double>(i), h);
    const int K = tgrid_entries(n_days, ns);
    double* tgrid = subh + ns;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const int d = k / ns;
        tgrid[k] = dadd(static_cast<double>(d), dmul(static_cast<double>(k - d * ns), h));
    }
    return TimeGrid{K > 0 ? tgrid : nullptr, subh};
}

// Cooperative copy of a window into shared memory (all threads call; ends
// with a barrier), in the WindowLayout of the dynamic segment.
template <int MET, int SUB>
__device__ __forceinline__ SmemWindow stage_window(const DevWindow* __restrict__ gw, DevWindow* sdesc,
                                                   unsigned char* smem) {
    if (threadIdx.x == 0) *sdesc = *gw;
    const int n = gw->n_days;
    const int ns = gw->substeps;
    const WindowLayout L = window_layout(n, ns, MET);
    double* times = reinterpret_cast<double*>(smem);
    ObsDay* obs = reinterpret_cast<ObsDay*>(smem + L.obs);
    ObsDay* robs = reinterpret_cast<ObsDay*>(smem + L.robs);
    unsigned char* flag = smem + L.flag;
    const double* src = reinterpret_cast<const double*>(gw->obs);
    double* dst = reinterpret_cast<double*>(obs);
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) dst[i] = src[i];
    TimeGrid tg;
    if (gw->times) {
        // Copy the host-built table (16-byte vectors; both ends 16-aligned).
        const int m = ns + tgrid_entries(n, ns);
        const double2* s2 = reinterpret_cast<const double2*>(gw->times);
        double2* d2 = reinterpret_cast<double2*>(times);
        for (int i = threadIdx.x; i < (m >> 1); i += blockDim.x) d2[i] = __ldg(s2 + i);
        if ((m & 1) && threadIdx.x == 0) times[m - 1] = gw->times[m - 1];
        tg = TimeGrid{m > ns ? times + ns : nullptr, times};
    } else {
        tg = stage_times(times, n, ns, gw->h);
    }
    if (MET == kMetMAPE) {
        const double* rsrc = reinterpret_cast<const double*>(gw->robs);
        double* rdst = reinterpret_cast<double*>(robs);
        for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) rdst[i] = rsrc[i];
        for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) flag[i] = gw->obs_flag[i];
    }
    __syncthreads();
    return SmemWindow{sdesc, obs, robs, flag, tg};
}

// Dynamic shared memory a kernel specialisation needs for a window.
__host__ __device__ inline size_t kernel_smem_bytes(int n_days, int substeps, int metric, bool fast) {
    (void)fast;
    return smem_window_bytes(n_days, substeps, metric);
}

// ---- boundary 1 -------------------------------------------------------------
// positions: row-major n x 6 (the BatchObjective layout, pso.hpp:33-37).
template <int FAM, int MET, int SUB>
__global__ void __launch_bounds__(kEvalThreads, 5) eval_costs_kernel(const DevWindow* __restrict__ win,
                                                                  const double* __restrict__ positions, size_t n,
                                                                  double* __restrict__ costs) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ DevWindow sdesc;
    const SmemWindow sw = stage_window<MET, SUB>(win, &sdesc, smem);
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double x[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) x[d] = positions[6 * k + d];
    costs[k] = eval_particle<FAM, MET, SUB>(x, *sw.w, sw.tg, sw.obs, sw.robs, sw.flag);
}

// ---- trajectories -------------------------------------------------------------
struct StoreSink {
    double* out;  // n_days x 4 for this item
    __device__ __forceinline__ void day(int d, double S, double I, double R, double D) {
        const bool fin = all_finite(S, I, R, D);
        const double nan = __longlong_as_double(0x7FF8000000000000LL);
        out[4 * d + 0] = fin ? S : nan;
        out[4 * d + 1] = fin ? I : nan;
        out[4 * d + 2] = fin ? R : nan;
        out[4 * d + 3] = fin ? D : nan;
    }
};

// integrate_euler (model.cpp:76-107) per item.  params row-major n x 6;
// init: one state (init_stride 0) or one per item (init_stride 4);
// hold_beta2: forecast_extension's held parameters {b2, b2, 0, 0, g, mu}
// (calibration.cpp:305-312).  states: n x n_days x 4, NaN after a blow-up.
template <int SUB>
__global__ void __launch_bounds__(kEvalThreads) integrate_kernel(DevWindow w, const double* __restrict__ params,
                                                                 const double* __restrict__ init, int init_stride,
                                                                 int hold_beta2, size_t n,
                                                                 double* __restrict__ states,
                                                                 unsigned char* __restrict__ finite) {
    extern __shared__ __align__(16) unsigned char smem[];
    const TimeGrid tg = stage_times(reinterpret_cast<double*>(smem), w.n_days, w.substeps, w.h);
    __syncthreads();
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double* p = params + 6 * k;
    const double* s0 = init + init_stride * k;
    double S = s0[0], I = s0[1], R = s0[2], D = s0[3];
    StoreSink sink{states + k * static_cast<size_t>(w.n_days) * 4};
    sink.out[0] = S;  // day 0 is the initial state, bit for bit (model.cpp:85)
    sink.out[1] = I;
    sink.out[2] = R;
    sink.out[3] = D;
    const bool init_ok = isfinite(dadd(dadd(dadd(S, I), R), D));  // SirdState::total (model.hpp:31)
    if (!init_ok) {
        const double nan = __longlong_as_double(0x7FF8000000000000LL);
        for (int d = 1; d < w.n_days; ++d)
            for (int c = 0; c < 4; ++c) sink.out[4 * d + c] = nan;
        finite[k] = 0;
        return;
    }
    const Particle part = hold_beta2 ? make_particle(p[1], p[1], 0.0, 0.0, p[4], p[5], w)
                                     : make_particle(p[0], p[1], p[2], p[3], p[4], p[5], w);
    integrate_days<SUB>(part, w, tg, S, I, R, D, sink);
    finite[k] = all_finite(S, I, R, D) ? 1 : 0;
}

// ---- particle swarm ---------------------------------------------------------------

// One swarm as the kernels see it (pso.hpp:14-32 config + bounds).
struct alignas(16) DevSwarm {  // bounds and coefficients first: 16-byte vector loads
    double lo[6], hi[6];
    double w, c1, c2;    // w, c1 adjacent and 16-byte aligned
    uint64_t seed;
    uint64_t n;          // particles
    uint64_t offset;     // first particle in the flattened SoA planes
    uint64_t max_iters;
    uint32_t cta_begin;  // first CTA of this swarm in pso_step_kernel's grid
    uint32_t n_ctas;
    int window;          // index into the window table
    int repair;          // repair_time_order hook (calibration.cpp:89-93)
    uint32_t group_begin;  // first fold group of this swarm (kFoldGroupCtas CTAs each)
    uint32_t n_groups;     // 1: the last warp folds every warp partial itself
};

// Swarms of more than kFoldGroupCtas CTAs fold their warp minima in two
// levels: the last warp of each group of CTAs folds the group's warps, the
// last group folds the groups (C3: 32768 warp partials would otherwise be
// read by one warp on the critical path of every iteration).
constexpr uint32_t kFoldGroupCtas = 32;

// Swarm-global state updated by the last CTA of every iteration.
struct DevSwarmState {
    double best_cost;    // Swarm::best_cost_ (pso.cpp:49, +inf initially)
    double best[6];      // Swarm::best_position_ (0 initially, pso.cpp:63)
    unsigned int arrived;
    unsigned int pad;
    unsigned long long ramp_substeps;  // telemetry: ramp substeps evaluated (roofline op count)
};

// Particle-block layout: particles come in blocks of 32 (one warp's worth);
// a block stores each field's 32 values contiguously, so a warp's access to
// one field is one 256-byte segment and every field of a particle sits at a
// compile-time offset (field * 32 elements) from the particle's base.
__host__ __device__ __forceinline__ size_t pblock_base(size_t p, int fields) {
    return (p >> 5) * (32 * static_cast<size_t>(fields)) + (p & 31);
}
__host__ __device__ inline size_t pblock_elems(size_t n, int fields) {
    return (n + 31) / 32 * 32 * static_cast<size_t>(fields);
}

struct PsoPlanes {
    double* x;           // particle blocks of 6 fields (pblock_base(p, 6) + d*32)
    double* v;
    double* pb;
    double* pbc;         // personal-best cost (the last evaluated costs never leave registers)
    uint64_t* mt;        // particle blocks of 312 engine words (pblock_base(p, 312) + w*32)
    size_t stride;       // total particles (plane length)
    double* part_cost;   // per warp of the step kernel
    unsigned long long* part_idx;
    double* gpart_cost;  // per fold group (swarms of n_groups > 1)
    unsigned long long* gpart_idx;
    unsigned int* group_arrived;  // per fold group: warps arrived this iteration
    double* history;     // per swarm, max_iters_max entries
    uint64_t hist_stride;
};

__device__ __forceinline__ void repair_order(double* x) {  // calibration.cpp:89-93
    if (x[2] > x[3]) {
        const double t = x[2];
        x[2] = x[3];
        x[3] = t;
    }
}

// std::clamp(v, lo, hi) == std::min(std::max(v, lo), hi) (stl_algo.h:3667-3670)
__device__ __forceinline__ double std_clamp(double v, double lo, double hi) {
    const double m = v < lo ? lo : v;
    return hi < m ? hi : m;
}

// Swarm::Swarm (pso.cpp:47-75) for particle i of a swarm (slot p):
// engine i = mt19937_64(mix_seed(seed, i)); x[d] = lo[d] + u*(hi[d]-lo[d])
// for d = 0..5 in order; repair; v = 0; pbest = x; pbest cost = +inf.
__device__ __forceinline__ void init_particle(const DevSwarm& sw, const PsoPlanes& P, size_t p, uint64_t i) {
    // seed: mt[0] = seed; mt[j] = f*(mt[j-1] ^ (mt[j-1] >> 62)) + j
    uint64_t* const mt = P.mt + pblock_base(p, kMtN);
    uint64_t m = mix_seed(sw.seed, i);
    mt[0] = m;
    for (int j = 1; j < kMtN; ++j) {
        m = kMtF * (m ^ (m >> 62)) + static_cast<uint64_t>(j);
        mt[32 * j] = m;
    }
    double u[6];
    mt_draw<6>(mt, 0, u);  // words 0..5 of the first generation
    double x[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) x[d] = dadd(sw.lo[d], dmul(u[d], dsub(sw.hi[d], sw.lo[d])));
    if (sw.repair) repair_order(x);
    const size_t b = pblock_base(p, 6);
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        P.x[b + 32 * d] = x[d];
        P.v[b + 32 * d] = 0.0;
        P.pb[b + 32 * d] = x[d];
    }
    P.pbc[p] = __longlong_as_double(0x7FF0000000000000LL);
}

#ifndef SG_FAMILY_TU  // engine.cu only (family.cu holds the templated kernels)
__global__ void __launch_bounds__(kStepThreads) pso_init_kernel(const DevSwarm* __restrict__ swarms,
                                                                const uint32_t* __restrict__ cta_swarm,
                                                                PsoPlanes P, DevSwarmState* __restrict__ state) {
    const int s = static_cast<int>(cta_swarm[blockIdx.x]);
    const DevSwarm& sw = swarms[s];
    const uint64_t first = static_cast<uint64_t>(blockIdx.x - sw.cta_begin) * blockDim.x * kNP;
    if (first + threadIdx.x == 0) {
        state[s].best_cost = __longlong_as_double(0x7FF0000000000000LL);
        for (int d = 0; d < 6; ++d) state[s].best[d] = 0.0;
        state[s].arrived = 0;
        state[s].ramp_substeps = 0;
    }
    for (int q = 0; q < kNP; ++q) {
        const uint64_t i = first + static_cast<uint64_t>(q) * blockDim.x + threadIdx.x;
        if (i < sw.n) init_particle(sw, P, sw.offset + i, i);
    }
}

#endif  // SG_FAMILY_TU

// (cost, index) ordering of the global-best scan (pso.cpp:90-96): the lowest
// cost wins, ties go to the lowest index; NaN never wins (pbest costs are never
// NaN: pbest only takes a cost that compared less, pso.cpp:84).
__device__ __forceinline__ bool better(double ca, unsigned long long ia, double cb, unsigned long long ib) {
    return ca < cb || (ca == cb && ia < ib);
}

// Swarm::move_particles for one particle (pso.cpp:103-127): 12 draws of the
// particle's engine (r1, r2 per dimension, always both), velocity and
// clamped position update, repair.  Reads the global best published after
// iteration it-1 and writes x, v; returns the new position in x.
__device__ __forceinline__ void move_particle(const DevSwarm& sw, double best_cost, const double* best,
                                              const PsoPlanes& P, size_t p, uint64_t it, double* x) {
    const bool have_best = best_cost < __longlong_as_double(0x7FF0000000000000LL);  // pso.cpp:106
    double lo[6], hi[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // 16-byte loads of the swarm's bounds
        const double2 l = reinterpret_cast<const double2*>(sw.lo)[k];
        const double2 h = reinterpret_cast<const double2*>(sw.hi)[k];
        lo[2 * k] = l.x;
        lo[2 * k + 1] = l.y;
        hi[2 * k] = h.x;
        hi[2 * k + 1] = h.y;
    }
    const double2 wc1 = *reinterpret_cast<const double2*>(&sw.w);
    double u[12];
    mt_draw<12>(P.mt + pblock_base(p, kMtN), move_draw_word(it), u);
    double* const vb = P.v + pblock_base(p, 6);
    const double* const pbb = P.pb + pblock_base(p, 6);
    double* const xb = P.x + pblock_base(p, 6);
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        const double r1 = u[2 * d];
        const double r2 = u[2 * d + 1];
        const double vd = vb[32 * d];
        const double pbd = pbb[32 * d];
        // vel = w*v + (c1*r1)*(pbest - x)   (pso.cpp:116)
        double vel = dadd(dmul(wc1.x, vd), dmul(dmul(wc1.y, r1), dsub(pbd, x[d])));
        if (have_best) vel = dadd(vel, dmul(dmul(sw.c2, r2), dsub(best[d], x[d])));  // pso.cpp:117-119
        vb[32 * d] = vel;
        x[d] = std_clamp(dadd(x[d], vel), lo[d], hi[d]);  // pso.cpp:121
    }
    if (sw.repair) repair_order(x);  // pso.cpp:123-125
#pragma unroll
    for (int d = 0; d < 6; ++d) xb[32 * d] = x[d];
}

// move_particle on register-resident state (the persistent cluster kernel):
// u holds the 12 draws of this move, drawn ahead of time.
__device__ __forceinline__ void move_particle_regs(const DevSwarm& sw, double best_cost, const double* best,
                                                   const double* u, double* x, double* v, const double* pb) {
    const bool have_best = best_cost < __longlong_as_double(0x7FF0000000000000LL);  // pso.cpp:106
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        double vel = dadd(dmul(sw.w, v[d]), dmul(dmul(sw.c1, u[2 * d]), dsub(pb[d], x[d])));  // pso.cpp:116
        if (have_best) vel = dadd(vel, dmul(dmul(sw.c2, u[2 * d + 1]), dsub(best[d], x[d])));  // pso.cpp:117-119
        v[d] = vel;
        x[d] = std_clamp(dadd(x[d], vel), sw.lo[d], sw.hi[d]);  // pso.cpp:121
    }
    if (sw.repair) repair_order(x);  // pso.cpp:123-125
}

// Personal best (pso.cpp:83-89), warp argmin of personal-best costs (lowest
// particle index on ties), and — in the last warp of the swarm to arrive —
// the global-best scan (pso.cpp:90-96) over the warp minima plus
// cost_history[it].  (cost, index) order makes the parallel fold equal the
// sequential lowest-index scan.  No CTA-wide barrier: warps retire on their own.
template <int NPT>
__device__ __forceinline__ void finish_step(const DevSwarm& sw, DevSwarmState& st, const PsoPlanes& P, int s,
                                            const bool* active, const size_t* p, const uint64_t* i, const double* c,
                                            const double (*x)[6], const double* pbc_in, uint32_t wslot, uint64_t it,
                                            const int* ramp) {
    unsigned int my_ramp = 0;
#pragma unroll
    for (int q = 0; q < NPT; ++q) my_ramp += active[q] ? static_cast<unsigned int>(ramp[q]) : 0u;
    const unsigned int wramp = __reduce_add_sync(0xFFFFFFFFu, my_ramp);
    if ((threadIdx.x & 31) == 0 && wramp) atomicAdd(&st.ramp_substeps, static_cast<unsigned long long>(wramp));
    double my_c = __longlong_as_double(0x7FF0000000000000LL);
    unsigned long long my_i = ~0ULL;
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
        if (!active[q]) continue;
        double pbc = pbc_in[q];
        if (c[q] < pbc) {
            pbc = c[q];
            P.pbc[p[q]] = c[q];
#pragma unroll
            for (int d = 0; d < 6; ++d) P.pb[pblock_base(p[q], 6) + 32 * d] = x[q][d];  // the position just evaluated
        }
        if (better(pbc, i[q], my_c, my_i)) {
            my_c = pbc;
            my_i = i[q];
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double oc = __shfl_down_sync(0xFFFFFFFFu, my_c, off);
        const unsigned long long oi = __shfl_down_sync(0xFFFFFFFFu, my_i, off);
        if (better(oc, oi, my_c, my_i)) {
            my_c = oc;
            my_i = oi;
        }
    }
    const int lane = threadIdx.x & 31;
    const uint32_t n_wslots = sw.n_ctas * kStepWarps;
    const size_t base = static_cast<size_t>(sw.cta_begin) * kStepWarps;
    if (lane == 0) {
        P.part_cost[base + wslot] = my_c;
        P.part_idx[base + wslot] = my_i;
    }
    // Every lane's personal-best stores and lane 0's partial are ordered
    // before the arrival (release); the last warp fences before reading (acquire).
    __threadfence();
    __syncwarp();
    uint32_t fold_begin = 0, fold_n = n_wslots;  // warp partials the last warp folds
    const double* fold_cost = P.part_cost + base;
    const unsigned long long* fold_idx = P.part_idx + base;
    if (sw.n_groups > 1) {
        constexpr uint32_t kGroupWarps = kFoldGroupCtas * kStepWarps;
        const uint32_t g = wslot / kGroupWarps;
        const uint32_t g_first = g * kGroupWarps;
        const uint32_t g_n = min(kGroupWarps, n_wslots - g_first);
        unsigned int t = 0;
        if (lane == 0) t = atomicAdd(&P.group_arrived[sw.group_begin + g], 1u);
        t = __shfl_sync(0xFFFFFFFFu, t, 0);
        SG_CHECK(t < g_n);  // the counter was reset by the previous iteration's last warp, each warp arrives once
        if (t != g_n - 1) return;
        __threadfence();
        double gc = __longlong_as_double(0x7FF0000000000000LL);
        unsigned long long gi = ~0ULL;
        for (uint32_t k = lane; k < g_n; k += 32) {
            const double cc = __ldcg(&P.part_cost[base + g_first + k]);
            const unsigned long long ix = __ldcg(&P.part_idx[base + g_first + k]);
            if (better(cc, ix, gc, gi)) {
                gc = cc;
                gi = ix;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double oc = __shfl_down_sync(0xFFFFFFFFu, gc, off);
            const unsigned long long oi = __shfl_down_sync(0xFFFFFFFFu, gi, off);
            if (better(oc, oi, gc, gi)) {
                gc = oc;
                gi = oi;
            }
        }
        SG_CHECK(lane != 0 || gi < sw.n);  // lane 0 holds the fold; every group has an active particle
        if (lane == 0) {
            P.gpart_cost[sw.group_begin + g] = gc;
            P.gpart_idx[sw.group_begin + g] = gi;
            P.group_arrived[sw.group_begin + g] = 0;  // every warp of the group has arrived
        }
        __threadfence();
        __syncwarp();
        fold_begin = 0;
        fold_n = sw.n_groups;
        fold_cost = P.gpart_cost + sw.group_begin;
        fold_idx = P.gpart_idx + sw.group_begin;
    }
    unsigned int ticket = 0;
    if (lane == 0) ticket = atomicAdd(&st.arrived, 1u);
    ticket = __shfl_sync(0xFFFFFFFFu, ticket, 0);
    SG_CHECK(ticket < fold_n);
    if (ticket != fold_n - 1) return;
    __threadfence();
    double bc = __longlong_as_double(0x7FF0000000000000LL);
    unsigned long long bi = ~0ULL;
    for (uint32_t k = fold_begin + lane; k < fold_n; k += 32) {
        const double cc = __ldcg(&fold_cost[k]);
        const unsigned long long ix = __ldcg(&fold_idx[k]);
        if (better(cc, ix, bc, bi)) {
            bc = cc;
            bi = ix;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double oc = __shfl_down_sync(0xFFFFFFFFu, bc, off);
        const unsigned long long oi = __shfl_down_sync(0xFFFFFFFFu, bi, off);
        if (better(oc, oi, bc, bi)) {
            bc = oc;
            bi = oi;
        }
    }
    SG_CHECK(lane != 0 || bi < sw.n);  // lane 0 holds the fold (shfl_down)
    SG_CHECK(it < P.hist_stride);
    if (lane == 0) {
        if (bc < st.best_cost) {  // strict: an equal later cost never replaces (pso.cpp:91)
            st.best_cost = bc;
            const size_t q = sw.offset + bi;
            for (int d = 0; d < 6; ++d) st.best[d] = __ldcg(&P.pb[pblock_base(q, 6) + 32 * d]);
        }
        P.history[static_cast<size_t>(s) * P.hist_stride + it] = st.best_cost;
        st.arrived = 0;
    }
}

// One CTA's share of a step launch, resolved on the host so that a CTA
// reaches everything it needs after ONE dependent load: its swarm, its
// particle range and the window's device block (descriptor, substep times,
// observations), which the CTA stages with bulk asynchronous copies.
struct CtaTask {
    uint32_t swarm;          // index into the group's DevSwarm / DevSwarmState arrays
    uint32_t n_valid;        // particles of this CTA (<= kStepThreads * kNP)
    uint64_t p0;             // plane slot of the CTA's first particle
    uint64_t i0;             // swarm-local index of the CTA's first particle
    uint64_t max_iters;      // the swarm's iteration count
    const DevWindow* win;    // window descriptor (device)
    const double* times;     // its substep-time table (device)
    const double* obs;       // obs | robs | flags, 16-byte padded sections (device)
    uint16_t times_x16;      // staged subh + t_k table bytes / 16 (the table is at most kMaxTgrid entries)
    uint16_t substeps;       // the window's substep count when it has a t_k table (<= kMaxTgrid), else 0
    uint32_t obs_bytes;      // 24 B per day: beyond 16 bits from 2,731 days on (still inside the 200 KB window)
};
static_assert(sizeof(CtaTask) == 64, "one 64-byte record per CTA");

// ---- bulk asynchronous global -> shared copies (TMA, non-tensor) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// Address of the same shared-memory location in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 16 bytes into another CTA's shared memory, completing that many bytes of
// the transaction count of its mbarrier (no fence, no cluster barrier).
__device__ __forceinline__ void st_async_16(uint32_t raddr, uint64_t a, uint64_t b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "l"(a), "l"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    }
}

#ifndef SG_PBC_PREFETCH
#define SG_PBC_PREFETCH 0
#endif
#ifndef SG_TMA_STAGE
#define SG_TMA_STAGE 1
#endif

// Asynchronous staging of the CTA's window (specialised kernels, static
// shared arrays): thread 0 arms the barrier and issues the bulk copies; the
// caller overlaps them with the particle moves and waits with mbar_wait.
template <int MET, int SUB>
__device__ __forceinline__ SmemWindow stage_window_async(const CtaTask& t, DevWindow* sdesc, uint64_t* bar,
                                                         unsigned char* smem) {
    // WindowLayout: times | obs | robs | flags, the section sizes in the task
    double* s_times = reinterpret_cast<double*>(smem);
    const uint32_t times_bytes = 16u * t.times_x16;
    ObsDay* s_obs = reinterpret_cast<ObsDay*>(smem + times_bytes);
    ObsDay* s_robs = reinterpret_cast<ObsDay*>(smem + times_bytes + t.obs_bytes);
    unsigned char* s_flag = smem + times_bytes + 2 * t.obs_bytes;
    if (threadIdx.x == 0) {
#if SG_CHECKED
        uint32_t dyn = 0;
        asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        SG_CHECK(times_bytes + (MET == kMetMAPE ? 2u : 1u) * t.obs_bytes <= dyn);
#endif
        const uint32_t b = smem_u32(bar);
        mbar_init(b, 1);
        // obs_bytes = round16(24 n) is the obs and the robs section size
        const uint32_t flag_bytes = MET == kMetMAPE ? (3u * (t.obs_bytes / 24u) + 15u) & ~15u : 0u;
        const uint32_t n_days_bytes = t.obs_bytes;
        mbar_expect_tx(b, static_cast<uint32_t>(sizeof(DevWindow)) + times_bytes + n_days_bytes +
                              (MET == kMetMAPE ? n_days_bytes + flag_bytes : 0u));
        bulk_g2s(smem_u32(sdesc), t.win, sizeof(DevWindow), b);
        bulk_g2s(smem_u32(s_times), t.times, times_bytes, b);
        bulk_g2s(smem_u32(s_obs), t.obs, n_days_bytes, b);
        if (MET == kMetMAPE) {
            const unsigned char* o = reinterpret_cast<const unsigned char*>(t.obs);
            bulk_g2s(smem_u32(s_robs), o + n_days_bytes, n_days_bytes, b);
            bulk_g2s(smem_u32(s_flag), o + 2 * n_days_bytes, flag_bytes, b);
        }
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    // the t_k table follows subh[substeps]: a compile-time offset for SUB = 24
    // (no table for SUB = kSub24NoTable: ramp times are computed from subh)
    const double* tgrid = SubKind<SUB>::kTable ? s_times + (SUB > 0 ? static_cast<uint32_t>(SUB) : t.substeps) : nullptr;
    return SmemWindow{sdesc, s_obs, s_robs, s_flag, TimeGrid{tgrid, s_times}};
}

// One Swarm::step (pso.cpp:77-101) for every swarm, iteration `it`, fused:
// the move of iteration it-1 (which closes step it-1 in the reference), then
// evaluate, personal best, and the global-best fold.  Thread t of a swarm's
// CTA range owns particle t for all iterations.  Used for large swarms.
#if SG_CTA_TIMES
static __device__ unsigned long long g_cta_times[6 * 8192][3];
#endif

template <int FAM, int MET, int SUB>
__global__ void __launch_bounds__(kStepThreads, SG_STEP_MIN_BLOCKS)
    pso_step_kernel(const CtaTask* __restrict__ tasks, const DevSwarm* __restrict__ swarms, PsoPlanes P,
                    DevSwarmState* __restrict__ state, uint64_t it, uint32_t cta_offset) {
#if SG_CTA_TIMES
    // diagnostic build (tools/cta_times.py): globaltimer at CTA start / end and
    // the SM of every CTA of iteration SG_CTA_TIMES
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(16) DevWindow sdesc;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t cta = blockIdx.x + cta_offset;
    const CtaTask task = tasks[cta];
    if (it >= task.max_iters) return;  // CTA-uniform
    SG_CHECK(task.n_valid >= 1 && task.n_valid <= kStepThreads * kNP && task.p0 + task.n_valid <= P.stride);
    constexpr bool kAsync = SUB != 0 && SG_TMA_STAGE;
    SmemWindow win;
    if constexpr (kAsync) win = stage_window_async<MET, SUB>(task, &sdesc, &bar, smem);
    else win = stage_window<MET, SUB>(task.win, &sdesc, smem);
    const int s = static_cast<int>(task.swarm);
    const DevSwarm& sw = swarms[s];
    // Thread t owns particles i0 + q*blockDim + t, q < kNP (coalesced per q).
    uint64_t i[kNP];
    bool active[kNP];
    size_t p[kNP];
    double x[kNP][6];
    double pbc[kNP];
#pragma unroll
    for (int q = 0; q < kNP; ++q) {
        const uint32_t local = static_cast<uint32_t>(q) * blockDim.x + threadIdx.x;
        active[q] = local < task.n_valid;
        i[q] = task.i0 + local;
        p[q] = task.p0 + (active[q] ? local : 0);
        if (active[q]) {
            if (SG_PBC_PREFETCH) pbc[q] = P.pbc[p[q]];
#pragma unroll
            for (int d = 0; d < 6; ++d) x[q][d] = P.x[pblock_base(p[q], 6) + 32 * d];
            if (it > 0) move_particle(sw, state[s].best_cost, state[s].best, P, p[q], it, x[q]);
        } else {
            pbc[q] = 0.0;
#pragma unroll
            for (int d = 0; d < 6; ++d) x[q][d] = x[0][d];  // idle slot mirrors slot 0 (result unused)
        }
    }
    if constexpr (kAsync) mbar_wait(smem_u32(&bar), 0);
    if (!SG_PBC_PREFETCH) {
#pragma unroll
        for (int q = 0; q < kNP; ++q) pbc[q] = active[q] ? P.pbc[p[q]] : 0.0;
    }
    double c[kNP];
    int ramp[kNP];
#pragma unroll
    for (int q = 0; q < kNP; ++q) {
        c[q] = 0.0;
        ramp[q] = 0;
    }
    if (active[0]) c[0] = eval_particle<FAM, MET, SUB>(x[0], *win.w, win.tg, win.obs, win.robs, win.flag, &ramp[0]);
    finish_step<kNP>(sw, state[s], P, s, active, p, i, c, x, pbc,
                     (cta - sw.cta_begin) * kStepWarps + (threadIdx.x >> 5), it, ramp);
#if SG_CTA_TIMES
    __syncthreads();
    const uint64_t rec = (it - SG_CTA_TIMES) * 8192 + cta;  // iterations SG_CTA_TIMES..+5, <= 8192 CTAs each
    if (threadIdx.x == 0 && it >= SG_CTA_TIMES && it < SG_CTA_TIMES + 6 && cta < 8192) {
        unsigned long long t_end;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cta_times[rec][0] = t_start;
        g_cta_times[rec][1] = t_end;
        g_cta_times[rec][2] = smid;
    }
#endif
}

// ---- small swarms: one persistent thread-block cluster per swarm ---------------
//
// Swarms of at most kPersistMax particles (C1: 256, tests) run their whole
// optimize() (pso.cpp:129-143) in one launch: seeding, then every
// iteration's move -> evaluate -> personal best -> argmin -> global best.
// Such a plan cannot fill the GPU, so the time per iteration is the Euler
// dependency chain of one particle (6 dependent FP64 ops per substep): the
// swarm is spread over a cluster of up to 8 CTAs (one per SM, at most one
// warp per SM sub-partition) instead of stacking warps on one SM.  CTA r of
// the cluster owns particles r*blockDim + t (+ k*cluster*blockDim).  Per
// iteration each CTA folds its warps' minima into a partial (cost, index,
// personal-best position) and pushes it into every rank's shared memory
// (st.async, completing on the receiver's mbarrier); each CTA then folds the
// partials of all ranks in rank order locally, so all CTAs hold the same
// global best.  The partials and their mbarriers are double-buffered by
// iteration parity.
constexpr int kSwarmThreadsMax = 128;
constexpr int kSwarmClusterMax = 8;
constexpr int kPersistMax = kSwarmThreadsMax * kSwarmClusterMax;  // 1024 particles per swarm

#if SG_C1_PROBE
// diagnostic build (tools/c1_probe.py): per (warp of the cluster, iteration)
// clock64 stamps of the iteration's phases
static __device__ unsigned long long g_c1[8][512][6];
#define SG_C1_STAMP(k)                                                                       \
    do {                                                                                     \
        const unsigned gw = rank * (blockDim.x >> 5) + (threadIdx.x >> 5);                   \
        if ((threadIdx.x & 31) == 0 && gw < 8 && it < 512) g_c1[gw][it][k] = clock64();     \
    } while (0)
#else
#define SG_C1_STAMP(k) \
    do {               \
    } while (0)
#endif

struct SwarmPartial {
    double cost;
    unsigned long long idx;
    double pos[6];
};

template <int FAM, int MET, int SUB>
__global__ void __launch_bounds__(kSwarmThreadsMax, 1) pso_swarm_kernel(const DevSwarm* __restrict__ swarms,
                                                                     const DevWindow* __restrict__ windows,
                                                                     PsoPlanes P, DevSwarmState* __restrict__ state,
                                                                     uint32_t swarm_offset) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ DevWindow sdesc;
    __shared__ double red_c[kSwarmThreadsMax / 32];
    __shared__ unsigned long long red_i[kSwarmThreadsMax / 32];
    __shared__ double red_pos[kSwarmThreadsMax / 32][6];
    // every rank's partial of the iteration, pushed by the ranks themselves
    // (st.async); double-buffered by iteration parity, one mbarrier each
    __shared__ __align__(16) SwarmPartial part[2][kSwarmClusterMax];
    __shared__ __align__(8) uint64_t part_bar[2];
    __shared__ double gbest[6];
    __shared__ double gbest_cost;
    const unsigned rank = cluster.block_rank();
    const unsigned n_ranks = cluster.num_blocks();
    static_assert(sizeof(SwarmPartial) == 64, "a partial is four 16-byte stores");
    const int s = static_cast<int>(blockIdx.x / n_ranks + swarm_offset);
    const DevSwarm& sw = swarms[s];
    const SmemWindow win = stage_window<MET, SUB>(windows + sw.window, &sdesc, smem);
    const uint32_t n = static_cast<uint32_t>(sw.n);
    // The host sizes the cluster so that every thread owns at most one
    // particle (cluster * blockDim >= n): its state lives in registers for
    // the whole optimize() and goes back to the planes at the end.
    const uint32_t i = rank * blockDim.x + threadIdx.x;
    const bool active = i < n;
    const size_t p = sw.offset + (active ? i : 0);
    double x[6], v[6], pb[6], pbc = __longlong_as_double(0x7FF0000000000000LL), c = pbc;
    double u[12];  // the next move's draws, taken one iteration ahead
    MtBatch<12> next;  // their engine words, loaded during the evaluation
    if (active) {
        init_particle(sw, P, p, i);
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            x[d] = P.x[pblock_base(p, 6) + 32 * d];
            v[d] = 0.0;
            pb[d] = x[d];
        }
    }
    if (threadIdx.x == 0) {
        gbest_cost = __longlong_as_double(0x7FF0000000000000LL);
        for (int d = 0; d < 6; ++d) gbest[d] = 0.0;
        if (rank == 0) state[s].ramp_substeps = 0;
        mbar_init(smem_u32(&part_bar[0]), 1);  // (fence.mbarrier_init: visible to the cluster's st.async)
        mbar_init(smem_u32(&part_bar[1]), 1);
    }
    unsigned long long ramp_acc = 0;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n_warps = (blockDim.x + 31) >> 5;
    cluster.sync();  // ramp counter cleared, gbest initialised, every rank's partial mbarriers initialised
    for (uint64_t it = 0; it < sw.max_iters; ++it) {
        double my_c = __longlong_as_double(0x7FF0000000000000LL);
        unsigned long long my_i = ~0ULL;
        SG_C1_STAMP(0);
        if (active) {
            if (it > 0) move_particle_regs(sw, gbest_cost, gbest, u, x, v, pb);
            int ramp = 0;
            SG_C1_STAMP(1);
            // the next move's engine words: loads in flight during the evaluation
            if (it + 1 < sw.max_iters) mt_load<12>(P.mt + pblock_base(p, kMtN), move_draw_word(it + 1), next);
            c = eval_particle<FAM, MET, SUB>(x, *win.w, win.tg, win.obs, win.robs, win.flag, &ramp);
            SG_C1_STAMP(2);
            ramp_acc += static_cast<unsigned long long>(ramp);
            if (c < pbc) {  // pso.cpp:83-89
                pbc = c;
#pragma unroll
                for (int d = 0; d < 6; ++d) pb[d] = x[d];
            }
            my_c = pbc;
            my_i = i;
        }
        unsigned long long w_i = my_i;  // warp argmin (cost, index)
        double w_c = my_c;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double oc = __shfl_xor_sync(0xFFFFFFFFu, w_c, off);
            const unsigned long long oi = __shfl_xor_sync(0xFFFFFFFFu, w_i, off);
            if (better(oc, oi, w_c, w_i)) {
                w_c = oc;
                w_i = oi;
            }
        }
        if (active && my_i == w_i) {  // the warp's winner publishes its personal best
            red_c[warp] = w_c;
            red_i[warp] = w_i;
#pragma unroll
            for (int d = 0; d < 6; ++d) red_pos[warp][d] = pb[d];
        } else if (lane == 0 && w_i == ~0ULL) {
            red_c[warp] = w_c;
            red_i[warp] = w_i;
        }
        SG_C1_STAMP(3);
        __syncthreads();  // warp minima visible in the CTA
        const int par = static_cast<int>(it & 1);
        const uint32_t bar = smem_u32(&part_bar[par]);
        if (threadIdx.x == 0) {
            // The CTA's partial, pushed into slot `rank` of every rank's
            // part[par] (itself included); each rank's mbarrier phase
            // completes when all n_ranks partials have landed.  A rank
            // pushes iteration it+2's partial (same slots) only after it has
            // received this rank's it+1 partial, which this rank sends after
            // its fold of iteration it — so no slot is overwritten early.
            int bw = 0;
            for (int k = 1; k < n_warps; ++k)
                if (better(red_c[k], red_i[k], red_c[bw], red_i[bw])) bw = k;
            uint64_t w8[8];
            w8[0] = static_cast<uint64_t>(__double_as_longlong(red_c[bw]));
            w8[1] = red_i[bw];
            for (int d = 0; d < 6; ++d)
                w8[2 + d] = red_i[bw] != ~0ULL ? static_cast<uint64_t>(__double_as_longlong(red_pos[bw][d])) : 0ULL;
            mbar_expect_tx(bar, n_ranks * static_cast<uint32_t>(sizeof(SwarmPartial)));
            const uint32_t slot = smem_u32(&part[par][rank]);
            for (unsigned r = 0; r < n_ranks; ++r) {
                const uint32_t dst = mapa_u32(slot, r), rbar = mapa_u32(bar, r);
#pragma unroll
                for (int q = 0; q < 4; ++q) st_async_16(dst + 16 * q, w8[2 * q], w8[2 * q + 1], rbar);
            }
        }
        // the next move's draws (engine words loaded during the evaluation),
        // while the other ranks' partials are on their way
        if (active && it + 1 < sw.max_iters) mt_finish<12>(P.mt + pblock_base(p, kMtN), move_draw_word(it + 1), next, u);
        mbar_wait(bar, static_cast<uint32_t>((it >> 1) & 1));  // every rank's partial of iteration `it` here
        SG_C1_STAMP(4);
        if (threadIdx.x == 0) {
            // Global-best scan (pso.cpp:90-96) over the ranks' partials in
            // rank order: identical in every CTA.
            const SwarmPartial* best = nullptr;
            for (unsigned r = 0; r < n_ranks; ++r) {
                const SwarmPartial* q = &part[par][r];
                SG_CHECK(q->idx == ~0ULL || q->idx < n);
                if (!best || better(q->cost, q->idx, best->cost, best->idx)) best = q;
            }
            SG_CHECK(best != nullptr && best->idx < n);
            const double bc = best->cost;
            if (bc < gbest_cost) {  // strict: an equal later cost never replaces
                gbest_cost = bc;
                for (int d = 0; d < 6; ++d) gbest[d] = best->pos[d];
            }
            if (rank == 0) P.history[static_cast<size_t>(s) * P.hist_stride + it] = gbest_cost;
        }
        __syncthreads();  // global best published for the next move
        SG_C1_STAMP(5);
    }
    if (active) {  // final particle state back to the planes
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            P.x[pblock_base(p, 6) + 32 * d] = x[d];
            P.v[pblock_base(p, 6) + 32 * d] = v[d];
            P.pb[pblock_base(p, 6) + 32 * d] = pb[d];
        }
        P.pbc[p] = pbc;
    }
    // per-thread count <= iterations * 840 < 2^32 / 32
    const unsigned long long wr = __reduce_add_sync(0xFFFFFFFFu, static_cast<unsigned int>(ramp_acc));
    if (threadIdx.x == 0 && rank == 0) {
        state[s].best_cost = gbest_cost;
        for (int d = 0; d < 6; ++d) state[s].best[d] = gbest[d];
        state[s].arrived = 0;
    }
    if (lane == 0) atomicAdd(&state[s].ramp_substeps, wr);
    cluster.sync();  // no CTA leaves while a push to it may still be in flight
}

#ifndef SG_FAMILY_TU  // engine.cu only (family.cu holds the templated kernels)
// ---- R^2 of the re-integrated deaths (fit_window's finish) ------------------------
//
// r_squared_d (objectives.cpp:122-144) per fit, one thread each, with the
// reference's sequential sums: mean of the observed series, then
// ss_res += e*e and ss_tot += c*c day by day; NaN where ss_tot == 0
// (ConstantObservedError, calibration.cpp:183-185).  states: n x n_days x 4.
__global__ void r2_kernel(const double* __restrict__ states, const double* __restrict__ obs_d, size_t n, int n_days,
                          double* __restrict__ r2) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double* y = obs_d + k * static_cast<size_t>(n_days);
    const double* st = states + k * static_cast<size_t>(n_days) * 4;
    double mean = 0.0;
    for (int d = 0; d < n_days; ++d) mean = dadd(mean, y[d]);
    mean = ddiv(mean, static_cast<double>(n_days));
    double ss_res = 0.0, ss_tot = 0.0;
    for (int d = 0; d < n_days; ++d) {
        const double e = dsub(y[d], st[4 * d + 3]);
        ss_res = dadd(ss_res, dmul(e, e));
        const double c = dsub(y[d], mean);
        ss_tot = dadd(ss_tot, dmul(c, c));
    }
    r2[k] = ss_tot == 0.0 ? __longlong_as_double(0x7FF8000000000000LL) : dsub(1.0, ddiv(ss_res, ss_tot));
}

#endif  // SG_FAMILY_TU

// ---- forecast-scenario ensemble ----------------------------------------------------
// Sample k: 6 uniform01 draws of mt19937_64(mix_seed(seed, k)) mapped into the
// box like Swarm::Swarm (pso.cpp:65-72) + repair; score it on the window
// (cost), then continue `horizon` days holding beta = beta2
// (forecast_extension, calibration.cpp:305-317) and write D per forecast day.
struct ForecastDSink {
    double* out;
    size_t dstride;
    __device__ __forceinline__ void day(int d, double S, double I, double R, double D) {
        (void)S;
        (void)I;
        (void)R;
        out[d * dstride] = D;
    }
};

// Sample k of an ensemble: the first 6 draws of mt19937_64(mix_seed(seed, k))
// mapped into the box like Swarm::Swarm (pso.cpp:65-72), then repaired.
__device__ __forceinline__ void x_of_sample(const double* lo, const double* hi, uint64_t seed, size_t k, double* x) {
    double u[6];
    mt_first_uniforms<6>(mix_seed(seed, k), u);
#pragma unroll
    for (int d = 0; d < 6; ++d) x[d] = dadd(lo[d], dmul(u[d], dsub(hi[d], lo[d])));
    repair_order(x);
}

// ---- quantile bands by selection (C5): shared declarations ---------------------
//
// build_quantile_bands (calibration.cpp:337-361) needs, per forecast day, the
// count k of finite values and the order statistics at ranks lo and lo+1 of
// h = (k-1)*p for 7 probabilities — at most 14 ranks out of 10^6.  Instead of
// sorting every day column, the values are mapped to order-preserving 64-bit
// keys, bucketed into 2^12 bins over each day's key range (monotone, so rank
// intervals of bins are exact), and only the bins holding a wanted rank are
// gathered and sorted — in one CTA's shared memory, with a finer histogram
// level for a bin too full to sort there.  The order statistics are values of
// the data, so the bands are the full sort's to the bit (ties between -0 and
// +0 follow the key order, as a radix sort of the column does).
constexpr int kBandP = 7;
constexpr int kBandRanks = 2 * kBandP;  // lo and lo+1 per probability
constexpr int kSelBinBits = 12;
constexpr int kSelBins = 1 << kSelBinBits;  // per day; a CTA histogram fits in shared memory

__host__ __device__ __forceinline__ uint64_t order_key(double x) {
#ifdef __CUDA_ARCH__
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t b;
    std::memcpy(&b, &x, sizeof b);
#endif
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__device__ __forceinline__ double key_value(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

struct SelDay {                   // per forecast day, device memory
    unsigned long long kmin, kmax, count;  // finite values: key range (a superset when fused) and k
    unsigned long long base;      // bin origin of the selection: bin = (key - base) >> shift
    int shift;
    int n_seg;                    // distinct bins holding wanted ranks
    // The ensemble kernel's fused histogram (band path): bins predicted from
    // the key range the slot's previous window had, widened by half its width
    // on both sides (sel_init_kernel); values outside counted apart.  A day
    // whose wanted ranks fall outside the predicted bins takes the histogram
    // pass over its exact range instead (full = 1).
    unsigned long long pbase;
    int pshift;                   // -1: no prediction
    int full;
    unsigned long long under, over;
    uint32_t seg_bin[kBandRanks];
    uint64_t seg_rank0[kBandRanks];   // rank of the bin's first value
    uint32_t seg_count[kBandRanks];
    uint32_t seg_fill[kBandRanks];
};

__host__ __device__ __forceinline__ int sel_shift(unsigned long long range) {
#ifdef __CUDA_ARCH__
    const int bits = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
#else
    const int bits = range ? 64 - __builtin_clzll(range) : 0;
#endif
    return bits > kSelBinBits ? bits - kSelBinBits : 0;
}

// Evaluation order of an ensemble: every sample's parameters into SoA
// planes, keys[k] = a key (day of t1, day of t2, each in steps of `q` days and
// capped at 63) and keys[n + k] = its rank among the samples of that key —
// samples with equal keys ramp on the same days, so grouping them makes a
// warp's lanes ramp together (the warp pays a ramp substep if any lane
// ramps).  The order never changes a result: every sample is evaluated by
// the same code into its own slot, and the bands only need each day's
// multiset.  Fused: the key histogram of the counting sort
// (ens_scan_kernel, ens_scatter_kernel).
constexpr int kOrderKeys = 4096;
__device__ __forceinline__ void sample_into(const double* __restrict__ lo, const double* __restrict__ hi,
                                            uint64_t seed, size_t n, int q, size_t k, double* __restrict__ planes,
                                            uint32_t* __restrict__ keys, unsigned int* __restrict__ key_count) {
    auto day = [q](double t) -> uint32_t {  // NaN and negatives -> 0, capped at 63 steps
        return t > 0.0 ? static_cast<uint32_t>(fmin(floor(t), 4096.0)) / q : 0u;
    };
    double x[6];
    x_of_sample(lo, hi, seed, k, x);
#pragma unroll
    for (int d = 0; d < 6; ++d) planes[d * n + k] = x[d];
    const uint32_t key = (min(day(x[2]), 63u) << 6) | min(day(x[3]), 63u);
    keys[k] = key;
    keys[n + k] = atomicAdd(&key_count[key], 1u);  // the sample's rank within its key
}

// A later window's samples drawn by an ensemble launch (the batch band
// pipeline): its seed and order buffers; planes == nullptr for none.
struct EnsNext {
    uint64_t seed;
    double* planes;
    uint32_t* keys;
    unsigned int* key_count;
    int q;
};

#ifndef SG_FAMILY_TU  // engine.cu only (family.cu holds the templated kernels)
// Thread counts of the selection stream's kernels (ordering and band
// selection).  They run beside the FP64-bound ensemble kernel of the next
// window and take CTA slots from it as they go (the hardware dispatches a
// lower-priority grid's CTAs only once the higher one has none left to
// place, so they cannot be confined to the registers the ensemble's 5 CTAs
// leave free — measured): each is sized for its shortest
// standalone time, which is the ensemble time it costs.
constexpr int kBgThreads = 128;       // small kernels (init, scan, locate, bands)
constexpr int kSampleThreads = 256;   // ens_sample / ens_scatter / sel_range / sel_gather / sel_finish
constexpr int kHistThreads = 1024;    // sel_hist (a CTA histogram in shared memory)

__global__ void __launch_bounds__(kSampleThreads) ens_sample_kernel(const double* __restrict__ lo,
                                                                   const double* __restrict__ hi, uint64_t seed,
                                                                   size_t n, int q, double* __restrict__ planes,
                                                                   uint32_t* __restrict__ keys,
                                                                   unsigned int* __restrict__ key_count) {
    for (size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x)
        sample_into(lo, hi, seed, n, q, k, planes, keys, key_count);
}

// Exclusive scan of the kOrderKeys key counts into bucket cursors
// (key_count[kOrderKeys + key]); the counts are zeroed for the next window.
// One CTA: thread t owns 32 consecutive keys.
__global__ void __launch_bounds__(kBgThreads) ens_scan_kernel(unsigned int* __restrict__ key_count) {
    constexpr int kPer = kOrderKeys / kBgThreads;
    __shared__ unsigned int warp_base[kBgThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4* const c = reinterpret_cast<uint4*>(key_count) + threadIdx.x * (kPer / 4);
    unsigned int total = 0;
#pragma unroll
    for (int i = 0; i < kPer / 4; ++i) {
        const uint4 u = c[i];
        total += u.x + u.y + u.z + u.w;
    }
    unsigned int incl = total;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned int o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) warp_base[warp] = incl;
    __syncthreads();
    unsigned int carry = incl - total;
    for (int w = 0; w < warp; ++w) carry += warp_base[w];
    uint4* const cur = reinterpret_cast<uint4*>(key_count + kOrderKeys) + threadIdx.x * (kPer / 4);
#pragma unroll 4
    for (int i = 0; i < kPer / 4; ++i) {
        const uint4 v = c[i];
        c[i] = make_uint4(0u, 0u, 0u, 0u);
        uint4 u;
        u.x = carry;
        u.y = u.x + v.x;
        u.z = u.y + v.y;
        u.w = u.z + v.z;
        carry = u.w + v.w;
        cur[i] = u;
    }
}

// Counting-sort scatter: sample k goes to its key's bucket start plus its
// rank within the key (taken by ens_sample_kernel's count), no atomics.
__global__ void __launch_bounds__(kSampleThreads) ens_scatter_kernel(const uint32_t* __restrict__ keys, size_t n,
                                                const unsigned int* __restrict__ cursor,
                                                uint32_t* __restrict__ perm) {
    for (size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x)
        perm[cursor[keys[k]] + keys[n + k]] = static_cast<uint32_t>(k);
}

// Reset a slot's day records for its next window; with `predict`, each
// day's fused-histogram bins come from the key range the slot's previous
// window had (two windows back in the pipeline), widened by half its width
// on each side.
__global__ void __launch_bounds__(kBgThreads) sel_init_kernel(SelDay* __restrict__ days, int n_days, int predict) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_days) return;
    SelDay& sd = days[d];
    sd.pshift = -1;
    if (predict && sd.count > 0 && sd.kmax >= sd.kmin) {
        const unsigned long long half = (sd.kmax - sd.kmin) / 2;
        const unsigned long long lo = sd.kmin > half ? sd.kmin - half : 0ULL;
        const unsigned long long hi = ~0ULL - sd.kmax > half ? sd.kmax + half : ~0ULL;
        sd.pbase = lo;
        sd.pshift = sel_shift(hi - lo);
    }
    sd.kmin = ~0ULL;
    sd.kmax = 0;
    sd.count = 0;
    sd.n_seg = 0;
    sd.full = 0;
    sd.under = 0;
    sd.over = 0;
}
#endif  // SG_FAMILY_TU

// Scores nothing: the band path needs no cost per sample.
struct NullSink {
    __device__ __forceinline__ void day(int, double, double, double, double) {}
};

// The band path's forecast sink: writes the deaths row (when `on`) and
// does the selection's first two passes as the days arrive, without
// re-reading the plane:
//   * each day's key range, reduced over the warp — the top 32 bits of the
//     order key by REDUX, so the range is a superset of the exact one by
//     < 2^32 key units, which only widens the bins of a histogram pass
//     (lane d keeps day d's warp range; horizon < 32);
//   * each day's histogram over the bins predicted for it (SelDay::pbase,
//     pshift), values outside the predicted bins counted apart.
// Every lane of the warp must run the loop: the reductions name the full warp.
struct BandDSink {
    double* out;
    size_t dstride;
    bool on;          // this lane's row is written and counted
    uint32_t lo, hi;  // lane d: day d's warp range (hi32 of the keys)
    const unsigned long long* pbase;  // shared memory, per day
    const int* pshift;                // shared memory, per day (-1: no prediction)
    unsigned int* hist;               // n_days x kSelBins
    SelDay* days;
    // One value into (+1) or out of (-1, a row that blows up later) the
    // day's predicted histogram.
    __device__ __forceinline__ void count(int d, unsigned long long key, int delta) {
        const int sh = pshift[d];
        if (sh < 0) return;
        const unsigned long long base = pbase[d];
        if (key < base) {
            atomicAdd(&days[d].under, static_cast<unsigned long long>(static_cast<long long>(delta)));
        } else if (((key - base) >> sh) >= static_cast<unsigned long long>(kSelBins)) {
            atomicAdd(&days[d].over, static_cast<unsigned long long>(static_cast<long long>(delta)));
        } else {
            atomicAdd(&hist[d * kSelBins + static_cast<int>((key - base) >> sh)], static_cast<unsigned>(delta));
        }
    }
    __device__ __forceinline__ void put(int d, double D) {
        if (on) out[d * dstride] = D;
        const bool fin = on && isfinite(D);
        const unsigned long long key = order_key(D);
        if (fin) count(d, key, 1);
        const uint32_t k32 = static_cast<uint32_t>(key >> 32);
        const uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, fin ? k32 : 0xFFFFFFFFu);
        const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, fin ? k32 : 0u);
        if ((threadIdx.x & 31) == static_cast<unsigned>(d)) {
            lo = mn;
            hi = mx;
        }
    }
    __device__ __forceinline__ void day(int d, double, double, double, double D) { put(d, D); }
};

template <int FAM, int MET, int SUB>
__global__ void __launch_bounds__(kEvalThreads, 5) ensemble_kernel(const DevWindow* __restrict__ win, DevWindow fwin,
                                                                const double* __restrict__ lo,
                                                                const double* __restrict__ hi, uint64_t seed,
                                                                size_t n, int horizon, double* __restrict__ costs,
                                                                double* __restrict__ params_out,
                                                                double* __restrict__ deaths_out, size_t sstride,
                                                                size_t dstride, const uint32_t* __restrict__ perm,
                                                                const double* __restrict__ planes, int out_by_slot,
                                                                SelDay* __restrict__ days,
                                                                unsigned int* __restrict__ hist,
                                                                unsigned long long* __restrict__ ramp_count,
                                                                EnsNext next) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ DevWindow sdesc;
    __shared__ unsigned long long s_pbase[32];
    __shared__ int s_pshift[32];
    if (next.planes) {  // a later window's sample of this slot (integer work before the FP64-bound part)
        const size_t s0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        if (s0 < n) sample_into(lo, hi, next.seed, n, next.q, s0, next.planes, next.keys, next.key_count);
    }
    if (days && static_cast<int>(threadIdx.x) <= horizon) {  // the band path (horizon < 32)
        s_pbase[threadIdx.x] = days[threadIdx.x].pbase;
        s_pshift[threadIdx.x] = days[threadIdx.x].pshift;
    }
    const SmemWindow sw = stage_window<MET, SUB>(win, &sdesc, smem);  // ends with a barrier
    // Thread slot -> sample k: identity, or the ramp-coherent order of
    // ens_sample_kernel + counting sort (perm), with the sample's parameters
    // read from its planes.  Costs and parameters always land at k; the
    // deaths row at k, or at the slot when the caller only needs the per-day
    // multiset (bands).
    const size_t slot = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = slot < n;
    const size_t k = live ? (perm ? perm[slot] : slot) : 0;
    // deaths of sample k, forecast day d at deaths_out[k*sstride + d*dstride]
    // (sample-major rows, or day-major columns for the on-device bands)
    double* drow = deaths_out + (out_by_slot ? slot : k) * sstride;
    const DevWindow& w = *sw.w;
    const double nan = __longlong_as_double(0x7FF8000000000000LL);
    if (!w.init_finite) {  // the whole launch (one window): no finite row, count 0
        if (live) {
            if (costs) costs[k] = __longlong_as_double(0x7FF0000000000000LL);
            for (int d = 0; d <= horizon; ++d) drow[d * dstride] = nan;
        }
        return;
    }
    double x[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (live) {
        if (planes) {
#pragma unroll
            for (int d = 0; d < 6; ++d) x[d] = planes[d * n + k];
        } else {
            x_of_sample(lo, hi, seed, k, x);
        }
        if (params_out) {
#pragma unroll
            for (int d = 0; d < 6; ++d) params_out[6 * k + d] = x[d];
        }
    }
    // The window (from its initial state to the junction), scored only when
    // the caller wants costs.  Lanes past n run it on zero parameters and
    // discard the result, so a band warp stays whole for its reductions.
    const Particle p = make_particle(x[0], x[1], x[2], x[3], x[4], x[5], w,
                                     SubKind<SUB>::kTable ? sw.tg.tgrid : nullptr);
    if (ramp_count) {  // telemetry: the window's ramp substeps (the roofline's ramp credit)
        const unsigned wr = __reduce_add_sync(0xFFFFFFFFu, live ? static_cast<unsigned>(p.k2 - p.k1) : 0u);
        if ((threadIdx.x & 31) == 0 && wr) atomicAdd(ramp_count, static_cast<unsigned long long>(wr));
    }
    double S = w.init[0], I = w.init[1], R = w.init[2], D = w.init[3];
    bool fin_w;
    if (costs) {
        ScoreSink<FAM, MET> score(w, sw.obs, sw.robs, sw.flag);  // starts from the day-0 contribution
        integrate_days<SUB>(p, w, sw.tg, S, I, R, D, score);
        fin_w = all_finite(S, I, R, D);
        if (live) costs[k] = score.finish(fin_w);
    } else {
        NullSink none;
        integrate_days<SUB>(p, w, sw.tg, S, I, R, D, none);
        fin_w = all_finite(S, I, R, D);
    }
    // forecast_extension re-checks the junction through integrate_euler's
    // isfinite(init.total()) (model.cpp:83); it throws NonFiniteError for a
    // non-finite junction or forecast (calibration.cpp:301-303, 318-320).
    const bool fin_j = fin_w && isfinite(dadd(dadd(dadd(S, I), R), D));
    // Forecast: fwin carries n_days = horizon + 1 and the same N, h,
    // substeps; held parameters never enter the ramp, so no time table is read.
    const Particle held = make_particle(x[1], x[1], 0.0, 0.0, x[4], x[5], fwin);
    const TimeGrid ftg{nullptr, sw.tg.subh};
    if (!days) {
        if (!live) return;
        if (!fin_j) {
            for (int d = 0; d <= horizon; ++d) drow[d * dstride] = nan;
            return;
        }
        drow[0] = D;
        ForecastDSink fs{drow, dstride};
        integrate_days<SUB>(held, fwin, ftg, S, I, R, D, fs);
        if (!all_finite(S, I, R, D)) {  // calibration.cpp:318-320
            for (int d = 0; d <= horizon; ++d) drow[d * dstride] = nan;
        }
        return;
    }
    // Band path with the selection's first pass fused (horizon < 32): every
    // lane runs the forecast, the warp reduces each day's key range as the
    // day arrives, and the finite rows are counted at the end (a row is all
    // finite or all NaN: non-finiteness is absorbing, model.cpp:101-104).
    BandDSink bs{drow, dstride, live && fin_j, 0xFFFFFFFFu, 0u, s_pbase, s_pshift, hist, days};
    bs.put(0, D);
    integrate_days<SUB>(held, fwin, ftg, S, I, R, D, bs);
    const bool row_ok = bs.on && all_finite(S, I, R, D);
    if (bs.on && !row_ok) {  // blew up after some finite days: take them back out of the histograms
        for (int d = 0; d <= horizon; ++d) {
            const double v = drow[d * dstride];
            if (isfinite(v)) bs.count(d, order_key(v), -1);
        }
    }
    if (live && !row_ok) {  // a non-finite junction or forecast: the whole row NaN
        for (int d = 0; d <= horizon; ++d) drow[d * dstride] = nan;
    }
    const unsigned n_ok = __popc(__ballot_sync(0xFFFFFFFFu, row_ok));
    const int lane = threadIdx.x & 31;
    if (lane <= horizon && bs.lo <= bs.hi) {
        atomicMin(&days[lane].kmin, static_cast<unsigned long long>(bs.lo) << 32);
        atomicMax(&days[lane].kmax, (static_cast<unsigned long long>(bs.hi) << 32) | 0xFFFFFFFFull);
    }
    if (lane <= horizon && n_ok) atomicAdd(&days[lane].count, static_cast<unsigned long long>(n_ok));
}

#ifndef SG_FAMILY_TU  // engine.cu only
__device__ __constant__ double kBandProbs[kBandP] = {0.5, 0.25, 0.75, 0.05, 0.95, 0.025, 0.975};  // 352-358


// The ranks quantile_sorted reads for k finite values (calibration.cpp:324-335).
__device__ __forceinline__ int band_ranks(uint64_t k, uint64_t* ranks) {
    int m = 0;
    for (int q = 0; q < kBandP; ++q) {
        const double hq = dmul(static_cast<double>(k - 1), kBandProbs[q]);
        const uint64_t lo = static_cast<uint64_t>(hq);
        if (lo + 1 >= k) {
            ranks[m++] = k - 1;
        } else {
            ranks[m++] = lo;
            ranks[m++] = lo + 1;
        }
    }
    return m;
}

// k and the key range of every day of a given plane (grid: chunks x days) —
// the ensemble kernel's fused epilogue as a kernel of its own, for bands of
// values that come from elsewhere (sg_quantile_bands).
__global__ void __launch_bounds__(kSampleThreads) sel_range_kernel(const double* __restrict__ col, size_t n, SelDay* __restrict__ days) {
    const int d = blockIdx.y;
    const double* c = col + static_cast<size_t>(d) * n;
    unsigned long long lo = ~0ULL, hi = 0, cnt = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double x = c[i];
        if (!isfinite(x)) continue;
        const unsigned long long k = order_key(x);
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
        ++cnt;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long olo = __shfl_xor_sync(0xFFFFFFFFu, lo, off);
        const unsigned long long ohi = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
        lo = olo < lo ? olo : lo;
        hi = ohi > hi ? ohi : hi;
        cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicMin(&days[d].kmin, lo);
        atomicMax(&days[d].kmax, hi);
        atomicAdd(&days[d].count, cnt);
    }
}

// Histogram pass over the plane for the days that need it (no prediction,
// or a wanted rank outside the predicted bins: SelDay::full), over the
// day's key range: per CTA in shared memory, then one global add per
// non-empty bin.
__global__ void __launch_bounds__(kHistThreads) sel_hist_kernel(const double* __restrict__ col, size_t n,
                                             const SelDay* __restrict__ days, unsigned int* __restrict__ hist) {
    __shared__ unsigned int sh[kSelBins];
    const int d = blockIdx.y;
    const SelDay& sd = days[d];
    if (sd.count == 0 || !sd.full) return;
    for (int b = threadIdx.x; b < kSelBins; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    const int shift = sd.shift;
    const unsigned long long base = sd.base;
    const double* c = col + static_cast<size_t>(d) * n;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    constexpr int kBatch = 8;  // loads in flight per thread
    for (size_t i0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i0 < n; i0 += kBatch * stride) {
        double xs[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const size_t i = i0 + u * stride;
            xs[u] = i < n ? c[i] : __longlong_as_double(0x7FF8000000000000LL);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
            if (isfinite(xs[u])) atomicAdd(&sh[static_cast<unsigned>((order_key(xs[u]) - base) >> shift)], 1u);
    }
    __syncthreads();
    unsigned int* h = hist + static_cast<size_t>(d) * kSelBins;
    for (int b = threadIdx.x; b < kSelBins; b += blockDim.x)
        if (sh[b]) atomicAdd(&h[b], sh[b]);
}

// One CTA per day: the bins holding the wanted ranks (deduplicated,
// ascending) and their rank offsets, from the day's histogram, which is
// left zero for the slot's next window.
//   pass 0: the fused histogram over the predicted bins, when every wanted
//           rank falls inside them (the counts outside come first: `under`);
//           else the day is marked for the histogram pass (full = 1) over
//           its key range;
//   pass 1: the days marked full, from the pass's histogram.
__global__ void __launch_bounds__(kBgThreads) sel_locate_kernel(unsigned int* __restrict__ hist, SelDay* __restrict__ days,
                                               int pass, unsigned long long* __restrict__ stats) {
    constexpr int kPer = kSelBins / kBgThreads;
    constexpr int kWarps = kBgThreads / 32;
    const int d = blockIdx.x;
    SelDay& sd = days[d];
    const unsigned long long k = sd.count;
    if (k == 0 || (pass == 1 && !sd.full)) {
        if (threadIdx.x == 0 && k == 0) sd.n_seg = 0;
        return;
    }
    unsigned int* h = hist + static_cast<size_t>(d) * kSelBins;
    __shared__ uint32_t warp_sum[kWarps];
    __shared__ uint64_t ranks[kBandRanks];
    __shared__ int n_ranks, s_ok;
    __shared__ uint32_t bins[kBandRanks];
    __shared__ uint64_t bin_rank0[kBandRanks];
    __shared__ uint32_t bin_count[kBandRanks];
    uint32_t mine = 0;
    for (int j = 0; j < kPer; ++j) mine += h[threadIdx.x * kPer + j];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) warp_sum[warp] = incl;
    const unsigned long long under = pass == 0 ? sd.under : 0ULL;
    if (threadIdx.x == 0) n_ranks = band_ranks(k, ranks);
    __syncthreads();
    uint64_t base = under + (incl - mine);  // values before this thread's bins
    uint64_t in_bins = 0;
    for (int w = 0; w < kWarps; ++w) {
        if (w < warp) base += warp_sum[w];
        in_bins += warp_sum[w];
    }
    if (threadIdx.x == 0) {
        bool ok = true;
        if (pass == 0) {
            // the prediction holds when it counted every finite value and
            // every wanted rank lies inside its bins
            ok = sd.pshift >= 0 && under + in_bins + sd.over == k;
            for (int r = 0; r < n_ranks && ok; ++r) ok = ranks[r] >= under && ranks[r] < under + in_bins;
        }
        s_ok = ok;
        if (pass == 0 && stats) atomicAdd(&stats[ok ? 0 : 1], 1ULL);
        if (!ok) {  // the histogram pass over the day's key range
            sd.full = 1;
            sd.base = sd.kmin;
            sd.shift = sel_shift(sd.kmax - sd.kmin);
            sd.n_seg = 0;
        } else if (pass == 0) {
            sd.base = sd.pbase;
            sd.shift = sd.pshift;
        }
    }
    __syncthreads();
    if (s_ok) {
        // the thread whose bins cover a wanted rank finds the exact bin
        for (int r = 0; r < n_ranks; ++r) {
            const uint64_t want = ranks[r];
            if (want >= base && want < base + mine) {
                uint64_t acc = base;
                for (int j = 0; j < kPer; ++j) {
                    const uint32_t c = h[threadIdx.x * kPer + j];
                    if (want < acc + c) {
                        bins[r] = threadIdx.x * kPer + j;
                        bin_rank0[r] = acc;
                        bin_count[r] = c;
                        break;
                    }
                    acc += c;
                }
            }
        }
    }
    __syncthreads();
    // the day's histogram is consumed: leave it zero for the pass / the next window
    for (int j = 0; j < kPer; ++j) h[threadIdx.x * kPer + j] = 0;
    if (threadIdx.x == 0 && s_ok) {
        // distinct bins in ascending order (ranks were produced unordered)
        int ns = 0;
        for (int r = 0; r < n_ranks; ++r) {
            bool seen = false;
            for (int t = 0; t < ns; ++t) seen = seen || sd.seg_bin[t] == bins[r];
            if (seen) continue;
            int at = ns++;
            while (at > 0 && sd.seg_bin[at - 1] > bins[r]) {
                sd.seg_bin[at] = sd.seg_bin[at - 1];
                sd.seg_rank0[at] = sd.seg_rank0[at - 1];
                sd.seg_count[at] = sd.seg_count[at - 1];
                --at;
            }
            sd.seg_bin[at] = bins[r];
            sd.seg_rank0[at] = bin_rank0[r];
            sd.seg_count[at] = bin_count[r];
        }
        for (int t = 0; t < ns; ++t) sd.seg_fill[t] = 0;
        sd.n_seg = ns;
    }
}

// Copy the values of the wanted bins into their segments (a shared-memory
// bin -> segment table, warp-aggregated slot reservation).  Segment j of day
// d occupies cand[d*n + sum of the earlier segments' counts ...].
__global__ void __launch_bounds__(kSampleThreads) sel_gather_kernel(const double* __restrict__ col, size_t n,
                                                         SelDay* __restrict__ days, double* __restrict__ cand) {
    __shared__ unsigned char seg_of[kSelBins];
    __shared__ uint64_t seg_off[kBandRanks];
    const int d = blockIdx.y;
    SelDay& sd = days[d];
    if (sd.count == 0) return;
    for (int b = threadIdx.x; b < kSelBins; b += blockDim.x) seg_of[b] = 0xFF;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t off = 0;
        for (int j = 0; j < sd.n_seg; ++j) {
            seg_of[sd.seg_bin[j]] = static_cast<unsigned char>(j);
            seg_off[j] = off;
            off += sd.seg_count[j];
        }
    }
    __syncthreads();
    const unsigned long long kmin = sd.base;
    const int shift = sd.shift;
    const double* c = col + static_cast<size_t>(d) * n;
    double* out = cand + static_cast<size_t>(d) * n;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t end = (n + stride - 1) / stride * stride;  // whole warps iterate together
    const unsigned lane = threadIdx.x & 31;
    constexpr int kBatch = 8;  // loads in flight per thread (one CTA per SM: latency needs ILP)
    for (size_t i0 = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i0 < end; i0 += kBatch * stride) {
        double xs[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const size_t i = i0 + u * stride;
            xs[u] = i < n ? c[i] : __longlong_as_double(0x7FF8000000000000LL);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const double x = xs[u];
            int seg = -1;
            const unsigned long long key = order_key(x);
            // finite and inside the bins (predicted bins need not cover every value)
            if (isfinite(x) && key >= kmin && ((key - kmin) >> shift) < static_cast<unsigned long long>(kSelBins)) {
                const unsigned char j = seg_of[static_cast<uint32_t>((key - kmin) >> shift)];
                if (j != 0xFF) seg = j;
            }
            const unsigned want = __ballot_sync(0xFFFFFFFFu, seg >= 0);
            if (want == 0) continue;
            const unsigned peers = __match_any_sync(0xFFFFFFFFu, seg);
            if (seg < 0) continue;
            const int leader = __ffs(peers) - 1;
            uint32_t base = 0;
            if (static_cast<int>(lane) == leader)
                base = atomicAdd(&sd.seg_fill[seg], static_cast<unsigned>(__popc(peers)));
            base = __shfl_sync(peers, base, leader);
            SG_CHECK(base + __popc(peers & ((1u << lane) - 1u)) < sd.seg_count[seg]);
            out[seg_off[seg] + base + __popc(peers & ((1u << lane) - 1u))] = x;
        }
    }
}

// ---- the wanted ranks of each gathered bin, one CTA per (day, bin) -----------------
constexpr int kSelDirect = 512;        // values ranked directly (all pairs) in shared memory

// Exclusive prefix sum of one value per thread over the CTA (<= 1024 threads).
__device__ __forceinline__ uint32_t block_exclusive_sum(uint32_t v) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, n_warps = (blockDim.x + 31) >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < n_warps ? warp_sums[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, wi, off);
            if (lane >= off) wi += o;
        }
        if (lane < n_warps) warp_sums[lane] = wi - w;
    }
    __syncthreads();
    const uint32_t r = warp_sums[warp] + incl - v;
    __syncthreads();  // warp_sums reusable by the next call
    return r;
}

// Rank selection among `count` (<= kSelDirect) keys in shared memory: the
// key of local rank r is the key with #(keys < key) <= r < #(keys <= key).
// Ties are equal keys, hence equal values.  Writes *out for every wanted
// local rank found (CTA-uniform call).
__device__ __forceinline__ void rank_select(const unsigned long long* keys, uint32_t count, const uint32_t* want,
                                            int n_want, double* const* out) {
    for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
        const unsigned long long x = keys[i];
        uint32_t lt = 0, le = 0;
        for (uint32_t j = 0; j < count; ++j) {
            const unsigned long long y = keys[j];  // broadcast read
            lt += y < x;
            le += y <= x;
        }
        for (int t = 0; t < n_want; ++t)
            if (want[t] >= lt && want[t] < le) *out[t] = key_value(x);
    }
}

// The values of local ranks want[0..n_want) among the `count` values of one
// bin (keys in [base, base + 2^shift)) at src: finer histogram levels of
// 2^12 sub-bins, each keeping the sub-bin that holds the (first) wanted
// rank — into shared memory once it fits, else into the scratch pair —
// until the rest is small enough to rank directly or is a single key.
// Called per group of wanted ranks that share every level's sub-bin; a rank
// leaving the group's sub-bin is resolved by its own call.  CTA-uniform.
__device__ void select_in_bin(const double* src, uint32_t count, unsigned long long base, int shift,
                              const uint32_t* want_in, int n_want_in, double* const* out_in, double* scratch_a,
                              double* scratch_b, unsigned long long* keys, unsigned int* hist) {
    __shared__ uint32_t s_bin, s_before, s_fill, s_want[kBandRanks];
    __shared__ double* s_out[kBandRanks];
    __shared__ int s_n;
    if (threadIdx.x == 0) {
        s_n = n_want_in;
        for (int t = 0; t < n_want_in; ++t) {
            s_want[t] = want_in[t];
            s_out[t] = out_in[t];
        }
    }
    __syncthreads();
    double* dst = scratch_a;
    bool in_smem = false;  // src values already staged as keys in shared memory
    while (true) {
        if (count <= static_cast<uint32_t>(kSelDirect)) {
            if (!in_smem)
                for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) keys[i] = order_key(src[i]);
            __syncthreads();
            rank_select(keys, count, s_want, s_n, s_out);
            __syncthreads();
            return;
        }
        if (shift == 0) {  // every value of the bin is this key
            if (threadIdx.x < static_cast<unsigned>(s_n)) *s_out[threadIdx.x] = key_value(base);
            __syncthreads();
            return;
        }
        const int sub = shift > kSelBinBits ? shift - kSelBinBits : 0;
        for (int b = threadIdx.x; b < kSelBins; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
            SG_CHECK(((order_key(src[i]) - base) >> sub) < static_cast<unsigned long long>(kSelBins));
            atomicAdd(&hist[static_cast<uint32_t>((order_key(src[i]) - base) >> sub)], 1u);
        }
        __syncthreads();
        // the sub-bin of the first wanted rank: a block scan of the bins
        // (each thread owns kSelBins / blockDim consecutive bins)
        {
            const int per = kSelBins / static_cast<int>(blockDim.x);
            uint32_t mine = 0;
            for (int b = 0; b < per; ++b) mine += hist[threadIdx.x * per + b];
            const uint32_t before_me = block_exclusive_sum(mine);
            const uint32_t want0 = s_want[0];
            if (want0 >= before_me && want0 < before_me + mine) {
                uint32_t acc = before_me;
                int b = threadIdx.x * per;
                while (acc + hist[b] <= want0) acc += hist[b++];
                s_bin = static_cast<uint32_t>(b);
                s_before = acc;
            }
            if (threadIdx.x == 0) s_fill = 0;
        }
        __syncthreads();
        const uint32_t bin = s_bin, before = s_before, c_bin = hist[bin];
        // ranks of this group outside the chosen sub-bin: split off (rare: lo
        // and lo+1 straddling a sub-bin boundary)
        if (threadIdx.x == 0) {
            int m = 0;
            for (int t = 0; t < s_n; ++t) {
                if (s_want[t] >= before && s_want[t] < before + c_bin) {
                    s_want[m] = s_want[t] - before;
                    s_out[m] = s_out[t];
                    ++m;
                }
            }
            s_n = m;
        }
        __syncthreads();
        const bool to_smem = c_bin <= static_cast<uint32_t>(kSelDirect);
        for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
            const double x = src[i];
            const unsigned long long key = order_key(x);
            if (static_cast<uint32_t>((key - base) >> sub) == bin) {
                const uint32_t slot = atomicAdd(&s_fill, 1u);
                SG_CHECK(slot < c_bin);
                if (to_smem) keys[slot] = key;
                else dst[slot] = x;
            }
        }
        __syncthreads();
        count = c_bin;
        base += static_cast<unsigned long long>(bin) << sub;
        shift = sub;
        in_smem = to_smem;
        src = dst;
        dst = dst == scratch_a ? scratch_b : scratch_a;
    }
}

// Segment j (a gathered bin) of day d: its wanted ranks, resolved in shared
// memory (CTA-uniform).
__device__ void finish_segment(const SelDay& sd, int d, int j, const double* __restrict__ cand,
                               double* __restrict__ scratch, size_t n, double* __restrict__ vals,
                               unsigned long long* keys, unsigned int* hist, uint64_t* ranks, uint32_t* want,
                               double** outp, int& n_ranks, int& n_want) {
    const uint32_t cnt = sd.seg_count[j];
    const uint64_t r0 = sd.seg_rank0[j];
    if (threadIdx.x == 0) {
        n_ranks = band_ranks(sd.count, ranks);
        int m = 0;
        for (int r = 0; r < n_ranks; ++r) {
            if (ranks[r] < r0 || ranks[r] >= r0 + cnt) continue;
            bool dup = false;  // lo of one probability may equal lo+1 of another
            for (int t = 0; t < m; ++t) dup = dup || want[t] == static_cast<uint32_t>(ranks[r] - r0);
            if (dup) continue;
            // ascending insertion: the group's first rank picks the sub-bin
            int at = m++;
            while (at > 0 && want[at - 1] > static_cast<uint32_t>(ranks[r] - r0)) {
                want[at] = want[at - 1];
                outp[at] = outp[at - 1];
                --at;
            }
            want[at] = static_cast<uint32_t>(ranks[r] - r0);
            outp[at] = vals + static_cast<size_t>(d) * kBandRanks + r;
        }
        n_want = m;
    }
    __syncthreads();
    uint64_t off = 0;
    for (int t = 0; t < j; ++t) off += sd.seg_count[t];
    SG_CHECK(off + cnt <= n && n_want >= 1);
    const double* src = cand + static_cast<size_t>(d) * n + off;
    // the scratch pair of this bin: 2 x cnt doubles of the day's 2 x n (the
    // CTAs of one day's bins run concurrently)
    double* sa = scratch + static_cast<size_t>(d) * 2 * n + 2 * off;
    const unsigned long long base = sd.base + (static_cast<unsigned long long>(sd.seg_bin[j]) << sd.shift);
    // All the segment's wanted ranks in one pass (ascending: the first picks
    // each level's sub-bin); a rank that leaves the group's sub-bin (rare:
    // lo and lo+1 straddling a sub-bin boundary) stays unresolved and goes
    // to the next pass.  Results are staged in shared memory with a NaN
    // sentinel (a selected value is always finite).
    constexpr long long kUnresolved = 0x7FF8DEADBEEF0001LL;
    __shared__ double res[kBandRanks];
    __shared__ uint32_t left_want[kBandRanks];
    __shared__ double* left_out[kBandRanks];
    __shared__ int n_left;
    if (threadIdx.x == 0)
        for (int t = 0; t < n_want; ++t) res[t] = __longlong_as_double(kUnresolved);
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) {
            int m = 0;
            for (int t = 0; t < n_want; ++t) {
                if (__double_as_longlong(res[t]) != kUnresolved) continue;
                left_want[m] = want[t];
                left_out[m] = &res[t];
                ++m;
            }
            n_left = m;
        }
        __syncthreads();
        if (n_left == 0) break;
        select_in_bin(src, cnt, base, sd.shift, left_want, n_left, left_out, sa, sa + cnt, keys, hist);
    }
    if (threadIdx.x == 0)
        for (int t = 0; t < n_want; ++t) *outp[t] = res[t];
}

// One CTA per (gathered bin, day): the bin's wanted ranks.  vals: 14 per day,
// indexed like band_ranks().  scratch: 2 x n doubles per day (only touched by
// bins that need more than one finer level outside shared memory).
__global__ void __launch_bounds__(kSampleThreads) sel_finish_kernel(int n_days, const SelDay* __restrict__ days,
                                                                        const double* __restrict__ cand,
                                                                        double* __restrict__ scratch, size_t n,
                                                                        double* __restrict__ vals) {
    __shared__ unsigned long long keys[kSelDirect];
    __shared__ unsigned int hist[kSelBins];
    __shared__ uint64_t ranks[kBandRanks];
    __shared__ uint32_t want[kBandRanks];
    __shared__ double* outp[kBandRanks];
    __shared__ int n_ranks, n_want;
    for (int pair = blockIdx.x; pair < kBandRanks * n_days; pair += gridDim.x) {
        const int d = pair / kBandRanks;
        const int j = pair - d * kBandRanks;
        const SelDay& sd = days[d];
        if (sd.count == 0 || j >= sd.n_seg) continue;  // CTA-uniform
        finish_segment(sd, d, j, cand, scratch, n, vals, keys, hist, ranks, want, outp, n_ranks, n_want);
        __syncthreads();  // the shared arrays are reused by the next pair
    }
}

// quantile_sorted (calibration.cpp:324-335) of every day from its resolved
// order statistics, with the reference's operation order.
__global__ void __launch_bounds__(kBgThreads) sel_bands_kernel(const SelDay* __restrict__ days, const double* __restrict__ vals,
                                 double* __restrict__ bands, unsigned long long* __restrict__ counts, int n_days) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_days) return;
    const uint64_t k = days[d].count;
    counts[d] = k;
    uint64_t ranks[kBandRanks];
    const int n_ranks = k ? band_ranks(k, ranks) : 0;
    const double* v = vals + static_cast<size_t>(d) * kBandRanks;
    auto at = [&](uint64_t r) {
        for (int t = 0; t < n_ranks; ++t)
            if (ranks[t] == r) return v[t];
        return __longlong_as_double(0x7FF8000000000000LL);  // unreachable
    };
    for (int q = 0; q < kBandP; ++q) {
        double x = __longlong_as_double(0x7FF8000000000000LL);
        if (k) {
            const double h = dmul(static_cast<double>(k - 1), kBandProbs[q]);
            const uint64_t lo = static_cast<uint64_t>(h);
            if (lo + 1 >= k) {
                x = at(k - 1);
            } else {
                const double a = at(lo), b = at(lo + 1);
                x = dadd(a, dmul(dsub(h, static_cast<double>(lo)), dsub(b, a)));
            }
        }
        bands[q * n_days + d] = x;
    }
}

// ---- quantile bands of a sorted column (n == 0 path) ------------------------------
//
// quantile_sorted (calibration.cpp:324-335) with the reference's operation
// order; bands_kernel cuts each column at its first non-finite entry.
__device__ __forceinline__ double quantile_sorted_dev(const double* sorted, size_t k, double p) {
    if (k == 0) return __longlong_as_double(0x7FF8000000000000LL);
    const double h = dmul(static_cast<double>(k - 1), p);
    const size_t lo = static_cast<size_t>(h);
    if (lo + 1 >= k) return sorted[k - 1];
    const double frac = dsub(h, static_cast<double>(lo));
    return dadd(sorted[lo], dmul(frac, dsub(sorted[lo + 1], sorted[lo])));
}

__global__ void bands_kernel(const double* __restrict__ sorted, size_t n, double* __restrict__ bands,
                             unsigned long long* __restrict__ counts, int n_days) {
    const int d = blockIdx.x;
    if (threadIdx.x != 0 || d >= n_days) return;
    const double* col = sorted + static_cast<size_t>(d) * n;
    // first non-finite entry (finite values precede NaN after the sort)
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = lo + (hi - lo) / 2;
        if (isfinite(col[mid])) lo = mid + 1;
        else hi = mid;
    }
    const size_t k = lo;
    counts[d] = k;
    const double ps[7] = {0.5, 0.25, 0.75, 0.05, 0.95, 0.025, 0.975};  // calibration.cpp:352-358
#pragma unroll
    for (int q = 0; q < 7; ++q) bands[q * n_days + d] = quantile_sorted_dev(col, k, ps[q]);
}

#endif  // SG_FAMILY_TU

}  // namespace sirdgpu
