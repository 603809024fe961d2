// sird_device.cuh — device-side arithmetic of the particle-window cost engine.
//
// Bit-exactness contract: every function here reproduces the reference's
// IEEE-754 double arithmetic operation by operation (the reference object
// code contains no FMA, SURVEY.md §0 key finding 2).  The file is compiled
// with -fmad=false and additionally spells every rounded operation with an
// explicit __dmul_rn/__dadd_rn/__dsub_rn intrinsic, so no contraction can
// ever be introduced.  The only fma() uses are the exact-division sequences
// div_exact() (3 ops) and div_by_N() (2 ops), whose results are proven equal
// to the correctly rounded quotient for the inputs that reach them
// (DESIGN.md §4).
#pragma once

#include <cstdint>

// SG_CHECKED=1 (a diagnostic build, tools/checked_build.py): device-side
// asserts of the invariants the lock-free folds, the cluster kernel and the
// bulk staging rely on.  compute-sanitizer is not available on the GPU pool,
// so these asserts, run under the GPU test suite, stand in for it.
#ifndef SG_CHECKED
#define SG_CHECKED 0
#endif
#if SG_CHECKED
#undef NDEBUG
#include <cassert>
#define SG_CHECK(cond) assert(cond)
#else
#define SG_CHECK(cond) ((void)0)
#endif

#ifndef SG_RAMP_MODE
#define SG_RAMP_MODE 1
#endif
#ifndef SG_DAY_COUNTERS
#define SG_DAY_COUNTERS 0
#endif
#ifndef SG_DAY_SPLIT
#define SG_DAY_SPLIT 2
#endif
#ifndef SG_CONST_UNROLL
#define SG_CONST_UNROLL 8
#endif
#ifndef SG_QUIET_UNROLL
#define SG_QUIET_UNROLL 8
#endif
#ifndef SG_SLOW_UNROLL
#define SG_SLOW_UNROLL 12
#endif
#ifndef SG_RAMP_UNROLL
#define SG_RAMP_UNROLL 12
#endif
#ifndef SG_OBS_ASM
#define SG_OBS_ASM 1
#endif
#if SG_DAY_COUNTERS
// Diagnostic build only: warp-days per class (0 constant, 1 switch, 2 ramp).
static __device__ unsigned long long g_day_class[3];  // one copy per object (family.cu reads its own)
#endif

namespace sirdgpu {

constexpr int kConstUnroll = SG_CONST_UNROLL;  // substep unroll of constant days
constexpr int kRampUnroll = SG_RAMP_UNROLL;    // ... of switch and ramp days
constexpr int kQuietUnroll = SG_QUIET_UNROLL;  // ... of the quiet-stretch loop
constexpr int kSlowUnroll = SG_SLOW_UNROLL;    // ... of ramp days with IEEE divisions
constexpr int kFamD = 0;
constexpr int kFamIRD = 1;
constexpr int kMetMXSE = 0;
constexpr int kMetMSE = 1;
constexpr int kMetMAE = 2;
constexpr int kMetMAPE = 3;

// Per-day observation flags (MAPE): skip (obs == 0), fast reciprocal division,
// or plain IEEE division.
constexpr unsigned char kObsSkip = 0;
constexpr unsigned char kObsFast = 1;
constexpr unsigned char kObsSlow = 2;

// One observed day, staged in shared memory (I, R, D).
struct ObsDay {
    double v[3];
};

// Window descriptor as the kernels see it (device memory, one per window).
// Built on the host by sg_window_create from the reference's
// make_window_objective inputs (calibration.cpp:120-139).
struct alignas(16) DevWindow {  // 16-byte multiple: staged by one bulk copy
    int n_days;
    int substeps;
    int family;
    int metric;
    double N;             // population
    double rN;            // RN(1/N)
    double rN_lo;         // RN(1/N - rN): rN + rN_lo is 1/N to ~2^-106 (ramp division, when fast_N)
    double h;             // 1.0 / substeps (model.cpp:90)
    int fast_N;           // N admits the exact 2-op ramp division
    int init_finite;      // isfinite(init.total()) (model.cpp:83)
    double init[4];       // S, I, R, D
    double scale[3];      // compartment_cost scale (objectives.cpp:61-69); 1 for D-only
    int mxse_abs;         // MXSE tracks max |obs - pred| (scale and square once at the end)
    double acc0[3];       // day-0 score contribution per compartment: the initial state is
                          // the same for every particle (model.cpp:85), so it is window-constant
    double kept[3];       // MAPE: number of days with obs != 0 (objectives.cpp:41-55)
    const ObsDay* obs;    // n_days
    const ObsDay* robs;   // RN(1/obs) per day (MAPE)
    const unsigned char* obs_flag;  // 3 per day (MAPE)
    const double* times;  // subh[substeps] then tgrid (tgrid_entries), host-built; null: kernels compute them
};

// ---- exact arithmetic ---------------------------------------------------------

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// std::max(a, b) == (a < b) ? b : a (stl_algobase.h), NaN-preserving order.
__device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }

// Pin a value in a register: the compiler may not recompute it from its
// operands.  Without this nvcc sinks the per-particle beta/N divisions into
// the per-substep regime select (div(sel(b1,b2), N) instead of
// sel(div(b1,N), div(b2,N))), paying a full division every substep.
__device__ __forceinline__ void opaque(double& x) { asm volatile("" : "+d"(x)); }

// Biased exponent of a double, from its high word (integer pipe only).
__device__ __forceinline__ int dexp(double a) {
    return (__double2hiint(a) >> 20) & 0x7FF;
}

// a / b, correctly rounded, given rb = RN(1/b) and a divisor b that passed the
// host-side admissibility test (divisor_admits_fast_path in engine.cu:
// |b| in [2^-60, 2^60] and the odd part of b's significand below 2^53/3).
// The Markstein step q0 = RN(a*rb); r = a - q0*b (exact by fma);
// q = RN(q0 + r*rb) then equals RN(a/b) for every dividend with
// |a| in [2^-700, 2^701) (proof in DESIGN.md §4: a quotient of such b lies at
// least ulp/(2*oddpart(b)) from any rounding boundary, farther than the
// sequence's error of 1.5 ulp * 2^-53).  Every other dividend (0, subnormal,
// huge, inf, NaN) goes through the IEEE division.
__device__ __forceinline__ double div_exact(double a, double b, double rb) {
    const int e = dexp(a);
    if (e >= 1023 - 700 && e <= 1023 + 700) {
        const double q0 = __dmul_rn(a, rb);
        const double r = __fma_rn(-q0, b, a);
        return __fma_rn(r, rb, q0);
    }
    return __ddiv_rn(a, b);
}

// ---- beta(t) regimes --------------------------------------------------------
//
// beta_at (model.cpp:55-64) compares t = (day-1) + sub*h (model.cpp:94)
// against t1 and t2.  t is non-decreasing in the substep index
// k = (day-1)*S + sub, so {k : t_k < x} is a prefix; the kernel resolves both
// comparisons once per particle into prefix lengths k1, k2 and then selects
// the regime with integer compares only.

__device__ __forceinline__ double t_of(int k, int S, double h) {
    const int day_m1 = k / S;
    const int sub = k - day_m1 * S;
    return dadd(static_cast<double>(day_m1), dmul(static_cast<double>(sub), h));
}

// Number of k in [0, K) with t_k < x (x may be NaN -> 0).  t_k is within a
// few ulps of k/S, so the search starts at floor(x*S) and walks the exact
// t_k to the boundary (one or two steps in practice; monotone, so exact).
// With a substep-time table (tgrid[k] == t_of(k), k < K) the walk reads it
// instead of recomputing t_k.
__device__ __forceinline__ int count_t_below(double x, int K, int S, double h, const double* tgrid = nullptr) {
    if (!(x > 0.0)) return 0;  // t_0 = 0: nothing below 0, -inf or NaN
    if (!(x <= static_cast<double>(K))) return K;  // +inf / beyond the window
    int k = static_cast<int>(x * static_cast<double>(S));  // estimate, any rounding
    k = k < 0 ? 0 : (k > K ? K : k);
    if (tgrid) {
        while (k < K && tgrid[k] < x) ++k;
        while (k > 0 && !(tgrid[k - 1] < x)) --k;
        return k;
    }
    while (k < K && t_of(k, S, h) < x) ++k;
    while (k > 0 && !(t_of(k - 1, S, h) < x)) --k;
    return k;
}

// Per-particle constants of the integration.
struct Particle {
    double b1, b2, t1, g, mu;
    double bp1, bp2;  // beta1/N, beta2/N (model.cpp:67, constant regimes)
    double slope;     // (beta2-beta1)/(t2-t1) (model.cpp:62)
    int k1, k2;       // regime prefix lengths: k<k1 -> beta1; k>=k2 -> beta2; else ramp
    bool fast;        // every ramp beta admits the 3-op division (see beta_in_fast_range)
};

// True when every beta the ramp can produce (beta1 + slope*(t - t1) for
// t in [t1, t2)) is +0 or has magnitude in [2^-700, 2^701), the dividend
// range of div_exact, so the per-substep exponent test can be skipped:
// beta1, beta2 each +0 or of magnitude [2^-600, 2^680], t1/t2/slope finite
// (DESIGN.md §4 bounds the ramp values by these).
__device__ __forceinline__ bool beta_in_fast_range(double b) {
    const long long bits = __double_as_longlong(b);
    if (bits == 0) return true;  // +0 (not -0)
    const int e = dexp(b);
    return e >= 1023 - 600 && e <= 1023 + 680;
}

// RN(beta/N) in two operations for an admissible N and beta:
// beta*(rN + rN_lo) is within 2^-105 relative of beta/N, closer than any
// rounding boundary of the quotient.
__device__ __forceinline__ double div_by_N(double beta, double rN, double rN_lo) {
    return __fma_rn(beta, rN, __dmul_rn(beta, rN_lo));
}

__device__ __forceinline__ Particle make_particle(double b1, double b2, double t1, double t2, double g, double mu,
                                                  const DevWindow& w, const double* tgrid = nullptr) {
    Particle p;
    p.b1 = b1;
    p.b2 = b2;
    p.t1 = t1;
    p.g = g;
    p.mu = mu;
    const bool fast1 = w.fast_N && beta_in_fast_range(b1);
    const bool fast2 = w.fast_N && beta_in_fast_range(b2);
    p.bp1 = fast1 ? div_by_N(b1, w.rN, w.rN_lo) : ddiv(b1, w.N);
    p.bp2 = fast2 ? div_by_N(b2, w.rN, w.rN_lo) : ddiv(b2, w.N);
    p.slope = ddiv(dsub(b2, b1), dsub(t2, t1));
    opaque(p.bp1);
    opaque(p.bp2);
    opaque(p.slope);
    const int K = (w.n_days - 1) * w.substeps;
    p.k1 = count_t_below(t1, K, w.substeps, w.h, tgrid);
    // "t >= t2" is the complement of "t < t2" except for NaN t2, where both
    // comparisons are false and the ramp branch is taken (model.cpp:59-63).
    p.k2 = (t2 != t2) ? K : count_t_below(t2, K, w.substeps, w.h, tgrid);
    if (p.k2 < p.k1) p.k2 = p.k1;  // t1 > t2: no ramp (k >= k1 implies t >= t2)
    p.fast = fast1 && fast2 && isfinite(t1) && isfinite(t2) && isfinite(p.slope);
    return p;
}

// One Euler substep of sird_rhs (model.cpp:66-74) + update (model.cpp:96-99),
// in the reference's exact operation order:
//   inf = ((beta/N)*S)*I;  dI = (inf - g*I) - mu*I
//   S += h*(-inf); I += h*dI; R += h*(g*I); D += h*(mu*I)
__device__ __forceinline__ void euler_substep(double bp, double g, double mu, double h, double& S, double& I,
                                              double& R, double& D) {
    const double inf = dmul(dmul(bp, S), I);
    const double gI = dmul(g, I);
    const double mI = dmul(mu, I);
    const double dI = dsub(dsub(inf, gI), mI);
    S = dsub(S, dmul(h, inf));  // S + h*(-inf) == S - h*inf exactly (RN is symmetric)
    I = dadd(I, dmul(h, dI));
    R = dadd(R, dmul(h, gI));
    D = dadd(D, dmul(h, mI));
}

// beta(t_k)/N for a ramp substep (model.cpp:62-63 then model.cpp:67); t is
// the substep time t_k = (day-1) + sub*h (model.cpp:94).
__device__ __forceinline__ double ramp_bp(const Particle& p, double t, double N, double rN, double rN_lo) {
    const double beta = dadd(p.b1, dmul(p.slope, dsub(t, p.t1)));
    if (p.fast) return div_by_N(beta, rN, rN_lo);  // no per-value range test needed
    return ddiv(beta, N);
}

// Substep-time source.  The specialised kernels (SUB == 24, the reference
// default) read t_k from a per-window table in shared memory (tgrid); the
// generic kernels (SUB == 0) compute t = RN(RN(day-1) + subh[sub]).
struct TimeGrid {
    const double* tgrid;  // (n_days-1)*substeps entries (SUB > 0 only)
    const double* subh;   // substeps entries: RN(sub*h)
};

// Largest t_k table kept in shared memory (entries, 47 KB): windows up to
// 251 days at 24 substeps stage it (four step CTAs per SM still fit from 202
// days on, five below).  Longer windows compute their ramp times from subh
// (kSub24NoTable), which beats a larger table at lower occupancy: measured
// 0.89-0.90 of P with the table up to 251 days against 0.88 computed, 0.86
// against 0.88 at 301 days (profiles/r02l_long_windows.txt).
constexpr int kMaxTgrid = 6000;

// A window's t_k table fits in shared memory (any substep count).
__host__ __device__ inline bool uses_time_table(int n_days, int substeps) {
    return substeps >= 1 && static_cast<long long>(n_days - 1) * substeps <= kMaxTgrid;
}

// ... and the window takes the kernels specialised for the reference's 24 substeps.
__host__ __device__ inline bool uses_fast_grid(int n_days, int substeps) {
    return substeps == 24 && uses_time_table(n_days, substeps);
}

// Kernel specialisations by substep handling (the SUB template parameter):
//   SUB > 0   the substep count fixed at compile time (24, the reference
//             default kDefaultSubsteps, model.hpp:12) with the t_k table in
//             shared memory;
//   -24       24 substeps at compile time for windows whose table does not
//             fit shared memory (over 201 days): ramp times are computed as
//             RN(RN(day-1) + subh[sub]) (model.cpp:94), like the generic path;
//   -1        a runtime count with the table;
//   0         a runtime count without it (generic).
constexpr int kSub24NoTable = -24;
template <int SUB>
struct SubKind {
    static constexpr int kCount = SUB > 0 ? SUB : (SUB == kSub24NoTable ? 24 : 0);  // 0: runtime
    static constexpr bool kTable = SUB > 0 || SUB == -1;  // reads the t_k table
    static constexpr bool kFast = SUB != 0;               // branch-free ramp days, bulk-copy staging
};

// Integrate days 1..n_days-1 (model.cpp:92-106), calling sink.day(day, S, I, R, D)
// after every day, with the substep handling of SubKind<SUB>.
template <int SUB, class Sink>
__device__ __forceinline__ void integrate_days(const Particle& p, const DevWindow& w, const TimeGrid& tg,
                                               double& S, double& I, double& R, double& D, Sink& sink) {
    using K = SubKind<SUB>;
    const int nsub = K::kCount > 0 ? K::kCount : w.substeps;
    const double h = w.h;
    const double g = p.g, mu = p.mu;
    const double N = w.N, rN = w.rN, rN_lo = w.rN_lo;
    const unsigned mask = __activemask();
    // Warp-uniform: every lane's ramp admits the 3-op division, so the ramp
    // days run without the per-value IEEE-division fallback.
    const bool warp_fast = __all_sync(mask, p.fast);
    // Warp-uniform quiet stretches.  A lane is in beta1 for all of day d iff
    // k1 >= d*nsub, and in beta2 for all of it iff k2 <= (d-1)*nsub
    // (k2 >= k1).  Days before d_first are beta1 days in every lane, days
    // after d_last beta2 days in every lane: they skip the class votes.
#if SG_DAY_SPLIT
    const int d_first = __reduce_min_sync(mask, p.k1 / nsub + 1);
    const int d_last = __reduce_max_sync(mask, (p.k2 + nsub - 1) / nsub);
#endif
    // One classified day (class votes, then the matching substep loop).
    auto classified_day = [&](int day, int kbase) {
        const int lo = p.k1 - kbase;  // sub < lo  -> beta1
        const int hi = p.k2 - kbase;  // sub >= hi -> beta2, else ramp
        // Warp-uniform day classes (the regime depends only on k, so a day
        // whose substeps all share one regime in every lane needs no
        // per-substep select): 2 = some lane ramps today, 1 = some lane
        // switches beta1 -> beta2 today, 0 = every lane constant all day.
        const bool ramp_today = lo < hi && lo < nsub && hi > 0;
        const bool switch_today = lo > 0 && lo < nsub;
#if SG_DAY_COUNTERS
        {
            const int cls = __any_sync(mask, ramp_today) ? 2 : (__any_sync(mask, switch_today) ? 1 : 0);
            if ((threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(&g_day_class[cls], 1ull);
        }
#endif
#if SG_DAY_SPLIT == 1
        const bool quiet = day < d_first || day > d_last;
#else
        constexpr bool quiet = false;  // SG_DAY_SPLIT 2: quiet days never reach here
#endif
        // t_k of substep `sub` today (model.cpp:94): the table, or computed
        const double dayf = static_cast<double>(day - 1);
        auto t_at = [&](int sub) -> double {
            if constexpr (K::kTable) return tg.tgrid[kbase + sub];
            else return dadd(dayf, tg.subh[sub]);
        };
        if (!quiet && __any_sync(mask, ramp_today)) {
            if (SG_RAMP_MODE >= 1 && K::kFast && warp_fast && __all_sync(mask, lo <= 0 && hi >= nsub)) {
                // Every lane ramps through the whole day: no selects at all.
#pragma unroll(K::kCount > 0 ? kRampUnroll : 4)
                for (int sub = 0; sub < nsub; ++sub) {
                    const double t = t_at(sub);
                    const double beta = dadd(p.b1, dmul(p.slope, dsub(t, p.t1)));
                    euler_substep(div_by_N(beta, rN, rN_lo), g, mu, h, S, I, R, D);
                }
            } else if (SG_RAMP_MODE >= 1 && K::kFast && warp_fast) {
                // Branch-free ramp day: every lane computes the ramp value
                // (the warp would issue it anyway once any lane needs it) and
                // selects; non-FP64 work per substep is two compares and
                // selects plus the t_k load.
#pragma unroll(K::kCount > 0 ? kRampUnroll : 4)
                for (int sub = 0; sub < nsub; ++sub) {
                    const double t = t_at(sub);
                    const double beta = dadd(p.b1, dmul(p.slope, dsub(t, p.t1)));
                    const double q = div_by_N(beta, rN, rN_lo);
                    const double bp = sub < lo ? p.bp1 : (sub < hi ? q : p.bp2);
                    euler_substep(bp, g, mu, h, S, I, R, D);
                }
            } else {
#pragma unroll(K::kCount > 0 ? kSlowUnroll : 4)  // rare path (a lane outside the 2-op division range)
                for (int sub = 0; sub < nsub; ++sub) {
                    double bp = sub < lo ? p.bp1 : p.bp2;
                    if (sub >= lo && sub < hi) bp = ramp_bp(p, t_at(sub), N, rN, rN_lo);
                    euler_substep(bp, g, mu, h, S, I, R, D);
                }
            }
        } else if (!quiet && __any_sync(mask, switch_today)) {
#pragma unroll(K::kCount > 0 ? kRampUnroll : 4)
            for (int sub = 0; sub < nsub; ++sub) euler_substep(sub < lo ? p.bp1 : p.bp2, g, mu, h, S, I, R, D);
        } else {
            const double bp = lo >= nsub ? p.bp1 : p.bp2;
#pragma unroll(K::kCount > 0 ? kConstUnroll : 4)
            for (int sub = 0; sub < nsub; ++sub) euler_substep(bp, g, mu, h, S, I, R, D);
        }
    };
#if SG_DAY_SPLIT >= 2
    // Three segments: quiet beta1 days, classified days, quiet beta2 days.
    // The quiet loop body exists once in the code (instruction-cache
    // footprint) and runs without votes or regime selects.
    const int n_days = w.n_days;
    int day = 1;
#pragma unroll 1
    for (int seg = 0; seg < 3; ++seg) {
        if (seg == 1) {
            const int end = d_last + 1 < n_days ? d_last + 1 : n_days;
            for (; day < end; ++day) {
                classified_day(day, (day - 1) * nsub);
                sink.day(day, S, I, R, D);
            }
            continue;
        }
        const int end = seg == 0 ? (d_first < n_days ? d_first : n_days) : n_days;
        const double bpq = seg == 0 ? p.bp1 : p.bp2;
        for (; day < end; ++day) {
#pragma unroll(K::kCount > 0 ? kQuietUnroll : 4)
            for (int sub = 0; sub < nsub; ++sub) euler_substep(bpq, g, mu, h, S, I, R, D);
            sink.day(day, S, I, R, D);
        }
    }
#else
    for (int day = 1; day < w.n_days; ++day) {
        classified_day(day, (day - 1) * nsub);
        sink.day(day, S, I, R, D);
    }
#endif
}

__device__ __forceinline__ bool all_finite(double S, double I, double R, double D) {
    return isfinite(S) && isfinite(I) && isfinite(R) && isfinite(D);
}

// ---- scoring (objectives.cpp:15-120), fused into the day loop ----------------
//
// Accumulates per compartment exactly like metric_on_scaled_residuals / mape
// do over k = 0..n-1, one day at a time, so trajectories never leave
// registers.  Non-finiteness is absorbing under x + h*dx, so checking the
// final state once equals the per-day check of model.cpp:101-104.
template <int FAM, int MET>
struct ScoreSink {
    const DevWindow* w;
    const ObsDay* obs;    // shared memory
    const ObsDay* robs;   // shared memory (MAPE)
    const unsigned char* flag;  // shared memory (MAPE)
    uint32_t obs_s;       // shared-window address of obs[next day] (days arrive as 1, 2, ... in order)
    bool abs_max;         // MXSE on max |obs - pred| (DevWindow::mxse_abs)
    double acc[3];

    ScoreSink() = default;
    __device__ __forceinline__ ScoreSink(const DevWindow& win, const ObsDay* o, const ObsDay* ro,
                                         const unsigned char* f)
        : w(&win), obs(o), robs(ro), flag(f), obs_s(static_cast<uint32_t>(__cvta_generic_to_shared(o + 1))),
          abs_max(MET == kMetMXSE && win.mxse_abs) {
        acc[0] = win.acc0[0];  // day 0 already scored (sg_window_create)
        acc[1] = win.acc0[1];
        acc[2] = win.acc0[2];
    }

    __device__ __forceinline__ void one(int c, int day, double pred) {
        double o;
        if (MET == kMetMAPE || !SG_OBS_ASM) {
            o = obs[day].v[c];
        } else {
            // 32-bit shared address + immediate offset (a generic pointer
            // makes nvcc rebuild the shared-window base every day)
            const uint32_t a = obs_s + 8u * c;
            asm("ld.shared.f64 %0, [%1];" : "=d"(o) : "r"(a));
        }
        if (MET == kMetMAPE) {
            const unsigned char f = flag[3 * day + c];
            if (f == kObsSkip) return;  // objectives.cpp:46-48
            const double num = dsub(o, pred);
            const double q = f == kObsFast ? div_exact(num, o, robs[day].v[c]) : ddiv(num, o);
            acc[c] = dadd(acc[c], fabs(q));
            return;
        }
        if (MET == kMetMXSE && abs_max) {
            // max_d RN(RN(d*s)^2) = RN(RN(max_d |d| * s)^2) for s > 0 finite:
            // both roundings are monotone in |d| (objectives.cpp:22-26)
            acc[c] = std_max(acc[c], fabs(dsub(o, pred)));
            return;
        }
        double e = dsub(o, pred);
        if (FAM == kFamIRD) e = dmul(e, w->scale[c]);  // D-only scales by 1.0: identity
        if (MET == kMetMXSE) acc[c] = std_max(acc[c], dmul(e, e));
        else if (MET == kMetMSE) acc[c] = dadd(acc[c], dmul(e, e));
        else acc[c] = dadd(acc[c], fabs(e));
    }

    __device__ __forceinline__ void day(int d, double S, double I, double R, double D) {
        (void)S;
        if (FAM == kFamIRD) {
            one(0, d, I);
            one(1, d, R);
        }
        one(2, d, D);
        obs_s += sizeof(ObsDay);
    }

    __device__ __forceinline__ double finish_one(int c) const {
        if (MET == kMetMAPE) {
            if (w->kept[c] == 0.0) return __longlong_as_double(0x7FF0000000000000LL);
            return ddiv(dmul(100.0, acc[c]), w->kept[c]);
        }
        if (MET == kMetMSE || MET == kMetMAE) return ddiv(acc[c], static_cast<double>(w->n_days));
        if (abs_max) {
            const double e = FAM == kFamIRD ? dmul(acc[c], w->scale[c]) : acc[c];
            return dmul(e, e);
        }
        return acc[c];
    }

    __device__ __forceinline__ double finish(bool finite) const {
        if (!finite) return __longlong_as_double(0x7FF0000000000000LL);  // objectives.cpp:101-103
        if (FAM == kFamD) return finish_one(2);
        double worst = finish_one(0);           // objectives.cpp:116-119
        worst = std_max(worst, finish_one(1));
        worst = std_max(worst, finish_one(2));
        return worst;
    }
};

// Full particle-window evaluation: objective_value(spec, slice,
// integrate_euler(params)) (calibration.cpp:148-152).
// *ramp receives the particle's number of ramp substeps (the R_ramp of the
// algorithmic operation count).
template <int FAM, int MET, int SUB>
__device__ __forceinline__ double eval_particle(const double* x, const DevWindow& w, const TimeGrid& tg,
                                                const ObsDay* obs, const ObsDay* robs, const unsigned char* flag,
                                                int* ramp = nullptr) {
    if (!w.init_finite) {
        if (ramp) *ramp = 0;
        return __longlong_as_double(0x7FF0000000000000LL);
    }
    const Particle p = make_particle(x[0], x[1], x[2], x[3], x[4], x[5], w, SubKind<SUB>::kTable ? tg.tgrid : nullptr);
    if (ramp) *ramp = p.k2 - p.k1;
    double S = w.init[0], I = w.init[1], R = w.init[2], D = w.init[3];
    ScoreSink<FAM, MET> sink(w, obs, robs, flag);  // starts from the day-0 contribution
    integrate_days<SUB>(p, w, tg, S, I, R, D, sink);
    return sink.finish(all_finite(S, I, R, D));
}

// ---- std::mt19937_64, structure-of-arrays ---------------------------------
//
// Each particle owns one engine (pso.hpp:79) seeded mix_seed(seed, i)
// (pso.cpp:55-57).  State word j of particle p lives at
// mt[pblock_base(p, 312) + 32*j], so a warp touches 32 consecutive words.  Every particle of a swarm has drawn the
// same number of values at any time, so the generation position `count` is
// uniform and the standard in-place twist is evaluated lazily, one word per
// draw: word i of the next generation depends on words i, i+1 (old) and
// (i+156)%312 (old for i<156, already new for i>=156) — exactly the order of
// the sequential twist.

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kMtF = 6364136223846793005ULL;

__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t base, uint64_t index) {  // pso.cpp:36-41
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

__device__ __forceinline__ uint64_t mt_twist_word(uint64_t cur, uint64_t next, uint64_t far) {
    const uint64_t y = (cur & 0xFFFFFFFF80000000ULL) | (next & 0x7FFFFFFFULL);
    return far ^ (y >> 1) ^ ((y & 1ULL) ? kMtA : 0ULL);
}

// uniform01 (pso.cpp:43-45)
__device__ __forceinline__ double to_uniform01(uint64_t x) {
    return dmul(static_cast<double>(x >> 11), 0x1.0p-53);
}

// Draw NDRAW consecutive values (NDRAW <= 12) from the engine whose word w
// lives at mt[32*w] (particle-block layout), starting at state word
// i0 = (values drawn so far) mod 312 — uniform over a swarm, so callers
// compute it once.  All 2*NDRAW+1 state words are loaded before any is
// rewritten: the batch's words are distinct (NDRAW < 156), every "next" word
// is read before it is twisted (old value, as the sequential twist reads
// it), and every "far" word lies outside the batch — so the loads are
// independent and overlap.  Word addresses are a row pointer plus a
// compile-time offset; the (warp-uniform) wrap past word 311 switches rows.
// Split in two (mt_load, then mt_finish) a caller can issue the loads long
// before it needs the values; mt_draw does both in one (its own code: the
// step kernel's register allocation is tuned on it).
template <int NDRAW>
struct MtBatch {
    uint64_t cur[NDRAW + 1];
    uint64_t far[NDRAW];
};

template <int NDRAW>
__device__ __forceinline__ void mt_load(const uint64_t* __restrict__ mt, int i0, MtBatch<NDRAW>& b) {
    static_assert(NDRAW >= 1 && NDRAW < kMtM, "batch must not reach its own far words");
    SG_CHECK(i0 >= 0 && i0 < kMtN);
    const uint64_t* const row = mt + 32 * i0;            // word i0 + j at row[32*j] ...
    const uint64_t* const row_w = row - 32 * kMtN;       // ... or, past word 311, at row_w[32*j]
    const int wrap = kMtN - i0;                          // first j that wraps
    const int f0 = i0 + kMtM < kMtN ? i0 + kMtM : i0 + kMtM - kMtN;  // far word of j = 0
    const uint64_t* const frow = mt + 32 * f0;
    const uint64_t* const frow_w = frow - 32 * kMtN;
    const int fwrap = kMtN - f0;
    if (wrap > NDRAW && fwrap >= NDRAW) {  // warp-uniform: no word of the batch wraps (24 moves in 26)
#pragma unroll
        for (int j = 0; j <= NDRAW; ++j) b.cur[j] = row[32 * j];
#pragma unroll
        for (int j = 0; j < NDRAW; ++j) b.far[j] = frow[32 * j];
        return;
    }
#pragma unroll
    for (int j = 0; j <= NDRAW; ++j) b.cur[j] = (j < wrap ? row : row_w)[32 * j];
#pragma unroll
    for (int j = 0; j < NDRAW; ++j) b.far[j] = (j < fwrap ? frow : frow_w)[32 * j];
}

template <int NDRAW>
__device__ __forceinline__ void mt_finish(uint64_t* __restrict__ mt, int i0, const MtBatch<NDRAW>& b, double* out) {
    uint64_t* const row = mt + 32 * i0;
    uint64_t* const row_w = row - 32 * kMtN;
    const int wrap = kMtN - i0;
#pragma unroll
    for (int j = 0; j < NDRAW; ++j) {
        const uint64_t v = mt_twist_word(b.cur[j], b.cur[j + 1], b.far[j]);
        (j < wrap ? row : row_w)[32 * j] = v;
        out[j] = to_uniform01(mt_temper(v));
    }
}

template <int NDRAW>
__device__ __forceinline__ void mt_draw(uint64_t* __restrict__ mt, int i0, double* out) {
    static_assert(NDRAW >= 1 && NDRAW < kMtM, "batch must not reach its own far words");
    SG_CHECK(i0 >= 0 && i0 < kMtN);
    uint64_t* const row = mt + 32 * i0;
    uint64_t* const row_w = row - 32 * kMtN;
    const int wrap = kMtN - i0;
    const int f0 = i0 + kMtM < kMtN ? i0 + kMtM : i0 + kMtM - kMtN;
    uint64_t* const frow = mt + 32 * f0;
    uint64_t* const frow_w = frow - 32 * kMtN;
    const int fwrap = kMtN - f0;
    uint64_t cur[NDRAW + 1];
    uint64_t far[NDRAW];
    if (wrap > NDRAW && fwrap >= NDRAW) {  // warp-uniform: no word of the batch wraps (24 moves in 26)
#pragma unroll
        for (int j = 0; j <= NDRAW; ++j) cur[j] = row[32 * j];
#pragma unroll
        for (int j = 0; j < NDRAW; ++j) far[j] = frow[32 * j];
#pragma unroll
        for (int j = 0; j < NDRAW; ++j) {
            const uint64_t v = mt_twist_word(cur[j], cur[j + 1], far[j]);
            row[32 * j] = v;
            out[j] = to_uniform01(mt_temper(v));
        }
        return;
    }
#pragma unroll
    for (int j = 0; j <= NDRAW; ++j) cur[j] = (j < wrap ? row : row_w)[32 * j];
#pragma unroll
    for (int j = 0; j < NDRAW; ++j) far[j] = (j < fwrap ? frow : frow_w)[32 * j];
#pragma unroll
    for (int j = 0; j < NDRAW; ++j) {
        const uint64_t v = mt_twist_word(cur[j], cur[j + 1], far[j]);
        (j < wrap ? row : row_w)[32 * j] = v;
        out[j] = to_uniform01(mt_temper(v));
    }
}

// Engine word where iteration it's move starts (it >= 1): 6 draws at
// Swarm::Swarm, then 12 per move_particles (pso.cpp:65-69, 114-115).
__host__ __device__ __forceinline__ int move_draw_word(uint64_t it) {
    return static_cast<int>((6 + 12 * ((it - 1) % 26)) % kMtN);
}

// First `n` (<= 156) outputs of mt19937_64(seed) without materialising the
// state: generation-1 word i needs seeded words i, i+1 and i+156 only.
template <int NDRAW>
__device__ __forceinline__ void mt_first_uniforms(uint64_t seed, double* out) {
    static_assert(NDRAW <= 155, "needs words i+1 and i+156 of the seeded state");
    uint64_t lowv[NDRAW + 1];
    uint64_t farv[NDRAW];
    uint64_t x = seed;
#pragma unroll
    for (int i = 0; i <= kMtM + NDRAW - 1; ++i) {
        if (i > 0) x = kMtF * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
        if (i <= NDRAW) lowv[i] = x;
        if (i >= kMtM) farv[i - kMtM] = x;
    }
#pragma unroll
    for (int j = 0; j < NDRAW; ++j) out[j] = to_uniform01(mt_temper(mt_twist_word(lowv[j], lowv[j + 1], farv[j])));
}

}  // namespace sirdgpu
