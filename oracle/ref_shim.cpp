// ref_shim.cpp — extern "C" adapter over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE (see oracle/oracle.h).  oracle/Makefile compiles this
// file together with /root/reference/proj/src/*.cpp (read in place, never
// copied) into oracle/_ref/libsirdref.so.  Every function forwards to the
// reference API it names; none re-implements arithmetic.  The extra ref_*
// entry points exist for fixture generation and the reference bench arm.

#include "oracle.h"

#include "sirdfit/calibration.hpp"
#include "sirdfit/csv.hpp"
#include "sirdfit/errors.hpp"
#include "sirdfit/model.hpp"
#include "sirdfit/objectives.hpp"
#include "sirdfit/pso.hpp"
#include "sirdfit/timeseries.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <span>
#include <string>
#include <vector>

using namespace sirdfit;

namespace {

thread_local std::string g_last_error;

int status_of(const std::exception& e) {
    g_last_error = e.what();
    if (dynamic_cast<const AllInfeasibleError*>(&e)) return 4;
    if (dynamic_cast<const InsufficientPopulationError*>(&e)) return 3;
    if (dynamic_cast<const NonFiniteError*>(&e)) return 5;
    if (dynamic_cast<const SchemeError*>(&e)) return 2;
    return 1;
}

ObjectiveSpec spec_of(int family, int metric) {
    return ObjectiveSpec{family == 0 ? Family::DOnly : Family::IRDJoint, static_cast<Metric>(metric)};
}

SirdState state_of(const double* s) { return SirdState{.S = s[0], .I = s[1], .R = s[2], .D = s[3]}; }

void write_states(const Trajectory& tr, double* out) {
    for (std::size_t k = 0; k < tr.states.size(); ++k) {
        out[4 * k + 0] = tr.states[k].S;
        out[4 * k + 1] = tr.states[k].I;
        out[4 * k + 2] = tr.states[k].R;
        out[4 * k + 3] = tr.states[k].D;
    }
}

EpiSeries series_of(const double* I, const double* R, const double* D, std::size_t n) {
    EpiSeries epi;
    epi.infectious.assign(I, I + n);
    epi.recovered_cum.assign(R, R + n);
    epi.deaths_cum.assign(D, D + n);
    epi.new_cases.assign(n, 0.0);
    return epi;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

uint64_t oracle_mix_seed(uint64_t base, uint64_t index) { return mix_seed(base, index); }

void oracle_mt_raw(uint64_t seed, uint64_t skip, size_t n, uint64_t* out) {
    std::mt19937_64 engine(seed);
    engine.discard(skip);
    for (size_t k = 0; k < n; ++k) out[k] = engine();
}

void oracle_uniform01(uint64_t seed, size_t n, double* out) {
    std::mt19937_64 engine(seed);
    for (size_t k = 0; k < n; ++k) out[k] = uniform01(engine);
}

int oracle_integrate(const double* p, const double* init4, double population, int n_days, int substeps,
                     double* states, int* finite) {
    try {
        const SirdParams params = params_from_position(std::span<const double>(p, 6));
        const Trajectory tr = integrate_euler(params, state_of(init4), population, n_days, substeps);
        write_states(tr, states);
        *finite = tr.finite ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int oracle_eval_costs(int family, int metric, const double* I, const double* R, const double* D, int n_days,
                      const double* init4, double population, int substeps, int n_threads,
                      const double* positions, size_t n, double* costs) {
    try {
        const WindowSlice slice{std::span<const double>(I, n_days), std::span<const double>(R, n_days),
                                std::span<const double>(D, n_days)};
        const BatchObjective objective = make_window_objective(spec_of(family, metric), slice, state_of(init4),
                                                               population, substeps, n_threads);
        objective(std::span<const double>(positions, n * 6), 6, std::span<double>(costs, n));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int oracle_fit_swarm(int family, int metric, const double* I, const double* R, const double* D, int n_days,
                     const double* init4, double population, int substeps, int n_threads, const double* lower6,
                     const double* upper6, uint64_t n_particles, uint64_t max_iters, double inertia,
                     double cognitive, double social, uint64_t seed, int repair, double* best6, double* best_cost,
                     double* history) {
    try {
        const WindowSlice slice{std::span<const double>(I, n_days), std::span<const double>(R, n_days),
                                std::span<const double>(D, n_days)};
        const BatchObjective objective = make_window_objective(spec_of(family, metric), slice, state_of(init4),
                                                               population, substeps, n_threads);
        PsoConfig config;
        config.n_particles = n_particles;
        config.max_iters = max_iters;
        config.inertia = inertia;
        config.cognitive = cognitive;
        config.social = social;
        config.seed = seed;
        const SearchBounds bounds{std::vector<double>(lower6, lower6 + 6), std::vector<double>(upper6, upper6 + 6)};
        // optimize() (pso.cpp:129-143) driven through the public Swarm API so
        // the history is available even when the swarm ends all-infeasible.
        Swarm swarm(config, bounds, repair ? RepairHook(repair_time_order) : RepairHook{});
        for (uint64_t it = 0; it < max_iters; ++it) {
            history[it] = swarm.step(objective);
        }
        const std::span<const double> best = swarm.best_position();
        std::copy(best.begin(), best.end(), best6);
        *best_cost = swarm.best_cost();
        if (!(swarm.best_cost() < std::numeric_limits<double>::infinity())) {
            g_last_error = AllInfeasibleError{}.what();
            return 4;
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int oracle_forecast(const double* p, const double* junction4, double population, int horizon, int substeps,
                    double* states, int* finite) {
    // forecast_extension needs a FitResult; build the minimal one it reads
    // (calibration.cpp:298-322: ok, trajectory.states.back(), population).
    try {
        FitResult fit;
        fit.ok = true;
        fit.params = params_from_position(std::span<const double>(p, 6));
        fit.trajectory.population = population;
        fit.trajectory.finite = true;
        fit.trajectory.states.push_back(state_of(junction4));
        fit.window = Window{.index = 0, .start = 0, .length = 1};
        const Forecast fc = forecast_extension(fit, static_cast<std::size_t>(horizon), substeps);
        write_states(fc.trajectory, states);
        *finite = 1;
        return 0;
    } catch (const NonFiniteError& e) {
        // forecast_extension throws on blow-up; report it as data like
        // oracle_integrate does, with the trajectory the integrator produced.
        const SirdParams held{.beta1 = p[1], .beta2 = p[1], .t1 = 0.0, .t2 = 0.0, .gamma = p[4], .mu = p[5]};
        const Trajectory tr = integrate_euler(held, state_of(junction4), population, horizon + 1, substeps);
        write_states(tr, states);
        *finite = 0;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// ---- reference-only entry points ------------------------------------------

// fit_window (calibration.cpp:157-188) on a series given as three columns.
// bounds7 = {beta_lo, beta_hi, gamma_lo, gamma_hi, mu_lo, mu_hi, t_margin}.
int ref_fit_window(const double* I, const double* R, const double* D, size_t n_series, size_t start,
                   size_t length, int family, int metric, const double* bounds7, double population, int substeps,
                   int n_threads, uint64_t n_particles, uint64_t max_iters, double inertia, double cognitive,
                   double social, uint64_t seed, double* best6, double* objective, double* r2, double* traj,
                   int* finite) {
    try {
        const EpiSeries epi = series_of(I, R, D, n_series);
        FitSettings settings;
        settings.spec = spec_of(family, metric);
        settings.bounds = ParamBounds{.beta_lo = bounds7[0], .beta_hi = bounds7[1], .gamma_lo = bounds7[2],
                                      .gamma_hi = bounds7[3], .mu_lo = bounds7[4], .mu_hi = bounds7[5],
                                      .t_margin = static_cast<std::size_t>(bounds7[6])};
        settings.population = population;
        settings.substeps = substeps;
        settings.n_threads = n_threads;
        settings.pso.n_particles = n_particles;
        settings.pso.max_iters = max_iters;
        settings.pso.inertia = inertia;
        settings.pso.cognitive = cognitive;
        settings.pso.social = social;
        const FitResult fit = fit_window(epi, Window{.index = 0, .start = start, .length = length}, settings, seed);
        const double p[6] = {fit.params.beta1, fit.params.beta2, fit.params.t1,
                             fit.params.t2,    fit.params.gamma, fit.params.mu};
        std::memcpy(best6, p, sizeof p);
        *objective = fit.objective;
        *r2 = fit.r2_d;
        write_states(fit.trajectory, traj);
        *finite = fit.trajectory.finite ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// fit_all_windows (calibration.cpp:190-216).  Per window w (count from
// make_windows): ok[w], best6[w*6..], objective[w], r2[w]; returns count in
// *n_windows (arrays must hold max_windows entries).
int ref_fit_all_windows(const double* I, const double* R, const double* D, size_t n_series, size_t tau,
                        size_t delta, int family, int metric, const double* bounds7, double population,
                        int substeps, int n_threads, uint64_t n_particles, uint64_t max_iters, double inertia,
                        double cognitive, double social, uint64_t base_seed, size_t max_windows,
                        size_t* n_windows, int* ok, double* best6, double* objective, double* r2,
                        double* mean_r2, size_t* failed) {
    try {
        const EpiSeries epi = series_of(I, R, D, n_series);
        FitSettings settings;
        settings.spec = spec_of(family, metric);
        settings.bounds = ParamBounds{.beta_lo = bounds7[0], .beta_hi = bounds7[1], .gamma_lo = bounds7[2],
                                      .gamma_hi = bounds7[3], .mu_lo = bounds7[4], .mu_hi = bounds7[5],
                                      .t_margin = static_cast<std::size_t>(bounds7[6])};
        settings.population = population;
        settings.substeps = substeps;
        settings.n_threads = n_threads;
        settings.pso.n_particles = n_particles;
        settings.pso.max_iters = max_iters;
        settings.pso.inertia = inertia;
        settings.pso.cognitive = cognitive;
        settings.pso.social = social;
        const FitAllResult all = fit_all_windows(epi, WindowScheme{.tau = tau, .delta = delta}, settings, base_seed);
        *n_windows = all.fits.size();
        if (all.fits.size() > max_windows) return 1;
        for (std::size_t w = 0; w < all.fits.size(); ++w) {
            const FitResult& f = all.fits[w];
            ok[w] = f.ok ? 1 : 0;
            const double p[6] = {f.params.beta1, f.params.beta2, f.params.t1, f.params.t2, f.params.gamma, f.params.mu};
            std::memcpy(best6 + 6 * w, p, sizeof p);
            objective[w] = f.objective;
            r2[w] = f.r2_d;
        }
        *mean_r2 = all.mean_r2_d;
        *failed = all.failed_count;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// stability_study (calibration.cpp:378-436) in the layout of
// sg_stability_study_series (include/sirdgpu.h): per repetition ok/params/
// objective; 5 day-band blocks x 7 rows; day counts; gamma/mu scalar bands.
int ref_stability_study(const double* I, const double* R, const double* D, size_t n_series, size_t start,
                        size_t length, int family, int metric, const double* bounds7, double population,
                        int substeps, uint64_t n_particles, uint64_t max_iters, double inertia, double cognitive,
                        double social, uint64_t repetitions, uint64_t horizon, uint64_t base_seed, int* ok,
                        double* params, double* objective, double* day_bands, uint64_t* day_counts,
                        double* scalar_bands, uint64_t* scalar_counts, uint64_t* failed) {
    try {
        const EpiSeries epi = series_of(I, R, D, n_series);
        FitSettings settings;
        settings.spec = spec_of(family, metric);
        settings.bounds = ParamBounds{.beta_lo = bounds7[0], .beta_hi = bounds7[1], .gamma_lo = bounds7[2],
                                      .gamma_hi = bounds7[3], .mu_lo = bounds7[4], .mu_hi = bounds7[5],
                                      .t_margin = static_cast<std::size_t>(bounds7[6])};
        settings.population = population;
        settings.substeps = substeps;
        settings.pso.n_particles = n_particles;
        settings.pso.max_iters = max_iters;
        settings.pso.inertia = inertia;
        settings.pso.cognitive = cognitive;
        settings.pso.social = social;
        const StabilityResult st = stability_study(epi, Window{.index = 0, .start = start, .length = length},
                                                   settings, repetitions, horizon, base_seed);
        for (std::size_t r = 0; r < st.fits.size(); ++r) {
            const FitResult& f = st.fits[r];
            ok[r] = f.ok ? 1 : 0;
            const double p[6] = {f.params.beta1, f.params.beta2, f.params.t1, f.params.t2, f.params.gamma, f.params.mu};
            std::memcpy(params + 6 * r, p, sizeof p);
            objective[r] = f.objective;
        }
        double* out = day_bands;
        uint64_t* cnt = day_counts;
        for (const QuantileBands* b : {&st.beta, &st.r0, &st.infectious, &st.recovered, &st.deaths}) {
            const std::size_t n = b->days();
            for (const std::vector<double>* v : {&b->median, &b->p50_lo, &b->p50_hi, &b->p90_lo, &b->p90_hi,
                                                 &b->p95_lo, &b->p95_hi}) {
                std::copy(v->begin(), v->end(), out);
                out += n;
            }
            for (std::size_t d = 0; d < n; ++d) *cnt++ = b->count[d];
        }
        const ScalarBands* sb[2] = {&st.gamma, &st.mu};
        for (int k = 0; k < 2; ++k) {
            const double v[7] = {sb[k]->median, sb[k]->p50_lo, sb[k]->p50_hi, sb[k]->p90_lo,
                                 sb[k]->p90_hi, sb[k]->p95_lo, sb[k]->p95_hi};
            std::copy(v, v + 7, scalar_bands + 7 * k);
            scalar_counts[k] = sb[k]->count;
        }
        *failed = st.failed;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// forecast_extension (calibration.cpp:298-322) of a fit_window result.
int ref_fit_window_forecast(const double* I, const double* R, const double* D, size_t n_series, size_t start,
                            size_t length, int family, int metric, const double* bounds7, double population,
                            int substeps, uint64_t n_particles, uint64_t max_iters, uint64_t seed, uint64_t horizon,
                            double* states) {
    try {
        const EpiSeries epi = series_of(I, R, D, n_series);
        FitSettings settings;
        settings.spec = spec_of(family, metric);
        settings.bounds = ParamBounds{.beta_lo = bounds7[0], .beta_hi = bounds7[1], .gamma_lo = bounds7[2],
                                      .gamma_hi = bounds7[3], .mu_lo = bounds7[4], .mu_hi = bounds7[5],
                                      .t_margin = static_cast<std::size_t>(bounds7[6])};
        settings.population = population;
        settings.substeps = substeps;
        settings.pso.n_particles = n_particles;
        settings.pso.max_iters = max_iters;
        const FitResult fit = fit_window(epi, Window{.index = 0, .start = start, .length = length}, settings, seed);
        const Forecast fc = forecast_extension(fit, horizon, substeps);
        write_states(fc.trajectory, states);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// format_double (csv.cpp:84-94) into buf (>= 32 bytes).
void ref_format_double(double v, char* buf) {
    const std::string s = format_double(v);
    std::memcpy(buf, s.c_str(), s.size() + 1);
}

// build_epi_series (+ smooth7) from raw rows with optional cells (NaN =
// missing) and day offsets from 2020-03-18; stats = {interpolated,
// negative, outflow}.  Outputs hold max_days values; *n_out the series length.
int ref_clean_raw(const int* day_offset, const double* c, const double* r, const double* d, size_t n_rows, int smooth,
                  size_t max_days, double* I, double* R, double* D, double* new_cases, size_t* n_out,
                  uint64_t* stats) {
    try {
        RawSeries raw;
        for (std::size_t k = 0; k < n_rows; ++k) {
            RawRecord rec;
            rec.date = Date{std::chrono::days(18339 + day_offset[k])};
            if (!std::isnan(c[k])) rec.confirmed_cum = c[k];
            if (!std::isnan(r[k])) rec.recovered_cum = r[k];
            if (!std::isnan(d[k])) rec.deaths_cum = d[k];
            raw.records.push_back(rec);
        }
        CleaningStats st;
        EpiSeries epi = build_epi_series(raw, &st);
        if (smooth) epi = smooth7(epi);
        *n_out = epi.size();
        if (epi.size() > max_days) return 1;
        std::copy(epi.infectious.begin(), epi.infectious.end(), I);
        std::copy(epi.recovered_cum.begin(), epi.recovered_cum.end(), R);
        std::copy(epi.deaths_cum.begin(), epi.deaths_cum.end(), D);
        std::copy(epi.new_cases.begin(), epi.new_cases.end(), new_cases);
        stats[0] = st.interpolated_cells;
        stats[1] = st.negative_corrections;
        stats[2] = st.outflow_corrections;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// build_envelope (calibration.cpp:218-245) per day over a row-major
// n_samples x n_days matrix (NaN = no sample).  out: 7 x n_days (outer_lo,
// band1_lo, band2_lo, median, band2_hi, band1_hi, outer_hi); count: n_days.
int ref_build_envelope(const double* values, size_t n_samples, size_t n_days, double* out, size_t* count) {
    try {
        std::vector<std::vector<double>> per_day(n_days);
        for (std::size_t s = 0; s < n_samples; ++s)
            for (std::size_t d = 0; d < n_days; ++d) per_day[d].push_back(values[s * n_days + d]);
        const Envelope e = build_envelope(per_day);
        for (std::size_t d = 0; d < n_days; ++d) {
            const double v[7] = {e.outer_lo[d], e.band1_lo[d], e.band2_lo[d], e.median[d],
                                 e.band2_hi[d], e.band1_hi[d], e.outer_hi[d]};
            for (int k = 0; k < 7; ++k) out[k * n_days + d] = v[k];
            count[d] = e.count[d];
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Cleaning pipeline for fixture generation: build_epi_series then smooth7
// (timeseries.cpp:127-179).  Raw rows are daily (no gaps), cumulative.
// Output columns have n values each.
int ref_clean_series(const double* confirmed, const double* recovered, const double* deaths, size_t n,
                     int smooth, double* I, double* R, double* D, double* new_cases) {
    try {
        RawSeries raw;
        raw.records.resize(n);
        for (std::size_t t = 0; t < n; ++t) {
            raw.records[t].date = Date{std::chrono::days(18339 + static_cast<int>(t))};
            raw.records[t].confirmed_cum = confirmed[t];
            raw.records[t].recovered_cum = recovered[t];
            raw.records[t].deaths_cum = deaths[t];
        }
        EpiSeries epi = build_epi_series(raw);
        if (smooth) epi = smooth7(epi);
        if (epi.size() != n) return 1;
        std::copy(epi.infectious.begin(), epi.infectious.end(), I);
        std::copy(epi.recovered_cum.begin(), epi.recovered_cum.end(), R);
        std::copy(epi.deaths_cum.begin(), epi.deaths_cum.end(), D);
        std::copy(epi.new_cases.begin(), epi.new_cases.end(), new_cases);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// build_quantile_bands (calibration.cpp:337-361) over n_days columns of a
// row-major n_samples x n_days matrix.  out: 7 x n_days
// (median, p50_lo, p50_hi, p90_lo, p90_hi, p95_lo, p95_hi); count: n_days.
int ref_quantile_bands(const double* values, size_t n_samples, size_t n_days, double* out, size_t* count) {
    try {
        std::vector<std::vector<double>> per_day(n_days);
        for (std::size_t s = 0; s < n_samples; ++s)
            for (std::size_t d = 0; d < n_days; ++d) per_day[d].push_back(values[s * n_days + d]);
        const QuantileBands b = build_quantile_bands(per_day);
        for (std::size_t d = 0; d < n_days; ++d) {
            out[0 * n_days + d] = b.median[d];
            out[1 * n_days + d] = b.p50_lo[d];
            out[2 * n_days + d] = b.p50_hi[d];
            out[3 * n_days + d] = b.p90_lo[d];
            out[4 * n_days + d] = b.p90_hi[d];
            out[5 * n_days + d] = b.p95_lo[d];
            out[6 * n_days + d] = b.p95_hi[d];
            count[d] = b.count[d];
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

} // extern "C"
