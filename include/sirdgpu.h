/*
 * sirdgpu.h — C-ABI of the B200 particle-window cost engine.
 *
 * This is the drop-in boundary for the reference's hot path (sirdfit, arXiv
 * 2204.12346, /root/reference/proj).  Every entry point below replaces one
 * reference interface; the citation after each declaration names it.
 *
 *   boundary 1 (cost only):   sirdfit::make_window_objective -> BatchObjective
 *                             (include/sirdfit/calibration.hpp:84-85,
 *                              src/calibration.cpp:120-155, pso.hpp:36-37)
 *   boundary 2 (optimizer):   sirdfit::optimize / fit_window / fit_all_windows /
 *                             stability_study / forecast_extension
 *                             (pso.hpp:92-93, calibration.hpp:89-100, 143, 188-189)
 *
 * Conventions
 *   - Plain C: POD structs, pointers and sizes; no torch or C++ types.
 *   - Every function returns an sg_status (0 = OK).  The text of the last
 *     error of a context is available from sg_last_error().  Status codes map
 *     one-to-one onto the reference's exception types (errors.hpp:8-50).
 *   - Host buffers are caller-owned and are fully consumed / filled before the
 *     call returns.  Device memory is owned by the context.
 *   - One context per device, shareable between host threads: every entry
 *     point serialises on a per-context lock (the reference's objectives and
 *     fit_window are reentrant), and sg_last_error() returns the calling
 *     thread's last error on that context.  Different contexts (devices)
 *     run concurrently.
 *   - Numerical blow-up is data, not an error: a particle whose trajectory
 *     leaves the finite range costs +inf (model.hpp:34-36,
 *     objectives.cpp:101-103), exactly as in the reference.
 *   - Results are bit-identical to the reference C++ built without FMA
 *     contraction (the reference object code has none).
 */
#ifndef SIRDGPU_H
#define SIRDGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 1

/* Status codes.  The C++ layer (sirdfit_b200.hpp) rethrows them as the
 * reference's exception classes (errors.hpp:8-50). */
typedef enum sg_status {
    SG_OK = 0,
    SG_ERR_INVALID_ARGUMENT = 1,        /* sirdfit::Error (e.g. calibration.cpp:141-143)   */
    SG_ERR_SCHEME = 2,                  /* sirdfit::SchemeError (calibration.cpp:39-44)    */
    SG_ERR_INSUFFICIENT_POPULATION = 3, /* InsufficientPopulationError (calibration.cpp:113)*/
    SG_ERR_ALL_INFEASIBLE = 4,          /* AllInfeasibleError (pso.cpp:137-139)            */
    SG_ERR_NON_FINITE = 5,              /* NonFiniteError (calibration.cpp:302, 318-320)   */
    SG_ERR_CUDA = 6,                    /* device failure (no reference counterpart)      */
    SG_ERR_NO_DEVICE = 7,               /* no sm_100 device / extension cannot run        */
    SG_ERR_OUT_OF_MEMORY = 8            /* device allocation failed                       */
} sg_status;

/* sirdfit::Family / sirdfit::Metric (objectives.hpp:12-13) */
enum { SG_FAMILY_D_ONLY = 0, SG_FAMILY_IRD_JOINT = 1 };
enum { SG_METRIC_MXSE = 0, SG_METRIC_MSE = 1, SG_METRIC_MAE = 2, SG_METRIC_MAPE = 3 };

/* sirdfit::SirdState (model.hpp:25-32) */
typedef struct sg_state {
    double S, I, R, D;
} sg_state;

typedef struct sg_ctx sg_ctx;
typedef struct sg_window sg_window;

int sg_abi_version(void);

/* --- context ------------------------------------------------------------ */
int sg_ctx_create(int device, sg_ctx** out);
void sg_ctx_destroy(sg_ctx* ctx);
const char* sg_last_error(const sg_ctx* ctx);
/* Number of CUDA kernels this context has launched (telemetry for bench). */
uint64_t sg_ctx_launch_count(const sg_ctx* ctx);
/* Host->device and device->host bytes copied by this context's calls so far
 * (telemetry for bench: the e2e transfer volume, counted at every copy). */
void sg_ctx_copy_bytes(const sg_ctx* ctx, uint64_t* h2d, uint64_t* d2h);

/* Band telemetry of the context's C5 calls (cumulative): forecast days
 * whose quantiles were resolved from the ensemble kernel's fused histogram
 * (bins predicted from the slot's previous window), days that took the
 * histogram pass over the deaths plane, and the ramp substeps of the
 * evaluated windows (the roofline's ramp credit, as sg_plan_ramp_substeps).
 * Any pointer may be NULL.  Synchronises the stream. */
int sg_ctx_band_stats(sg_ctx* ctx, uint64_t* fused_days, uint64_t* pass_days, uint64_t* ramp_substeps);
/* Underlying cudaStream_t used by every call of this context. */
void* sg_ctx_stream(const sg_ctx* ctx);

/* --- boundary 1: the window objective ------------------------------------
 * sg_window_create replaces the construction half of make_window_objective
 * (calibration.cpp:120-139): it owns copies of the observed slices, the
 * initial state, the population and the substep count, and precomputes the
 * window-constant parts of objective_value (objectives.cpp:61-69: the
 * per-compartment min-max scale; objectives.cpp:41-55: MAPE reciprocals).
 * The three series hold n_days >= 1 values each (the window length, tau+1).
 * Fails with SG_ERR_INVALID_ARGUMENT when integrate_euler would throw
 * (model.cpp:78-80: n_days < 1, substeps < 1, population <= 0). */
int sg_window_create(sg_ctx* ctx, const double* infectious, const double* recovered_cum,
                     const double* deaths_cum, int n_days, sg_state init, double population, int substeps,
                     int family, int metric, sg_window** out);
void sg_window_destroy(sg_window* window);

/* The BatchObjective body (calibration.cpp:140-154): costs[k] =
 * objective_value(spec, slice, integrate_euler(params_from_position(pos[k])))
 * for k < n.  positions is row-major n x dim host memory; dim must be 6. */
int sg_eval_costs(sg_window* window, const double* positions, size_t n, size_t dim, double* costs);

/* Same on device memory (row-major n x 6 doubles -> n doubles) on the given
 * cudaStream_t (NULL = the context stream).  Asynchronous. */
int sg_eval_costs_device(sg_window* window, const double* d_positions, size_t n, double* d_costs,
                         void* cuda_stream);

/* --- integrator -------------------------------------------------------------
 * integrate_batch (model.cpp:116-125) / integrate_euler (model.cpp:76-107):
 * one trajectory per parameter set, row-major params n x 6 in SirdParams
 * order [beta1, beta2, t1, t2, gamma, mu].  states receives n x n_days x 4
 * doubles (S,I,R,D per day, NaN after a blow-up exactly as model.cpp:84-104),
 * finite receives n flags (Trajectory::finite). */
int sg_integrate_batch(sg_ctx* ctx, const double* params, size_t n, sg_state init, double population,
                       int n_days, int substeps, double* states, uint8_t* finite);

/* Same with one initial state per item (inits: n states), as fit_window's
 * final re-integration of every fitted window needs (calibration.cpp:175-176). */
int sg_integrate_states(sg_ctx* ctx, const double* params, const sg_state* inits, size_t n, double population,
                        int n_days, int substeps, double* states, uint8_t* finite);

/* fit_window's finish for n fits on the device (calibration.cpp:175-185):
 * the re-integration of sg_integrate_states plus r_squared_d of the
 * trajectory's D against the observed deaths (objectives.cpp:122-144,
 * observed_d: n x n_days), r2[k] = NaN where the observed series is
 * constant (the ConstantObservedError branch). */
int sg_integrate_states_r2(sg_ctx* ctx, const double* params, const sg_state* inits, const double* observed_d,
                           size_t n, double population, int n_days, int substeps, double* states, uint8_t* finite,
                           double* r2);

/* --- boundary 2: the particle swarm --------------------------------------
 * One descriptor per independent swarm (Swarm::Swarm + optimize,
 * pso.cpp:47-143).  Swarms may use different windows, sizes and seeds;
 * all swarms of one call run concurrently on the device. */
typedef struct sg_swarm_desc {
    const sg_window* window;  /* objective: the window's BatchObjective       */
    double lower[6];          /* SearchBounds (pso.hpp:26-32)                 */
    double upper[6];
    uint64_t n_particles;     /* PsoConfig (pso.hpp:14-23)                    */
    uint64_t max_iters;
    double inertia;
    double cognitive;
    double social;
    uint64_t seed;            /* particle i draws from mt19937_64(mix_seed(seed,i)) */
    int repair_time_order;    /* 1: RepairHook = repair_time_order (calibration.cpp:89-93) */
} sg_swarm_desc;

typedef struct sg_swarm_result {
    double best_position[6];  /* PsoResult::best_position (pso.hpp:50-54)     */
    double best_cost;         /* PsoResult::best_cost                         */
    double* cost_history;     /* caller-owned, max_iters slots, or NULL       */
    int status;               /* SG_OK or SG_ERR_ALL_INFEASIBLE / SG_ERR_INVALID_ARGUMENT */
} sg_swarm_result;

/* Runs every swarm for its max_iters iterations.  Per-swarm failures are
 * reported in results[k].status (the call itself returns SG_OK); a config
 * that PsoConfig::validate / SearchBounds::validate would reject
 * (pso.cpp:16-34) makes that swarm fail with SG_ERR_INVALID_ARGUMENT. */
int sg_fit_swarms(sg_ctx* ctx, const sg_swarm_desc* swarms, size_t n_swarms, sg_swarm_result* results);

/* Reusable plan: the same work as sg_fit_swarms split into setup (validate,
 * allocate, upload descriptors), an asynchronous device run on the context
 * stream (engine seeding + max_iters fused step launches, no host round
 * trips), and result collection.  Lets callers time or graph the device part
 * alone; a plan may be run repeatedly (each run restarts from the seeds).
 * The plan reads its windows' device data at every run: destroy a plan
 * before the windows it was created from (and both before the context). */
typedef struct sg_plan sg_plan;
int sg_plan_create(sg_ctx* ctx, const sg_swarm_desc* swarms, size_t n_swarms, sg_plan** out);
int sg_plan_run(sg_plan* plan);
/* Same as sg_plan_run, synchronous, and reports device time measured with
 * CUDA events on the context stream: *seed_ms for the engine-seeding
 * launches, *steps_ms for all fused step launches (max_iters per group). */
int sg_plan_run_timed(sg_plan* plan, double* seed_ms, double* steps_ms);
int sg_plan_results(sg_plan* plan, sg_swarm_result* results);
uint64_t sg_plan_evals(const sg_plan* plan);  /* sum of n_particles * max_iters */
uint64_t sg_plan_step_launches(const sg_plan* plan);  /* fused step launches per run */
/* Ramp substeps evaluated by the last run (beta in its linear ramp,
 * model.cpp:62-63): the R_ramp term of the algorithmic FP64 operation count
 * (DESIGN.md §5).  Synchronous; 0 before the first run. */
uint64_t sg_plan_ramp_substeps(sg_plan* plan);
void sg_plan_destroy(sg_plan* plan);

/* --- the general swarm: Swarm / optimize for any objective -----------------
 * Swarm (pso.hpp:56-86, pso.cpp:47-127) of any dimension with its state in
 * device memory: positions, velocities and personal bests row-major n x dim,
 * one mt19937_64(mix_seed(seed, i)) per particle.  A step is: put the costs
 * of the current positions (sg_gswarm_set_costs from a host objective, or
 * sg_gswarm_eval_window for a window objective, evaluated on the device),
 * then sg_gswarm_step = personal bests, global best, move (+ repair when
 * repair_time_order).  An arbitrary host repair hook is applied by the caller
 * between steps through get/set_positions.  Bit-identical to the reference's
 * Swarm for the same seeds.  (The fused many-swarm plans above are the fast
 * path for window objectives.) */
typedef struct sg_gswarm sg_gswarm;
int sg_gswarm_create(sg_ctx* ctx, int dim, const double* lower, const double* upper, uint64_t n_particles,
                     double inertia, double cognitive, double social, uint64_t seed, int repair_time_order,
                     sg_gswarm** out);
void sg_gswarm_destroy(sg_gswarm* swarm);
const double* sg_gswarm_positions_device(const sg_gswarm* swarm);  /* n x dim, row-major */
double* sg_gswarm_costs_device(sg_gswarm* swarm);                  /* n                    */
int sg_gswarm_get_positions(sg_gswarm* swarm, double* positions);  /* n x dim host copy    */
int sg_gswarm_set_positions(sg_gswarm* swarm, const double* positions);
/* Initial positions after a host repair hook: also resets the personal-best
 * positions to them (Swarm::Swarm repairs before pbest = x, pso.cpp:70-74). */
int sg_gswarm_set_initial_positions(sg_gswarm* swarm, const double* positions);
int sg_gswarm_set_costs(sg_gswarm* swarm, const double* costs);
int sg_gswarm_eval_window(sg_gswarm* swarm, sg_window* window);   /* dim 6: costs on the device */
/* pso.cpp:83-98 (everything of Swarm::step after the objective); *best_cost
 * (optional) receives best_cost_ after the step. */
int sg_gswarm_step(sg_gswarm* swarm, double* best_cost);
int sg_gswarm_best(sg_gswarm* swarm, double* best_position, double* best_cost);

/* --- scoring of given trajectories ---------------------------------------
 * objective_value (objectives.cpp:95-120) of n trajectories (states: n x
 * n_days x 4; finite: n flags or NULL) against one observed window (three
 * series of n_days), on the device. */
int sg_objective_values(sg_ctx* ctx, int family, int metric, const double* infectious, const double* recovered_cum,
                        const double* deaths_cum, size_t n_days, const double* states, const uint8_t* finite, size_t n,
                        double* costs);
/* metric_value (objectives.cpp:72-81) of n series pairs (observed,
 * predicted: n x n_days each). */
int sg_metric_values(sg_ctx* ctx, int metric, const double* observed, const double* predicted, size_t n_days,
                     size_t n, double* out);
/* sird_rhs (model.cpp:66-74) for n (state, beta, gamma, mu) at one population. */
int sg_sird_rhs_batch(sg_ctx* ctx, const sg_state* states, const double* beta, const double* gamma, const double* mu,
                      double population, size_t n, sg_state* out);

/* --- forecast ---------------------------------------------------------------
 * forecast_extension (calibration.cpp:298-322), batched: for each k, holds
 * beta = beta2 and integrates horizon+1 days from junction[k] (the fitted
 * window's last state).  states receives n x (horizon+1) x 4; finite n flags
 * (a blow-up is NonFiniteError in the reference: the caller decides). */
int sg_forecast_batch(sg_ctx* ctx, const double* params, const sg_state* junction, size_t n,
                      double population, int horizon, int substeps, double* states, uint8_t* finite);

/* Forecast-scenario ensemble on one window: n parameter sets drawn exactly
 * like the Swarm's initial sample (pso.cpp:55-73 + repair_time_order:
 * set k = 6 uniform01 draws of mt19937_64(mix_seed(seed, k))), each
 * integrated over the window and then `horizon` days with beta held at beta2
 * (calibration.cpp:305-317).  Writes the window cost of each set (costs, n,
 * optional), the parameter sets (params_out, n x 6, optional) and the deaths
 * series of the forecast (deaths_out, n x (horizon+1), day 0 = junction;
 * NaN rows for sets whose window or forecast blew up). */
int sg_forecast_ensemble(sg_window* window, const double lower[6], const double upper[6], uint64_t seed,
                         size_t n, int horizon, double* costs, double* params_out, double* deaths_out);

/* --- calibration layer (C++ host side, src: csrc/host_api.cpp) --------------
 * The reference's window scheduler / restart driver as C entry points, for
 * bindings (Python, CLI).  They run the C++ API of include/sirdfit_b200.hpp
 * on the given context.  Series are the cleaned EpiSeries columns
 * (timeseries.hpp:37-46) of n_series days. */
typedef struct sg_fit_settings {  /* FitSettings (calibration.hpp:58-65) */
    int family, metric;           /* ObjectiveSpec                            */
    double beta_lo, beta_hi, gamma_lo, gamma_hi, mu_lo, mu_hi;  /* ParamBounds */
    uint64_t t_margin;
    uint64_t n_particles, max_iters;  /* PsoConfig                            */
    double inertia, cognitive, social;
    double population;
    int substeps;
} sg_fit_settings;

typedef struct sg_fit_record {    /* FitResult (calibration.hpp:67-76)        */
    uint64_t index, start, length;
    double params[6];             /* beta1, beta2, t1, t2, gamma, mu          */
    double objective;
    double r2_d;
    int ok;
    int status;                   /* sg_status of the failure (0 when ok)     */
    char failure[192];            /* FitResult::failure (truncated)           */
} sg_fit_record;

/* fit_window (calibration.cpp:157-188).  Returns the status of the exception
 * the reference would throw (record->failure holds its message).
 * trajectory: length x 4 doubles or NULL; history: max_iters doubles or NULL. */
int sg_fit_window_series(sg_ctx* ctx, const double* infectious, const double* recovered_cum,
                         const double* deaths_cum, size_t n_series, uint64_t start, uint64_t length,
                         const sg_fit_settings* settings, uint64_t seed, sg_fit_record* record, double* trajectory,
                         double* history);

/* fit_all_windows (calibration.cpp:190-216): window w is fitted with seed
 * mix_seed(base_seed, w); failures are recorded per window.  records holds
 * max_windows entries, trajectories (optional) max_windows x (tau+1) x 4.
 * Returns SG_ERR_SCHEME when make_windows throws. */
int sg_fit_all_windows_series(sg_ctx* ctx, const double* infectious, const double* recovered_cum,
                              const double* deaths_cum, size_t n_series, uint64_t tau, uint64_t delta,
                              const sg_fit_settings* settings, uint64_t base_seed, size_t max_windows,
                              size_t* n_windows, sg_fit_record* records, double* trajectories, double* mean_r2_d,
                              size_t* failed_count);

/* fit_all_windows restricted to windows [first_window, first_window +
 * max_windows) of the scheme — one rank's share of a sweep sharded over GPUs
 * (SURVEY.md §8e): the same windows, seeds mix_seed(base_seed, w) and
 * per-window failure records as the whole sweep (calibration.cpp:190-216),
 * so the shards merged in window order equal sg_fit_all_windows_series.
 * *n_windows receives the number of records written. */
int sg_fit_window_range_series(sg_ctx* ctx, const double* infectious, const double* recovered_cum,
                               const double* deaths_cum, size_t n_series, uint64_t tau, uint64_t delta,
                               const sg_fit_settings* settings, uint64_t base_seed, uint64_t first_window,
                               uint64_t max_windows, size_t* n_windows, sg_fit_record* records,
                               double* trajectories);

/* stability_study (calibration.cpp:378-436): repetitions fits of one window
 * (seeds mix_seed(base_seed, rep)) + forecast_extension(horizon).
 * records: repetitions entries.  day_bands: 5 blocks (beta, r0: length days;
 * infectious, recovered, deaths: length + horizon days), each block 7 rows
 * (median, p50_lo, p50_hi, p90_lo, p90_hi, p95_lo, p95_hi) of its days,
 * laid out consecutively; day_counts: the per-day sample counts of the same
 * 5 blocks; scalar_bands: gamma then mu, 7 values each; scalar_counts: 2. */
int sg_stability_study_series(sg_ctx* ctx, const double* infectious, const double* recovered_cum,
                              const double* deaths_cum, size_t n_series, uint64_t start, uint64_t length,
                              const sg_fit_settings* settings, uint64_t repetitions, uint64_t horizon,
                              uint64_t base_seed, sg_fit_record* records, double* day_bands, uint64_t* day_counts,
                              double* scalar_bands, uint64_t* scalar_counts, uint64_t* failed);

/* --- diagnostics -----------------------------------------------------------
 * Measured FP64 issue rate of this device: a kernel of independent
 * DADD/DMUL chains (no FMA), timed with CUDA events.  *ops_per_s receives
 * double-precision lane operations per second (the roofline denominator of
 * the non-FMA integrate-and-score kernel). */
int sg_probe_fp64_rate(sg_ctx* ctx, double* ops_per_s);

/* The same ensemble reduced on the device to the per-day quantile bands of
 * the forecast deaths — build_quantile_bands (calibration.cpp:337-361) over
 * the n samples of each forecast day, non-finite samples (blown-up sets)
 * dropped as append_finite_sorted does (calibration.cpp:17-25) — so an
 * ensemble of 10^6 sets per window never leaves HBM.  bands: 7 x (horizon+1)
 * doubles, rows median, p50_lo, p50_hi, p90_lo, p90_hi, p95_lo, p95_hi;
 * counts: finite samples per day (horizon+1); costs: n window costs or NULL.
 * n must fit in an int. */
int sg_forecast_ensemble_bands(sg_window* window, const double lower[6], const double upper[6], uint64_t seed,
                               size_t n, int horizon, double* bands, uint64_t* counts, double* costs);

/* build_quantile_bands (calibration.cpp:337-361) of n_days columns of n
 * values each (values: day-major, n_days x n, host), on the device by the
 * same order-statistic selection as the ensemble bands (non-finite values
 * dropped, calibration.cpp:17-25).  bands: 7 x n_days (median, p50_lo,
 * p50_hi, p90_lo, p90_hi, p95_lo, p95_hi); counts: n_days. */
int sg_quantile_bands(sg_ctx* ctx, const double* values, size_t n, int n_days, double* bands, uint64_t* counts);

/* The same for many windows in one call (C5: every window of the sweep):
 * window k uses seeds[k]; bands: n_windows x 7 x (horizon + 1), counts:
 * n_windows x (horizon + 1).  Windows are pipelined on two streams (the
 * band selection at a higher priority), so one window's band selection
 * overlaps the next window's evaluation. */
int sg_forecast_ensemble_bands_batch(sg_window* const* windows, size_t n_windows, const double lower[6],
                                     const double upper[6], const uint64_t* seeds, size_t n, int horizon,
                                     double* bands, uint64_t* counts);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SIRDGPU_H */
