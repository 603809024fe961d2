// sirdfit_b200.hpp — C++ calibration API over the B200 engine.
//
// Mirrors the reference's public C++ surface for the hot path — every
// declaration of /root/reference/proj/include/sirdfit/{model,objectives,pso,
// calibration,errors}.hpp — with the same names, argument meaning and
// exception types, so a caller of the reference's window scheduler / PSO
// driver / cost and forecast entry points can switch namespaces (the
// reference's data-cleaning and CSV headers are outside this path; EpiSeries
// carries the cleaned columns).  Every integration, objective evaluation and
// PSO update runs on the GPU through include/sirdgpu.h (Swarm included, for
// any objective); this layer only slices windows, validates, batches
// independent swarms into one device launch, does the reference's small
// host post-processing (quantiles, envelopes) and turns status codes back
// into exceptions.  Differences from the reference are documented in
// DESIGN.md §2 (threads are ignored: the device decides parallelism; results
// are bit-identical to the reference for any thread count, as the reference
// guarantees itself, README.md:16-19).
#pragma once

#include "sirdgpu.h"

#include <cstddef>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace sirdfit_b200 {

// ---- errors.hpp:8-50 ---------------------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct EmptySeriesError : Error {
    EmptySeriesError() : Error("series has no records") {}
};
struct MissingEndpointError : Error {
    using Error::Error;
};
struct ParseError : Error {
    using Error::Error;
};
struct DegenerateRangeError : Error {
    DegenerateRangeError() : Error("min-max normalization range is zero") {}
};
struct SchemeError : Error {
    using Error::Error;
};
struct DegenerateRatesError : Error {
    DegenerateRatesError() : Error("gamma + mu must be positive") {}
};
struct ConstantObservedError : Error {
    ConstantObservedError() : Error("observed series is constant; R^2 undefined") {}
};
struct AllInfeasibleError : Error {
    AllInfeasibleError() : Error("no particle produced a finite cost") {}
};
struct InsufficientPopulationError : Error {
    using Error::Error;
};
struct NonFiniteError : Error {
    NonFiniteError() : Error("trajectory left the finite range") {}
};
struct DeviceError : Error {
    using Error::Error;
};

// ---- model.hpp ------------------------------------------------------------------
inline constexpr int kDefaultSubsteps = 24;  // model.hpp:12

struct SirdParams {  // model.hpp:16-23
    double beta1 = 0.0, beta2 = 0.0, t1 = 0.0, t2 = 0.0, gamma = 0.0, mu = 0.0;
};

struct SirdState {  // model.hpp:25-32
    double S = 0.0, I = 0.0, R = 0.0, D = 0.0;
    double total() const { return S + I + R + D; }
};

struct Trajectory {  // model.hpp:37-43
    std::vector<SirdState> states;
    double population = 0.0;
    bool finite = true;
    std::size_t days() const { return states.size(); }
};

double beta_at(const SirdParams& params, double t);  // model.cpp:55-64 (host helper)
double basic_reproduction_number(double beta, double gamma, double mu);

// sird_rhs (model.cpp:66-74), on the device (sg_sird_rhs_batch).
SirdState sird_rhs(const SirdState& state, double beta, double gamma, double mu, double population);

// integrate_euler / integrate_batch (model.cpp:76-125), on the device.
Trajectory integrate_euler(const SirdParams& params, const SirdState& init, double population, int n_days,
                           int substeps = kDefaultSubsteps);
void integrate_euler_into(const SirdParams& params, const SirdState& init, double population, int n_days,
                          int substeps, Trajectory& out);
std::vector<Trajectory> integrate_batch(std::span<const SirdParams> batch, const SirdState& init, double population,
                                        int n_days, int substeps = kDefaultSubsteps, int n_threads = 0);

// ---- objectives.hpp ---------------------------------------------------------------
enum class Metric { MXSE, MSE, MAE, MAPE };
enum class Family { DOnly, IRDJoint };

struct ObjectiveSpec {
    Family family = Family::IRDJoint;
    Metric metric = Metric::MXSE;
};

struct WindowSlice {
    std::span<const double> infectious;
    std::span<const double> recovered_cum;
    std::span<const double> deaths_cum;
};

// objectives.cpp:72-120: metric_value and objective_value score on the
// device (sg_metric_values / sg_objective_values); minmax_normalize is the
// reference's elementwise host helper.
double metric_value(Metric metric, std::span<const double> observed, std::span<const double> predicted);
std::vector<double> minmax_normalize(std::span<const double> values, double ref_min, double ref_max);
double objective_value(const ObjectiveSpec& spec, const WindowSlice& observed, const Trajectory& predicted);

double r_squared_d(std::span<const double> observed_d, std::span<const double> predicted_d);
ObjectiveSpec parse_objective(std::string_view name);
std::string objective_name(const ObjectiveSpec& spec);
std::string metric_name(Metric metric);

// ---- pso.hpp ------------------------------------------------------------------------
struct PsoConfig {
    std::size_t n_particles = 10000;
    double inertia = 0.5;
    double cognitive = 0.5;
    double social = 0.5;
    std::size_t max_iters = 100;
    std::uint64_t seed = 0;
    void validate() const;
};

struct SearchBounds {
    std::vector<double> lower;
    std::vector<double> upper;
    std::size_t dim() const { return lower.size(); }
    void validate() const;
};

using BatchObjective =
    std::function<void(std::span<const double> positions, std::size_t dim, std::span<double> costs)>;

using RepairHook = std::function<void(std::span<double> position)>;  // pso.hpp:39-41

std::uint64_t mix_seed(std::uint64_t base, std::uint64_t index);  // pso.cpp:36-41

double uniform01(std::mt19937_64& engine);  // pso.cpp:43-45 (a host engine's draw)

struct PsoResult {
    std::vector<double> best_position;
    double best_cost = 0.0;
    std::vector<double> cost_history;
};

// The BatchObjective make_window_objective returns: a device window (the
// engine evaluates it where the positions live).  Swarm and optimize look
// for it with BatchObjective::target<WindowObjective>().
struct WindowObjective {
    sg_ctx* ctx = nullptr;
    std::shared_ptr<sg_window> window;  // null when the construction inputs were invalid ...
    std::string deferred;               // ... and this error is thrown at the first call (model.cpp:78-80)
    void operator()(std::span<const double> positions, std::size_t dim, std::span<double> costs) const;
};

// Swarm (pso.hpp:56-86) with its state on the device (sg_gswarm): any
// dimension, any objective.  A window objective is evaluated on the device;
// any other BatchObjective is called with the positions (host copy) once per
// step, like the reference calls it (pso.cpp:81).  repair_time_order runs on
// the device; any other RepairHook on the host copy between steps.
class Swarm {
public:
    Swarm(const PsoConfig& config, SearchBounds bounds, RepairHook repair = {});
    ~Swarm();
    Swarm(const Swarm&) = delete;
    Swarm& operator=(const Swarm&) = delete;
    Swarm(Swarm&& other) noexcept;
    Swarm& operator=(Swarm&& other) noexcept;

    double step(const BatchObjective& objective);

    std::size_t n_particles() const { return config_.n_particles; }
    std::size_t dim() const { return bounds_.dim(); }
    std::span<const double> positions() const;
    std::span<const double> best_position() const;
    double best_cost() const { return best_cost_; }
    std::size_t iterations_done() const { return iterations_done_; }

private:
    void apply_host_repair(bool initial);

    PsoConfig config_;
    SearchBounds bounds_;
    RepairHook repair_;
    bool device_repair_ = false;
    sg_gswarm* swarm_ = nullptr;
    std::vector<double> costs_;
    mutable std::vector<double> positions_, best_position_;
    mutable bool positions_fresh_ = false, best_fresh_ = false;
    double best_cost_;
    std::size_t iterations_done_ = 0;
};

// optimize (pso.cpp:129-143).  A window objective with the reference's
// repair (or none) runs as one fused device swarm (sg_fit_swarms); any other
// objective steps a device Swarm.  Results are the reference's bit for bit.
PsoResult optimize(const PsoConfig& config, const SearchBounds& bounds, const BatchObjective& objective,
                   RepairHook repair = {});

// ---- calibration.hpp --------------------------------------------------------------
struct EpiSeries {  // timeseries.hpp:37-46 (dates kept as an opaque day number)
    int start_day = 0;
    std::vector<double> infectious, recovered_cum, deaths_cum, new_cases;
    std::size_t size() const { return infectious.size(); }
};

struct WindowScheme {
    std::size_t tau = 35;
    std::size_t delta = 3;
};

struct Window {
    std::size_t index = 0, start = 0, length = 0;
    std::size_t last_day() const { return start + length - 1; }
};

std::vector<Window> make_windows(std::size_t n_days, const WindowScheme& scheme);

struct ParamBounds {
    double beta_lo = 0.0, beta_hi = 10.0;
    double gamma_lo = 0.0, gamma_hi = 10.0;
    double mu_lo = 0.0, mu_hi = 10.0;
    std::size_t t_margin = 0;
    static ParamBounds stage1();
    static ParamBounds stage2();
    SearchBounds to_search_bounds(std::size_t tau) const;
    bool contains(const SirdParams& params, std::size_t tau) const;
};

SirdParams params_from_position(std::span<const double> position);
void repair_time_order(std::span<double> position);

struct FitSettings {
    ObjectiveSpec spec;
    ParamBounds bounds = ParamBounds::stage2();
    PsoConfig pso;
    double population = 0.0;
    int substeps = kDefaultSubsteps;
    int n_threads = 1;  // accepted for API compatibility; the device decides
};

struct FitResult {
    Window window;
    SirdParams params;
    ObjectiveSpec spec;
    double objective = std::numeric_limits<double>::quiet_NaN();
    double r2_d = std::numeric_limits<double>::quiet_NaN();
    Trajectory trajectory;
    bool ok = false;
    std::string failure;
    std::vector<double> cost_history;  // extension: optimize()'s history
};

WindowSlice slice_window(const EpiSeries& data, const Window& window);
SirdState window_initial_state(const EpiSeries& data, std::size_t day, double population);

// Boundary 1: the BatchObjective runs sg_eval_costs on the device.
BatchObjective make_window_objective(const ObjectiveSpec& spec, const WindowSlice& observed, const SirdState& init,
                                     double population, int substeps, int n_threads);

FitResult fit_window(const EpiSeries& data, const Window& window, const FitSettings& settings, std::uint64_t seed);

struct FitAllResult {
    std::vector<FitResult> fits;
    double mean_r2_d = 0.0;
    std::size_t failed_count = 0;
};

// All windows run as concurrent swarms in one device launch sequence.
FitAllResult fit_all_windows(const EpiSeries& data, const WindowScheme& scheme, const FitSettings& settings,
                             std::uint64_t base_seed);

// Rank envelopes over the overlapping windows (calibration.cpp:218-296):
// host post-processing of the fits, O(windows x days).
struct Envelope {
    std::vector<std::size_t> count;
    std::vector<double> outer_lo, outer_hi;
    std::vector<double> band1_lo, band1_hi;
    std::vector<double> band2_lo, band2_hi;
    std::vector<double> median;
    std::size_t days() const { return count.size(); }
};

Envelope build_envelope(const std::vector<std::vector<double>>& values_per_day);

struct ParameterEnvelopes {
    Envelope beta, gamma, mu, r0;
};

ParameterEnvelopes parameter_envelopes(std::span<const FitResult> fits, std::size_t n_days);

struct CompartmentEnvelopes {
    Envelope infectious, recovered, deaths;
};

CompartmentEnvelopes compartment_envelopes(std::span<const FitResult> fits, std::size_t n_days);

struct Forecast {
    std::size_t junction_day = 0;
    std::size_t horizon = 0;
    Trajectory trajectory;
};

Forecast forecast_extension(const FitResult& fit, std::size_t horizon, int substeps = kDefaultSubsteps);

struct QuantileBands {
    std::vector<std::size_t> count;
    std::vector<double> median, p50_lo, p50_hi, p90_lo, p90_hi, p95_lo, p95_hi;
    std::size_t days() const { return count.size(); }
};

struct ScalarBands {
    std::size_t count = 0;
    double median = 0.0, p50_lo = 0.0, p50_hi = 0.0, p90_lo = 0.0, p90_hi = 0.0, p95_lo = 0.0, p95_hi = 0.0;
};

double quantile_sorted(std::span<const double> sorted, double p);
QuantileBands build_quantile_bands(const std::vector<std::vector<double>>& values_per_day);
ScalarBands build_scalar_bands(std::vector<double> values);

struct StabilityResult {
    Window window;
    std::size_t horizon = 0, repetitions = 0, failed = 0;
    QuantileBands beta, r0, infectious, recovered, deaths;
    ScalarBands gamma, mu;
    std::vector<FitResult> fits;
};

// Repetitions run as concurrent swarms on the device.
StabilityResult stability_study(const EpiSeries& data, const Window& window, const FitSettings& settings,
                                std::size_t repetitions, std::size_t horizon, std::uint64_t base_seed);

// The engine context used by the functions above (one per device, created
// on first use).  select_device() picks the device for this thread.
sg_ctx* engine_context();
void select_device(int device);

}  // namespace sirdfit_b200
