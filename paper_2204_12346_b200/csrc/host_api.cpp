// host_api.cpp — the reference's calibration API (window scheduler, restart
// driver, cost and forecast entry points) over the B200 engine.
//
// Host-side logic only: window slicing and validation in the reference's
// order (so the same exception surfaces), batching of independent swarms into
// one sg_fit_swarms call, status -> exception mapping, and the small O(days)
// post-processing the reference also does on the host (R^2, quantile bands).
// Every SIRD integration and every particle-window cost runs on the device.
// Compiled with -ffp-contract=off like the reference.
#include "sirdfit_b200.hpp"

#include "engine_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>

namespace sirdfit_b200 {

namespace {

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
constexpr double kInf = std::numeric_limits<double>::infinity();

thread_local int t_device = 0;
thread_local sg_ctx* t_override = nullptr;
std::mutex g_ctx_mu;
std::map<int, sg_ctx*>& contexts() {
    static std::map<int, sg_ctx*> m;
    return m;
}

[[noreturn]] void throw_status(int rc, const std::string& msg) {
    switch (rc) {
    case SG_ERR_SCHEME: throw SchemeError(msg);
    case SG_ERR_INSUFFICIENT_POPULATION: throw InsufficientPopulationError(msg);
    case SG_ERR_ALL_INFEASIBLE: throw AllInfeasibleError();
    case SG_ERR_NON_FINITE: throw NonFiniteError();
    case SG_ERR_CUDA:
    case SG_ERR_NO_DEVICE:
    case SG_ERR_OUT_OF_MEMORY: throw DeviceError(msg);
    default: throw Error(msg);
    }
}

void check(sg_ctx* ctx, int rc) {
    if (rc) throw_status(rc, sg_last_error(ctx));
}

struct WindowHandle {
    sg_window* w = nullptr;
    ~WindowHandle() { sg_window_destroy(w); }
};

int family_code(Family f) { return f == Family::DOnly ? SG_FAMILY_D_ONLY : SG_FAMILY_IRD_JOINT; }
int metric_code(Metric m) { return static_cast<int>(m); }

void params_to(const SirdParams& p, double* out) {
    out[0] = p.beta1;
    out[1] = p.beta2;
    out[2] = p.t1;
    out[3] = p.t2;
    out[4] = p.gamma;
    out[5] = p.mu;
}

void states_to_trajectory(const double* states, int n_days, bool finite, double population, Trajectory& out) {
    out.states.resize(static_cast<std::size_t>(n_days));
    for (int d = 0; d < n_days; ++d)
        out.states[static_cast<std::size_t>(d)] =
            SirdState{states[4 * d + 0], states[4 * d + 1], states[4 * d + 2], states[4 * d + 3]};
    out.finite = finite;
    out.population = population;
}

void append_finite_sorted(std::vector<double>& out, const std::vector<double>& values) {  // calibration.cpp:17-25
    out.clear();
    for (const double v : values)
        if (std::isfinite(v)) out.push_back(v);
    std::sort(out.begin(), out.end());
}

}  // namespace

// ---- context -------------------------------------------------------------------------

void select_device(int device) { t_device = device; }

sg_ctx* engine_context() {
    if (t_override) return t_override;
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    auto it = contexts().find(t_device);
    if (it != contexts().end()) return it->second;
    sg_ctx* ctx = nullptr;
    const int rc = sg_ctx_create(t_device, &ctx);
    if (rc) throw DeviceError("no usable sm_100 device " + std::to_string(t_device) + " (status " +
                              std::to_string(rc) + ")");
    contexts()[t_device] = ctx;
    return ctx;
}

// ---- model -----------------------------------------------------------------------------

double beta_at(const SirdParams& p, double t) {  // model.cpp:55-64
    if (t < p.t1) return p.beta1;
    if (t >= p.t2) return p.beta2;
    const double slope = (p.beta2 - p.beta1) / (p.t2 - p.t1);
    return p.beta1 + slope * (t - p.t1);
}

double basic_reproduction_number(double beta, double gamma, double mu) {  // model.cpp:127-133
    const double removal = gamma + mu;
    if (removal <= 0.0) throw DegenerateRatesError{};
    return beta / removal;
}

std::vector<Trajectory> integrate_batch(std::span<const SirdParams> batch, const SirdState& init, double population,
                                        int n_days, int substeps, int /*n_threads*/) {
    if (n_days < 1 || substeps < 1 || !(population > 0.0))  // model.cpp:78-80
        throw Error("integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
    std::vector<Trajectory> out(batch.size());
    if (batch.empty()) return out;
    std::vector<double> params(6 * batch.size());
    for (std::size_t k = 0; k < batch.size(); ++k) params_to(batch[k], params.data() + 6 * k);
    std::vector<double> states(batch.size() * static_cast<std::size_t>(n_days) * 4);
    std::vector<uint8_t> finite(batch.size());
    sg_ctx* ctx = engine_context();
    check(ctx, sg_integrate_batch(ctx, params.data(), batch.size(), sg_state{init.S, init.I, init.R, init.D},
                                  population, n_days, substeps, states.data(), finite.data()));
    for (std::size_t k = 0; k < batch.size(); ++k)
        states_to_trajectory(states.data() + k * n_days * 4, n_days, finite[k] != 0, population, out[k]);
    return out;
}

Trajectory integrate_euler(const SirdParams& params, const SirdState& init, double population, int n_days,
                           int substeps) {
    return std::move(integrate_batch(std::span<const SirdParams>(&params, 1), init, population, n_days, substeps)[0]);
}

void integrate_euler_into(const SirdParams& params, const SirdState& init, double population, int n_days,
                          int substeps, Trajectory& out) {  // model.cpp:76-107
    out = integrate_euler(params, init, population, n_days, substeps);
}

SirdState sird_rhs(const SirdState& state, double beta, double gamma, double mu, double population) {
    const sg_state in{state.S, state.I, state.R, state.D};
    sg_state out{};
    sg_ctx* ctx = engine_context();
    check(ctx, sg_sird_rhs_batch(ctx, &in, &beta, &gamma, &mu, population, 1, &out));
    return SirdState{out.S, out.I, out.R, out.D};
}

// ---- objectives ------------------------------------------------------------------------

double metric_value(Metric metric, std::span<const double> observed, std::span<const double> predicted) {
    if (observed.empty() || observed.size() != predicted.size())  // objectives.cpp:72-81
        throw Error("metric_value: series must be non-empty and of equal length");
    double v = 0.0;
    sg_ctx* ctx = engine_context();
    check(ctx, sg_metric_values(ctx, metric_code(metric), observed.data(), predicted.data(), observed.size(), 1, &v));
    return v;
}

std::vector<double> minmax_normalize(std::span<const double> values, double ref_min, double ref_max) {
    if (!(ref_max > ref_min)) throw DegenerateRangeError{};  // objectives.cpp:83-93
    const double scale = 1.0 / (ref_max - ref_min);
    std::vector<double> out;
    out.reserve(values.size());
    for (const double v : values) out.push_back((v - ref_min) * scale);
    return out;
}

double objective_value(const ObjectiveSpec& spec, const WindowSlice& observed, const Trajectory& predicted) {
    const std::size_t n = observed.deaths_cum.size();  // objectives.cpp:95-120
    if (n == 0 || observed.infectious.size() != n || observed.recovered_cum.size() != n || predicted.days() != n)
        throw Error("objective_value: observed and predicted must cover the same days");
    if (!predicted.finite) return kInf;
    std::vector<double> states(4 * n);
    for (std::size_t d = 0; d < n; ++d) {
        const SirdState& s = predicted.states[d];
        states[4 * d + 0] = s.S;
        states[4 * d + 1] = s.I;
        states[4 * d + 2] = s.R;
        states[4 * d + 3] = s.D;
    }
    double v = 0.0;
    sg_ctx* ctx = engine_context();
    check(ctx, sg_objective_values(ctx, family_code(spec.family), metric_code(spec.metric), observed.infectious.data(),
                                   observed.recovered_cum.data(), observed.deaths_cum.data(), n, states.data(), nullptr,
                                   1, &v));
    return v;
}

double r_squared_d(std::span<const double> observed_d, std::span<const double> predicted_d) {  // objectives.cpp:122-144
    if (observed_d.empty() || observed_d.size() != predicted_d.size())
        throw Error("r_squared_d: series must be non-empty and of equal length");
    double mean = 0.0;
    for (const double y : observed_d) mean += y;
    mean /= static_cast<double>(observed_d.size());
    double ss_res = 0.0, ss_tot = 0.0;
    for (std::size_t k = 0; k < observed_d.size(); ++k) {
        const double e = observed_d[k] - predicted_d[k];
        ss_res += e * e;
        const double c = observed_d[k] - mean;
        ss_tot += c * c;
    }
    if (ss_tot == 0.0) throw ConstantObservedError{};
    return 1.0 - ss_res / ss_tot;
}

ObjectiveSpec parse_objective(std::string_view name) {  // objectives.cpp:146-170
    ObjectiveSpec spec;
    std::string_view metric = name;
    if (name.starts_with("d-")) {
        spec.family = Family::DOnly;
        metric = name.substr(2);
    } else if (name.starts_with("ird-")) {
        spec.family = Family::IRDJoint;
        metric = name.substr(4);
    } else {
        throw ParseError("unknown objective '" + std::string(name) + "'");
    }
    if (metric == "mxse") spec.metric = Metric::MXSE;
    else if (metric == "mse") spec.metric = Metric::MSE;
    else if (metric == "mae") spec.metric = Metric::MAE;
    else if (metric == "mape") spec.metric = Metric::MAPE;
    else throw ParseError("unknown objective '" + std::string(name) + "'");
    return spec;
}

std::string metric_name(Metric m) {
    switch (m) {
    case Metric::MXSE: return "mxse";
    case Metric::MSE: return "mse";
    case Metric::MAE: return "mae";
    default: return "mape";
    }
}

std::string objective_name(const ObjectiveSpec& spec) {
    return (spec.family == Family::DOnly ? "d-" : "ird-") + metric_name(spec.metric);
}

// ---- pso -------------------------------------------------------------------------------

void PsoConfig::validate() const {  // pso.cpp:16-23
    if (n_particles == 0 || max_iters == 0) throw Error("pso: n_particles and max_iters must be positive");
    if (!std::isfinite(inertia) || !std::isfinite(cognitive) || !std::isfinite(social))
        throw Error("pso: coefficients must be finite");
}

void SearchBounds::validate() const {  // pso.cpp:25-34
    if (lower.empty() || lower.size() != upper.size())
        throw Error("pso: bounds must be non-empty and of equal dimension");
    for (std::size_t d = 0; d < lower.size(); ++d)
        if (!std::isfinite(lower[d]) || !std::isfinite(upper[d]) || lower[d] > upper[d])
            throw Error("pso: bound " + std::to_string(d) + " is invalid");
}

std::uint64_t mix_seed(std::uint64_t base, std::uint64_t index) {  // pso.cpp:36-41
    std::uint64_t z = base + 0x9E3779B97F4A7C15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double uniform01(std::mt19937_64& engine) {  // pso.cpp:43-45: the top 53 bits scaled by 2^-53
    return static_cast<double>(engine() >> 11) * 0x1.0p-53;
}

namespace {

// The reference's repair hook (calibration.cpp:89-93) runs on the device;
// std::function keeps it as a plain function pointer.
bool is_repair_time_order(const RepairHook& repair) {
    using Fn = void (*)(std::span<double>);
    const Fn* f = repair.target<Fn>();
    return f && *f == &repair_time_order;
}

sg_window* device_window(const WindowObjective& wo) {
    if (!wo.window) throw Error(wo.deferred);
    return wo.window.get();
}

}  // namespace

void WindowObjective::operator()(std::span<const double> positions, std::size_t dim, std::span<double> costs) const {
    if (dim != 6 || positions.size() != costs.size() * dim)  // calibration.cpp:141-143
        throw Error("window objective expects 6-dim positions");
    if (costs.empty()) return;
    sg_window* w = device_window(*this);
    check(ctx, sg_eval_costs(w, positions.data(), costs.size(), dim, costs.data()));
}

Swarm::Swarm(const PsoConfig& config, SearchBounds bounds, RepairHook repair)  // pso.cpp:47-75
    : config_(config), bounds_(std::move(bounds)), repair_(std::move(repair)), best_cost_(kInf) {
    config_.validate();
    bounds_.validate();
    device_repair_ = repair_ && is_repair_time_order(repair_) && bounds_.dim() >= 4;
    sg_ctx* ctx = engine_context();
    check(ctx, sg_gswarm_create(ctx, static_cast<int>(bounds_.dim()), bounds_.lower.data(), bounds_.upper.data(),
                                config_.n_particles, config_.inertia, config_.cognitive, config_.social, config_.seed,
                                device_repair_ ? 1 : 0, &swarm_));
    costs_.assign(config_.n_particles, kInf);
    best_position_.assign(bounds_.dim(), 0.0);
    best_fresh_ = true;
    if (repair_ && !device_repair_) apply_host_repair(true);
}

Swarm::~Swarm() { sg_gswarm_destroy(swarm_); }

Swarm::Swarm(Swarm&& o) noexcept
    : config_(o.config_), bounds_(std::move(o.bounds_)), repair_(std::move(o.repair_)),
      device_repair_(o.device_repair_), swarm_(o.swarm_), costs_(std::move(o.costs_)),
      positions_(std::move(o.positions_)), best_position_(std::move(o.best_position_)),
      positions_fresh_(o.positions_fresh_), best_fresh_(o.best_fresh_), best_cost_(o.best_cost_),
      iterations_done_(o.iterations_done_) {
    o.swarm_ = nullptr;
}

Swarm& Swarm::operator=(Swarm&& o) noexcept {
    if (this != &o) {
        sg_gswarm_destroy(swarm_);
        config_ = o.config_;
        bounds_ = std::move(o.bounds_);
        repair_ = std::move(o.repair_);
        device_repair_ = o.device_repair_;
        swarm_ = o.swarm_;
        o.swarm_ = nullptr;
        costs_ = std::move(o.costs_);
        positions_ = std::move(o.positions_);
        best_position_ = std::move(o.best_position_);
        positions_fresh_ = o.positions_fresh_;
        best_fresh_ = o.best_fresh_;
        best_cost_ = o.best_cost_;
        iterations_done_ = o.iterations_done_;
    }
    return *this;
}

// A RepairHook the device does not know: applied to each particle of the
// host copy in particle order, exactly where the reference calls it (after
// the initial draw, pso.cpp:70-72, and after each move, pso.cpp:123-125).
void Swarm::apply_host_repair(bool initial) {
    sg_ctx* ctx = engine_context();
    const std::size_t dim = bounds_.dim();
    positions_.resize(config_.n_particles * dim);
    check(ctx, sg_gswarm_get_positions(swarm_, positions_.data()));
    for (std::size_t i = 0; i < config_.n_particles; ++i) repair_(std::span<double>(positions_.data() + i * dim, dim));
    check(ctx, initial ? sg_gswarm_set_initial_positions(swarm_, positions_.data())
                       : sg_gswarm_set_positions(swarm_, positions_.data()));
    positions_fresh_ = true;
}

std::span<const double> Swarm::positions() const {
    if (!positions_fresh_) {
        positions_.resize(config_.n_particles * bounds_.dim());
        check(engine_context(), sg_gswarm_get_positions(swarm_, positions_.data()));
        positions_fresh_ = true;
    }
    return positions_;
}

std::span<const double> Swarm::best_position() const {
    if (!best_fresh_) {
        double cost = 0.0;
        check(engine_context(), sg_gswarm_best(swarm_, best_position_.data(), &cost));
        best_fresh_ = true;
    }
    return best_position_;
}

double Swarm::step(const BatchObjective& objective) {  // pso.cpp:77-101
    sg_ctx* ctx = engine_context();
    const std::size_t dim = bounds_.dim();
    if (const WindowObjective* wo = objective.target<WindowObjective>()) {
        if (dim != 6) throw Error("window objective expects 6-dim positions");
        check(ctx, sg_gswarm_eval_window(swarm_, device_window(*wo)));  // costs stay on the device
    } else {
        objective(positions(), dim, costs_);
        check(ctx, sg_gswarm_set_costs(swarm_, costs_.data()));
    }
    check(ctx, sg_gswarm_step(swarm_, &best_cost_));
    positions_fresh_ = false;
    best_fresh_ = false;
    if (repair_ && !device_repair_) apply_host_repair(false);
    ++iterations_done_;
    return best_cost_;
}

PsoResult optimize(const PsoConfig& config, const SearchBounds& bounds, const BatchObjective& objective,
                   RepairHook repair) {  // pso.cpp:129-143
    const WindowObjective* wo = objective.target<WindowObjective>();
    if (wo && bounds.dim() == 6 && (!repair || is_repair_time_order(repair))) {
        // the fused device swarm of sg_fit_swarms: same trajectory, no host round trip per step
        config.validate();  // Swarm::Swarm (pso.cpp:49-50)
        bounds.validate();
        sg_swarm_desc d{};
        d.window = device_window(*wo);
        for (int k = 0; k < 6; ++k) {
            d.lower[k] = bounds.lower[k];
            d.upper[k] = bounds.upper[k];
        }
        d.n_particles = config.n_particles;
        d.max_iters = config.max_iters;
        d.inertia = config.inertia;
        d.cognitive = config.cognitive;
        d.social = config.social;
        d.seed = config.seed;
        d.repair_time_order = repair ? 1 : 0;
        PsoResult result;
        result.cost_history.assign(config.max_iters, 0.0);
        sg_swarm_result r{};
        r.cost_history = result.cost_history.data();
        sg_ctx* ctx = wo->ctx;
        check(ctx, sg_fit_swarms(ctx, &d, 1, &r));
        if (r.status == SG_ERR_ALL_INFEASIBLE) throw AllInfeasibleError{};  // pso.cpp:137-139
        if (r.status != SG_OK) throw_status(r.status, sg_last_error(ctx));
        result.best_cost = r.best_cost;
        result.best_position.assign(r.best_position, r.best_position + 6);
        return result;
    }
    Swarm swarm(config, bounds, std::move(repair));
    PsoResult result;
    result.cost_history.reserve(config.max_iters);
    for (std::size_t it = 0; it < config.max_iters; ++it) result.cost_history.push_back(swarm.step(objective));
    if (!(swarm.best_cost() < kInf)) throw AllInfeasibleError{};
    result.best_cost = swarm.best_cost();
    const auto best = swarm.best_position();
    result.best_position.assign(best.begin(), best.end());
    return result;
}

// ---- calibration -------------------------------------------------------------------------

std::vector<Window> make_windows(std::size_t n_days, const WindowScheme& scheme) {  // calibration.cpp:37-52
    if (scheme.tau < 1 || scheme.delta < 1) throw SchemeError("window scheme needs tau >= 1 and delta >= 1");
    if (n_days < scheme.tau + 1)
        throw SchemeError("series has " + std::to_string(n_days) + " days; a window needs " +
                          std::to_string(scheme.tau + 1));
    const std::size_t count = 1 + (n_days - 1 - scheme.tau) / scheme.delta;
    std::vector<Window> windows(count);
    for (std::size_t i = 0; i < count; ++i) windows[i] = Window{i, i * scheme.delta, scheme.tau + 1};
    return windows;
}

ParamBounds ParamBounds::stage1() { return ParamBounds{}; }

ParamBounds ParamBounds::stage2() {  // calibration.cpp:58-65
    ParamBounds b;
    b.beta_hi = 2.0;
    b.gamma_hi = 1.0;
    b.mu_hi = 0.1;
    b.t_margin = 7;
    return b;
}

SearchBounds ParamBounds::to_search_bounds(std::size_t tau) const {  // calibration.cpp:67-76
    if (t_margin > tau) throw SchemeError("t_margin exceeds the window length");
    const double t_hi = static_cast<double>(tau - t_margin);
    return SearchBounds{{beta_lo, beta_lo, 0.0, 0.0, gamma_lo, mu_lo}, {beta_hi, beta_hi, t_hi, t_hi, gamma_hi, mu_hi}};
}

bool ParamBounds::contains(const SirdParams& p, std::size_t tau) const {  // calibration.cpp:78-83
    const double t_hi = static_cast<double>(tau) - static_cast<double>(t_margin);
    return p.beta1 >= beta_lo && p.beta1 <= beta_hi && p.beta2 >= beta_lo && p.beta2 <= beta_hi && p.t1 >= 0.0 &&
           p.t2 >= p.t1 && p.t2 <= t_hi && p.gamma >= gamma_lo && p.gamma <= gamma_hi && p.mu >= mu_lo &&
           p.mu <= mu_hi;
}

SirdParams params_from_position(std::span<const double> x) { return SirdParams{x[0], x[1], x[2], x[3], x[4], x[5]}; }

void repair_time_order(std::span<double> position) {  // calibration.cpp:89-93
    if (position[2] > position[3]) std::swap(position[2], position[3]);
}

WindowSlice slice_window(const EpiSeries& data, const Window& window) {  // calibration.cpp:95-104
    if (window.length == 0 || window.start + window.length > data.size())
        throw SchemeError("window " + std::to_string(window.index) + " falls outside the series");
    return WindowSlice{std::span(data.infectious).subspan(window.start, window.length),
                       std::span(data.recovered_cum).subspan(window.start, window.length),
                       std::span(data.deaths_cum).subspan(window.start, window.length)};
}

SirdState window_initial_state(const EpiSeries& data, std::size_t day, double population) {  // 106-118
    if (day >= data.size()) throw SchemeError("initial day outside the series");
    const double I = data.infectious[day], R = data.recovered_cum[day], D = data.deaths_cum[day];
    const double S = population - I - R - D;
    if (S < 0.0) throw InsufficientPopulationError("population smaller than I+R+D at day " + std::to_string(day));
    return SirdState{S, I, R, D};
}

BatchObjective make_window_objective(const ObjectiveSpec& spec, const WindowSlice& observed, const SirdState& init,
                                     double population, int substeps, int /*n_threads*/) {
    WindowObjective wo;
    wo.ctx = engine_context();
    // The reference validates n_days / substeps / population only when the
    // objective integrates (model.cpp:78-80); keep that timing.
    sg_window* w = nullptr;
    const int rc = sg_window_create(wo.ctx, observed.infectious.data(), observed.recovered_cum.data(),
                                    observed.deaths_cum.data(), static_cast<int>(observed.deaths_cum.size()),
                                    sg_state{init.S, init.I, init.R, init.D}, population, substeps,
                                    family_code(spec.family), metric_code(spec.metric), &w);
    if (rc == SG_ERR_INVALID_ARGUMENT) wo.deferred = sg_last_error(wo.ctx);
    else check(wo.ctx, rc);
    if (w) wo.window = std::shared_ptr<sg_window>(w, sg_window_destroy);
    return wo;
}

namespace {

// One fit request of the batched scheduler.
struct Job {
    Window window;
    std::uint64_t seed;
};

struct JobOutcome {
    FitResult fit;
    int status = SG_OK;  // exception the reference's fit_window would throw
};

void fail_job(JobOutcome& o, int status, const std::string& msg) {
    o.status = status;
    o.fit.ok = false;
    o.fit.failure = msg;
}

int status_of(const Error& e) {
    if (dynamic_cast<const SchemeError*>(&e)) return SG_ERR_SCHEME;
    if (dynamic_cast<const InsufficientPopulationError*>(&e)) return SG_ERR_INSUFFICIENT_POPULATION;
    if (dynamic_cast<const AllInfeasibleError*>(&e)) return SG_ERR_ALL_INFEASIBLE;
    if (dynamic_cast<const NonFiniteError*>(&e)) return SG_ERR_NON_FINITE;
    if (dynamic_cast<const DeviceError*>(&e)) return SG_ERR_CUDA;
    return SG_ERR_INVALID_ARGUMENT;
}

// fit_window (calibration.cpp:157-188) for many (window, seed) pairs: the
// per-window checks run on the host in the reference's order; every valid
// swarm then runs concurrently in one sg_fit_swarms call, and the best fits
// are re-integrated on the device in one batch.
std::vector<JobOutcome> fit_jobs(const EpiSeries& data, const std::vector<Job>& jobs, const FitSettings& settings) {
    sg_ctx* ctx = engine_context();
    std::vector<JobOutcome> out(jobs.size());
    std::map<std::pair<std::size_t, std::size_t>, std::shared_ptr<WindowHandle>> windows;
    std::vector<sg_swarm_desc> descs;
    std::vector<std::size_t> desc_job;
    std::vector<SirdState> inits(jobs.size());
    std::vector<std::vector<double>> histories(jobs.size());
    for (std::size_t j = 0; j < jobs.size(); ++j) {
        JobOutcome& o = out[j];
        o.fit.window = jobs[j].window;
        o.fit.spec = settings.spec;
        try {
            const WindowSlice observed = slice_window(data, jobs[j].window);
            inits[j] = window_initial_state(data, jobs[j].window.start, settings.population);
            const std::size_t tau = jobs[j].window.length - 1;
            const SearchBounds bounds = settings.bounds.to_search_bounds(tau);
            settings.pso.validate();  // Swarm::Swarm (pso.cpp:49-50)
            bounds.validate();
            auto key = std::make_pair(jobs[j].window.start, jobs[j].window.length);
            auto it = windows.find(key);
            if (it == windows.end()) {
                auto h = std::make_shared<WindowHandle>();
                const SirdState& s0 = inits[j];
                const int rc = sg_window_create(ctx, observed.infectious.data(), observed.recovered_cum.data(),
                                                observed.deaths_cum.data(), static_cast<int>(jobs[j].window.length),
                                                sg_state{s0.S, s0.I, s0.R, s0.D}, settings.population,
                                                settings.substeps, family_code(settings.spec.family),
                                                metric_code(settings.spec.metric), &h->w);
                if (rc) throw_status(rc, sg_last_error(ctx));
                it = windows.emplace(key, h).first;
            }
            sg_swarm_desc d{};
            d.window = it->second->w;
            for (int k = 0; k < 6; ++k) {
                d.lower[k] = bounds.lower[k];
                d.upper[k] = bounds.upper[k];
            }
            d.n_particles = settings.pso.n_particles;
            d.max_iters = settings.pso.max_iters;
            d.inertia = settings.pso.inertia;
            d.cognitive = settings.pso.cognitive;
            d.social = settings.pso.social;
            d.seed = jobs[j].seed;
            d.repair_time_order = 1;
            descs.push_back(d);
            desc_job.push_back(j);
        } catch (const DeviceError&) {
            throw;
        } catch (const Error& e) {
            fail_job(o, status_of(e), e.what());
        }
    }
    sg_trace_phase("fit_jobs: windows built");
    if (descs.empty()) return out;
    std::vector<sg_swarm_result> res(descs.size());
    for (std::size_t k = 0; k < descs.size(); ++k) {
        histories[desc_job[k]].assign(settings.pso.max_iters, 0.0);
        res[k].cost_history = histories[desc_job[k]].data();
    }
    check(ctx, sg_fit_swarms(ctx, descs.data(), descs.size(), res.data()));
    sg_trace_phase("fit_jobs: swarms done");
    // Re-integrate every successful best fit (calibration.cpp:175-176).
    std::vector<std::size_t> done;
    std::vector<double> params;
    std::vector<sg_state> s0;
    for (std::size_t k = 0; k < descs.size(); ++k) {
        JobOutcome& o = out[desc_job[k]];
        if (res[k].status == SG_ERR_ALL_INFEASIBLE) {
            fail_job(o, SG_ERR_ALL_INFEASIBLE, AllInfeasibleError{}.what());
            continue;
        }
        if (res[k].status != SG_OK) {
            fail_job(o, res[k].status, sg_last_error(ctx));
            continue;
        }
        o.fit.params = params_from_position(std::span<const double>(res[k].best_position, 6));
        o.fit.objective = res[k].best_cost;
        o.fit.cost_history = std::move(histories[desc_job[k]]);
        done.push_back(desc_job[k]);
        params.insert(params.end(), res[k].best_position, res[k].best_position + 6);
        const SirdState& s = inits[desc_job[k]];
        s0.push_back(sg_state{s.S, s.I, s.R, s.D});
    }
    // Group by window length (one integrate call per distinct length).
    std::map<std::size_t, std::vector<std::size_t>> by_len;
    for (std::size_t q = 0; q < done.size(); ++q) by_len[out[done[q]].fit.window.length].push_back(q);
    for (const auto& [len, qs] : by_len) {
        std::vector<double> p(6 * qs.size());
        std::vector<sg_state> st(qs.size());
        for (std::size_t i = 0; i < qs.size(); ++i) {
            std::copy_n(params.data() + 6 * qs[i], 6, p.data() + 6 * i);
            st[i] = s0[qs[i]];
        }
        std::vector<double> states(qs.size() * len * 4);
        std::vector<uint8_t> fin(qs.size());
        std::vector<double> obs_d(qs.size() * len), r2(qs.size());
        for (std::size_t i = 0; i < qs.size(); ++i) {
            const WindowSlice observed = slice_window(data, out[done[qs[i]]].fit.window);
            std::copy(observed.deaths_cum.begin(), observed.deaths_cum.end(), obs_d.begin() + i * len);
        }
        // re-integration (calibration.cpp:175-176) and R^2 (182-185) on the device
        check(ctx, sg_integrate_states_r2(ctx, p.data(), st.data(), obs_d.data(), qs.size(), settings.population,
                                          static_cast<int>(len), settings.substeps, states.data(), fin.data(),
                                          r2.data()));
        for (std::size_t i = 0; i < qs.size(); ++i) {
            JobOutcome& o = out[done[qs[i]]];
            states_to_trajectory(states.data() + i * len * 4, static_cast<int>(len), fin[i] != 0, settings.population,
                                 o.fit.trajectory);
            o.fit.r2_d = r2[i];  // NaN for a constant observed series (ConstantObservedError)
            o.fit.ok = true;
        }
    }
    sg_trace_phase("fit_jobs: re-integrated");
    return out;
}

}  // namespace

FitResult fit_window(const EpiSeries& data, const Window& window, const FitSettings& settings, std::uint64_t seed) {
    std::vector<JobOutcome> o = fit_jobs(data, {Job{window, seed}}, settings);
    if (o[0].status != SG_OK) throw_status(o[0].status, o[0].fit.failure);
    return std::move(o[0].fit);
}

FitAllResult fit_all_windows(const EpiSeries& data, const WindowScheme& scheme, const FitSettings& settings,
                             std::uint64_t base_seed) {  // calibration.cpp:190-216
    FitAllResult result;
    const std::vector<Window> windows = make_windows(data.size(), scheme);
    std::vector<Job> jobs;
    jobs.reserve(windows.size());
    for (const Window& w : windows) jobs.push_back(Job{w, mix_seed(base_seed, w.index)});
    std::vector<JobOutcome> outcomes = fit_jobs(data, jobs, settings);
    double r2_sum = 0.0;
    std::size_t r2_count = 0;
    for (JobOutcome& o : outcomes) {
        if (o.status == SG_OK) {
            if (std::isfinite(o.fit.r2_d)) {
                r2_sum += o.fit.r2_d;
                ++r2_count;
            }
        } else {
            ++result.failed_count;
        }
        result.fits.push_back(std::move(o.fit));
    }
    result.mean_r2_d = r2_count > 0 ? r2_sum / static_cast<double>(r2_count) : kNaN;
    return result;
}

Forecast forecast_extension(const FitResult& fit, std::size_t horizon, int substeps) {  // calibration.cpp:298-322
    if (!fit.ok || fit.trajectory.days() == 0) throw Error("cannot extend a failed fit");
    if (!fit.trajectory.finite) throw NonFiniteError{};
    const SirdState& j = fit.trajectory.states.back();
    const double params[6] = {fit.params.beta1, fit.params.beta2, fit.params.t1, fit.params.t2, fit.params.gamma,
                              fit.params.mu};
    const sg_state junction{j.S, j.I, j.R, j.D};
    const int n_days = static_cast<int>(horizon) + 1;
    if (substeps < 1 || !(fit.trajectory.population > 0.0))
        throw Error("integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
    std::vector<double> states(static_cast<std::size_t>(n_days) * 4);
    uint8_t fin = 0;
    sg_ctx* ctx = engine_context();
    check(ctx, sg_forecast_batch(ctx, params, &junction, 1, fit.trajectory.population, static_cast<int>(horizon),
                                 substeps, states.data(), &fin));
    Forecast f;
    f.junction_day = fit.window.last_day();
    f.horizon = horizon;
    states_to_trajectory(states.data(), n_days, fin != 0, fit.trajectory.population, f.trajectory);
    if (!f.trajectory.finite) throw NonFiniteError{};
    return f;
}

double quantile_sorted(std::span<const double> sorted, double p) {  // calibration.cpp:324-335
    if (sorted.empty()) return kNaN;
    const double h = static_cast<double>(sorted.size() - 1) * p;
    const std::size_t lo = static_cast<std::size_t>(h);
    if (lo + 1 >= sorted.size()) return sorted.back();
    const double frac = h - static_cast<double>(lo);
    return sorted[lo] + frac * (sorted[lo + 1] - sorted[lo]);
}

QuantileBands build_quantile_bands(const std::vector<std::vector<double>>& values_per_day) {  // 337-361
    const std::size_t n_days = values_per_day.size();
    QuantileBands b;
    b.count.assign(n_days, 0);
    for (auto* v : {&b.median, &b.p50_lo, &b.p50_hi, &b.p90_lo, &b.p90_hi, &b.p95_lo, &b.p95_hi})
        v->assign(n_days, kNaN);
    std::vector<double> sorted;
    for (std::size_t day = 0; day < n_days; ++day) {
        append_finite_sorted(sorted, values_per_day[day]);
        b.count[day] = sorted.size();
        if (sorted.empty()) continue;
        b.median[day] = quantile_sorted(sorted, 0.5);
        b.p50_lo[day] = quantile_sorted(sorted, 0.25);
        b.p50_hi[day] = quantile_sorted(sorted, 0.75);
        b.p90_lo[day] = quantile_sorted(sorted, 0.05);
        b.p90_hi[day] = quantile_sorted(sorted, 0.95);
        b.p95_lo[day] = quantile_sorted(sorted, 0.025);
        b.p95_hi[day] = quantile_sorted(sorted, 0.975);
    }
    return b;
}

ScalarBands build_scalar_bands(std::vector<double> values) {  // calibration.cpp:363-376
    std::vector<double> sorted;
    append_finite_sorted(sorted, values);
    ScalarBands b;
    b.count = sorted.size();
    b.median = quantile_sorted(sorted, 0.5);
    b.p50_lo = quantile_sorted(sorted, 0.25);
    b.p50_hi = quantile_sorted(sorted, 0.75);
    b.p90_lo = quantile_sorted(sorted, 0.05);
    b.p90_hi = quantile_sorted(sorted, 0.95);
    b.p95_lo = quantile_sorted(sorted, 0.025);
    b.p95_hi = quantile_sorted(sorted, 0.975);
    return b;
}

Envelope build_envelope(const std::vector<std::vector<double>>& values_per_day) {  // calibration.cpp:218-245
    Envelope env;
    const std::size_t n_days = values_per_day.size();
    env.count.assign(n_days, 0);
    for (auto* col : {&env.outer_lo, &env.outer_hi, &env.band1_lo, &env.band1_hi, &env.band2_lo, &env.band2_hi,
                      &env.median})
        col->assign(n_days, kNaN);
    std::vector<double> v;
    for (std::size_t day = 0; day < n_days; ++day) {
        append_finite_sorted(v, values_per_day[day]);
        const std::size_t k = v.size();
        env.count[day] = k;
        if (k == 0) continue;
        // rank envelopes: extremes, second ranks from 3 values, third ranks from 5
        env.outer_lo[day] = v[0];
        env.outer_hi[day] = v[k - 1];
        env.band1_lo[day] = k < 3 ? v[0] : v[1];
        env.band1_hi[day] = k < 3 ? v[k - 1] : v[k - 2];
        if (k >= 5) {
            env.band2_lo[day] = v[2];
            env.band2_hi[day] = v[k - 3];
        }
        env.median[day] = (k & 1) ? v[k / 2] : 0.5 * (v[k / 2 - 1] + v[k / 2]);  // calibration.cpp:27-33
    }
    return env;
}

ParameterEnvelopes parameter_envelopes(std::span<const FitResult> fits, std::size_t n_days) {  // 247-274
    std::vector<std::vector<double>> beta(n_days), gamma(n_days), mu(n_days), r0(n_days);
    for (const FitResult& f : fits) {
        if (!f.ok) continue;
        const double rate = f.params.gamma + f.params.mu;
        for (std::size_t local = 0; local < f.window.length && f.window.start + local < n_days; ++local) {
            const std::size_t day = f.window.start + local;
            const double b = beta_at(f.params, static_cast<double>(local));
            beta[day].push_back(b);
            gamma[day].push_back(f.params.gamma);
            mu[day].push_back(f.params.mu);
            r0[day].push_back(rate > 0.0 ? b / rate : kNaN);
        }
    }
    return ParameterEnvelopes{build_envelope(beta), build_envelope(gamma), build_envelope(mu), build_envelope(r0)};
}

CompartmentEnvelopes compartment_envelopes(std::span<const FitResult> fits, std::size_t n_days) {  // 276-296
    std::vector<std::vector<double>> I(n_days), R(n_days), D(n_days);
    for (const FitResult& f : fits) {
        if (!f.ok) continue;
        const std::size_t len = std::min(f.window.length, f.trajectory.days());
        for (std::size_t local = 0; local < len && f.window.start + local < n_days; ++local) {
            const SirdState& s = f.trajectory.states[local];
            I[f.window.start + local].push_back(s.I);
            R[f.window.start + local].push_back(s.R);
            D[f.window.start + local].push_back(s.D);
        }
    }
    return CompartmentEnvelopes{build_envelope(I), build_envelope(R), build_envelope(D)};
}

StabilityResult stability_study(const EpiSeries& data, const Window& window, const FitSettings& settings,
                                std::size_t repetitions, std::size_t horizon, std::uint64_t base_seed) {
    // calibration.cpp:378-436, with the repetitions run as concurrent swarms
    // and their forecasts integrated in one device batch.
    if (repetitions < 1) throw Error("stability study needs at least one repetition");
    StabilityResult out;
    out.window = window;
    out.horizon = horizon;
    out.repetitions = repetitions;
    const std::size_t window_days = window.length;
    const std::size_t total_days = window_days + horizon;
    std::vector<std::vector<double>> beta(window_days), r0(window_days), I(total_days), R(total_days), D(total_days);
    std::vector<double> gammas, mus;

    std::vector<Job> jobs;
    for (std::size_t rep = 0; rep < repetitions; ++rep) jobs.push_back(Job{window, mix_seed(base_seed, rep)});
    std::vector<JobOutcome> fits = fit_jobs(data, jobs, settings);

    // forecast_extension for every successful repetition, one device batch.
    std::vector<std::size_t> ok_reps;
    std::vector<double> params;
    std::vector<sg_state> junctions;
    for (std::size_t rep = 0; rep < repetitions; ++rep) {
        JobOutcome& o = fits[rep];
        if (o.status != SG_OK) continue;
        if (!o.fit.trajectory.finite) {  // calibration.cpp:301-303
            fail_job(o, SG_ERR_NON_FINITE, NonFiniteError{}.what());
            continue;
        }
        ok_reps.push_back(rep);
        double p[6];
        params_to(o.fit.params, p);
        params.insert(params.end(), p, p + 6);
        const SirdState& j = o.fit.trajectory.states.back();
        junctions.push_back(sg_state{j.S, j.I, j.R, j.D});
    }
    std::vector<double> fstates(ok_reps.size() * (horizon + 1) * 4);
    std::vector<uint8_t> ffin(ok_reps.size());
    if (!ok_reps.empty()) {
        if (settings.substeps < 1 || !(settings.population > 0.0))
            throw Error("integrate_euler needs n_days >= 1, substeps >= 1 and a positive population");
        sg_ctx* ctx = engine_context();
        check(ctx, sg_forecast_batch(ctx, params.data(), junctions.data(), ok_reps.size(), settings.population,
                                     static_cast<int>(horizon), settings.substeps, fstates.data(), ffin.data()));
    }
    std::size_t q = 0;
    for (std::size_t rep = 0; rep < repetitions; ++rep) {
        JobOutcome& o = fits[rep];
        if (q < ok_reps.size() && ok_reps[q] == rep) {
            const double* fs = fstates.data() + q * (horizon + 1) * 4;
            const bool ffinite = ffin[q] != 0;
            ++q;
            if (!ffinite) {  // calibration.cpp:318-320
                fail_job(o, SG_ERR_NON_FINITE, NonFiniteError{}.what());
            } else {
                const FitResult& fit = o.fit;
                const double rate = fit.params.gamma + fit.params.mu;
                for (std::size_t local = 0; local < window_days; ++local) {
                    const double b = beta_at(fit.params, static_cast<double>(local));
                    beta[local].push_back(b);
                    r0[local].push_back(rate > 0.0 ? b / rate : kNaN);
                    const SirdState& s = fit.trajectory.states[local];
                    I[local].push_back(s.I);
                    R[local].push_back(s.R);
                    D[local].push_back(s.D);
                }
                for (std::size_t k = 1; k <= horizon; ++k) {
                    I[window_days - 1 + k].push_back(fs[4 * k + 1]);
                    R[window_days - 1 + k].push_back(fs[4 * k + 2]);
                    D[window_days - 1 + k].push_back(fs[4 * k + 3]);
                }
                gammas.push_back(fit.params.gamma);
                mus.push_back(fit.params.mu);
            }
        }
        if (o.status != SG_OK) {
            // the reference records a fresh failed FitResult (calibration.cpp:418-425)
            FitResult failed;
            failed.window = window;
            failed.spec = settings.spec;
            failed.failure = o.fit.failure;
            out.fits.push_back(std::move(failed));
            ++out.failed;
        } else {
            out.fits.push_back(std::move(o.fit));
        }
    }
    out.beta = build_quantile_bands(beta);
    out.r0 = build_quantile_bands(r0);
    out.infectious = build_quantile_bands(I);
    out.recovered = build_quantile_bands(R);
    out.deaths = build_quantile_bands(D);
    out.gamma = build_scalar_bands(std::move(gammas));
    out.mu = build_scalar_bands(std::move(mus));
    return out;
}

}  // namespace sirdfit_b200

// ---- C entry points -------------------------------------------------------------------------

namespace {

using namespace sirdfit_b200;

struct ContextScope {  // run the C++ layer on the caller's context
    explicit ContextScope(sg_ctx* ctx) { t_override = ctx; }
    ~ContextScope() { t_override = nullptr; }
};

FitSettings settings_of(const sg_fit_settings& s) {
    FitSettings f;
    f.spec.family = s.family == SG_FAMILY_D_ONLY ? Family::DOnly : Family::IRDJoint;
    if (s.metric < 0 || s.metric > 3) throw Error("unknown objective metric");
    f.spec.metric = static_cast<Metric>(s.metric);
    f.bounds = ParamBounds{s.beta_lo, s.beta_hi, s.gamma_lo, s.gamma_hi, s.mu_lo, s.mu_hi,
                           static_cast<std::size_t>(s.t_margin)};
    f.pso.n_particles = s.n_particles;
    f.pso.max_iters = s.max_iters;
    f.pso.inertia = s.inertia;
    f.pso.cognitive = s.cognitive;
    f.pso.social = s.social;
    f.population = s.population;
    f.substeps = s.substeps;
    return f;
}

EpiSeries series_of(const double* I, const double* R, const double* D, std::size_t n) {
    EpiSeries e;
    e.infectious.assign(I, I + n);
    e.recovered_cum.assign(R, R + n);
    e.deaths_cum.assign(D, D + n);
    e.new_cases.assign(n, 0.0);
    return e;
}

void record_of(const FitResult& f, int status, sg_fit_record* r) {
    r->index = f.window.index;
    r->start = f.window.start;
    r->length = f.window.length;
    params_to(f.params, r->params);
    r->objective = f.objective;
    r->r2_d = f.r2_d;
    r->ok = f.ok ? 1 : 0;
    r->status = status;
    std::snprintf(r->failure, sizeof r->failure, "%s", f.failure.c_str());
}

void trajectory_out(const FitResult& f, double* out) {
    for (std::size_t d = 0; d < f.window.length; ++d) {
        const bool have = d < f.trajectory.states.size();
        const SirdState s = have ? f.trajectory.states[d] : SirdState{kNaN, kNaN, kNaN, kNaN};
        out[4 * d + 0] = s.S;
        out[4 * d + 1] = s.I;
        out[4 * d + 2] = s.R;
        out[4 * d + 3] = s.D;
    }
}

int public_status(const Error& e) {
    if (dynamic_cast<const SchemeError*>(&e)) return SG_ERR_SCHEME;
    if (dynamic_cast<const InsufficientPopulationError*>(&e)) return SG_ERR_INSUFFICIENT_POPULATION;
    if (dynamic_cast<const AllInfeasibleError*>(&e)) return SG_ERR_ALL_INFEASIBLE;
    if (dynamic_cast<const NonFiniteError*>(&e)) return SG_ERR_NON_FINITE;
    if (dynamic_cast<const DeviceError*>(&e)) return SG_ERR_CUDA;
    return SG_ERR_INVALID_ARGUMENT;
}

template <class F>
int guarded(sg_ctx* ctx, F&& fn) {
    try {
        ContextScope scope(ctx);
        fn();
        return SG_OK;
    } catch (const Error& e) {
        sg_set_last_error(ctx, e.what());
        return public_status(e);
    } catch (const std::bad_alloc&) {
        sg_set_last_error(ctx, "host allocation failed");
        return SG_ERR_OUT_OF_MEMORY;
    }
}

}  // namespace

extern "C" {

int sg_fit_window_series(sg_ctx* ctx, const double* I, const double* R, const double* D, size_t n_series,
                         uint64_t start, uint64_t length, const sg_fit_settings* s, uint64_t seed,
                         sg_fit_record* record, double* trajectory, double* history) {
    if (!ctx || !I || !R || !D || !s || !record) return SG_ERR_INVALID_ARGUMENT;
    FitResult fit;
    fit.window = Window{0, static_cast<std::size_t>(start), static_cast<std::size_t>(length)};
    const int rc = guarded(ctx, [&] {
        const EpiSeries data = series_of(I, R, D, n_series);
        fit = fit_window(data, fit.window, settings_of(*s), seed);
    });
    if (rc) fit.failure = sg_last_error(ctx);
    record_of(fit, rc, record);
    if (!rc && trajectory) trajectory_out(fit, trajectory);
    if (!rc && history) std::copy(fit.cost_history.begin(), fit.cost_history.end(), history);
    return rc;
}

int sg_fit_all_windows_series(sg_ctx* ctx, const double* I, const double* R, const double* D, size_t n_series,
                              uint64_t tau, uint64_t delta, const sg_fit_settings* s, uint64_t base_seed,
                              size_t max_windows, size_t* n_windows, sg_fit_record* records, double* trajectories,
                              double* mean_r2_d, size_t* failed_count) {
    if (!ctx || !I || !R || !D || !s || !n_windows || !records || !mean_r2_d || !failed_count)
        return SG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        sg_trace_phase("fit_all_windows_series: in");
        const EpiSeries data = series_of(I, R, D, n_series);
        const WindowScheme scheme{static_cast<std::size_t>(tau), static_cast<std::size_t>(delta)};
        *n_windows = make_windows(data.size(), scheme).size();
        if (*n_windows > max_windows) throw Error("records array holds fewer entries than there are windows");
        const FitAllResult all = fit_all_windows(data, scheme, settings_of(*s), base_seed);
        for (std::size_t w = 0; w < all.fits.size(); ++w) {
            const FitResult& f = all.fits[w];
            int st = SG_OK;
            if (!f.ok) st = f.failure == AllInfeasibleError{}.what() ? SG_ERR_ALL_INFEASIBLE : SG_ERR_INVALID_ARGUMENT;
            record_of(f, st, records + w);
            if (trajectories) trajectory_out(f, trajectories + w * (tau + 1) * 4);
        }
        *mean_r2_d = all.mean_r2_d;
        *failed_count = all.failed_count;
        sg_trace_phase("fit_all_windows_series: out");
    });
}

int sg_fit_window_range_series(sg_ctx* ctx, const double* I, const double* R, const double* D, size_t n_series,
                               uint64_t tau, uint64_t delta, const sg_fit_settings* s, uint64_t base_seed,
                               uint64_t first_window, uint64_t max_windows, size_t* n_windows, sg_fit_record* records,
                               double* trajectories) {
    if (!ctx || !I || !R || !D || !s || !n_windows || (max_windows && !records)) return SG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        const EpiSeries data = series_of(I, R, D, n_series);
        const WindowScheme scheme{static_cast<std::size_t>(tau), static_cast<std::size_t>(delta)};
        const std::vector<Window> all = make_windows(data.size(), scheme);  // calibration.cpp:193
        const std::size_t begin = std::min<std::size_t>(first_window, all.size());
        const std::size_t end = std::min<std::size_t>(begin + max_windows, all.size());
        std::vector<Job> jobs;
        for (std::size_t w = begin; w < end; ++w) jobs.push_back(Job{all[w], mix_seed(base_seed, all[w].index)});
        const std::vector<JobOutcome> out = fit_jobs(data, jobs, settings_of(*s));
        for (std::size_t k = 0; k < out.size(); ++k) {
            record_of(out[k].fit, out[k].status, records + k);
            if (trajectories) trajectory_out(out[k].fit, trajectories + k * (tau + 1) * 4);
        }
        *n_windows = out.size();
    });
}

int sg_stability_study_series(sg_ctx* ctx, const double* I, const double* R, const double* D, size_t n_series,
                              uint64_t start, uint64_t length, const sg_fit_settings* s, uint64_t repetitions,
                              uint64_t horizon, uint64_t base_seed, sg_fit_record* records, double* day_bands,
                              uint64_t* day_counts, double* scalar_bands, uint64_t* scalar_counts, uint64_t* failed) {
    if (!ctx || !I || !R || !D || !s || !records || !day_bands || !day_counts || !scalar_bands || !scalar_counts ||
        !failed)
        return SG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        const EpiSeries data = series_of(I, R, D, n_series);
        const Window window{0, static_cast<std::size_t>(start), static_cast<std::size_t>(length)};
        const StabilityResult st = stability_study(data, window, settings_of(*s), repetitions, horizon, base_seed);
        for (std::size_t r = 0; r < st.fits.size(); ++r) record_of(st.fits[r], st.fits[r].ok ? SG_OK : 1, records + r);
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
    });
}

}  // extern "C"
