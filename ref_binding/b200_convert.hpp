// b200_convert.hpp — conversions between the reference's types (namespace
// sirdfit, /root/reference/proj/include/sirdfit/*.hpp) and the engine's C++
// API (namespace sirdfit_b200, include/sirdfit_b200.hpp), and the mapping of
// the engine's exceptions back to the reference's classes with the same
// messages (errors.hpp:8-50).
//
// Part of the reference-side binding (ref_binding/*.cpp): the files a
// maintainer of the reference compiles IN PLACE OF src/model.cpp,
// src/objectives.cpp and src/calibration.cpp to run the reference's own
// callers (tools, bindings/module.cpp, tests/acceptance) on the B200 engine.
// See INTEGRATION.md §2.
#pragma once

#include "sirdfit/calibration.hpp"
#include "sirdfit/errors.hpp"
#include "sirdfit/model.hpp"
#include "sirdfit/objectives.hpp"

#include "sirdfit_b200.hpp"

#include <utility>
#include <vector>

namespace sirdfit::b200 {

namespace sf = sirdfit_b200;

// Runs fn(); an engine exception becomes the reference exception of the
// same class and message.
template <class F>
auto translated(F&& fn) -> decltype(fn()) {
    try {
        return fn();
    } catch (const sf::SchemeError& e) {
        throw SchemeError(e.what());
    } catch (const sf::InsufficientPopulationError& e) {
        throw InsufficientPopulationError(e.what());
    } catch (const sf::AllInfeasibleError&) {
        throw AllInfeasibleError{};
    } catch (const sf::NonFiniteError&) {
        throw NonFiniteError{};
    } catch (const sf::DegenerateRatesError&) {
        throw DegenerateRatesError{};
    } catch (const sf::DegenerateRangeError&) {
        throw DegenerateRangeError{};
    } catch (const sf::ConstantObservedError&) {
        throw ConstantObservedError{};
    } catch (const sf::ParseError& e) {
        throw ParseError(e.what());
    } catch (const sf::Error& e) {
        throw Error(e.what());
    }
}

inline sf::SirdParams to_b200(const SirdParams& p) { return {p.beta1, p.beta2, p.t1, p.t2, p.gamma, p.mu}; }
inline SirdParams from_b200(const sf::SirdParams& p) {
    return SirdParams{.beta1 = p.beta1, .beta2 = p.beta2, .t1 = p.t1, .t2 = p.t2, .gamma = p.gamma, .mu = p.mu};
}
inline sf::SirdState to_b200(const SirdState& s) { return {s.S, s.I, s.R, s.D}; }
inline SirdState from_b200(const sf::SirdState& s) { return SirdState{.S = s.S, .I = s.I, .R = s.R, .D = s.D}; }

inline Trajectory from_b200(const sf::Trajectory& t) {
    Trajectory out;
    out.states.reserve(t.states.size());
    for (const sf::SirdState& s : t.states) out.states.push_back(from_b200(s));
    out.population = t.population;
    out.finite = t.finite;
    return out;
}
inline sf::Trajectory to_b200(const Trajectory& t) {
    sf::Trajectory out;
    out.states.reserve(t.states.size());
    for (const SirdState& s : t.states) out.states.push_back(to_b200(s));
    out.population = t.population;
    out.finite = t.finite;
    return out;
}

inline sf::Metric to_b200(Metric m) { return static_cast<sf::Metric>(static_cast<int>(m)); }
inline sf::ObjectiveSpec to_b200(const ObjectiveSpec& s) {
    return {s.family == Family::DOnly ? sf::Family::DOnly : sf::Family::IRDJoint, to_b200(s.metric)};
}
inline ObjectiveSpec from_b200(const sf::ObjectiveSpec& s) {
    return ObjectiveSpec{s.family == sf::Family::DOnly ? Family::DOnly : Family::IRDJoint,
                         static_cast<Metric>(static_cast<int>(s.metric))};
}
inline sf::WindowSlice to_b200(const WindowSlice& w) { return {w.infectious, w.recovered_cum, w.deaths_cum}; }

inline sf::Window to_b200(const Window& w) { return {w.index, w.start, w.length}; }
inline Window from_b200(const sf::Window& w) { return Window{.index = w.index, .start = w.start, .length = w.length}; }

inline sf::EpiSeries to_b200(const EpiSeries& e) {
    sf::EpiSeries out;
    out.infectious = e.infectious;
    out.recovered_cum = e.recovered_cum;
    out.deaths_cum = e.deaths_cum;
    out.new_cases = e.new_cases;
    return out;
}

inline sf::ParamBounds to_b200(const ParamBounds& b) {
    return {b.beta_lo, b.beta_hi, b.gamma_lo, b.gamma_hi, b.mu_lo, b.mu_hi, b.t_margin};
}
inline ParamBounds from_b200(const sf::ParamBounds& b) {
    ParamBounds out;
    out.beta_lo = b.beta_lo;
    out.beta_hi = b.beta_hi;
    out.gamma_lo = b.gamma_lo;
    out.gamma_hi = b.gamma_hi;
    out.mu_lo = b.mu_lo;
    out.mu_hi = b.mu_hi;
    out.t_margin = b.t_margin;
    return out;
}

inline sf::FitSettings to_b200(const FitSettings& s) {
    sf::FitSettings out;
    out.spec = to_b200(s.spec);
    out.bounds = to_b200(s.bounds);
    out.pso.n_particles = s.pso.n_particles;
    out.pso.inertia = s.pso.inertia;
    out.pso.cognitive = s.pso.cognitive;
    out.pso.social = s.pso.social;
    out.pso.max_iters = s.pso.max_iters;
    out.pso.seed = s.pso.seed;
    out.population = s.population;
    out.substeps = s.substeps;
    out.n_threads = s.n_threads;
    return out;
}

inline FitResult from_b200(const sf::FitResult& f) {
    FitResult out;
    out.window = from_b200(f.window);
    out.params = from_b200(f.params);
    out.spec = from_b200(f.spec);
    out.objective = f.objective;
    out.r2_d = f.r2_d;
    out.trajectory = from_b200(f.trajectory);
    out.ok = f.ok;
    out.failure = f.failure;
    return out;
}
inline sf::FitResult to_b200(const FitResult& f) {
    sf::FitResult out;
    out.window = to_b200(f.window);
    out.params = to_b200(f.params);
    out.spec = to_b200(f.spec);
    out.objective = f.objective;
    out.r2_d = f.r2_d;
    out.trajectory = to_b200(f.trajectory);
    out.ok = f.ok;
    out.failure = f.failure;
    return out;
}
inline std::vector<sf::FitResult> to_b200(std::span<const FitResult> fits) {
    std::vector<sf::FitResult> out;
    out.reserve(fits.size());
    for (const FitResult& f : fits) out.push_back(to_b200(f));
    return out;
}

inline Envelope from_b200(const sf::Envelope& e) {
    Envelope out;
    out.count = e.count;
    out.outer_lo = e.outer_lo;
    out.outer_hi = e.outer_hi;
    out.band1_lo = e.band1_lo;
    out.band1_hi = e.band1_hi;
    out.band2_lo = e.band2_lo;
    out.band2_hi = e.band2_hi;
    out.median = e.median;
    return out;
}

inline QuantileBands from_b200(const sf::QuantileBands& b) {
    QuantileBands out;
    out.count = b.count;
    out.median = b.median;
    out.p50_lo = b.p50_lo;
    out.p50_hi = b.p50_hi;
    out.p90_lo = b.p90_lo;
    out.p90_hi = b.p90_hi;
    out.p95_lo = b.p95_lo;
    out.p95_hi = b.p95_hi;
    return out;
}
inline ScalarBands from_b200(const sf::ScalarBands& b) {
    ScalarBands out;
    out.count = b.count;
    out.median = b.median;
    out.p50_lo = b.p50_lo;
    out.p50_hi = b.p50_hi;
    out.p90_lo = b.p90_lo;
    out.p90_hi = b.p90_hi;
    out.p95_lo = b.p95_lo;
    out.p95_hi = b.p95_hi;
    return out;
}

}  // namespace sirdfit::b200
