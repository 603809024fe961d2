// api_parity.cpp — the engine's C++ API (sirdfit_b200, include/sirdfit_b200.hpp)
// against the UNMODIFIED reference (namespace sirdfit, its src/*.cpp compiled
// in place by oracle/Makefile) in one process, bit for bit:
//
//   optimize / Swarm      host objectives of several dimensions (the draws of a
//                         100-d move cross the MT19937-64 twist), a host repair
//                         hook, the window objective on the fused path and on
//                         a stepped Swarm, and the reference's acceptance
//                         sphere (pso.cpp:47-143, acceptance/main.cpp:148-177)
//   objective_value, metric_value, minmax_normalize, sird_rhs,
//   integrate_euler_into  (objectives.cpp:72-120, model.cpp:66-107)
//   envelopes             build_envelope / parameter_envelopes /
//                         compartment_envelopes (calibration.cpp:218-296)
//
// TEST INFRASTRUCTURE: tests/test_gpu_refbinding.py runs it on a B200.
// Prints one line per check ("ok <name>" / "MISMATCH <name> ..."); exit 1 on
// any mismatch.
#include "sirdfit/calibration.hpp"
#include "sirdfit/errors.hpp"
#include "sirdfit/model.hpp"
#include "sirdfit/objectives.hpp"
#include "sirdfit/pso.hpp"

#include "sirdfit_b200.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <vector>

namespace ref = sirdfit;
namespace sf = sirdfit_b200;

static int g_bad = 0;

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0 || (std::isnan(a) && std::isnan(b)); }

static bool same(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t k = 0; k < a.size(); ++k)
        if (!same(a[k], b[k])) return false;
    return true;
}

static void report(const std::string& name, bool ok, const std::string& detail = "") {
    std::printf("%s %s%s%s\n", ok ? "ok" : "MISMATCH", name.c_str(), detail.empty() ? "" : " ", detail.c_str());
    if (!ok) ++g_bad;
}

static bool same_result(const ref::PsoResult& a, const sf::PsoResult& b) {
    return same(a.best_cost, b.best_cost) && same(a.best_position, b.best_position) &&
           same(a.cost_history, b.cost_history);
}

// the same objective body for both namespaces (the std::function types coincide)
static void sphere(std::span<const double> x, std::size_t dim, std::span<double> c) {
    for (std::size_t k = 0; k < c.size(); ++k) {
        double acc = 0.0;
        for (std::size_t d = 0; d < dim; ++d) acc += x[k * dim + d] * x[k * dim + d];
        c[k] = acc;
    }
}

static void rosenbrock(std::span<const double> x, std::size_t dim, std::span<double> c) {
    for (std::size_t k = 0; k < c.size(); ++k) {
        double acc = 0.0;
        for (std::size_t d = 0; d + 1 < dim; ++d) {
            const double a = x[k * dim + d], b = x[k * dim + d + 1];
            acc += 100.0 * (b - a * a) * (b - a * a) + (1.0 - a) * (1.0 - a);
        }
        c[k] = acc;
    }
}

template <class Box>
static void pso_case(const std::string& name, std::size_t n, std::size_t iters, const Box& box, uint64_t seed,
                     const ref::BatchObjective& f, const ref::RepairHook& repair = {}, double w = 0.5,
                     double c1 = 0.5, double c2 = 0.5) {
    ref::PsoConfig rc;
    rc.n_particles = n;
    rc.max_iters = iters;
    rc.seed = seed;
    rc.inertia = w;
    rc.cognitive = c1;
    rc.social = c2;
    sf::PsoConfig sc;
    sc.n_particles = n;
    sc.max_iters = iters;
    sc.seed = seed;
    sc.inertia = w;
    sc.cognitive = c1;
    sc.social = c2;
    const ref::SearchBounds rb{box.first, box.second};
    const sf::SearchBounds sb{box.first, box.second};
    const ref::PsoResult want = ref::optimize(rc, rb, f, repair);
    const sf::PsoResult got = sf::optimize(sc, sb, f, repair);
    report(name, same_result(want, got),
           "best " + std::to_string(want.best_cost) + " vs " + std::to_string(got.best_cost));
}

int main() {
    try {
        // ---- optimize / Swarm with host objectives -------------------------------
        const auto box = [](std::size_t dim, double lo, double hi) {
            return std::make_pair(std::vector<double>(dim, lo), std::vector<double>(dim, hi));
        };
        for (uint64_t seed : {0ull, 7ull})  // the acceptance sphere (#3): default PsoConfig, 6-d [0, 10]
            pso_case("optimize.sphere6.default.seed" + std::to_string(seed), 10000, 100, box(6, 0.0, 10.0), seed,
                     sphere);
        pso_case("optimize.rosenbrock3", 500, 60, box(3, -2.0, 2.0), 11, rosenbrock, {}, 0.7298, 1.4962, 1.4962);
        pso_case("optimize.sphere1", 33, 25, box(1, -5.0, 3.0), 3, sphere);
        pso_case("optimize.sphere100.twist_crossing", 64, 12, box(100, -1.0, 1.0), 5, sphere);
        const ref::RepairHook sort2 = [](std::span<double> x) {
            if (x[0] > x[1]) std::swap(x[0], x[1]);
        };
        pso_case("optimize.rosenbrock8.host_repair", 300, 30, box(8, -2.0, 2.0), 13, rosenbrock, sort2);
        int calls = 0;
        const ref::BatchObjective infeasible = [&](std::span<const double>, std::size_t, std::span<double> c) {
            ++calls;
            for (double& v : c) v = std::numeric_limits<double>::quiet_NaN();
        };
        bool threw_ref = false, threw_sf = false;
        try {
            ref::optimize(ref::PsoConfig{.n_particles = 20, .max_iters = 3}, ref::SearchBounds{{0.0}, {1.0}}, infeasible);
        } catch (const ref::AllInfeasibleError&) {
            threw_ref = true;
        }
        try {
            sf::optimize(sf::PsoConfig{.n_particles = 20, .max_iters = 3}, sf::SearchBounds{{0.0}, {1.0}}, infeasible);
        } catch (const sf::AllInfeasibleError&) {
            threw_sf = true;
        }
        report("optimize.all_infeasible_throws", threw_ref && threw_sf && calls == 6);
        {  // Swarm accessors after a few steps (pso.hpp:60-69)
            ref::Swarm rs(ref::PsoConfig{.n_particles = 50, .max_iters = 5, .seed = 9}, ref::SearchBounds{{-1, -1}, {1, 1}});
            sf::Swarm ss(sf::PsoConfig{.n_particles = 50, .max_iters = 5, .seed = 9}, sf::SearchBounds{{-1, -1}, {1, 1}});
            bool ok = true;
            for (int it = 0; it < 5; ++it) {
                ok = ok && same(rs.step(sphere), ss.step(sphere));
                ok = ok && same(std::vector<double>(rs.positions().begin(), rs.positions().end()),
                                std::vector<double>(ss.positions().begin(), ss.positions().end()));
                ok = ok && same(std::vector<double>(rs.best_position().begin(), rs.best_position().end()),
                                std::vector<double>(ss.best_position().begin(), ss.best_position().end()));
            }
            report("swarm.step_positions_best", ok && rs.iterations_done() == ss.iterations_done());
        }

        // ---- window objectives -----------------------------------------------------
        const double N = 1e6;
        const ref::SirdParams gen{.beta1 = 0.6, .beta2 = 0.3, .t1 = 8.0, .t2 = 16.0, .gamma = 0.1, .mu = 0.012};
        const ref::Trajectory truth = ref::integrate_euler(gen, ref::SirdState{.S = N - 100.0, .I = 100.0}, N, 40);
        std::vector<double> I, R, D;
        for (const auto& s : truth.states) {
            I.push_back(s.I);
            R.push_back(s.R);
            D.push_back(s.D * 1.01);
        }
        const ref::WindowSlice slice{std::span(I).subspan(2, 30), std::span(R).subspan(2, 30), std::span(D).subspan(2, 30)};
        const sf::WindowSlice sslice{slice.infectious, slice.recovered_cum, slice.deaths_cum};
        const ref::SirdState init{.S = N - I[2] - R[2] - D[2], .I = I[2], .R = R[2], .D = D[2]};
        const sf::SirdState sinit{init.S, init.I, init.R, init.D};
        const ref::SearchBounds wb = ref::ParamBounds::stage2().to_search_bounds(29);
        const sf::SearchBounds swb{wb.lower, wb.upper};
        for (const char* spec : {"ird-mxse", "d-mape"}) {
            const ref::BatchObjective rf = ref::make_window_objective(ref::parse_objective(spec), slice, init, N, 24, 1);
            const sf::BatchObjective gf = sf::make_window_objective(sf::parse_objective(spec), sslice, sinit, N, 24, 1);
            ref::PsoConfig rc{.n_particles = 700, .max_iters = 25, .seed = 21};
            sf::PsoConfig sc{.n_particles = 700, .max_iters = 25, .seed = 21};
            const ref::PsoResult want = ref::optimize(rc, wb, rf, ref::repair_time_order);
            report(std::string("optimize.window_fused.") + spec,
                   same_result(want, sf::optimize(sc, swb, gf, sf::repair_time_order)));
            // a stepped device Swarm on the window objective (device evaluation, no host copy)
            sf::Swarm sw(sc, swb, sf::repair_time_order);
            std::vector<double> hist;
            for (int it = 0; it < 25; ++it) hist.push_back(sw.step(gf));
            report(std::string("swarm.window_stepped.") + spec,
                   same(hist, want.cost_history) &&
                       same(std::vector<double>(sw.best_position().begin(), sw.best_position().end()),
                            want.best_position));
            // the window objective with a hook the device does not know (host repair)
            const ref::RepairHook flip = [](std::span<double> x) {
                if (x[2] > x[3]) std::swap(x[2], x[3]);
                if (x[4] < 0.05) x[4] = 0.05;
            };
            report(std::string("optimize.window_host_repair.") + spec,
                   same_result(ref::optimize(rc, wb, rf, flip), sf::optimize(sc, swb, gf, flip)));
        }

        // ---- objectives and model on the device ----------------------------------------
        std::mt19937_64 rng(5);
        std::uniform_real_distribution<double> u(0.0, 1.0);
        bool ok_obj = true, ok_metric = true, ok_rhs = true, ok_int = true;
        for (int k = 0; k < 40; ++k) {
            const ref::SirdParams p{.beta1 = 2 * u(rng), .beta2 = 2 * u(rng), .t1 = 29 * u(rng), .t2 = 29 * u(rng),
                                    .gamma = u(rng), .mu = 0.1 * u(rng)};
            ref::Trajectory tr;
            ref::integrate_euler_into(p, init, N, 30, 24, tr);
            sf::Trajectory str;
            sf::integrate_euler_into(sf::SirdParams{p.beta1, p.beta2, p.t1, p.t2, p.gamma, p.mu}, sinit, N, 30, 24, str);
            for (std::size_t d = 0; d < 30; ++d)
                ok_int = ok_int && same(tr.states[d].S, str.states[d].S) && same(tr.states[d].I, str.states[d].I) &&
                         same(tr.states[d].R, str.states[d].R) && same(tr.states[d].D, str.states[d].D);
            ok_int = ok_int && tr.finite == str.finite;
            for (const char* spec : {"d-mxse", "d-mse", "d-mae", "d-mape", "ird-mxse", "ird-mse", "ird-mae", "ird-mape"})
                ok_obj = ok_obj && same(ref::objective_value(ref::parse_objective(spec), slice, tr),
                                        sf::objective_value(sf::parse_objective(spec), sslice, str));
            std::vector<double> pred;
            for (const auto& s : tr.states) pred.push_back(s.D);
            for (auto m : {ref::Metric::MXSE, ref::Metric::MSE, ref::Metric::MAE, ref::Metric::MAPE})
                ok_metric = ok_metric && same(ref::metric_value(m, slice.deaths_cum, pred),
                                              sf::metric_value(static_cast<sf::Metric>(static_cast<int>(m)),
                                                               slice.deaths_cum, pred));
        }
        {
            std::mt19937_64 r1(77), r2(77);
            for (int k = 0; k < 40; ++k) {
                const ref::SirdState st{.S = N * u(r1), .I = 1e4 * u(r1), .R = 1e3 * u(r1), .D = 10 * u(r1)};
                const double b = 3 * u(r1), g = u(r1), m = 0.1 * u(r1);
                const ref::SirdState a = ref::sird_rhs(st, b, g, m, N);
                const sf::SirdState c = sf::sird_rhs(sf::SirdState{st.S, st.I, st.R, st.D}, b, g, m, N);
                ok_rhs = ok_rhs && same(a.S, c.S) && same(a.I, c.I) && same(a.R, c.R) && same(a.D, c.D);
            }
        }
        report("integrate_euler_into", ok_int);
        report("objective_value.8specs", ok_obj);
        report("metric_value.4metrics", ok_metric);
        report("sird_rhs", ok_rhs);
        {
            const std::vector<double> v = {3.0, -1.0, 2.5, 7.0};
            report("minmax_normalize", same(ref::minmax_normalize(v, -1.0, 7.0), sf::minmax_normalize(v, -1.0, 7.0)));
            bool both = false;
            try {
                ref::minmax_normalize(v, 1.0, 1.0);
            } catch (const ref::DegenerateRangeError&) {
                try {
                    sf::minmax_normalize(v, 1.0, 1.0);
                } catch (const sf::DegenerateRangeError&) {
                    both = true;
                }
            }
            report("minmax_normalize.degenerate", both);
        }

        // ---- envelopes ------------------------------------------------------------------
        {
            std::vector<std::vector<double>> cols(9);
            for (std::size_t d = 0; d < cols.size(); ++d)
                for (std::size_t k = 0; k < d; ++k) cols[d].push_back(k % 3 == 2 ? std::nan("") : u(rng) - 0.5);
            const ref::Envelope a = ref::build_envelope(cols);
            const sf::Envelope b = sf::build_envelope(cols);
            report("build_envelope", a.count == b.count && same(a.outer_lo, b.outer_lo) && same(a.outer_hi, b.outer_hi) &&
                                         same(a.band1_lo, b.band1_lo) && same(a.band1_hi, b.band1_hi) &&
                                         same(a.band2_lo, b.band2_lo) && same(a.band2_hi, b.band2_hi) &&
                                         same(a.median, b.median));
        }
    } catch (const std::exception& e) {
        std::printf("MISMATCH exception %s\n", e.what());
        return 1;
    }
    return g_bad ? 1 : 0;
}
