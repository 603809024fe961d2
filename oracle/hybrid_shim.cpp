// hybrid_shim.cpp — the INTEGRATION.md §1 drop-in, compiled for real.
//
// TEST INFRASTRUCTURE.  The reference's own Swarm / optimize (pso.cpp, read
// unmodified from /root/reference/proj/src) driven by a BatchObjective whose
// body is the GPU engine's sg_eval_costs (include/sirdgpu.h) instead of the
// reference's make_window_objective.  tests/test_gpu_dropin.py checks that
// this hybrid follows the pure-reference trajectory bit for bit.
#include "oracle.h"
#include "sirdgpu.h"

#include "sirdfit/calibration.hpp"
#include "sirdfit/errors.hpp"
#include "sirdfit/pso.hpp"

#include <algorithm>
#include <limits>
#include <memory>
#include <span>
#include <vector>

using namespace sirdfit;

namespace {

sg_ctx* engine() {
    static sg_ctx* ctx = [] {
        sg_ctx* c = nullptr;
        return sg_ctx_create(0, &c) == SG_OK ? c : nullptr;
    }();
    return ctx;
}

// make_window_objective with the GPU body.
BatchObjective gpu_window_objective(int family, int metric, const double* I, const double* R, const double* D,
                                    int n_days, const double* init4, double population, int substeps) {
    sg_ctx* ctx = engine();
    if (!ctx) throw Error("no sm_100 device");
    sg_window* w = nullptr;
    if (sg_window_create(ctx, I, R, D, n_days, sg_state{init4[0], init4[1], init4[2], init4[3]}, population,
                         substeps, family, metric, &w) != SG_OK)
        throw Error(sg_last_error(ctx));
    std::shared_ptr<sg_window> win(w, sg_window_destroy);
    return [win, ctx](std::span<const double> positions, std::size_t dim, std::span<double> costs) {
        if (dim != 6 || positions.size() != costs.size() * dim) throw Error("window objective expects 6-dim positions");
        if (sg_eval_costs(win.get(), positions.data(), costs.size(), dim, costs.data()) != SG_OK)
            throw Error(sg_last_error(ctx));
    };
}

}  // namespace

extern "C" int hybrid_fit_swarm(int family, int metric, const double* I, const double* R, const double* D,
                                int n_days, const double* init4, double population, int substeps,
                                int /*n_threads*/, const double* lower6, const double* upper6, uint64_t n_particles, uint64_t max_iters,
                                double inertia, double cognitive, double social, uint64_t seed, int repair,
                                double* best6, double* best_cost, double* history) {
    try {
        const BatchObjective objective =
            gpu_window_objective(family, metric, I, R, D, n_days, init4, population, substeps);
        PsoConfig config;
        config.n_particles = n_particles;
        config.max_iters = max_iters;
        config.inertia = inertia;
        config.cognitive = cognitive;
        config.social = social;
        config.seed = seed;
        const SearchBounds bounds{std::vector<double>(lower6, lower6 + 6), std::vector<double>(upper6, upper6 + 6)};
        Swarm swarm(config, bounds, repair ? RepairHook(repair_time_order) : RepairHook{});
        for (uint64_t it = 0; it < max_iters; ++it) history[it] = swarm.step(objective);
        const std::span<const double> best = swarm.best_position();
        std::copy(best.begin(), best.end(), best6);
        *best_cost = swarm.best_cost();
        return swarm.best_cost() < std::numeric_limits<double>::infinity() ? 0 : 4;
    } catch (const std::exception&) {
        return 1;
    }
}
