// model_b200.cpp — the reference's model.hpp API (/root/reference/proj/
// include/sirdfit/model.hpp:48-72) on the B200 engine.  Compiled in place of
// src/model.cpp (see b200_convert.hpp): every integration runs on the device
// (sg_integrate_batch, sg_sird_rhs_batch); the closed-form scalar helpers
// beta_at and basic_reproduction_number stay host functions, as in the
// engine's own C++ API.
#include "b200_convert.hpp"

namespace sirdfit {

using namespace sirdfit::b200;

double beta_at(const SirdParams& params, double t) {  // model.cpp:55-64
    return sf::beta_at(to_b200(params), t);
}

SirdState sird_rhs(const SirdState& state, double beta, double gamma, double mu, double population) {  // 66-74
    return translated([&] { return from_b200(sf::sird_rhs(to_b200(state), beta, gamma, mu, population)); });
}

void integrate_euler_into(const SirdParams& params, const SirdState& init, double population, int n_days,
                          int substeps, Trajectory& out) {  // model.cpp:76-107
    out = translated([&] { return from_b200(sf::integrate_euler(to_b200(params), to_b200(init), population, n_days,
                                                                 substeps)); });
}

Trajectory integrate_euler(const SirdParams& params, const SirdState& init, double population, int n_days,
                           int substeps) {  // model.cpp:109-114
    Trajectory out;
    integrate_euler_into(params, init, population, n_days, substeps, out);
    return out;
}

std::vector<Trajectory> integrate_batch(std::span<const SirdParams> batch, const SirdState& init, double population,
                                        int n_days, int substeps, int n_threads) {  // model.cpp:116-125
    return translated([&] {
        std::vector<sf::SirdParams> params;
        params.reserve(batch.size());
        for (const SirdParams& p : batch) params.push_back(to_b200(p));
        const std::vector<sf::Trajectory> trs =
            sf::integrate_batch(params, to_b200(init), population, n_days, substeps, n_threads);
        std::vector<Trajectory> out;
        out.reserve(trs.size());
        for (const sf::Trajectory& t : trs) out.push_back(from_b200(t));
        return out;
    });
}

double basic_reproduction_number(double beta, double gamma, double mu) {  // model.cpp:127-133
    return translated([&] { return sf::basic_reproduction_number(beta, gamma, mu); });
}

}  // namespace sirdfit
