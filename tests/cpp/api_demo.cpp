// api_demo.cpp — the C++ calibration API (include/sirdfit_b200.hpp) used the
// way a reference maintainer would after `namespace sf = sirdfit_b200;`
// (INTEGRATION.md §2).  TEST INFRASTRUCTURE: tests/test_cpp_api.py compiles it
// on the CPU and, on a B200, runs it and compares every printed value with the
// Python API on the same inputs.
//
//   api_demo <poland_like.csv>   -> "key hex-double" lines
#include "sirdfit_b200.hpp"

#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

namespace sf = sirdfit_b200;

static void put(const char* key, double v) { std::printf("%s %a\n", key, v); }

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    sf::EpiSeries data;
    std::ifstream in(argv[1]);
    std::string line;
    std::getline(in, line);  // header: day,new_cases,infectious,recovered_cum,deaths_cum (any order below)
    std::vector<std::string> cols;
    {
        std::stringstream ss(line);
        std::string c;
        while (std::getline(ss, c, ',')) cols.push_back(c);
    }
    while (std::getline(in, line)) {
        std::stringstream ss(line);
        std::string c;
        for (std::size_t k = 0; std::getline(ss, c, ','); ++k) {
            const double v = std::stod(c);
            if (cols[k] == "infectious") data.infectious.push_back(v);
            else if (cols[k] == "recovered_cum") data.recovered_cum.push_back(v);
            else if (cols[k] == "deaths_cum") data.deaths_cum.push_back(v);
            else if (cols[k] == "new_cases") data.new_cases.push_back(v);
        }
    }
    try {
        sf::FitSettings s;
        s.spec = sf::parse_objective("ird-mxse");
        s.population = 38e6;
        s.pso.n_particles = 256;
        s.pso.max_iters = 60;
        const sf::Window w0{0, 0, 21};
        const sf::FitResult fit = sf::fit_window(data, w0, s, 2204);
        put("fit.objective", fit.objective);
        put("fit.r2_d", fit.r2_d);
        put("fit.beta1", fit.params.beta1);
        put("fit.t2", fit.params.t2);
        put("fit.mu", fit.params.mu);
        const sf::Forecast fc = sf::forecast_extension(fit, 7);
        put("forecast.D7", fc.trajectory.states.back().D);

        s.pso.n_particles = 300;
        s.pso.max_iters = 20;
        const sf::FitAllResult all = sf::fit_all_windows(data, sf::WindowScheme{35, 60}, s, 7);
        std::printf("all.n %zu\n", all.fits.size());
        for (std::size_t k = 0; k < all.fits.size(); ++k) put(("all.objective." + std::to_string(k)).c_str(),
                                                              all.fits[k].objective);
        put("all.mean_r2_d", all.mean_r2_d);

        s.spec = sf::parse_objective("d-mse");
        s.pso.n_particles = 128;
        s.pso.max_iters = 15;
        const sf::StabilityResult st = sf::stability_study(data, sf::Window{0, 100, 21}, s, 6, 5, 11);
        put("stability.deaths_median_last", st.deaths.median.back());
        put("stability.gamma_median", st.gamma.median);

        const sf::WindowSlice obs = sf::slice_window(data, sf::Window{0, 40, 36});
        const sf::BatchObjective f = sf::make_window_objective(sf::parse_objective("ird-mape"), obs,
                                                               sf::window_initial_state(data, 40, 38e6), 38e6, 24, 8);
        const std::vector<double> pos = {0.3, 0.2, 5.0, 20.0, 0.1, 0.01, 1.5, 0.05, 30.0, 2.0, 0.5, 0.002};
        std::vector<double> costs(2);
        f(pos, 6, costs);
        put("objective.cost0", costs[0]);
        put("objective.cost1", costs[1]);
    } catch (const sf::Error& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
    return 0;
}
