// threads_demo.cpp — reentrancy of the C++ layer (one process-wide
// context per device is shared by every host thread).  The reference's
// make_window_objective closures and fit_window are reentrant; here four
// threads hammer objectives of the shared context at once — one objective
// shared by all threads, one private per thread, batch sizes that force the
// context's scratch buffers to regrow — while a fifth runs fit_window.
// Every result must equal the single-threaded result bit for bit.
// TEST INFRASTRUCTURE: tests/test_cpp_api.py builds and runs it on a B200.
//
//   threads_demo <poland_like.csv>   -> "threads ok <calls>" or a mismatch line
#include "sirdfit_b200.hpp"

#include <atomic>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

namespace sf = sirdfit_b200;

static sf::EpiSeries load(const char* path) {
    sf::EpiSeries data;
    std::ifstream in(path);
    std::string line;
    std::getline(in, line);
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
    return data;
}

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const sf::EpiSeries data = load(argv[1]);
    const double N = 38e6;
    constexpr int kThreads = 4;
    constexpr int kRounds = 60;
    const std::size_t sizes[] = {37, 4096, 300, 9000, 1};
    try {
        auto objective_at = [&](std::size_t start, const char* spec) {
            const sf::WindowSlice obs = sf::slice_window(data, sf::Window{0, start, 36});
            return sf::make_window_objective(sf::parse_objective(spec), obs, sf::window_initial_state(data, start, N),
                                             N, 24, 1);
        };
        const sf::BatchObjective shared = objective_at(60, "ird-mxse");
        std::vector<sf::BatchObjective> own;
        const char* specs[kThreads] = {"ird-mse", "d-mape", "ird-mae", "d-mxse"};
        for (int t = 0; t < kThreads; ++t) own.push_back(objective_at(30 * t, specs[t]));
        // inputs and single-threaded answers
        std::vector<std::vector<double>> pos(std::size(sizes));
        std::mt19937_64 rng(11);
        std::uniform_real_distribution<double> u(0.0, 1.0);
        const double hi[6] = {2.0, 2.0, 28.0, 28.0, 1.0, 0.1};
        for (std::size_t k = 0; k < std::size(sizes); ++k) {
            pos[k].resize(6 * sizes[k]);
            for (std::size_t i = 0; i < pos[k].size(); ++i) pos[k][i] = u(rng) * hi[i % 6];
        }
        auto eval = [](const sf::BatchObjective& f, const std::vector<double>& p) {
            std::vector<double> c(p.size() / 6);
            f(p, 6, c);
            return c;
        };
        std::vector<std::vector<double>> want_shared, want_own[kThreads];
        for (const auto& p : pos) want_shared.push_back(eval(shared, p));
        for (int t = 0; t < kThreads; ++t)
            for (const auto& p : pos) want_own[t].push_back(eval(own[t], p));
        sf::FitSettings s;
        s.population = N;
        s.pso.n_particles = 512;
        s.pso.max_iters = 40;
        const sf::FitResult want_fit = sf::fit_window(data, sf::Window{0, 200, 36}, s, 99);

        std::atomic<int> bad{0};
        std::atomic<long> calls{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < kThreads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (int r = 0; r < kRounds; ++r) {
                        const std::size_t k = static_cast<std::size_t>(r + t) % std::size(sizes);
                        if (!same_bits(eval(shared, pos[k]), want_shared[k])) ++bad;
                        if (!same_bits(eval(own[t], pos[k]), want_own[t][k])) ++bad;
                        calls += 2;
                    }
                } catch (const sf::Error& e) {
                    std::printf("thread error %s\n", e.what());
                    ++bad;
                }
            });
        }
        pool.emplace_back([&] {
            try {
                for (int r = 0; r < 3; ++r) {
                    const sf::FitResult f = sf::fit_window(data, sf::Window{0, 200, 36}, s, 99);
                    if (f.objective != want_fit.objective || !same_bits(f.cost_history, want_fit.cost_history)) ++bad;
                    ++calls;
                }
            } catch (const sf::Error& e) {
                std::printf("thread error %s\n", e.what());
                ++bad;
            }
        });
        for (std::thread& th : pool) th.join();
        if (bad) {
            std::printf("threads mismatch %d of %ld calls\n", bad.load(), calls.load());
            return 1;
        }
        std::printf("threads ok %ld\n", calls.load());
    } catch (const sf::Error& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
    return 0;
}
