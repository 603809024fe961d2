// calibration_b200.cpp — the reference's calibration.hpp API (/root/reference/
// proj/include/sirdfit/calibration.hpp:34-189) on the B200 engine.  Compiled
// in place of src/calibration.cpp (see b200_convert.hpp), it lets the
// reference's OWN callers — tools/main.cpp, bindings/module.cpp,
// tests/acceptance/main.cpp — run the window scheduler, the restart driver,
// the window objective and the forecast on the device, unchanged:
//
//   make_window_objective  -> a device window (sg_window_create / sg_eval_costs)
//   fit_window / fit_all_windows / stability_study
//                          -> concurrent device swarms (sg_fit_swarms) plus the
//                             device re-integration, R^2 and forecasts
//   forecast_extension     -> sg_forecast_batch
//   envelopes, quantile bands and the small window/bounds helpers
//                          -> the engine's host post-processing
//
// Results are the reference's bit for bit (tests/test_gpu_refbinding.py runs
// the reference's acceptance criteria and python smoke test on this binding
// and compares them with the pure-reference build).
#include "b200_convert.hpp"

namespace sirdfit {

using namespace sirdfit::b200;

std::vector<Window> make_windows(std::size_t n_days, const WindowScheme& scheme) {  // calibration.cpp:37-52
    return translated([&] {
        std::vector<Window> out;
        for (const sf::Window& w : sf::make_windows(n_days, sf::WindowScheme{scheme.tau, scheme.delta}))
            out.push_back(from_b200(w));
        return out;
    });
}

ParamBounds ParamBounds::stage1() { return from_b200(sf::ParamBounds::stage1()); }  // calibration.cpp:54-56

ParamBounds ParamBounds::stage2() { return from_b200(sf::ParamBounds::stage2()); }  // calibration.cpp:58-65

SearchBounds ParamBounds::to_search_bounds(std::size_t tau) const {  // calibration.cpp:67-76
    return translated([&] {
        const sf::SearchBounds b = to_b200(*this).to_search_bounds(tau);
        return SearchBounds{.lower = b.lower, .upper = b.upper};
    });
}

bool ParamBounds::contains(const SirdParams& params, std::size_t tau) const {  // calibration.cpp:78-83
    return to_b200(*this).contains(to_b200(params), tau);
}

SirdParams params_from_position(std::span<const double> position) {  // calibration.cpp:85-87
    return from_b200(sf::params_from_position(position));
}

void repair_time_order(std::span<double> position) { sf::repair_time_order(position); }  // calibration.cpp:89-93

// The slices must view the caller's own series (calibration.cpp:95-104):
// validated by the engine's rule, cut here.
WindowSlice slice_window(const EpiSeries& data, const Window& window) {
    if (window.length == 0 || window.start + window.length > data.size())
        throw SchemeError("window " + std::to_string(window.index) + " falls outside the series");
    return WindowSlice{.infectious = std::span(data.infectious).subspan(window.start, window.length),
                       .recovered_cum = std::span(data.recovered_cum).subspan(window.start, window.length),
                       .deaths_cum = std::span(data.deaths_cum).subspan(window.start, window.length)};
}

SirdState window_initial_state(const EpiSeries& data, std::size_t day, double population) {  // 106-118
    return translated([&] { return from_b200(sf::window_initial_state(to_b200(data), day, population)); });
}

BatchObjective make_window_objective(const ObjectiveSpec& spec, const WindowSlice& observed, const SirdState& init,
                                     double population, int substeps, int n_threads) {  // calibration.cpp:120-155
    BatchObjective device = translated([&] {
        return sf::make_window_objective(to_b200(spec), to_b200(observed), to_b200(init), population, substeps,
                                         n_threads);
    });
    return [device = std::move(device)](std::span<const double> positions, std::size_t dim, std::span<double> costs) {
        translated([&] { device(positions, dim, costs); });
    };
}

FitResult fit_window(const EpiSeries& data, const Window& window, const FitSettings& settings,
                     std::uint64_t seed) {  // calibration.cpp:157-188
    return translated([&] { return from_b200(sf::fit_window(to_b200(data), to_b200(window), to_b200(settings), seed)); });
}

FitAllResult fit_all_windows(const EpiSeries& data, const WindowScheme& scheme, const FitSettings& settings,
                             std::uint64_t base_seed) {  // calibration.cpp:190-216
    return translated([&] {
        const sf::FitAllResult r = sf::fit_all_windows(to_b200(data), sf::WindowScheme{scheme.tau, scheme.delta},
                                                       to_b200(settings), base_seed);
        FitAllResult out;
        for (const sf::FitResult& f : r.fits) out.fits.push_back(from_b200(f));
        out.mean_r2_d = r.mean_r2_d;
        out.failed_count = r.failed_count;
        return out;
    });
}

Envelope build_envelope(const std::vector<std::vector<double>>& values_per_day) {  // calibration.cpp:218-245
    return from_b200(sf::build_envelope(values_per_day));
}

ParameterEnvelopes parameter_envelopes(std::span<const FitResult> fits, std::size_t n_days) {  // 247-274
    const std::vector<sf::FitResult> f = to_b200(fits);
    const sf::ParameterEnvelopes e = sf::parameter_envelopes(f, n_days);
    return ParameterEnvelopes{.beta = from_b200(e.beta), .gamma = from_b200(e.gamma), .mu = from_b200(e.mu),
                              .r0 = from_b200(e.r0)};
}

CompartmentEnvelopes compartment_envelopes(std::span<const FitResult> fits, std::size_t n_days) {  // 276-296
    const std::vector<sf::FitResult> f = to_b200(fits);
    const sf::CompartmentEnvelopes e = sf::compartment_envelopes(f, n_days);
    return CompartmentEnvelopes{.infectious = from_b200(e.infectious), .recovered = from_b200(e.recovered),
                                .deaths = from_b200(e.deaths)};
}

Forecast forecast_extension(const FitResult& fit, std::size_t horizon, int substeps) {  // calibration.cpp:298-322
    return translated([&] {
        const sf::Forecast f = sf::forecast_extension(to_b200(fit), horizon, substeps);
        Forecast out;
        out.junction_day = f.junction_day;
        out.horizon = f.horizon;
        out.trajectory = from_b200(f.trajectory);
        return out;
    });
}

double quantile_sorted(std::span<const double> sorted, double p) { return sf::quantile_sorted(sorted, p); }  // 324-335

QuantileBands build_quantile_bands(const std::vector<std::vector<double>>& values_per_day) {  // 337-361
    return from_b200(sf::build_quantile_bands(values_per_day));
}

ScalarBands build_scalar_bands(std::vector<double> values) {  // calibration.cpp:363-376
    return from_b200(sf::build_scalar_bands(std::move(values)));
}

StabilityResult stability_study(const EpiSeries& data, const Window& window, const FitSettings& settings,
                                std::size_t repetitions, std::size_t horizon,
                                std::uint64_t base_seed) {  // calibration.cpp:378-436
    return translated([&] {
        const sf::StabilityResult r = sf::stability_study(to_b200(data), to_b200(window), to_b200(settings),
                                                          repetitions, horizon, base_seed);
        StabilityResult out;
        out.window = from_b200(r.window);
        out.horizon = r.horizon;
        out.repetitions = r.repetitions;
        out.failed = r.failed;
        out.beta = from_b200(r.beta);
        out.r0 = from_b200(r.r0);
        out.infectious = from_b200(r.infectious);
        out.recovered = from_b200(r.recovered);
        out.deaths = from_b200(r.deaths);
        out.gamma = from_b200(r.gamma);
        out.mu = from_b200(r.mu);
        for (const sf::FitResult& f : r.fits) out.fits.push_back(from_b200(f));
        return out;
    });
}

}  // namespace sirdfit
