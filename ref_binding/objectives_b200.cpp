// objectives_b200.cpp — the reference's objectives.hpp API (/root/reference/
// proj/include/sirdfit/objectives.hpp:25-50) on the B200 engine.  Compiled in
// place of src/objectives.cpp (see b200_convert.hpp): metric_value and
// objective_value score on the device (sg_metric_values,
// sg_objective_values); r_squared_d, the name parsing and minmax_normalize
// are the engine's host helpers.
#include "b200_convert.hpp"

namespace sirdfit {

using namespace sirdfit::b200;

double metric_value(Metric metric, std::span<const double> observed, std::span<const double> predicted) {
    return translated([&] { return sf::metric_value(to_b200(metric), observed, predicted); });
}

std::vector<double> minmax_normalize(std::span<const double> values, double ref_min, double ref_max) {
    return translated([&] { return sf::minmax_normalize(values, ref_min, ref_max); });
}

double objective_value(const ObjectiveSpec& spec, const WindowSlice& observed, const Trajectory& predicted) {
    return translated([&] { return sf::objective_value(to_b200(spec), to_b200(observed), to_b200(predicted)); });
}

double r_squared_d(std::span<const double> observed_d, std::span<const double> predicted_d) {
    return translated([&] { return sf::r_squared_d(observed_d, predicted_d); });
}

ObjectiveSpec parse_objective(std::string_view name) {
    return translated([&] { return from_b200(sf::parse_objective(name)); });
}

std::string objective_name(const ObjectiveSpec& spec) { return sf::objective_name(to_b200(spec)); }

std::string metric_name(Metric metric) { return sf::metric_name(to_b200(metric)); }

}  // namespace sirdfit
