// Drop-in replacement for proj/src/laplace.cpp (laplace.hpp:20-59): grid
// arithmetic on the host, fsm_invert / rational_invert on the B200.
#include <cmath>
#include <numbers>

#include "fdsweep_b200_shim.hpp"

namespace fdsweep {

FsmGrid::FsmGrid(double T, int ns) : period(T), sample_count(ns) {
    if (!(period > 0.0)) throw ValidationError("FsmGrid: period must be positive");
    if (sample_count < 2 || sample_count % 2 != 0) throw ValidationError("FsmGrid: sample count must be even and positive");
}
double FsmGrid::delta_omega() const { return 2.0 * std::numbers::pi / period; }
double FsmGrid::delta_t() const { return period / sample_count; }
double FsmGrid::omega_max() const { return std::numbers::pi / delta_t(); }
int FsmGrid::contour_count() const { return sample_count / 2 + 1; }
std::vector<Complex> FsmGrid::contour(double eta) const {
    std::vector<Complex> s(contour_count());
    for (int k = 0; k < contour_count(); ++k) s[k] = Complex(eta, k * delta_omega());
    return s;
}
std::vector<double> FsmGrid::time_grid() const {
    std::vector<double> t(sample_count);
    for (int n = 0; n < sample_count; ++n) t[n] = n * delta_t();
    return t;
}

double damping_eta(double kappa, double T) {
    if (!(T > 0.0)) throw ValidationError("damping_eta: period must be positive");
    return kappa * std::log(10.0) / T;
}

double hanning_window(int k, int ns) {
    if (k < 0 || k >= ns) throw ValidationError("hanning_window: index out of range");
    return 0.5 * (1.0 + std::cos(2.0 * std::numbers::pi * k / ns));
}

std::vector<Complex> conjugate_fill(std::span<const Complex> half) {
    if (half.size() < 2) throw ValidationError("conjugate_fill: need at least two entries");
    const int n = 2 * (static_cast<int>(half.size()) - 1);
    std::vector<Complex> full(n);
    full[0] = Complex(half[0].real(), 0.0);
    full[n / 2] = Complex(half[n / 2].real(), 0.0);
    for (int k = 1; k < n / 2; ++k) {
        full[k] = half[k];
        full[n - k] = std::conj(half[k]);
    }
    return full;
}

TimeSeries fsm_invert(const FsmGrid& grid, double eta, const std::vector<std::vector<Complex>>& half,
                      std::vector<std::string> labels, bool hanning) {
    return b200::fsm_invert(grid, eta, half, std::move(labels), hanning);
}

TimeSeries rational_invert(const RationalModel& model, std::span<const double> t) {
    return b200::rational_invert(model, t);
}

}  // namespace fdsweep
