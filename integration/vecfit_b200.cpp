// Drop-in replacement for proj/src/vecfit.cpp: the reference's vecfit.hpp API
// (vecfit.hpp:48-86) implemented by forwarding to libfdsweep_b200 (GPU).
// Linked instead of vecfit.cpp, it makes the reference's own run_afs
// (afs.cpp:226-396) fit on the B200, eval_model / fit_error_evf included; the
// O(M) pole utilities (conjugate closure, canonical order, starting poles)
// are host bookkeeping and keep the reference semantics here.
#include <algorithm>
#include <cmath>

#include "fdsweep_b200_shim.hpp"

namespace fdsweep {

bool is_conjugate_closed(std::span<const Complex> poles, double rel_tol) {  // vecfit.cpp:116-132
    std::vector<char> used(poles.size(), 0);
    for (size_t i = 0; i < poles.size(); ++i) {
        if (used[i] || poles[i].imag() == 0.0) continue;
        bool hit = false;
        for (size_t k = 0; k < poles.size() && !hit; ++k) {
            if (k == i || used[k]) continue;
            const double sc = std::max({std::abs(poles[i]), std::abs(poles[k]), 1e-300});
            if (std::abs(poles[i] - std::conj(poles[k])) <= rel_tol * sc) { used[i] = used[k] = 1; hit = true; }
        }
        if (!hit) return false;
    }
    return true;
}

std::vector<Complex> canonical_poles(std::span<const Complex> poles) {  // vecfit.cpp:134-169
    std::vector<Complex> heads, reals;
    std::vector<char> used(poles.size(), 0);
    for (size_t i = 0; i < poles.size(); ++i) {
        if (used[i]) continue;
        if (poles[i].imag() == 0.0) { reals.push_back(poles[i]); used[i] = 1; continue; }
        size_t k = i + 1;
        for (; k < poles.size(); ++k) {
            if (used[k] || poles[k].imag() == 0.0) continue;
            const double sc = std::max({std::abs(poles[i]), std::abs(poles[k]), 1e-300});
            if (std::abs(poles[i] - std::conj(poles[k])) <= 1e-9 * sc) break;
        }
        if (k == poles.size()) throw ValidationError("pole set is not closed under conjugation");
        heads.push_back(poles[i].imag() > 0.0 ? poles[i] : poles[k]);
        used[i] = used[k] = 1;
    }
    std::vector<Complex> out;
    for (Complex h : heads) { out.push_back(h); out.push_back(std::conj(h)); }
    out.insert(out.end(), reals.begin(), reals.end());
    return out;
}

std::vector<Complex> initial_poles(double omega_max, int order) {  // vecfit.cpp:171-186
    if (order < 1) throw ValidationError("initial_poles: order must be >= 1");
    if (!(omega_max > 0.0)) throw ValidationError("initial_poles: omega_max must be positive");
    std::vector<Complex> p;
    for (int i = 1; i <= order / 2; ++i) {
        const double beta = omega_max * static_cast<double>(i) / (order / 2);
        p.emplace_back(-beta / 100.0, beta);
        p.emplace_back(-beta / 100.0, -beta);
    }
    if (order % 2) p.emplace_back(-omega_max / 100.0, 0.0);
    return p;
}

std::vector<Complex> relocate_poles(std::span<const FrequencySample> samples, std::span<const Complex> poles,
                                    RelocationStats* stats) {
    if (samples.empty()) throw ValidationError("relocate_poles: no samples");
    return b200::relocate_poles(samples, poles, stats);
}

std::vector<Complex> identify_residues(std::span<const Complex> freqs, std::span<const Complex> values,
                                       std::span<const Complex> poles, double* residual_rms) {
    if (values.size() != freqs.size()) throw ValidationError("identify_residues: freqs/values size mismatch");
    return b200::identify_residues(freqs, values, poles, residual_rms);
}

std::pair<RationalModel, FitReport> vector_fit(std::span<const FrequencySample> samples, std::span<const int> orf,
                                               int order, int n_relocations, std::vector<std::string> labels) {
    if (samples.empty()) throw ValidationError("vector_fit: no samples");
    const int K = static_cast<int>(samples[0].values.size());
    if (!labels.empty() && static_cast<int>(labels.size()) != K) throw ValidationError("vector_fit: label count mismatch");
    return b200::vector_fit(samples, orf, order, n_relocations, std::move(labels));
}

// One (channel, s) point: M complex divisions. The reference's channel_errors
// (afs.cpp:118-145) calls this G x K times per iteration, where a device round
// trip per call would cost ~10^3 times the arithmetic, so the scalar form stays
// on the host; every batched evaluation (eval_model over the channels,
// fit_error_evf over the samples, fds_eval_model over a grid, the GPU AFS
// driver's channel errors) runs on the device.
Complex eval_model_channel(const RationalModel& model, int channel, Complex s) {  // vecfit.cpp:490-501
    if (channel < 0 || channel >= model.channel_count()) throw ValidationError("eval_model_channel: channel out of range");
    Complex acc(0.0, 0.0);
    for (int m = 0; m < model.order(); ++m) {
        const Complex d = s - model.poles[m];
        if (d == 0.0) throw NumericError("eval_model: s coincides with a pole");
        acc += model.residues[channel][m] / d;
    }
    return acc;
}

std::vector<Complex> eval_model(const RationalModel& model, Complex s) {  // vecfit.cpp:503-509
    const int K = model.channel_count(), M = model.order();
    std::vector<Complex> res(static_cast<size_t>(K) * M), out(K);
    for (int k = 0; k < K; ++k) std::copy(model.residues[k].begin(), model.residues[k].end(), res.begin() + static_cast<size_t>(k) * M);
    b200::check(fds_eval_model(M, b200::c(model.poles.data()), K, b200::c(res.data()), 1, b200::c(&s), b200::c(out.data())));
    return out;
}

double fit_error_evf(const RationalModel& model, int channel, std::span<const FrequencySample> samples) {  // :511-526
    if (samples.empty()) throw ValidationError("fit_error_evf: no samples");
    if (channel < 0 || channel >= model.channel_count()) throw ValidationError("eval_model_channel: channel out of range");
    const int J = static_cast<int>(samples.size()), M = model.order();
    std::vector<Complex> s(J), v(J);
    for (int j = 0; j < J; ++j) {
        s[j] = samples[j].s;
        v[j] = samples[j].values.at(channel);
    }
    double e = 0.0;
    b200::check(fds_fit_error_evf(M, b200::c(model.poles.data()), 1, b200::c(model.residues[channel].data()), 0, J,
                                  b200::c(s.data()), b200::c(v.data()), &e));
    return e;
}

}  // namespace fdsweep
