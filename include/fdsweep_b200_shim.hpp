// Drop-in C++ shim for the reference toolkit (fdsweep, arXiv:1511.04355).
//
// Header-only; compiled INSIDE the reference's build against its own headers
// (proj/include/fdsweep/*.hpp) and linked with libfdsweep_b200.so. It provides
//   * fdsweep::b200::BemSystem — a FrequencySystem (systems.hpp:34-42) whose
//     evaluate(s) is one GPU BEM solve (fds_bem_evaluate), plus evaluate_batch;
//   * fdsweep::b200::{vector_fit, identify_residues, relocate_poles,
//     fsm_invert, rational_invert, channel_errors} with the reference
//     signatures (vecfit.hpp:48-86, laplace.hpp:40-59, afs.hpp:66-79) routed to
//     the C-ABI, rethrowing FDS_E* statuses as the reference's exception classes
//     (types.hpp:14-36).
// The reference's run_afs (afs.cpp:226) drives a BemSystem unchanged; a
// maintainer who also wants the GPU fits inside run_afs swaps vecfit.cpp /
// laplace.cpp for thin forwarding files that call these functions
// (INTEGRATION.md §2).
#pragma once

#include <memory>
#include <span>
#include <string>
#include <vector>

#include "fdsweep/afs.hpp"
#include "fdsweep/laplace.hpp"
#include "fdsweep/systems.hpp"
#include "fdsweep/types.hpp"
#include "fdsweep/vecfit.hpp"
#include "fdsweep_b200.h"

namespace fdsweep::b200 {

inline void check(int rc) {
    if (rc == FDS_OK) return;
    const std::string msg = fds_last_error();
    switch (rc) {
        case FDS_EVALIDATION: throw ValidationError(msg);
        case FDS_ENUMERIC: throw NumericError(msg);
        case FDS_EIO: throw IoError(msg);
        case FDS_ECONVERGENCE: throw ConvergenceError(msg);
        default: throw Error("fdsweep_b200 device failure: " + msg);
    }
}

inline const fds_c64* c(const Complex* p) { return reinterpret_cast<const fds_c64*>(p); }
inline fds_c64* c(Complex* p) { return reinterpret_cast<fds_c64*>(p); }

struct BemMesh {
    std::vector<double> vertices;  // [nv][3]
    std::vector<int> triangles;    // [ne][3], (v1-v0)x(v2-v0) = domain-outward normal
    double shear_modulus = 1.0, poisson_ratio = 0.25, density = 1.0;
    std::vector<double> traction;  // [ne][3], times the Heaviside factor 1/s
    std::vector<int> channels;     // output DOFs (element-major u[3e+i]); empty => all
};

class BemSystem : public FrequencySystem {
  public:
    explicit BemSystem(const BemMesh& m) {
        fds_bem_desc d{};
        d.n_vertices = static_cast<int>(m.vertices.size() / 3);
        d.vertices = m.vertices.data();
        d.n_elements = static_cast<int>(m.triangles.size() / 3);
        d.triangles = m.triangles.data();
        d.shear_modulus = m.shear_modulus;
        d.poisson_ratio = m.poisson_ratio;
        d.density = m.density;
        d.traction = m.traction.data();
        d.n_channels = static_cast<int>(m.channels.size());
        d.channels = m.channels.empty() ? nullptr : m.channels.data();
        fds_bem* h = nullptr;
        check(fds_bem_create(&d, &h));
        h_.reset(h);
        desc_.channel_count = fds_bem_channels(h);
        for (int k = 0; k < desc_.channel_count; ++k)
            desc_.channel_labels.push_back("u" + std::to_string(m.channels.empty() ? k : m.channels[k]));
    }
    const SystemDescriptor& descriptor() const override { return desc_; }
    std::vector<Complex> evaluate(Complex s) const override {
        std::vector<Complex> out(desc_.channel_count);
        check(fds_bem_evaluate(h_.get(), fds_c64{s.real(), s.imag()}, c(out.data())));
        return out;
    }
    fds_bem* handle() const { return h_.get(); }
    // Solver of later evaluations: LU (default) or GMRES (fds_bem_set_solver).
    void set_solver(bool gmres, double tol = 1e-12, int restart = 60, int max_iter = 1000) {
        check(fds_bem_set_solver(h_.get(), gmres ? 1 : 0, tol, restart, max_iter));
    }
    // B independent solves in one batched assembly + LU (e.g. the FSM contour).
    std::vector<std::vector<Complex>> evaluate_batch(std::span<const Complex> s) const {
        std::vector<Complex> flat(s.size() * desc_.channel_count);
        check(fds_bem_evaluate_batch(h_.get(), c(s.data()), static_cast<int>(s.size()), c(flat.data())));
        std::vector<std::vector<Complex>> out(s.size());
        for (size_t b = 0; b < s.size(); ++b)
            out[b].assign(flat.begin() + b * desc_.channel_count, flat.begin() + (b + 1) * desc_.channel_count);
        return out;
    }

  private:
    struct Del {
        void operator()(fds_bem* p) const { fds_bem_destroy(p); }
    };
    std::unique_ptr<fds_bem, Del> h_;
    SystemDescriptor desc_;
};

// run_afs (afs.cpp:226-396) of a BemSystem on the library's own driver: the J0
// initial frequencies are one batched solve and the fits stay on the device.
// Same AfsResult as the reference driver (identical sampled frequencies; see
// tests/test_gpu_vf.py and tests/test_cli.py).
inline AfsResult run_afs_bem(const BemSystem& sys, const AfsConfig& cfg) {
    const int K = sys.descriptor().channel_count;
    fds_afs_config a{};
    a.initial_count = cfg.initial_count;
    a.alpha_high = cfg.alpha_high;
    a.alpha_low = cfg.alpha_low;
    a.e1_threshold = cfg.e1_threshold;
    a.e2_threshold = cfg.e2_threshold;
    a.validation_steps = cfg.validation_steps;
    a.n_orf = static_cast<int>(cfg.orf_indices.size());
    a.orf_indices = cfg.orf_indices.data();
    a.n_test = static_cast<int>(cfg.test_indices.size());
    a.test_indices = cfg.test_indices.data();
    a.omega_max = cfg.omega_max;
    a.eta = cfg.eta;
    a.period = cfg.period;
    a.grid_points = cfg.grid_points;
    a.time_points = cfg.time_points;
    a.max_iterations = cfg.max_iterations;
    a.seed = cfg.seed;
    a.n_relocations = cfg.n_relocations;
    const int cap = cfg.initial_count + cfg.max_iterations + cfg.validation_steps + 16;
    std::vector<Complex> s(cap), vals(static_cast<size_t>(cap) * K), poles(cap), res(static_cast<size_t>(cap) * K);
    std::vector<double> hist(static_cast<size_t>(cap) * 8);
    fds_afs_summary sm{};
    check(fds_run_afs_bem(sys.handle(), &a, cap, c(s.data()), c(vals.data()), hist.data(), c(poles.data()),
                          c(res.data()), &sm));
    AfsResult r;
    r.n_c = sm.n_c;
    r.converged = sm.converged != 0;
    r.solver_calls = sm.solver_calls;
    r.seed = cfg.seed;
    for (int j = 0; j < sm.n_c; ++j)
        r.samples.push_back(FrequencySample{s[j], std::vector<Complex>(vals.begin() + static_cast<size_t>(j) * K,
                                                                       vals.begin() + static_cast<size_t>(j + 1) * K)});
    const int M = sm.order;
    r.model_high.poles.assign(poles.begin(), poles.begin() + M);
    for (int k = 0; k < K; ++k)
        r.model_high.residues.emplace_back(res.begin() + static_cast<size_t>(k) * M,
                                           res.begin() + static_cast<size_t>(k + 1) * M);
    r.model_high.channel_labels = sys.descriptor().channel_labels;
    for (int i = 0; i < sm.n_history; ++i) {
        const double* h = &hist[8 * static_cast<size_t>(i)];
        AfsIteration it;
        it.sample_count = static_cast<int>(h[0]);
        it.order_high = static_cast<int>(h[1]);
        it.order_low = static_cast<int>(h[2]);
        if (h[3] != 0.0) it.s_new = Complex(h[4], h[5]);
        it.e1 = h[6];
        it.e2 = h[7];
        r.history.push_back(it);
    }
    r.orf_indices = cfg.orf_indices;
    if (r.orf_indices.empty())  // drawn by the driver (afs.cpp:234-236)
        r.orf_indices.assign(sm.orf_indices, sm.orf_indices + std::min(sm.n_orf, 8));
    if (cfg.test_indices.empty())
        for (int k = 0; k < K; ++k) r.test_indices.push_back(k);
    else
        r.test_indices = cfg.test_indices;
    return r;
}

inline std::vector<Complex> relocate_poles(std::span<const FrequencySample> samples,
                                           std::span<const Complex> poles, RelocationStats* stats = nullptr) {
    const int J = static_cast<int>(samples.size());
    const int K = J ? static_cast<int>(samples[0].values.size()) : 0;
    std::vector<Complex> s(J), v(static_cast<size_t>(J) * K), out(poles.size());
    for (int j = 0; j < J; ++j) {
        s[j] = samples[j].s;
        std::copy(samples[j].values.begin(), samples[j].values.end(), v.begin() + static_cast<size_t>(j) * K);
    }
    std::vector<double> rms(K);
    double mv = 0.0;
    check(fds_vf_relocate(J, K, c(s.data()), c(v.data()), static_cast<int>(poles.size()), c(poles.data()),
                          c(out.data()), rms.data(), &mv));
    if (stats) {
        stats->per_channel_rms = rms;
        stats->pole_movement = mv;
    }
    return out;
}

inline std::vector<Complex> identify_residues(std::span<const Complex> freqs, std::span<const Complex> values,
                                              std::span<const Complex> poles, double* residual_rms = nullptr) {
    std::vector<Complex> res(poles.size());
    double rms = 0.0;
    check(fds_vf_identify_residues(static_cast<int>(freqs.size()), 1, c(freqs.data()), c(values.data()),
                                   static_cast<int>(poles.size()), c(poles.data()), c(res.data()), &rms));
    if (residual_rms) *residual_rms = rms;
    return res;
}

inline std::pair<RationalModel, FitReport> vector_fit(std::span<const FrequencySample> samples,
                                                      std::span<const int> orf, int order, int n_relocations = 3,
                                                      std::vector<std::string> labels = {}) {
    const int J = static_cast<int>(samples.size());
    const int K = J ? static_cast<int>(samples[0].values.size()) : 0;
    std::vector<Complex> s(J), v(static_cast<size_t>(J) * K), poles(order), res(static_cast<size_t>(K) * order);
    for (int j = 0; j < J; ++j) {
        s[j] = samples[j].s;
        std::copy(samples[j].values.begin(), samples[j].values.end(), v.begin() + static_cast<size_t>(j) * K);
    }
    int ri[2] = {0, 0};
    double rd[1] = {0.0};
    FitReport rep;
    rep.per_channel_rms.resize(K);
    rep.relocation_rms.resize(orf.size());
    check(fds_vector_fit(J, K, c(s.data()), c(v.data()), static_cast<int>(orf.size()), orf.data(), order,
                         n_relocations, c(poles.data()), c(res.data()), ri, rd, rep.per_channel_rms.data(),
                         rep.relocation_rms.data()));
    rep.iterations_used = ri[0];
    rep.unstable_pole_count = ri[1];
    rep.pole_movement = rd[0];
    RationalModel m;
    m.poles = poles;
    for (int k = 0; k < K; ++k) m.residues.emplace_back(res.begin() + static_cast<size_t>(k) * order,
                                                        res.begin() + static_cast<size_t>(k + 1) * order);
    if (labels.empty())
        for (int k = 0; k < K; ++k) labels.push_back("ch" + std::to_string(k));
    m.channel_labels = std::move(labels);
    return {std::move(m), std::move(rep)};
}

inline TimeSeries fsm_invert(const FsmGrid& grid, double eta, const std::vector<std::vector<Complex>>& half,
                             std::vector<std::string> labels, bool hanning = true) {
    if (labels.size() != half.size()) throw ValidationError("fsm_invert: label count mismatch");
    const int K = static_cast<int>(half.size()), Nc = grid.contour_count(), Ns = grid.sample_count;
    std::vector<Complex> flat(static_cast<size_t>(K) * Nc);
    for (int k = 0; k < K; ++k) {
        if (static_cast<int>(half[k].size()) != Nc) throw ValidationError("fsm_invert: half spectrum length mismatch");
        std::copy(half[k].begin(), half[k].end(), flat.begin() + static_cast<size_t>(k) * Nc);
    }
    std::vector<double> out(static_cast<size_t>(K) * Ns);
    check(fds_fsm_invert(grid.period, Ns, eta, K, c(flat.data()), hanning ? 1 : 0, out.data()));
    TimeSeries ts;
    ts.t = grid.time_grid();
    ts.channel_labels = std::move(labels);
    for (int k = 0; k < K; ++k) ts.values.emplace_back(out.begin() + static_cast<size_t>(k) * Ns,
                                                       out.begin() + static_cast<size_t>(k + 1) * Ns);
    return ts;
}

inline TimeSeries rational_invert(const RationalModel& model, std::span<const double> t) {
    const int K = model.channel_count(), M = model.order(), T = static_cast<int>(t.size());
    std::vector<Complex> res(static_cast<size_t>(K) * M);
    for (int k = 0; k < K; ++k) std::copy(model.residues[k].begin(), model.residues[k].end(), res.begin() + static_cast<size_t>(k) * M);
    std::vector<double> out(static_cast<size_t>(K) * T);
    check(fds_rational_invert(M, c(model.poles.data()), K, c(res.data()), T, t.data(), out.data()));
    TimeSeries ts;
    ts.t.assign(t.begin(), t.end());
    ts.channel_labels = model.channel_labels;
    for (int k = 0; k < K; ++k) ts.values.emplace_back(out.begin() + static_cast<size_t>(k) * T,
                                                       out.begin() + static_cast<size_t>(k + 1) * T);
    return ts;
}

inline std::vector<double> channel_errors(const RationalModel& high, const RationalModel& low,
                                          std::span<const Complex> grid) {
    if (high.channel_count() != low.channel_count()) throw ValidationError("channel_errors: channel count mismatch");
    const int K = high.channel_count(), MH = high.order(), ML = low.order();
    std::vector<Complex> rh(static_cast<size_t>(K) * MH), rl(static_cast<size_t>(K) * ML);
    for (int k = 0; k < K; ++k) {
        std::copy(high.residues[k].begin(), high.residues[k].end(), rh.begin() + static_cast<size_t>(k) * MH);
        std::copy(low.residues[k].begin(), low.residues[k].end(), rl.begin() + static_cast<size_t>(k) * ML);
    }
    std::vector<double> e(K);
    check(fds_channel_errors(MH, c(high.poles.data()), c(rh.data()), ML, c(low.poles.data()), c(rl.data()), K,
                             static_cast<int>(grid.size()), c(grid.data()), e.data()));
    return e;
}

}  // namespace fdsweep::b200
