// AFS driver interface (host) — see afs.cpp.
#pragma once

#include <functional>
#include <vector>

#include "vf.cuh"

namespace fdsb {

struct AfsCfg {
    int initial_count = 16;
    double alpha_high = 2.0, alpha_low = 2.3;
    double e1_threshold = 1e-4, e2_threshold = 2e-3;
    int validation_steps = 3;
    std::vector<int> orf, test;
    double omega_max = 0.0, eta = 0.0, period = 0.0;
    int grid_points = 4096, time_points = 512, max_iterations = 500;
    uint64_t seed = 0;
    int n_relocations = 3;
};

struct AfsIter {
    int J, MH, ML;
    bool has_s_new;
    Cx s_new;
    double e1, e2;
};

struct AfsOut {
    std::vector<Cx> samples;   // in sampling order
    std::vector<Cx> values;    // [j][channels]
    std::vector<AfsIter> history;
    bool converged = false;
    int solver_calls = 0;
    std::vector<int> orf, test;
    std::vector<Cx> poles, residues;  // final model, residues [k][m]
};

// Evaluates a batch of frequencies: out[b*channels + k].
using BatchEval = std::function<void(const std::vector<Cx>&, std::vector<Cx>&)>;

// Fills r as it goes: when the reference algorithm throws, r keeps the
// samples and history of the iterations completed before the failure.
void run_afs_impl(const BatchEval& eval, int channels, const AfsCfg& cfg, AfsOut& r);
std::vector<int> draw_channels(int n, int k, uint64_t seed);
std::vector<Cx> afs_initial_frequencies(int j0, double eta, double omega_max);
std::pair<int, int> afs_fit_orders(int J, double ah, double al);
double afs_error_e1(const std::vector<double>& t, const std::vector<double>& cur, const std::vector<double>& prev, int K);

}  // namespace fdsb
