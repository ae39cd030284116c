// ORACLE — test infrastructure only. extern "C" surface over the CPU oracle so
// that pytest (ctypes) can drive it as the checker for the B200 product path.
//
// Linked into oracle/_ref/libfdsweep_oracle.so together with:
//   * the CPU restatement oracle/vecfit_oracle.cpp, oracle/laplace_oracle.cpp,
//   * the reference's own, unmodified proj/src/afs.cpp, systems.cpp, io.cpp,
//     compiled straight from /root/reference (see oracle/Makefile),
//   * the new BEM oracle oracle/bem_oracle.cpp.
// Status codes follow the reference's error classes (proj/include/fdsweep/types.hpp:14-36):
// 0 ok, 1 ValidationError, 2 NumericError, 3 IoError, 4 ConvergenceError, 9 other.
#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "bem_oracle.hpp"
#include "linalg.hpp"
#include "fdsweep/afs.hpp"
#include "fdsweep/io.hpp"
#include "fdsweep/laplace.hpp"
#include "fdsweep/systems.hpp"
#include "fdsweep/vecfit.hpp"

using fdsweep::Complex;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const fdsweep::ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const fdsweep::NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const fdsweep::IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const fdsweep::ConvergenceError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

std::vector<Complex> cvec(const double* p, int n) {
    std::vector<Complex> v(n);
    for (int i = 0; i < n; ++i) v[i] = Complex(p[2 * i], p[2 * i + 1]);
    return v;
}
void cput(const std::vector<Complex>& v, double* p) {
    for (size_t i = 0; i < v.size(); ++i) { p[2 * i] = v[i].real(); p[2 * i + 1] = v[i].imag(); }
}

// samples laid out [j][k] interleaved complex (the reference's per-frequency AoS)
std::vector<fdsweep::FrequencySample> samples_of(int J, int K, const double* s, const double* v) {
    std::vector<fdsweep::FrequencySample> out(J);
    for (int j = 0; j < J; ++j) {
        out[j].s = Complex(s[2 * j], s[2 * j + 1]);
        out[j].values = cvec(v + 2 * static_cast<size_t>(j) * K, K);
    }
    return out;
}

fdsweep::RationalModel model_of(int M, const double* poles, int K, const double* res) {
    fdsweep::RationalModel m;
    m.poles = cvec(poles, M);
    for (int k = 0; k < K; ++k) {
        m.residues.push_back(cvec(res + 2 * static_cast<size_t>(k) * M, M));
        m.channel_labels.push_back("ch" + std::to_string(k));
    }
    return m;
}

// A FrequencySystem backed by the BEM oracle: output = displacement at the
// requested DOFs (element-major [e][x,y,z]).
class OracleBemSystem : public fdsweep::FrequencySystem {
  public:
    OracleBemSystem(std::shared_ptr<oracle::BemOracle> bem, std::vector<int> dofs)
        : bem_(std::move(bem)), dofs_(std::move(dofs)) {
        desc_.channel_count = static_cast<int>(dofs_.size());
        for (int d : dofs_) desc_.channel_labels.push_back("u" + std::to_string(d));
    }
    const fdsweep::SystemDescriptor& descriptor() const override { return desc_; }
    std::vector<Complex> evaluate(Complex s) const override {
        const std::vector<Complex> u = bem_->solve(s);
        std::vector<Complex> out(dofs_.size());
        for (size_t i = 0; i < dofs_.size(); ++i) out[i] = u[dofs_[i]];
        return out;
    }

  private:
    std::shared_ptr<oracle::BemOracle> bem_;
    std::vector<int> dofs_;
    fdsweep::SystemDescriptor desc_;
};

// A FrequencySystem whose evaluate() calls back into the test harness, so the
// reference's own run_afs (afs.cpp, compiled unmodified) can be driven by
// responses produced elsewhere (the GPU product's solves) at sizes where the
// oracle BEM is too slow. evaluate() is serialised: the callback may hold a GIL.
using orc_eval_cb = int (*)(void* ctx, double sr, double si, double* out);
class OracleCallbackSystem : public fdsweep::FrequencySystem {
  public:
    OracleCallbackSystem(int channels, orc_eval_cb cb, void* ctx) : cb_(cb), ctx_(ctx) {
        desc_.channel_count = channels;
        for (int k = 0; k < channels; ++k) desc_.channel_labels.push_back("c" + std::to_string(k));
    }
    const fdsweep::SystemDescriptor& descriptor() const override { return desc_; }
    std::vector<Complex> evaluate(Complex s) const override {
        std::vector<Complex> out(static_cast<size_t>(desc_.channel_count));
        std::lock_guard<std::mutex> lk(mu_);
        if (cb_(ctx_, s.real(), s.imag(), reinterpret_cast<double*>(out.data())) != 0)
            throw fdsweep::NumericError("callback system: evaluate failed");
        return out;
    }

  private:
    orc_eval_cb cb_;
    void* ctx_;
    mutable std::mutex mu_;
    fdsweep::SystemDescriptor desc_;
};

struct OracleSystem {
    std::unique_ptr<fdsweep::FrequencySystem> sys;
};

// OpenBLAS (scipy's bundled build, 32-bit ints) for the CPU-baseline LU.
using zgetrf_t = void (*)(const int*, const int*, double*, const int*, int*, int*);
using zgetrs_t = void (*)(const char*, const int*, const int*, const double*, const int*,
                          const int*, double*, const int*, int*, long);
zgetrf_t g_zgetrf = nullptr;
zgetrs_t g_zgetrs = nullptr;

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- vecfit
int orc_initial_poles(double omega_max, int order, double* out) {
    return guarded([&] { cput(fdsweep::initial_poles(omega_max, order), out); });
}

int orc_is_conjugate_closed(int M, const double* poles, double tol, int* out) {
    return guarded([&] { *out = fdsweep::is_conjugate_closed(cvec(poles, M), tol) ? 1 : 0; });
}

int orc_canonical_poles(int M, const double* poles, double* out) {
    return guarded([&] { cput(fdsweep::canonical_poles(cvec(poles, M)), out); });
}

int orc_relocate_poles(int J, int K, const double* s, const double* vals, int M,
                       const double* poles_in, double* poles_out, double* rms_out,
                       double* movement) {
    return guarded([&] {
        fdsweep::RelocationStats st;
        const auto smp = samples_of(J, K, s, vals);
        const auto p = fdsweep::relocate_poles(smp, cvec(poles_in, M), &st);
        cput(p, poles_out);
        if (rms_out) for (int k = 0; k < K; ++k) rms_out[k] = st.per_channel_rms[k];
        if (movement) *movement = st.pole_movement;
    });
}

// ---- linear-algebra test hooks (tests/test_oracle_crosscheck.py) ----
// Dimensions of the last relocation's stacked sigma system; has_h = 1 when the
// companion matrix was formed (the rank test passed).
int orc_last_relocation_dims(int* rows, int* cols, int* has_h) {
    return guarded([&] {
        const auto& c = oracle::reloc_capture();
        *rows = c.stacked.rows;
        *cols = c.stacked.cols;
        *has_h = c.has_h ? 1 : 0;
    });
}
int orc_last_relocation(double* stacked, double* rhs, double* h) {
    return guarded([&] {
        const auto& c = oracle::reloc_capture();
        std::copy(c.stacked.a.begin(), c.stacked.a.end(), stacked);
        std::copy(c.rhs.begin(), c.rhs.end(), rhs);
        if (c.has_h && h) std::copy(c.h.a.begin(), c.h.a.end(), h);
    });
}
// The oracle's ColPivHouseholderQR on a column-major m x n matrix: |R_ii| in
// factor order, the column permutation, Eigen's rank, nonzero pivots, max
// pivot, and the basic least-squares solution for rhs b.
int orc_colpivqr(int m, int n, const double* a, const double* b, double* rdiag, int* perm, int* rank,
                 int* nonzero_pivots, double* maxpivot, double* x) {
    return guarded([&] {
        oracle::Mat A(m, n);
        std::copy(a, a + static_cast<size_t>(m) * n, A.a.begin());
        const oracle::ColPivQR qr(std::move(A));
        const int size = std::min(m, n);
        for (int i = 0; i < size; ++i) rdiag[i] = std::abs(qr.qr(i, i));
        for (int j = 0; j < n; ++j) perm[j] = qr.perm[j];
        *rank = qr.rank();
        *nonzero_pivots = qr.nonzero_pivots;
        *maxpivot = qr.maxpivot;
        if (x) {
            const auto y = qr.solve(std::vector<double>(b, b + m));
            std::copy(y.begin(), y.end(), x);
        }
    });
}
// The oracle's EigenSolver restatement (Hessenberg + Francis double shift).
int orc_real_eigenvalues(int n, const double* h, double* ev) {
    return guarded([&] {
        oracle::Mat H(n, n);
        std::copy(h, h + static_cast<size_t>(n) * n, H.a.begin());
        std::vector<Complex> e;
        if (!oracle::real_eigenvalues(std::move(H), e)) throw fdsweep::NumericError("eigenvalue iteration failed");
        cput(e, ev);
    });
}

int orc_identify_residues(int J, const double* s, const double* vals, int M,
                          const double* poles, double* res_out, double* rms) {
    return guarded([&] {
        const auto r = fdsweep::identify_residues(cvec(s, J), cvec(vals, J), cvec(poles, M), rms);
        cput(r, res_out);
    });
}

// CPU baseline of identify_residues over K channels (vecfit.cpp:356-408, one
// call per channel as the reference's final fit does, afs.cpp:386-393) on
// `threads` OpenMP threads. vals [j][k]; residues out [k][m].
int orc_identify_residues_many(int J, int K, const double* s, const double* vals, int M, const double* poles,
                               int threads, double* res_out) {
    return guarded([&] {
        const std::vector<Complex> sv = cvec(s, J), pv = cvec(poles, M);
        std::string err;
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int k = 0; k < K; ++k) {
            std::vector<Complex> v(J);
            for (int j = 0; j < J; ++j)
                v[j] = Complex(vals[2 * (static_cast<size_t>(j) * K + k)], vals[2 * (static_cast<size_t>(j) * K + k) + 1]);
            try {
                const auto r = fdsweep::identify_residues(sv, v, pv, nullptr);
                cput(r, res_out + 2 * static_cast<size_t>(k) * M);
            } catch (const std::exception& e) {
#pragma omp critical
                err = e.what();
            }
        }
        if (!err.empty()) throw fdsweep::NumericError(err);
    });
}

int orc_vector_fit(int J, int K, const double* s, const double* vals, int n_orf, const int* orf,
                   int order, int n_reloc, double* poles_out, double* res_out, int* iters,
                   double* movement, int* unstable, double* rms_out, double* reloc_rms_out) {
    return guarded([&] {
        const auto smp = samples_of(J, K, s, vals);
        const std::vector<int> o(orf, orf + n_orf);
        auto [model, rep] = fdsweep::vector_fit(smp, o, order, n_reloc);
        cput(model.poles, poles_out);
        for (int k = 0; k < K; ++k) cput(model.residues[k], res_out + 2 * static_cast<size_t>(k) * order);
        if (iters) *iters = rep.iterations_used;
        if (movement) *movement = rep.pole_movement;
        if (unstable) *unstable = rep.unstable_pole_count;
        if (rms_out) for (int k = 0; k < K; ++k) rms_out[k] = rep.per_channel_rms[k];
        if (reloc_rms_out)
            for (size_t k = 0; k < rep.relocation_rms.size(); ++k) reloc_rms_out[k] = rep.relocation_rms[k];
    });
}

int orc_eval_model(int M, const double* poles, int K, const double* res, double sr, double si,
                   double* out) {
    return guarded([&] { cput(fdsweep::eval_model(model_of(M, poles, K, res), Complex(sr, si)), out); });
}

int orc_fit_error_evf(int M, const double* poles, int K, const double* res, int ch, int J,
                      const double* s, const double* vals, double* out) {
    return guarded([&] {
        *out = fdsweep::fit_error_evf(model_of(M, poles, K, res), ch, samples_of(J, K, s, vals));
    });
}

// ---------------------------------------------------------------- laplace
int orc_damping_eta(double kappa, double T, double* out) {
    return guarded([&] { *out = fdsweep::damping_eta(kappa, T); });
}
int orc_hanning_window(int k, int ns, double* out) {
    return guarded([&] { *out = fdsweep::hanning_window(k, ns); });
}
int orc_conjugate_fill(int nh, const double* half, double* out) {
    return guarded([&] { cput(fdsweep::conjugate_fill(cvec(half, nh)), out); });
}
int orc_fsm_grid(double T, int ns, double* dw, double* dt, double* wmax, int* nc) {
    return guarded([&] {
        fdsweep::FsmGrid g(T, ns);
        *dw = g.delta_omega();
        *dt = g.delta_t();
        *wmax = g.omega_max();
        *nc = g.contour_count();
    });
}

// half: [k][Nc] interleaved complex; out: [k][Ns]
int orc_fsm_invert(double T, int ns, double eta, int K, const double* half, int hanning,
                   double* out) {
    return guarded([&] {
        fdsweep::FsmGrid g(T, ns);
        const int nc = ns / 2 + 1;
        std::vector<std::vector<Complex>> hs(K);
        std::vector<std::string> labels(K);
        for (int k = 0; k < K; ++k) hs[k] = cvec(half + 2 * static_cast<size_t>(k) * nc, nc);
        const auto ts = fdsweep::fsm_invert(g, eta, hs, labels, hanning != 0);
        for (int k = 0; k < K; ++k) std::memcpy(out + static_cast<size_t>(k) * ns, ts.values[k].data(), sizeof(double) * ns);
    });
}

int orc_rational_invert(int M, const double* poles, int K, const double* res, int nt,
                        const double* t, double* out) {
    return guarded([&] {
        const auto ts = fdsweep::rational_invert(model_of(M, poles, K, res), std::vector<double>(t, t + nt));
        for (int k = 0; k < K; ++k) std::memcpy(out + static_cast<size_t>(k) * nt, ts.values[k].data(), sizeof(double) * nt);
    });
}

// ---------------------------------------------------------------- afs (reference afs.cpp)
int orc_initial_frequencies(int j0, double eta, double wmax, double* out) {
    return guarded([&] { cput(fdsweep::initial_frequencies(j0, eta, wmax), out); });
}
int orc_fit_orders(int J, double ah, double al, int* mh, int* ml) {
    return guarded([&] {
        const auto [h, l] = fdsweep::fit_orders(J, ah, al);
        *mh = h;
        *ml = l;
    });
}
int orc_channel_errors(int MH, const double* ph, int ML, const double* pl, int K,
                       const double* rh, const double* rl, int G, const double* grid, double* out) {
    return guarded([&] {
        const auto e = fdsweep::channel_errors(model_of(MH, ph, K, rh), model_of(ML, pl, K, rl), cvec(grid, G));
        std::memcpy(out, e.data(), sizeof(double) * K);
    });
}
int orc_select_new_frequency(int MH, const double* ph, int ML, const double* pl, int K,
                             const double* rh, const double* rl, int G, const double* grid,
                             int ne, const double* existing, int no, const int* orf_pos,
                             double radius, double* out) {
    return guarded([&] {
        const Complex c = fdsweep::select_new_frequency(
            model_of(MH, ph, K, rh), model_of(ML, pl, K, rl), cvec(grid, G), cvec(existing, ne),
            std::vector<int>(orf_pos, orf_pos + no), radius);
        out[0] = c.real();
        out[1] = c.imag();
    });
}
int orc_error_e1(int K, int nt, const double* t, const double* cur, const double* prev, double* out) {
    return guarded([&] {
        fdsweep::TimeSeries a, b;
        a.t.assign(t, t + nt);
        b.t = a.t;
        for (int k = 0; k < K; ++k) {
            a.values.emplace_back(cur + static_cast<size_t>(k) * nt, cur + static_cast<size_t>(k + 1) * nt);
            b.values.emplace_back(prev + static_cast<size_t>(k) * nt, prev + static_cast<size_t>(k + 1) * nt);
        }
        *out = fdsweep::error_e1(a, b);
    });
}

// ---------------------------------------------------------------- systems
int orc_system_from_json(const char* json, void** out) {
    return guarded([&] {
        auto h = new OracleSystem;
        h->sys = fdsweep::make_system_from_json(json);
        *out = h;
    });
}
int orc_system_bem(void* bem, int n_dofs, const int* dofs, void** out) {
    return guarded([&] {
        auto h = new OracleSystem;
        auto sp = std::shared_ptr<oracle::BemOracle>(static_cast<oracle::BemOracle*>(bem), [](oracle::BemOracle*) {});
        h->sys = std::make_unique<OracleBemSystem>(sp, std::vector<int>(dofs, dofs + n_dofs));
        *out = h;
    });
}
int orc_system_callback(int channels, orc_eval_cb cb, void* ctx, void** out) {
    return guarded([&] {
        auto h = new OracleSystem;
        h->sys = std::make_unique<OracleCallbackSystem>(channels, cb, ctx);
        *out = h;
    });
}
void orc_system_destroy(void* h) { delete static_cast<OracleSystem*>(h); }
int orc_system_channels(void* h) { return static_cast<OracleSystem*>(h)->sys->descriptor().channel_count; }
int orc_system_evaluate(void* h, double sr, double si, double* out) {
    return guarded([&] { cput(static_cast<OracleSystem*>(h)->sys->evaluate(Complex(sr, si)), out); });
}

// cfg_d: [alpha_high, alpha_low, e1_thr, e2_thr, omega_max, eta, period]
// cfg_i: [initial_count, validation_steps, grid_points, time_points, max_iterations, seed, n_reloc]
// outputs: samples_s (2*cap), n_c, converged, solver_calls, history (cap rows x 7:
//   J, MH, ML, has_snew, snew_re, snew_im, e1, e2 -> 8 doubles), n_hist,
//   final poles (2*cap) + order, orf/test indices used.
int orc_run_afs(void* h, const double* cfg_d, const int* cfg_i, int n_orf, const int* orf,
                int n_test, const int* test, int cap, double* samples_s, int* n_c, int* converged,
                int* solver_calls, double* hist, int* n_hist, double* poles_out, int* order_out,
                int* orf_used, int* n_orf_used, double* res_out) {
    return guarded([&] {
        fdsweep::AfsConfig cfg;
        cfg.alpha_high = cfg_d[0];
        cfg.alpha_low = cfg_d[1];
        cfg.e1_threshold = cfg_d[2];
        cfg.e2_threshold = cfg_d[3];
        cfg.omega_max = cfg_d[4];
        cfg.eta = cfg_d[5];
        cfg.period = cfg_d[6];
        cfg.initial_count = cfg_i[0];
        cfg.validation_steps = cfg_i[1];
        cfg.grid_points = cfg_i[2];
        cfg.time_points = cfg_i[3];
        cfg.max_iterations = cfg_i[4];
        cfg.seed = static_cast<std::uint64_t>(cfg_i[5]);
        cfg.n_relocations = cfg_i[6];
        cfg.orf_indices.assign(orf, orf + n_orf);
        cfg.test_indices.assign(test, test + n_test);
        // on_sample (afs.cpp:296) records every solved frequency as it happens, so
        // the samples taken before a reference exception stay visible to the caller
        *n_c = 0;
        *solver_calls = 0;
        *n_hist = 0;
        auto on_sample = [&](const fdsweep::FrequencySample& smp) {
            if (*n_c < cap) {
                samples_s[2 * *n_c] = smp.s.real();
                samples_s[2 * *n_c + 1] = smp.s.imag();
            }
            ++*n_c;
            ++*solver_calls;
        };
        const auto r = fdsweep::run_afs(*static_cast<OracleSystem*>(h)->sys, cfg, {}, on_sample);
        const int nc = static_cast<int>(r.samples.size());
        if (nc > cap || static_cast<int>(r.history.size()) > cap || r.model_high.order() > cap)
            throw fdsweep::ValidationError("orc_run_afs: output capacity too small");
        for (int i = 0; i < nc; ++i) { samples_s[2 * i] = r.samples[i].s.real(); samples_s[2 * i + 1] = r.samples[i].s.imag(); }
        *n_c = r.n_c;
        *converged = r.converged ? 1 : 0;
        *solver_calls = r.solver_calls;
        *n_hist = static_cast<int>(r.history.size());
        for (size_t i = 0; i < r.history.size(); ++i) {
            const auto& it = r.history[i];
            double* row = hist + 8 * i;
            row[0] = it.sample_count;
            row[1] = it.order_high;
            row[2] = it.order_low;
            row[3] = it.s_new ? 1.0 : 0.0;
            row[4] = it.s_new ? it.s_new->real() : 0.0;
            row[5] = it.s_new ? it.s_new->imag() : 0.0;
            row[6] = it.e1;
            row[7] = it.e2;
        }
        *order_out = r.model_high.order();
        cput(r.model_high.poles, poles_out);
        *n_orf_used = static_cast<int>(r.orf_indices.size());
        for (size_t i = 0; i < r.orf_indices.size(); ++i) orf_used[i] = r.orf_indices[i];
        if (res_out) {
            const int M = r.model_high.order();
            for (size_t k = 0; k < r.model_high.residues.size(); ++k)
                cput(r.model_high.residues[k], res_out + 2 * k * M);
        }
    });
}

// ---------------------------------------------------------------- BEM oracle
int orc_bem_create(int nv, const double* verts, int ne, const int* tris, double mu, double nu,
                   double rho, const double* traction, void** out) {
    return guarded([&] {
        *out = new oracle::BemOracle(std::vector<double>(verts, verts + 3 * nv),
                                     std::vector<int>(tris, tris + 3 * ne), mu, nu, rho,
                                     std::vector<double>(traction, traction + 3 * ne));
    });
}
void orc_bem_destroy(void* h) { delete static_cast<oracle::BemOracle*>(h); }

int orc_bem_assemble(void* h, double sr, double si, double* A_out, double* b_out) {
    return guarded([&] {
        std::vector<Complex> A, b;
        static_cast<oracle::BemOracle*>(h)->assemble(Complex(sr, si), A, b);
        cput(A, A_out);
        cput(b, b_out);
    });
}
int orc_bem_entries(void* h, double sr, double si, int count, const int* rows, const int* cols, double* out) {
    return guarded([&] {
        auto* bem = static_cast<oracle::BemOracle*>(h);
        std::vector<Complex> v(count);
#pragma omp parallel for schedule(dynamic, 16)
        for (int i = 0; i < count; ++i) v[i] = bem->entry(rows[i], cols[i], Complex(sr, si));
        cput(v, out);
    });
}
int orc_bem_rhs_rows(void* h, double sr, double si, int count, const int* rows, double* out) {
    return guarded([&] {
        auto* bem = static_cast<oracle::BemOracle*>(h);
        std::vector<Complex> v(count);
#pragma omp parallel for schedule(dynamic, 1)
        for (int i = 0; i < count; ++i) v[i] = bem->rhs(rows[i], Complex(sr, si));
        cput(v, out);
    });
}
int orc_bem_solve(void* h, double sr, double si, double* u_out) {
    return guarded([&] { cput(static_cast<oracle::BemOracle*>(h)->solve(Complex(sr, si)), u_out); });
}
int orc_bem_self_block(void* h, int e, double sr, double si, double* U, double* T) {
    return guarded([&] {
        Complex u[9], t[9];
        static_cast<oracle::BemOracle*>(h)->self_block(e, Complex(sr, si), u, t);
        for (int i = 0; i < 9; ++i) { U[2 * i] = u[i].real(); U[2 * i + 1] = u[i].imag(); T[2 * i] = t[i].real(); T[2 * i + 1] = t[i].imag(); }
    });
}
int orc_kernel_ut(double mu, double nu, double rho, const double* rv, const double* n, double sr,
                  double si, double* U, double* T) {
    return guarded([&] {
        oracle::KernelCoeffs kc(mu, nu, rho);
        Complex u[9], t[9];
        kc.ut(rv, n, Complex(sr, si), u, t);
        for (int i = 0; i < 9; ++i) { U[2 * i] = u[i].real(); U[2 * i + 1] = u[i].imag(); T[2 * i] = t[i].real(); T[2 * i + 1] = t[i].imag(); }
    });
}
int orc_kernel_abcd(double mu, double nu, double rho, double zr, double zi, double* out) {
    return guarded([&] {
        oracle::KernelCoeffs kc(mu, nu, rho);
        Complex a, b, c, d;
        kc.abcd(Complex(zr, zi), a, b, c, d);
        cput({a, b, c, d}, out);
    });
}
int orc_lu_solve(int n, const double* A, const double* b, double* x) {
    return guarded([&] {
        std::vector<Complex> a = cvec(A, n * n), bb = cvec(b, n);
        std::vector<int> piv;
        if (oracle::lu_factor(n, a, piv) != 0) throw fdsweep::NumericError("singular matrix");
        oracle::lu_solve(n, a, piv, bb);
        cput(bb, x);
    });
}

// CPU-baseline solve: oracle assembly (OpenMP) + OpenBLAS zgetrf/zgetrs.
// Returns assembly / factor+solve seconds through t_out[2].
int orc_bem_solve_openblas(void* h, const char* openblas_path, double sr, double si,
                           double* u_out, double* t_out) {
    return guarded([&] {
        if (!g_zgetrf) {
            void* lib = dlopen(openblas_path, RTLD_NOW | RTLD_LOCAL);
            if (!lib) throw std::runtime_error(std::string("dlopen openblas: ") + dlerror());
            g_zgetrf = reinterpret_cast<zgetrf_t>(dlsym(lib, "scipy_zgetrf_"));
            g_zgetrs = reinterpret_cast<zgetrs_t>(dlsym(lib, "scipy_zgetrs_"));
            if (!g_zgetrf || !g_zgetrs) throw std::runtime_error("openblas: zgetrf/zgetrs not found");
        }
        auto* bem = static_cast<oracle::BemOracle*>(h);
        const int n = 3 * bem->elements();
        std::vector<Complex> A, b;
        const auto t0 = std::chrono::steady_clock::now();
        bem->assemble(Complex(sr, si), A, b);
        const auto t1 = std::chrono::steady_clock::now();
        std::vector<int> piv(n);
        int info = 0, one = 1;
        g_zgetrf(&n, &n, reinterpret_cast<double*>(A.data()), &n, piv.data(), &info);
        if (info != 0) throw fdsweep::NumericError("zgetrf failed");
        const char tr = 'N';
        g_zgetrs(&tr, &n, &one, reinterpret_cast<double*>(A.data()), &n, piv.data(),
                 reinterpret_cast<double*>(b.data()), &n, &info, 1);
        const auto t2 = std::chrono::steady_clock::now();
        cput(b, u_out);
        if (t_out) {
            t_out[0] = std::chrono::duration<double>(t1 - t0).count();
            t_out[1] = std::chrono::duration<double>(t2 - t1).count();
        }
    });
}

}  // extern "C"
