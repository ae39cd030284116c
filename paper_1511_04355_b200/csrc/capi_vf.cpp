// C-ABI for vector fitting, time reconstruction and the AFS driver
// (include/fdsweep_b200.h). Host buffers in the reference's layouts; all
// channel-parallel work runs in the CUDA kernels of vf.cu / laplace.cu.
#include <cstring>

#include "afs.h"
#include "capi_util.h"
#include "vf.cuh"

using namespace fdsb;

namespace {

std::vector<Cx> cv(const fds_c64* p, int n) {
    std::vector<Cx> v(n);
    for (int i = 0; i < n; ++i) v[i] = Cx(p[i].re, p[i].im);
    return v;
}

void put(const std::vector<Cx>& v, fds_c64* p) {
    for (size_t i = 0; i < v.size(); ++i) p[i] = {v[i].real(), v[i].imag()};
}

const Cx* as_cx(const fds_c64* p) { return reinterpret_cast<const Cx*>(p); }

void need(bool ok, const char* what) {
    if (!ok) throw ValidationError(what);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.0f;
    FDS_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
        FDS_CUDA(cudaEventCreate(&a));
        FDS_CUDA(cudaEventCreate(&b));
    }
    ~EventPair() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

}  // namespace

extern "C" {

int fds_vf_relocate(int J, int K, const fds_c64* s, const fds_c64* values, int M, const fds_c64* poles_in,
                    fds_c64* poles_out, double* rms, double* movement) {
    return fds_guard([&] {
        need(J >= 0 && K >= 0 && M >= 0, "relocate_poles: negative size");
        need(J == 0 || (s && values), "relocate_poles: null input");
        const RelocResult r = vf_relocate(cv(s, J), as_cx(values), K, cv(poles_in, M));
        put(r.poles, poles_out);
        if (rms) std::memcpy(rms, r.rms.data(), sizeof(double) * K);
        if (movement) *movement = r.movement;
    });
}

int fds_vf_identify_residues(int J, int K, const fds_c64* s, const fds_c64* values, int M, const fds_c64* poles,
                             fds_c64* residues, double* rms) {
    return fds_guard([&] {
        need(J >= 0 && K >= 0 && M >= 0, "identify_residues: negative size");
        if (J < 1) throw ValidationError("identify_residues: no samples");
        const std::vector<Cx> canon = canonical_order(cv(poles, M));
        if (K == 0) return;
        auto& cx = VfContext::get();
        cplx* dv = static_cast<cplx*>(cx.values.get(sizeof(cplx) * J * static_cast<size_t>(K)));
        cplx* dr = static_cast<cplx*>(cx.out.get(sizeof(cplx) * M * static_cast<size_t>(K)));
        double* drms = static_cast<double*>(cx.rms.get(sizeof(double) * K));
        FDS_CUDA(cudaMemcpyAsync(dv, values, sizeof(cplx) * J * static_cast<size_t>(K), cudaMemcpyHostToDevice, cx.st));
        vf_residues_device(cv(s, J), dv, K, canon, dr, rms ? drms : nullptr, cx.st);
        std::vector<Cx> rmk(static_cast<size_t>(M) * K);
        FDS_CUDA(cudaMemcpyAsync(rmk.data(), dr, rmk.size() * sizeof(cplx), cudaMemcpyDeviceToHost, cx.st));
        if (rms) FDS_CUDA(cudaMemcpyAsync(rms, drms, K * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
        FDS_CUDA(cudaStreamSynchronize(cx.st));
        for (int k = 0; k < K; ++k)
            for (int m = 0; m < M; ++m) {
                const Cx v = rmk[static_cast<size_t>(m) * K + k];
                residues[static_cast<size_t>(k) * M + m] = {v.real(), v.imag()};
            }
    });
}

int fds_vector_fit(int J, int K, const fds_c64* s, const fds_c64* values, int n_orf, const int* orf, int order,
                   int n_reloc, fds_c64* poles_out, fds_c64* residues_out, int* report_i, double* report_d,
                   double* rms, double* reloc_rms) {
    return fds_guard([&] {
        need(J >= 0 && K >= 0 && n_orf >= 0, "vector_fit: negative size");
        std::vector<Cx> poles, res;
        FitReportC rep;
        vf_vector_fit(cv(s, J), as_cx(values), K, std::vector<int>(orf, orf + n_orf), order, n_reloc, poles, res, &rep);
        put(poles, poles_out);
        put(res, residues_out);
        if (report_i) { report_i[0] = rep.iterations; report_i[1] = rep.unstable; }
        if (report_d) report_d[0] = rep.movement;
        if (rms) std::memcpy(rms, rep.rms.data(), sizeof(double) * K);
        if (reloc_rms) std::memcpy(reloc_rms, rep.reloc_rms.data(), sizeof(double) * rep.reloc_rms.size());
    });
}

int fds_vf_release_workspace(void) {
    return fds_guard([&] { VfContext::get().release(); });
}

int fds_eval_model(int M, const fds_c64* poles, int K, const fds_c64* residues, int G, const fds_c64* s, fds_c64* out) {
    // eval_model (vecfit.cpp:490-509) on the device (vf_eval_kernel)
    return fds_guard([&] {
        need(M >= 0 && K >= 0 && G >= 0, "eval_model: negative size");
        need((M == 0 || poles) && (K * M == 0 || residues) && (G == 0 || (s && out)), "eval_model: null argument");
        vf_eval_model(cv(poles, M), reinterpret_cast<const Cx*>(residues), K, cv(s, G), reinterpret_cast<Cx*>(out));
    });
}

int fds_fit_error_evf(int M, const fds_c64* poles, int K, const fds_c64* residues, int channel, int J,
                      const fds_c64* s, const fds_c64* values, double* out) {
    // fit_error_evf (vecfit.cpp:511-526) on the device (vf_evf_kernel)
    return fds_guard([&] {
        need(out && M >= 0 && K > 0 && J >= 0, "fit_error_evf: bad argument");
        if (channel < 0 || channel >= K) throw ValidationError("eval_model_channel: channel out of range");
        *out = vf_fit_error_evf(cv(poles, M), reinterpret_cast<const Cx*>(residues) + static_cast<size_t>(channel) * M,
                                cv(s, J), reinterpret_cast<const Cx*>(values) + channel, K);
    });
}

int fds_channel_errors(int MH, const fds_c64* ph, const fds_c64* rh, int ML, const fds_c64* pl, const fds_c64* rl,
                       int K, int G, const fds_c64* grid, double* errors) {
    return fds_guard([&] {
        need(K >= 0 && G >= 0, "channel_errors: negative size");
        const auto e = vf_channel_errors(cv(ph, MH), cv(rh, MH * K), cv(pl, ML), cv(rl, ML * K), K, cv(grid, G));
        std::memcpy(errors, e.data(), sizeof(double) * K);
    });
}

int fds_select_new_frequency(int MH, const fds_c64* ph, const fds_c64* rh, int ML, const fds_c64* pl,
                             const fds_c64* rl, int K, int G, const fds_c64* grid, int n_existing,
                             const fds_c64* existing, int n_orf, const int* orf_positions, double radius,
                             fds_c64* s_new) {
    return fds_guard([&] {
        const Cx c = vf_select_new_frequency(cv(ph, MH), cv(rh, MH * K), cv(pl, ML), cv(rl, ML * K), K, cv(grid, G),
                                             cv(existing, n_existing),
                                             std::vector<int>(orf_positions, orf_positions + n_orf), radius, nullptr);
        *s_new = {c.real(), c.imag()};
    });
}

int fds_fsm_invert(double period, int Ns, double eta, int K, const fds_c64* half, int hanning, double* out) {
    return fds_guard([&] {
        if (!(period > 0.0)) throw ValidationError("FsmGrid: period must be positive");
        if (Ns < 2 || Ns % 2 != 0) throw ValidationError("FsmGrid: sample count must be even and positive");
        need(K >= 0, "fsm_invert: negative channel count");
        if (K == 0) return;
        const int Nc = Ns / 2 + 1;
        auto& cx = VfContext::get();
        cplx* dh = static_cast<cplx*>(cx.values.get(sizeof(cplx) * Nc * static_cast<size_t>(K)));
        double* dout = static_cast<double*>(cx.out.get(sizeof(double) * Ns * static_cast<size_t>(K)));
        FDS_CUDA(cudaMemcpyAsync(dh, half, sizeof(cplx) * Nc * static_cast<size_t>(K), cudaMemcpyHostToDevice, cx.st));
        fsm_invert_device(period, Ns, eta, K, dh, Nc, 1, hanning != 0, dout, cx.st);
        FDS_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * Ns * static_cast<size_t>(K), cudaMemcpyDeviceToHost, cx.st));
        FDS_CUDA(cudaStreamSynchronize(cx.st));
    });
}

int fds_rational_invert(int M, const fds_c64* poles, int K, const fds_c64* residues, int T, const double* t,
                        double* out) {
    return fds_guard([&] {
        need(M >= 0 && K >= 0 && T >= 0, "rational_invert: negative size");
        rat_invert_host(cv(poles, M), cv(residues, M * K), K, std::vector<double>(t, t + T), out);
    });
}

// ---------------------------------------------------------------- device-resident (bench)
int fds_vf_identify_residues_device(int J, int K, const fds_c64* s_host, const fds_c64* values_dev, int M,
                                    const fds_c64* poles_host, fds_c64* residues_dev, double* ms) {
    return fds_guard([&] {
        auto& cx = VfContext::get();
        EventPair ev;
        const std::vector<Cx> canon = canonical_order(cv(poles_host, M));
        FDS_CUDA(cudaEventRecord(ev.a, cx.st));
        vf_residues_device(cv(s_host, J), reinterpret_cast<const cplx*>(values_dev), K, canon,
                           reinterpret_cast<cplx*>(residues_dev), nullptr, cx.st);
        FDS_CUDA(cudaEventRecord(ev.b, cx.st));
        FDS_CUDA(cudaEventSynchronize(ev.b));
        if (ms) *ms = elapsed(ev.a, ev.b);
    });
}

int fds_vf_identify_residues_device_heads(int J, int K, const fds_c64* s_host, const fds_c64* values_dev, int M,
                                    const fds_c64* poles_host, fds_c64* residues_dev, double* ms) {
    return fds_guard([&] {
        auto& cx = VfContext::get();
        EventPair ev;
        const std::vector<Cx> canon = canonical_order(cv(poles_host, M));
        FDS_CUDA(cudaEventRecord(ev.a, cx.st));
        vf_residues_device(cv(s_host, J), reinterpret_cast<const cplx*>(values_dev), K, canon,
                           reinterpret_cast<cplx*>(residues_dev), nullptr, cx.st, true);
        FDS_CUDA(cudaEventRecord(ev.b, cx.st));
        FDS_CUDA(cudaEventSynchronize(ev.b));
        if (ms) *ms = elapsed(ev.a, ev.b);
    });
}

int fds_rational_invert_device(int M, const fds_c64* poles_host, int K, const fds_c64* residues_dev, int T,
                               const double* t_host, double* out_dev, double* ms) {
    return fds_guard([&] {
        auto& cx = VfContext::get();
        EventPair ev;
        FDS_CUDA(cudaEventRecord(ev.a, cx.st));
        rat_invert_device(cv(poles_host, M), reinterpret_cast<const cplx*>(residues_dev), K,
                          std::vector<double>(t_host, t_host + T), out_dev, true, cx.st);
        FDS_CUDA(cudaEventRecord(ev.b, cx.st));
        FDS_CUDA(cudaEventSynchronize(ev.b));
        if (ms) *ms = elapsed(ev.a, ev.b);
    });
}

int fds_fsm_invert_device(double period, int Ns, double eta, int K, const fds_c64* half_dev, int hanning,
                          double* out_dev, double* ms) {
    return fds_guard([&] {
        auto& cx = VfContext::get();
        EventPair ev;
        FDS_CUDA(cudaEventRecord(ev.a, cx.st));
        fsm_invert_device(period, Ns, eta, K, reinterpret_cast<const cplx*>(half_dev), 1, static_cast<size_t>(K),
                          hanning != 0, out_dev, cx.st);
        FDS_CUDA(cudaEventRecord(ev.b, cx.st));
        FDS_CUDA(cudaEventSynchronize(ev.b));
        if (ms) *ms = elapsed(ev.a, ev.b);
    });
}

int fds_fsm_invert_device_strided(double period, int Ns, double eta, int K, const fds_c64* half_dev,
                                  long long stride_k, long long stride_i, int hanning, double* out_dev, double* ms) {
    return fds_guard([&] {
        need(stride_k >= 0 && stride_i >= 0, "fsm_invert: negative stride");
        auto& cx = VfContext::get();
        EventPair ev;
        FDS_CUDA(cudaEventRecord(ev.a, cx.st));
        fsm_invert_device(period, Ns, eta, K, reinterpret_cast<const cplx*>(half_dev), static_cast<size_t>(stride_k),
                          static_cast<size_t>(stride_i), hanning != 0, out_dev, cx.st);
        FDS_CUDA(cudaEventRecord(ev.b, cx.st));
        FDS_CUDA(cudaEventSynchronize(ev.b));
        if (ms) *ms = elapsed(ev.a, ev.b);
    });
}

// ---------------------------------------------------------------- AFS
namespace {

AfsCfg cfg_of(const fds_afs_config* c) {
    AfsCfg a;
    a.initial_count = c->initial_count;
    a.alpha_high = c->alpha_high;
    a.alpha_low = c->alpha_low;
    a.e1_threshold = c->e1_threshold;
    a.e2_threshold = c->e2_threshold;
    a.validation_steps = c->validation_steps;
    if (c->n_orf > 0) a.orf.assign(c->orf_indices, c->orf_indices + c->n_orf);
    if (c->n_test > 0) a.test.assign(c->test_indices, c->test_indices + c->n_test);
    a.omega_max = c->omega_max;
    a.eta = c->eta;
    a.period = c->period;
    a.grid_points = c->grid_points;
    a.time_points = c->time_points;
    a.max_iterations = c->max_iterations;
    a.seed = c->seed;
    a.n_relocations = c->n_relocations;
    return a;
}

void export_afs(const AfsOut& r, int channels, int cap, fds_c64* samples, fds_c64* values, double* hist,
                fds_c64* poles, fds_c64* residues, fds_afs_summary* sum) {
    const int nc = static_cast<int>(r.samples.size());
    if (nc > cap || static_cast<int>(r.history.size()) > cap || static_cast<int>(r.poles.size()) > cap)
        throw ValidationError("run_afs: output capacity too small");
    put(r.samples, samples);
    if (values) put(r.values, values);
    for (size_t i = 0; i < r.history.size(); ++i) {
        const auto& h = r.history[i];
        double* row = hist + 8 * i;
        row[0] = h.J; row[1] = h.MH; row[2] = h.ML; row[3] = h.has_s_new ? 1.0 : 0.0;
        row[4] = h.s_new.real(); row[5] = h.s_new.imag(); row[6] = h.e1; row[7] = h.e2;
    }
    put(r.poles, poles);
    if (residues) put(r.residues, residues);
    sum->n_c = nc;
    sum->converged = r.converged ? 1 : 0;
    sum->solver_calls = r.solver_calls;
    sum->n_history = static_cast<int>(r.history.size());
    sum->order = static_cast<int>(r.poles.size());
    sum->n_orf = static_cast<int>(r.orf.size());
    for (int i = 0; i < 8; ++i) sum->orf_indices[i] = i < sum->n_orf ? r.orf[i] : -1;
    (void)channels;
}

// Runs the driver; on an exception the completed iterations are exported
// before the error propagates (fds_run_afs_* contract in fdsweep_b200.h).
void run_and_export(const BatchEval& eval, int channels, const fds_afs_config* cfg, int cap, fds_c64* samples,
                    fds_c64* values, double* hist, fds_c64* poles, fds_c64* residues, fds_afs_summary* sum) {
    AfsOut r;
    try {
        run_afs_impl(eval, channels, cfg_of(cfg), r);
    } catch (...) {
        r.poles.clear();
        r.residues.clear();
        r.converged = false;
        if (static_cast<int>(r.samples.size()) <= cap && static_cast<int>(r.history.size()) <= cap)
            export_afs(r, channels, cap, samples, values, hist, poles, residues, sum);
        throw;
    }
    export_afs(r, channels, cap, samples, values, hist, poles, residues, sum);
}

}  // namespace

int fds_run_afs_bem(fds_bem* bem, const fds_afs_config* cfg, int cap, fds_c64* samples, fds_c64* values,
                    double* hist, fds_c64* poles, fds_c64* residues, fds_afs_summary* sum) {
    return fds_guard([&] {
        need(bem && cfg && sum, "run_afs: null argument");
        const int K = fds_bem_channels(bem);
        BatchEval eval = [&](const std::vector<Cx>& s, std::vector<Cx>& out) {
            const int rc = fds_bem_evaluate_batch(bem, reinterpret_cast<const fds_c64*>(s.data()),
                                                  static_cast<int>(s.size()), reinterpret_cast<fds_c64*>(out.data()));
            if (rc == FDS_ENUMERIC) throw NumericError(fds_last_error());
            if (rc == FDS_EVALIDATION) throw ValidationError(fds_last_error());
            if (rc == FDS_ECONVERGENCE) throw ConvergenceError(fds_last_error());
            if (rc != FDS_OK) throw CudaError(fds_last_error());
        };
        run_and_export(eval, K, cfg, cap, samples, values, hist, poles, residues, sum);
    });
}

int fds_run_afs_callback(fds_system_fn fn, void* user, int channels, const fds_afs_config* cfg, int cap,
                         fds_c64* samples, fds_c64* values, double* hist, fds_c64* poles, fds_c64* residues,
                         fds_afs_summary* sum) {
    return fds_guard([&] {
        need(fn && cfg && sum && channels > 0, "run_afs: bad argument");
        BatchEval eval = [&](const std::vector<Cx>& s, std::vector<Cx>& out) {
            for (size_t b = 0; b < s.size(); ++b) {  // reference order: one evaluate per frequency
                if (fn(user, {s[b].real(), s[b].imag()}, reinterpret_cast<fds_c64*>(out.data() + b * channels)) != 0)
                    throw NumericError("run_afs: system evaluation failed");
            }
        };
        run_and_export(eval, channels, cfg, cap, samples, values, hist, poles, residues, sum);
    });
}

}  // extern "C"
