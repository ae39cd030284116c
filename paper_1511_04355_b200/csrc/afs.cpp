// AFS driver (host C++) — replaces run_afs (proj/src/afs.cpp:226-396) with the
// same control flow, constants and error classes; every dense-grid / fitting /
// inversion kernel inside the loop runs on the GPU (vf.cu, laplace.cu), and the
// J0 initial frequencies of a BEM system are solved as one batched launch.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <future>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <limits>
#include <map>
#include <numbers>
#include <optional>
#include <set>

#include "afs.h"
#include "vf.cuh"

namespace fdsb {

namespace {

double trapezoid(const std::vector<double>& t, const double* y) {  // afs.cpp:18-24
    double acc = 0.0;
    for (size_t i = 1; i < t.size(); ++i) acc += 0.5 * (t[i] - t[i - 1]) * (y[i] + y[i - 1]);
    return acc;
}

void validate(const AfsCfg& c) {  // afs.cpp:59-84
    if (c.initial_count < 4) throw ValidationError("afs: initial_count must be >= 4");
    if (!(c.alpha_high > 1.0) || !(c.alpha_low > c.alpha_high)) throw ValidationError("afs: need 1 < alpha_high < alpha_low");
    if (!(c.e1_threshold > 0.0) || !(c.e2_threshold > 0.0)) throw ValidationError("afs: thresholds must be positive");
    if (c.validation_steps < 0) throw ValidationError("afs: validation_steps must be >= 0");
    if (!(c.omega_max > 0.0)) throw ValidationError("afs: omega_max must be positive");
    if (!(c.period > 0.0)) throw ValidationError("afs: period must be positive");
    if (c.grid_points < 2) throw ValidationError("afs: grid_points must be >= 2");
    if (c.time_points < 2) throw ValidationError("afs: time_points must be >= 2");
    if (c.max_iterations < 1) throw ValidationError("afs: max_iterations must be >= 1");
    if (c.n_relocations < 1) throw ValidationError("afs: n_relocations must be >= 1");
}

// growable device allocation owned by one run_afs call (contents not kept on growth)
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { if (p) cudaFree(p); }
    template <class T>
    T* get(size_t count) {
        const size_t need = std::max<size_t>(count, 1) * sizeof(T);
        if (need > bytes) {
            if (p) FDS_CUDA(cudaFree(p));
            p = nullptr;
            FDS_CUDA(cudaMalloc(&p, need));
            bytes = need;
        }
        return static_cast<T*>(p);
    }
};

}  // namespace

std::vector<int> draw_channels(int n, int k, uint64_t seed) {  // afs.cpp:28-46
    std::vector<int> pool(n);
    for (int i = 0; i < n; ++i) pool[i] = i;
    uint64_t st = seed ^ 0x9e3779b97f4a7c15ULL;
    std::vector<int> out;
    for (int i = 0; i < k; ++i) {
        st ^= st << 13;
        st ^= st >> 7;
        st ^= st << 17;
        const int j = i + static_cast<int>(st % static_cast<uint64_t>(pool.size() - i));
        std::swap(pool[i], pool[j]);
        out.push_back(pool[i]);
    }
    std::sort(out.begin(), out.end());
    return out;
}

std::vector<Cx> afs_initial_frequencies(int j0, double eta, double omega_max) {  // afs.cpp:88-100
    if (j0 < 2) throw ValidationError("initial_frequencies: j0 must be >= 2");
    if (!(omega_max > 0.0)) throw ValidationError("initial_frequencies: omega_max must be positive");
    std::vector<Cx> s(j0);
    for (int j = 0; j < j0; ++j)
        s[j] = Cx(eta, omega_max * (1.0 - std::cos(j * std::numbers::pi / (2.0 * (j0 - 1)))));
    return s;
}

std::pair<int, int> afs_fit_orders(int J, double ah, double al) {  // afs.cpp:102-116
    const int mh = static_cast<int>(std::floor(J / ah));
    int ml = static_cast<int>(std::floor(J / al));
    if (ml < 1) throw NumericError("fit_orders: degenerate low order for J = " + std::to_string(J));
    if (ml == mh) ml = std::max(mh - 1, 1);
    if (!(ml >= 1 && ml < mh)) throw NumericError("fit_orders: cannot separate the two orders for J = " + std::to_string(J));
    return {mh, ml};
}

double afs_error_e1(const std::vector<double>& t, const std::vector<double>& cur, const std::vector<double>& prev,
                    int K) {  // afs.cpp:189-216
    if (K == 0) throw ValidationError("error_e1: no channels");
    const size_t T = t.size();
    std::vector<double> d2(T), c2(T);
    double worst = 0.0;
    for (int k = 0; k < K; ++k) {
        for (size_t i = 0; i < T; ++i) {
            const double a = cur[k * T + i], b = prev[k * T + i];
            d2[i] = (a - b) * (a - b);
            c2[i] = a * a;
        }
        const double den = trapezoid(t, c2.data());
        if (den == 0.0) throw NumericError("error_e1: test channel " + std::to_string(k) + " has zero energy");
        worst = std::max(worst, trapezoid(t, d2.data()) / den);
    }
    return worst;
}

namespace {

// One host worker thread for the run: the low-order fit of each iteration runs
// on it (its own thread-local VfContext: stream, scratch, solve-operator cache)
// while the calling thread fits the high-order model. The two fits are
// independent (afs.cpp:337-340), so the results are those of the sequential
// order; an exception is reported in that order too (high first).
class FitWorker {
  public:
    explicit FitWorker(int device) : dev_(device), th_([this] { loop(); }) {}
    ~FitWorker() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    std::future<void> submit(std::function<void()> f) {
        auto task = std::make_shared<std::packaged_task<void()>>(std::move(f));
        std::future<void> fut = task->get_future();
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back([task] { (*task)(); });
        }
        cv_.notify_one();
        return fut;
    }

  private:
    void loop() {
        cudaSetDevice(dev_);
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;
                job = std::move(q_.front());
                q_.pop_front();
            }
            job();
        }
    }
    int dev_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    bool stop_ = false;
    std::thread th_;
};

}  // namespace

void run_afs_impl(const BatchEval& eval, int channels, const AfsCfg& cfg, AfsOut& r) {
    // FDSWEEP_AFS_TIMING=1: per-phase host wall times on stderr (development aid)
    static const bool timing = [] {
        const char* e = std::getenv("FDSWEEP_AFS_TIMING");
        return e && std::atoi(e) == 1;
    }();
    double t_eval = 0, t_upload = 0, t_fit = 0, t_err = 0, t_e1 = 0, t_sel = 0;
    using clk = std::chrono::steady_clock;
    auto since = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
    struct Report {
        bool on;
        double *a, *b, *c, *d, *e, *f;
        ~Report() {
            if (on)
                std::fprintf(stderr, "afs timing: eval %.3f upload %.3f fits %.3f errors %.3f e1 %.3f select %.3f s\n", *a,
                             *b, *c, *d, *e, *f);
        }
    } report{timing, &t_eval, &t_upload, &t_fit, &t_err, &t_e1, &t_sel};
    validate(cfg);
    r = AfsOut{};
    r.orf = cfg.orf.empty() ? draw_channels(channels, std::min(5, channels), cfg.seed) : cfg.orf;
    if (cfg.test.empty()) {
        r.test.resize(channels);
        for (int k = 0; k < channels; ++k) r.test[k] = k;
    } else {
        r.test = cfg.test;
    }
    for (const auto* set : {&r.orf, &r.test}) {
        std::set<int> seen;
        for (int k : *set) {
            if (k < 0 || k >= channels) throw ValidationError("afs: channel index out of range");
            if (!seen.insert(k).second) throw ValidationError("afs: duplicate channel index");
        }
    }
    std::vector<int> fitc;
    {
        std::set<int> u(r.orf.begin(), r.orf.end());
        u.insert(r.test.begin(), r.test.end());
        fitc.assign(u.begin(), u.end());
    }
    auto pos_of = [&](const std::vector<int>& idx) {
        std::vector<int> p;
        for (int k : idx) p.push_back(static_cast<int>(std::find(fitc.begin(), fitc.end(), k) - fitc.begin()));
        return p;
    };
    const std::vector<int> orf_pos = pos_of(r.orf), test_pos = pos_of(r.test);
    const int KF = static_cast<int>(fitc.size());

    std::map<std::pair<double, double>, std::vector<Cx>> cache;
    auto evaluate = [&](const std::vector<Cx>& ss) {  // afs.cpp:289-302 (batched misses)
        std::vector<Cx> miss;
        for (Cx s : ss)
            if (!cache.count({s.real(), s.imag()}) &&
                std::find(miss.begin(), miss.end(), s) == miss.end())
                miss.push_back(s);
        if (!miss.empty()) {
            std::vector<Cx> vals(miss.size() * static_cast<size_t>(channels));
            const auto t0 = clk::now();
            eval(miss, vals);
            t_eval += since(t0);
            for (size_t i = 0; i < miss.size(); ++i) {
                cache[{miss[i].real(), miss[i].imag()}] =
                    std::vector<Cx>(vals.begin() + i * channels, vals.begin() + (i + 1) * channels);
                ++r.solver_calls;
            }
        }
        for (Cx s : ss) {
            r.samples.push_back(s);
            const auto& v = cache[{s.real(), s.imag()}];
            r.values.insert(r.values.end(), v.begin(), v.end());
        }
    };
    evaluate(afs_initial_frequencies(cfg.initial_count, cfg.eta, cfg.omega_max));

    std::vector<Cx> grid(cfg.grid_points);  // afs.cpp:308-317
    for (int i = 0; i < cfg.grid_points; ++i)
        grid[i] = Cx(cfg.eta, cfg.omega_max * i / (cfg.grid_points - 1));
    const double radius = cfg.omega_max / (4.0 * cfg.grid_points);
    std::vector<double> e1_grid(cfg.time_points);
    for (int i = 0; i < cfg.time_points; ++i) e1_grid[i] = cfg.period * i / (cfg.time_points - 1);

    // GPU-resident iteration: the fit-channel samples,
    // both models' residues, the channel errors and the E1 series stay in HBM.
    // Per iteration only the new sample row goes up; E2, the worst ORF channel,
    // the per-channel E1 ratios and the selected grid index come back.
    auto& vcx = VfContext::get();
    const cudaStream_t st = vcx.st;
    int device = 0;
    FDS_CUDA(cudaGetDevice(&device));
    FitWorker worker(device);
    DevMem samp[2], res_h, res_l, res_t, ce, pos, red, ser[2];
    int samp_cur = 0, jcap = 0, j_dev = 0;
    const bool test_all = static_cast<int>(test_pos.size()) == KF &&
                          std::is_sorted(test_pos.begin(), test_pos.end()) && (KF == 0 || test_pos.back() == KF - 1);
    const int KT = static_cast<int>(test_pos.size()), KO = static_cast<int>(orf_pos.size());
    int* dtest = pos.get<int>(static_cast<size_t>(KT) + KO);
    int* dorf = dtest + KT;
    FDS_CUDA(cudaMemcpyAsync(dtest, test_pos.data(), KT * sizeof(int), cudaMemcpyHostToDevice, st));
    FDS_CUDA(cudaMemcpyAsync(dorf, orf_pos.data(), KO * sizeof(int), cudaMemcpyHostToDevice, st));
    double* dce = ce.get<double>(2 * static_cast<size_t>(KF));
    AfsErrReduce* dred = red.get<AfsErrReduce>(1);
    auto upload_samples = [&]() {  // append rows j_dev..J-1 of the fit channels
        const int J = static_cast<int>(r.samples.size());
        if (J > jcap) {
            const int cap = std::max(2 * jcap, J + 8);
            cplx* dst = samp[samp_cur ^ 1].get<cplx>(static_cast<size_t>(cap) * KF);
            if (j_dev > 0)
                FDS_CUDA(cudaMemcpyAsync(dst, samp[samp_cur].p, sizeof(cplx) * j_dev * static_cast<size_t>(KF),
                                         cudaMemcpyDeviceToDevice, st));
            samp_cur ^= 1;
            jcap = cap;
        }
        std::vector<Cx> rows(static_cast<size_t>(J - j_dev) * KF);
        for (int j = j_dev; j < J; ++j)
            for (int q = 0; q < KF; ++q)
                rows[static_cast<size_t>(j - j_dev) * KF + q] = r.values[static_cast<size_t>(j) * channels + fitc[q]];
        FDS_CUDA(cudaMemcpyAsync(static_cast<cplx*>(samp[samp_cur].p) + static_cast<size_t>(j_dev) * KF, rows.data(),
                                 rows.size() * sizeof(Cx), cudaMemcpyHostToDevice, st));
        FDS_CUDA(cudaStreamSynchronize(st));  // rows is a host temporary
        j_dev = J;
    };
    bool have_prev = false;
    int cur_slot = 0;
    int streak = 0;
    std::vector<Cx> ph;
    while (true) {  // afs.cpp:323-377
        if (static_cast<int>(r.history.size()) >= cfg.max_iterations)
            throw ConvergenceError("afs: no convergence within max_iterations");
        const int J = static_cast<int>(r.samples.size());
        const auto [MH, ML] = afs_fit_orders(J, cfg.alpha_high, cfg.alpha_low);
        auto t0 = clk::now();
        upload_samples();
        t_upload += since(t0);
        t0 = clk::now();
        const cplx* dsamp = static_cast<const cplx*>(samp[samp_cur].p);
        std::vector<Cx> ov(static_cast<size_t>(J) * KO);  // ORF samples for the host relocation step
        for (int j = 0; j < J; ++j)
            for (int q = 0; q < KO; ++q) ov[static_cast<size_t>(j) * KO + q] = r.values[static_cast<size_t>(j) * channels + r.orf[q]];
        cplx* drh = res_h.get<cplx>(static_cast<size_t>(MH) * KF);
        cplx* drl = res_l.get<cplx>(static_cast<size_t>(ML) * KF);
        // afs.cpp:337-340: the high- and low-order fits, concurrently
        std::vector<Cx> p_h, p_l;
        std::future<void> low = worker.submit([&] {
            auto& wcx = VfContext::get();
            p_l = vf_vector_fit_device(r.samples, ov.data(), dsamp, KF, orf_pos, ML, cfg.n_relocations, drl, wcx.st);
            FDS_CUDA(cudaStreamSynchronize(wcx.st));  // drl complete before the caller's stream reads it
        });
        std::exception_ptr fail;
        try {
            p_h = vf_vector_fit_device(r.samples, ov.data(), dsamp, KF, orf_pos, MH, cfg.n_relocations, drh, st);
        } catch (...) {
            fail = std::current_exception();
        }
        try {
            low.get();
        } catch (...) {
            if (!fail) fail = std::current_exception();
        }
        if (fail) std::rethrow_exception(fail);
        t_fit += since(t0);
        t0 = clk::now();
        vf_channel_errors_device(p_h, drh, p_l, drl, KF, grid, dtest, KT, dorf, KO, dce, dred, st);
        AfsErrReduce er;
        FDS_CUDA(cudaMemcpyAsync(&er, dred, sizeof(er), cudaMemcpyDeviceToHost, st));
        FDS_CUDA(cudaStreamSynchronize(st));
        if (er.zero_k >= 0)
            throw NumericError("channel_errors: channel " + std::to_string(er.zero_k) +
                               " has identically zero high-order fit");
        if (test_pos.empty()) throw ValidationError("error_e2: no test channels");
        const double e2 = er.e2;
        t_err += since(t0);
        t0 = clk::now();
        const cplx* drt = drh;
        if (!test_all) {
            cplx* g = res_t.get<cplx>(static_cast<size_t>(MH) * KT);
            vf_gather_channels(drh, KF, MH, dtest, KT, g, st);
            drt = g;
        }
        double* cur = ser[cur_slot].get<double>(static_cast<size_t>(KT) * e1_grid.size());
        rat_invert_mk_device(p_h, drt, KT, e1_grid, cur, st);
        const double e1 = have_prev ? afs_error_e1_device(e1_grid, cur, static_cast<double*>(ser[cur_slot ^ 1].p), KT, st)
                                    : std::numeric_limits<double>::infinity();
        have_prev = true;
        cur_slot ^= 1;
        t_e1 += since(t0);
        r.history.push_back({J, MH, ML, false, Cx(0, 0), e1, e2});
        ph = p_h;
        if (e1 <= cfg.e1_threshold && e2 <= cfg.e2_threshold) {
            if (++streak > cfg.validation_steps) {
                r.converged = true;
                break;
            }
        } else {
            streak = 0;
        }
        // select_new_frequency (afs.cpp:147-187) reuses this iteration's channel
        // errors (the reference recomputes identical values, afs.cpp:156)
        t0 = clk::now();
        const int sel = vf_select_device(p_h, drh + er.kmax, p_l, drl + er.kmax, static_cast<size_t>(KF), grid,
                                         r.samples, radius, st);
        const Cx s_new = grid[sel];
        t_sel += since(t0);
        r.history.back().has_s_new = true;
        r.history.back().s_new = s_new;
        evaluate({s_new});
    }
    // Final model over every system channel with the identified poles (afs.cpp:379-393).
    r.poles = ph;
    const int J = static_cast<int>(r.samples.size());
    const int M = static_cast<int>(ph.size());
    auto& cx = VfContext::get();
    cplx* dres = static_cast<cplx*>(cx.out.get(sizeof(cplx) * M * static_cast<size_t>(channels)));
    const cplx* dvals = nullptr;
    if (KF == channels && j_dev == J) {  // every channel is a fit channel: samples already in HBM
        dvals = static_cast<const cplx*>(samp[samp_cur].p);
    } else {
        cplx* v = static_cast<cplx*>(cx.values.get(sizeof(cplx) * J * static_cast<size_t>(channels)));
        FDS_CUDA(cudaMemcpyAsync(v, r.values.data(), sizeof(cplx) * J * static_cast<size_t>(channels),
                                 cudaMemcpyHostToDevice, cx.st));
        dvals = v;
    }
    vf_residues_device(r.samples, dvals, channels, canonical_order(ph), dres, nullptr, cx.st);
    std::vector<Cx> rmk(static_cast<size_t>(M) * channels);
    FDS_CUDA(cudaMemcpyAsync(rmk.data(), dres, rmk.size() * sizeof(cplx), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    r.residues.assign(static_cast<size_t>(channels) * M, Cx(0, 0));
    for (int k = 0; k < channels; ++k)
        for (int m = 0; m < M; ++m) r.residues[static_cast<size_t>(k) * M + m] = rmk[static_cast<size_t>(m) * channels + k];
}

}  // namespace fdsb
