// fdsweep_b200 — command-line front end of the sweep toolkit (SPEC.md "cli"
// module: sweep-fsm | sweep-afs | fit | invert | compare).
//
// Everything the reference defines is used as the reference defines it: the
// system factory (systems.cpp make_system_from_json), run_afs (afs.cpp), the
// archive / model JSON / CSV writers and content hashes (io.cpp) are the
// reference's own, unmodified translation units; vector_fit, fsm_invert and
// rational_invert resolve to whichever implementation of vecfit.hpp /
// laplace.hpp the binary links (integration/*_b200.cpp -> libfdsweep_b200.so
// for the product binary; the CPU oracle for oracle/_ref/fdsweep_oracle_cli).
// The one addition is the "bem" system type (cli_bem.hpp).
//
// Config JSON (all keys optional unless noted):
//   sweep-fsm: {"period": T (req), "samples": N_s (req, even), "eta": η | "kappa": κ (default 3),
//               "hanning": true}
//   sweep-afs: AfsConfig keys (afs.hpp:18-36: initial_count, alpha_high, alpha_low, e1_threshold,
//               e2_threshold, validation_steps, omega_max, eta, period, grid_points, time_points,
//               max_iterations, n_relocations) + "samples": N_s of the FSM-equivalent time grid
//               (default round(omega_max T / π) to even); --seed/--orf/--test override
//   fit:       {"period", "samples", "eta" | "kappa"} (contour) or "frequencies": [[re, im], ...];
//               "order": M (req), "n_relocations": 3
//   invert:    {"model": path (req), "period": T, "samples": N_s} or "t": [...]
//   compare:   {"fsm": dir (req), "afs": dir (req)}
// sweep-afs also takes --resume <archive.json> (reuse its samples) and
// --checkpoint (rewrite <out>/archive.json after every new sample).
// Exit codes: 0 ok; 2 usage; 3 ValidationError; 4 NumericError; 5 IoError;
// 6 ConvergenceError or an AFS run that did not converge; 7 other errors.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "cli_bem.hpp"
#include "fdsweep/afs.hpp"
#include "fdsweep/io.hpp"
#include "fdsweep/laplace.hpp"
#include "fdsweep/systems.hpp"
#include "fdsweep/vecfit.hpp"

namespace fs = std::filesystem;
using json = nlohmann::json;
using namespace fdsweep;

namespace {

struct Args {
    std::string command, system, config, out, resume;
    bool checkpoint = false;
    std::optional<std::uint64_t> seed;
    std::optional<std::vector<int>> orf, test;
};

std::vector<int> parse_list(const std::string& s) {
    std::vector<int> v;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ','))
        if (!item.empty()) v.push_back(std::stoi(item));
    return v;
}

json read_json(const std::string& path) {
    try {
        return json::parse(read_file(path));
    } catch (const json::exception& e) {
        throw ValidationError("malformed JSON in " + path + ": " + e.what());
    }
}

// ---------------------------------------------------------------- systems
cli::BemSpec bem_spec(const json& j) {
    cli::BemSpec b;
    const json mesh = j.value("mesh", json::object());
    const std::string kind = mesh.value("kind", "icosphere");
    if (kind == "icosphere") {
        cli::icosphere(mesh.value("level", 2), mesh.value("radius", 1.0), b.vertices, b.triangles);
    } else if (kind == "cube") {
        cli::cube_cavity(mesh.value("n", 8), b.vertices, b.triangles);
    } else if (kind == "explicit") {
        for (const auto& v : mesh.at("vertices"))
            for (int d = 0; d < 3; ++d) b.vertices.push_back(v.at(d).get<double>());
        for (const auto& t : mesh.at("triangles"))
            for (int d = 0; d < 3; ++d) b.triangles.push_back(t.at(d).get<int>());
    } else {
        throw ValidationError("bem: unknown mesh kind '" + kind + "'");
    }
    const json mat = j.value("material", json::object());
    b.shear_modulus = mat.value("shear_modulus", 1.0);
    b.poisson_ratio = mat.value("poisson_ratio", 0.25);
    b.density = mat.value("density", 1.0);
    const size_t ne = b.triangles.size() / 3;
    const json load = j.value("load", json::object());
    const std::string lk = load.value("kind", "pressure");
    if (lk == "pressure") {
        b.traction = cli::pressure_traction(b.vertices, b.triangles, load.value("p0", 1.0));
    } else if (lk == "random") {
        b.traction = cli::random_traction(ne, load.value("seed", 0ull));
    } else if (lk == "explicit") {
        for (const auto& t : load.at("traction"))
            for (int d = 0; d < 3; ++d) b.traction.push_back(t.at(d).get<double>());
        if (b.traction.size() != 3 * ne) throw ValidationError("bem: traction needs one 3-vector per element");
    } else {
        throw ValidationError("bem: unknown load kind '" + lk + "'");
    }
    if (j.contains("channels")) b.channels = j.at("channels").get<std::vector<int>>();
    if (j.contains("collocation_points"))
        for (int e : j.at("collocation_points").get<std::vector<int>>())
            for (int d = 0; d < 3; ++d) b.channels.push_back(3 * e + d);
    b.max_batch = j.value("max_batch", 0);
    if (j.contains("solver")) {
        const json& sv = j.at("solver");
        b.solver = sv.value("kind", "lu");
        if (b.solver != "lu" && b.solver != "gmres") throw ValidationError("bem: solver kind must be lu or gmres");
        b.tol = sv.value("tol", b.tol);
        b.restart = sv.value("restart", b.restart);
        b.max_iter = sv.value("max_iter", b.max_iter);
    }
    return b;
}

std::unique_ptr<FrequencySystem> load_any_system(const std::string& path) {
    const std::string text = read_file(path);
    json j;
    try {
        j = json::parse(text);
    } catch (const json::exception& e) {
        throw ValidationError("malformed system JSON: " + std::string(e.what()));
    }
    if (j.value("type", "") == "bem") return cli::make_bem_system(bem_spec(j));
    return make_system_from_json(text);
}

std::vector<FrequencySample> sample(const FrequencySystem& sys, std::span<const Complex> s) {
    const auto vals = cli::evaluate_many(sys, s);
    std::vector<FrequencySample> out(s.size());
    for (size_t i = 0; i < s.size(); ++i) out[i] = FrequencySample{s[i], vals[i]};
    return out;
}

double eta_of(const json& c, double period) {
    if (c.contains("eta")) return c.at("eta").get<double>();
    return damping_eta(c.value("kappa", 3.0), period);
}

// ---------------------------------------------------------------- output
struct Outputs {
    fs::path dir;
    json files = json::object();
    void put(const std::string& name, const std::string& content) {
        write_file_atomic(dir / name, content);
        files[name] = content_hash(content);
    }
    void report(json r) {
        r["files"] = files;
        write_file_atomic(dir / "report.json", r.dump(1) + "\n");
    }
};

json complex_list(std::span<const Complex> v) {
    json a = json::array();
    for (const Complex z : v) a.push_back({z.real(), z.imag()});
    return a;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------------- commands
int cmd_sweep_fsm(const Args& a) {
    const auto t0 = std::chrono::steady_clock::now();
    const auto sys = load_any_system(a.system);
    const double t_system = seconds_since(t0);
    const json c = read_json(a.config);
    const FsmGrid grid(c.at("period").get<double>(), c.at("samples").get<int>());
    const double eta = eta_of(c, grid.period);
    const std::vector<Complex> s = grid.contour(eta);
    const auto t1 = std::chrono::steady_clock::now();
    const auto samples = sample(*sys, s);
    const double t_solve = seconds_since(t1);
    const auto& labels = sys->descriptor().channel_labels;
    const int K = sys->descriptor().channel_count;
    std::vector<std::vector<Complex>> half(K, std::vector<Complex>(s.size()));
    for (size_t i = 0; i < s.size(); ++i)
        for (int k = 0; k < K; ++k) half[k][i] = samples[i].values[k];
    const TimeSeries ts = fsm_invert(grid, eta, half, labels, c.value("hanning", true));
    Outputs o{a.out};
    o.put("spectrum.csv", spectrum_csv(samples, labels));
    o.put("time.csv", timeseries_csv(ts));
    o.report({{"command", "sweep-fsm"}, {"solver", cli::solver_name()}, {"n_c", grid.contour_count()},
              {"period", grid.period}, {"samples", grid.sample_count}, {"eta", eta},
              {"channels", K}, {"wall_s", seconds_since(t0)}, {"system_s", t_system}, {"solve_s", t_solve}});
    return 0;
}

int cmd_sweep_afs(const Args& a) {
    const auto t0 = std::chrono::steady_clock::now();
    const auto sys = load_any_system(a.system);
    const json c = read_json(a.config);
    AfsConfig cfg;
    cfg.initial_count = c.value("initial_count", cfg.initial_count);
    cfg.alpha_high = c.value("alpha_high", cfg.alpha_high);
    cfg.alpha_low = c.value("alpha_low", cfg.alpha_low);
    auto thr = [&](const char* key, double def) -> double {
        if (!c.contains(key)) return def;
        if (c.at(key).is_string() && c.at(key).get<std::string>() == "inf") return INFINITY;
        return c.at(key).get<double>();
    };
    cfg.e1_threshold = thr("e1_threshold", cfg.e1_threshold);
    cfg.e2_threshold = thr("e2_threshold", cfg.e2_threshold);
    cfg.validation_steps = c.value("validation_steps", cfg.validation_steps);
    cfg.omega_max = c.value("omega_max", cfg.omega_max);
    cfg.period = c.value("period", cfg.period);
    cfg.eta = c.contains("eta") || c.contains("kappa") ? eta_of(c, cfg.period) : cfg.eta;
    cfg.grid_points = c.value("grid_points", cfg.grid_points);
    cfg.time_points = c.value("time_points", cfg.time_points);
    cfg.max_iterations = c.value("max_iterations", cfg.max_iterations);
    cfg.n_relocations = c.value("n_relocations", cfg.n_relocations);
    if (c.contains("orf_indices")) cfg.orf_indices = c.at("orf_indices").get<std::vector<int>>();
    if (c.contains("test_indices")) cfg.test_indices = c.at("test_indices").get<std::vector<int>>();
    cfg.seed = c.value("seed", 0ull);
    if (a.seed) cfg.seed = *a.seed;
    if (a.orf) cfg.orf_indices = *a.orf;
    if (a.test) cfg.test_indices = *a.test;
    int ns = c.value("samples", 0);
    if (ns <= 0) {
        ns = static_cast<int>(std::lround(cfg.omega_max * cfg.period / M_PI));
        ns += ns % 2;
    }
    const FsmGrid grid(cfg.period, ns);

    // explicit ORF set (afs.cpp:234-238 draws the same one from the seed)
    const int K = sys->descriptor().channel_count;
    if (cfg.orf_indices.empty()) cfg.orf_indices = cli::draw_indices(K, std::min(5, K), cfg.seed);
    Outputs o{a.out};
    // --resume: samples of an earlier (interrupted) run are reused, never re-solved
    // (afs.cpp:281-302); --checkpoint: the archive is rewritten after every new
    // sample, so an interrupted run can be resumed.
    std::vector<FrequencySample> resume;
    if (!a.resume.empty()) resume = load_archive(a.resume).samples;
    std::vector<FrequencySample> done = resume;
    std::function<void(const FrequencySample&)> on_sample;
    if (a.checkpoint)
        on_sample = [&](const FrequencySample& smp) {
            done.push_back(smp);
            SweepArchive ar;
            ar.config = cfg;
            ar.samples = done;
            save_archive(ar, o.dir / "archive.json");
        };
    std::optional<AfsResult> native;
    if (resume.empty() && !a.checkpoint) native = cli::run_afs_native(*sys, cfg);
    AfsResult r;
    if (native) {
        r = std::move(*native);
    } else {
        try {
            r = run_afs(*sys, cfg, resume, on_sample);
        } catch (const ConvergenceError&) {  // budget exhausted: the checkpoint archive is the partial result
            if (a.checkpoint) std::fprintf(stderr, "fdsweep_b200: partial archive in %s\n", (o.dir / "archive.json").c_str());
            throw;
        }
    }
    const auto& labels = sys->descriptor().channel_labels;
    const TimeSeries ts = rational_invert(r.model_high, grid.time_grid());
    o.put("spectrum.csv", spectrum_csv(r.samples, labels));
    o.put("time.csv", timeseries_csv(ts));
    o.put("model.json", model_to_json(r.model_high));
    if (!r.converged) {  // partial archive for resume (io.hpp SweepArchive)
        SweepArchive ar;
        ar.config = cfg;
        ar.samples = r.samples;
        ar.model = r.model_high;
        save_archive(ar, o.dir / "archive.json");
        o.files["archive.json"] = content_hash(read_file(o.dir / "archive.json"));
    }
    json hist = json::array();
    for (const auto& h : r.history) {
        json it = {{"sample_count", h.sample_count}, {"order_high", h.order_high}, {"order_low", h.order_low},
                   {"e1", h.e1}, {"e2", h.e2}};
        if (h.s_new) it["s_new"] = {h.s_new->real(), h.s_new->imag()};
        hist.push_back(it);
    }
    std::vector<Complex> seq;
    for (const auto& smp : r.samples) seq.push_back(smp.s);
    o.report({{"command", "sweep-afs"}, {"solver", cli::solver_name()}, {"n_c", r.n_c}, {"converged", r.converged},
              {"solver_calls", r.solver_calls}, {"seed", r.seed}, {"orf_indices", r.orf_indices},
              {"test_indices", r.test_indices}, {"period", cfg.period}, {"samples", ns}, {"eta", cfg.eta},
              {"omega_max", cfg.omega_max}, {"frequencies", complex_list(seq)}, {"history", hist}});
    // wall time kept out of report.json so fixed-seed reports are byte-identical
    write_file_atomic(o.dir / "timing.json", json({{"wall_s", seconds_since(t0)}}).dump() + "\n");
    return r.converged ? 0 : 6;
}

int cmd_fit(const Args& a) {
    const auto t0 = std::chrono::steady_clock::now();
    const auto sys = load_any_system(a.system);
    const json c = read_json(a.config);
    std::vector<Complex> s;
    if (c.contains("frequencies")) {
        for (const auto& z : c.at("frequencies")) s.emplace_back(z.at(0).get<double>(), z.at(1).get<double>());
    } else {
        const FsmGrid grid(c.at("period").get<double>(), c.at("samples").get<int>());
        s = grid.contour(eta_of(c, grid.period));
    }
    const auto samples = sample(*sys, s);
    const int K = sys->descriptor().channel_count;
    std::vector<int> orf = a.orf ? *a.orf : c.value("orf_indices", std::vector<int>{});
    if (orf.empty())
        for (int k = 0; k < std::min(K, 5); ++k) orf.push_back(k);
    const auto& labels = sys->descriptor().channel_labels;
    const auto [model, rep] = vector_fit(samples, orf, c.at("order").get<int>(), c.value("n_relocations", 3), labels);
    std::vector<double> evf(K);
    for (int k = 0; k < K; ++k) evf[k] = fit_error_evf(model, k, samples);
    Outputs o{a.out};
    o.put("spectrum.csv", spectrum_csv(samples, labels));
    o.put("model.json", model_to_json(model));
    o.report({{"command", "fit"}, {"solver", cli::solver_name()}, {"n_c", static_cast<int>(s.size())},
              {"order", c.at("order").get<int>()}, {"orf_indices", orf}, {"iterations_used", rep.iterations_used},
              {"pole_movement", rep.pole_movement}, {"unstable_pole_count", rep.unstable_pole_count},
              {"e_vf", evf}, {"wall_s", seconds_since(t0)}});
    return 0;
}

int cmd_invert(const Args& a) {
    const json c = read_json(a.config);
    const RationalModel model = load_model(c.at("model").get<std::string>());
    std::vector<double> t;
    if (c.contains("t")) {
        t = c.at("t").get<std::vector<double>>();
    } else {
        t = FsmGrid(c.at("period").get<double>(), c.at("samples").get<int>()).time_grid();
    }
    const TimeSeries ts = rational_invert(model, t);
    Outputs o{a.out};
    o.put("time.csv", timeseries_csv(ts));
    o.report({{"command", "invert"}, {"solver", cli::solver_name()}, {"poles", static_cast<int>(model.poles.size())},
              {"channels", static_cast<int>(ts.channel_count())}, {"time_steps", static_cast<int>(t.size())}});
    return 0;
}

int cmd_compare(const Args& a) {
    const json c = read_json(a.config);
    const fs::path fd = c.at("fsm").get<std::string>(), ad = c.at("afs").get<std::string>();
    const json rf = json::parse(read_file(fd / "report.json")), ra = json::parse(read_file(ad / "report.json"));
    const TimeSeries f = load_timeseries_csv(fd / "time.csv"), g = load_timeseries_csv(ad / "time.csv");
    const double T = rf.at("period").get<double>();
    if (std::abs(ra.value("period", T) - T) > 1e-12 * std::abs(T) || f.t.size() != g.t.size())
        throw ValidationError("compare: grid mismatch (time grids differ)");
    for (size_t n = 0; n < f.t.size(); ++n)
        if (std::abs(f.t[n] - g.t[n]) > 1e-12 * std::max(1.0, std::abs(f.t[n])))
            throw ValidationError("compare: grid mismatch (time grids differ)");
    if (f.channel_labels != g.channel_labels) throw ValidationError("compare: channel sets differ");
    json per = json::object();
    for (size_t k = 0; k < f.channel_count(); ++k) {
        double se = 0.0, pk = 0.0;
        int cnt = 0;
        for (size_t n = 0; n < f.t.size(); ++n) {
            if (f.t[n] > 0.9 * T) break;
            const double d = f.values[k][n] - g.values[k][n];
            se += d * d;
            pk = std::max(pk, std::abs(f.values[k][n]));
            ++cnt;
        }
        const double rms = cnt ? std::sqrt(se / cnt) : 0.0;
        per[f.channel_labels[k]] = {{"rms_diff", rms}, {"rms_diff_over_peak", pk > 0.0 ? rms / pk : 0.0}};
    }
    const double ncf = rf.at("n_c").get<double>(), nca = ra.at("n_c").get<double>();
    const json out = {{"nc_fsm", ncf}, {"nc_afs", nca}, {"nc_ratio", nca > 0 ? ncf / nca : 0.0},
                      {"per_channel", per}, {"metadata", {{"horizon", "[0, 0.9T]"}, {"period", T}}}};
    fs::create_directories(a.out);
    write_file_atomic(fs::path(a.out) / "comparison.json", out.dump(1) + "\n");
    return 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage: fdsweep_b200 {sweep-fsm|sweep-afs|fit|invert|compare} [--system s.json] --config c.json "
                 "--out dir [--seed n] [--orf i,j,..] [--test i,j,..] [--resume archive.json] [--checkpoint]\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    Args a;
    a.command = argv[1];
    for (int i = 2; i < argc; ++i) {
        const std::string f = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw ValidationError("missing value for " + f);
            return argv[++i];
        };
        try {
            if (f == "--system") a.system = val();
            else if (f == "--config") a.config = val();
            else if (f == "--out") a.out = val();
            else if (f == "--seed") a.seed = std::stoull(val());
            else if (f == "--orf") a.orf = parse_list(val());
            else if (f == "--test") a.test = parse_list(val());
            else if (f == "--resume") a.resume = val();
            else if (f == "--checkpoint") a.checkpoint = true;
            else {
                usage();
                return 2;
            }
        } catch (const std::exception& e) {
            std::fprintf(stderr, "fdsweep_b200: %s\n", e.what());
            return 2;
        }
    }
    const bool needs_system = a.command == "sweep-fsm" || a.command == "sweep-afs" || a.command == "fit";
    if (a.config.empty() || a.out.empty() || (needs_system && a.system.empty())) {
        usage();
        return 2;
    }
    try {
        fs::create_directories(a.out);
        if (a.command == "sweep-fsm") return cmd_sweep_fsm(a);
        if (a.command == "sweep-afs") return cmd_sweep_afs(a);
        if (a.command == "fit") return cmd_fit(a);
        if (a.command == "invert") return cmd_invert(a);
        if (a.command == "compare") return cmd_compare(a);
        usage();
        return 2;
    } catch (const ValidationError& e) {
        std::fprintf(stderr, "fdsweep_b200: validation error: %s\n", e.what());
        return 3;
    } catch (const NumericError& e) {
        std::fprintf(stderr, "fdsweep_b200: numeric error: %s\n", e.what());
        return 4;
    } catch (const IoError& e) {
        std::fprintf(stderr, "fdsweep_b200: io error: %s\n", e.what());
        return 5;
    } catch (const ConvergenceError& e) {
        std::fprintf(stderr, "fdsweep_b200: convergence error: %s\n", e.what());
        return 6;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "fdsweep_b200: error: %s\n", e.what());
        return 7;
    }
}
