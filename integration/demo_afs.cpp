// The reference's own run_afs (proj/src/afs.cpp, unmodified) and system factory
// (proj/src/systems.cpp) driving the B200 library through the drop-in shim:
//   demo_afs modal <json>           -> reference ModalSystem, GPU vector fitting
//   demo_afs bem <level> <J0> <Jc>  -> GPU BemSystem (icosphere, random traction)
// Prints one JSON line {n_c, samples: [[re,im],...], converged}.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "fdsweep_b200_shim.hpp"

using namespace fdsweep;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    try {
        std::unique_ptr<FrequencySystem> sys;
        AfsConfig cfg;
        const std::string mode = argv[1];
        if (mode == "modal") {
            std::ifstream f(argv[2]);
            std::stringstream ss;
            ss << f.rdbuf();
            sys = make_system_from_json(ss.str());
            cfg.omega_max = 1.5 * 29.8;
            cfg.eta = 0.35;
            cfg.period = 20.0;
            cfg.orf_indices = {0, 1, 2};
            cfg.test_indices = {3, 4, 5};
            cfg.grid_points = 1024;
            cfg.time_points = 256;
            cfg.e1_threshold = 1e-2;
            cfg.e2_threshold = 5e-2;
        } else {
            // mesh passed as a binary file written by the test: nv, ne, V, F, traction, K, dofs
            std::ifstream f(argv[2], std::ios::binary);
            int nv = 0, ne = 0, K = 0;
            f.read(reinterpret_cast<char*>(&nv), sizeof(int));
            f.read(reinterpret_cast<char*>(&ne), sizeof(int));
            b200::BemMesh m;
            m.vertices.resize(3 * nv);
            m.triangles.resize(3 * ne);
            m.traction.resize(3 * ne);
            f.read(reinterpret_cast<char*>(m.vertices.data()), sizeof(double) * 3 * nv);
            f.read(reinterpret_cast<char*>(m.triangles.data()), sizeof(int) * 3 * ne);
            f.read(reinterpret_cast<char*>(m.traction.data()), sizeof(double) * 3 * ne);
            f.read(reinterpret_cast<char*>(&K), sizeof(int));
            m.channels.resize(K);
            f.read(reinterpret_cast<char*>(m.channels.data()), sizeof(int) * K);
            sys = std::make_unique<b200::BemSystem>(m);
            cfg.omega_max = 3.14159265358979323846 * 256 / 20.0;
            cfg.eta = 0.25;
            cfg.period = 20.0;
            cfg.initial_count = 12;
            cfg.validation_steps = 6;
            cfg.e1_threshold = INFINITY;
            cfg.e2_threshold = INFINITY;
        }
        const AfsResult r = run_afs(*sys, cfg);
        std::printf("{\"n_c\": %d, \"converged\": %s, \"solver_calls\": %d, \"samples\": [", r.n_c,
                    r.converged ? "true" : "false", r.solver_calls);
        for (size_t i = 0; i < r.samples.size(); ++i)
            std::printf("%s[%.17g, %.17g]", i ? ", " : "", r.samples[i].s.real(), r.samples[i].s.imag());
        std::printf("]}\n");
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
