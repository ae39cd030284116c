// BEM system description for the fdsweep_b200 CLI ("type": "bem" system JSON).
//
// The reference's system factory (systems.hpp:112, make_system_from_json) knows
// "rational" | "rod" | "modal"; the CLI adds "bem": a Laplace-domain elastodynamic
// cavity whose evaluate(s) is one collocation BEM solve. The
// mesh / load generators restate paper_1511_04355_b200/mesh.py so the CLI and
// the Python API see the same discretisation for the same JSON.
//
// The solve itself comes from one of two translation units with the same
// interface: integration/cli_bem_gpu.cpp (the B200 library, batched contour
// solves) or oracle/cli_bem_cpu.cpp (the CPU oracle; test infrastructure).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <tuple>
#include <vector>

#include "fdsweep/afs.hpp"
#include "fdsweep/systems.hpp"
#include "fdsweep/types.hpp"

namespace fdsweep::cli {

struct BemSpec {
    std::vector<double> vertices;  // [nv][3]
    std::vector<int> triangles;    // [ne][3], (v1-v0)x(v2-v0) points into the cavity
    double shear_modulus = 1.0, poisson_ratio = 0.25, density = 1.0;
    std::vector<double> traction;  // [ne][3], times the Heaviside factor 1/s
    std::vector<int> channels;     // output DOFs u[3e+i]; empty => all
    int max_batch = 0;             // 0 => library default
    // "solver": {"kind": "lu" | "gmres", "tol": 1e-12, "restart": 60, "max_iter": 1000}
    std::string solver = "lu";
    double tol = 1e-12;
    int restart = 60, max_iter = 1000;
};

// FrequencySystem over a BemSpec, plus a many-frequency evaluation that the
// GPU build runs as batched solves: out[b][k].
std::unique_ptr<FrequencySystem> make_bem_system(const BemSpec& spec);
std::vector<std::vector<Complex>> evaluate_many(const FrequencySystem& system, std::span<const Complex> s);
// "b200" or "cpu-oracle": which solver this binary links.
const char* solver_name();
// The linked library's own AFS driver for its BEM systems (GPU build: J0
// batched, fits on the device); empty => the caller runs the reference run_afs.
std::optional<AfsResult> run_afs_native(const FrequencySystem& system, const AfsConfig& cfg);

// ORF draw of afs.cpp:28-46 (sorted partial Fisher–Yates, xorshift64 without the
// zero-state guard), so explicit and drawn ORF sets are interchangeable.
inline std::vector<int> draw_indices(int n, int k, std::uint64_t seed) {
    std::vector<int> pool(n);
    for (int i = 0; i < n; ++i) pool[i] = i;
    std::uint64_t state = seed ^ 0x9e3779b97f4a7c15ULL;
    std::vector<int> out;
    for (int i = 0; i < k; ++i) {
        state ^= state << 13;
        state ^= state >> 7;
        state ^= state << 17;
        const int j = i + static_cast<int>(state % (pool.size() - i));
        std::swap(pool[i], pool[j]);
        out.push_back(pool[i]);
    }
    std::sort(out.begin(), out.end());
    return out;
}

// ---------------------------------------------------------------- generators
// xorshift64 of proj/src/afs.cpp:31-37 (state = seed ^ 0x9e3779b97f4a7c15).
struct XorShift64 {
    std::uint64_t state;
    explicit XorShift64(std::uint64_t seed) : state(seed ^ 0x9E3779B97F4A7C15ull) {
        if (state == 0) state = 1;
    }
    std::uint64_t next() {
        std::uint64_t s = state;
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return state = s;
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double normal() {  // Box–Muller, as mesh.py
        const double u1 = std::max(uniform(), 0x1.0p-60);
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
    }
};

// Unit icosphere, recursive 4-way midpoint subdivision (mesh.py icosphere).
inline void icosphere(int level, double radius, std::vector<double>& V, std::vector<int>& F) {
    const double t = (1.0 + std::sqrt(5.0)) / 2.0;
    const double b[12][3] = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                             {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
    std::vector<std::array<double, 3>> verts;
    for (const auto& p : b) {
        const double nrm = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
        verts.push_back({p[0] / nrm, p[1] / nrm, p[2] / nrm});
    }
    std::vector<std::array<int, 3>> f = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                         {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                         {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                         {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
    for (int l = 0; l < level; ++l) {
        std::map<std::pair<int, int>, int> cache;
        auto mid = [&](int a, int c) {
            const auto key = a < c ? std::make_pair(a, c) : std::make_pair(c, a);
            auto it = cache.find(key);
            if (it != cache.end()) return it->second;
            std::array<double, 3> p;
            for (int d = 0; d < 3; ++d) p[d] = (verts[a][d] + verts[c][d]) * 0.5;
            const double nrm = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
            for (int d = 0; d < 3; ++d) p[d] /= nrm;
            const int id = static_cast<int>(verts.size());
            verts.push_back(p);
            cache.emplace(key, id);
            return id;
        };
        std::vector<std::array<int, 3>> nf;
        for (const auto& tri : f) {
            const int a = tri[0], bb = tri[1], c = tri[2];
            const int ab = mid(a, bb), bc = mid(bb, c), ca = mid(c, a);
            nf.push_back({a, ab, ca});
            nf.push_back({bb, bc, ab});
            nf.push_back({c, ca, bc});
            nf.push_back({ab, bc, ca});
        }
        f = nf;
    }
    V.clear();
    for (const auto& p : verts)
        for (int d = 0; d < 3; ++d) V.push_back(p[d] * radius);
    F.clear();
    for (const auto& tri : f) {  // flip: normals into the cavity
        F.push_back(tri[0]);
        F.push_back(tri[2]);
        F.push_back(tri[1]);
    }
}

// Unit cube cavity, n x n squares per face, diagonal (i,j)->(i+1,j+1) (mesh.py cube_cavity).
inline void cube_cavity(int n, std::vector<double>& V, std::vector<int>& F) {
    std::map<std::tuple<long, long, long>, int> ids;
    V.clear();
    F.clear();
    auto vid = [&](const double p[3]) {
        const auto key = std::make_tuple(std::lround(p[0] * n), std::lround(p[1] * n), std::lround(p[2] * n));
        auto it = ids.find(key);
        if (it != ids.end()) return it->second;
        const int id = static_cast<int>(V.size() / 3);
        V.push_back(static_cast<double>(std::get<0>(key)) / n);
        V.push_back(static_cast<double>(std::get<1>(key)) / n);
        V.push_back(static_cast<double>(std::get<2>(key)) / n);
        ids.emplace(key, id);
        return id;
    };
    for (int a = 0; a < 3; ++a) {
        const int u = (a + 1) % 3, w = (a + 2) % 3;
        for (int side = 0; side < 2; ++side)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    auto P = [&](int ii, int jj) {
                        double p[3] = {0.0, 0.0, 0.0};
                        p[a] = static_cast<double>(side);
                        p[u] = static_cast<double>(ii) / n;
                        p[w] = static_cast<double>(jj) / n;
                        return vid(p);
                    };
                    const int p00 = P(i, j), p10 = P(i + 1, j), p11 = P(i + 1, j + 1), p01 = P(i, j + 1);
                    int t1[3] = {p00, p10, p11}, t2[3] = {p00, p11, p01};
                    if (side == 1) {
                        std::swap(t1[0], t1[2]);
                        std::swap(t2[0], t2[2]);
                    }
                    F.insert(F.end(), t1, t1 + 3);
                    F.insert(F.end(), t2, t2 + 3);
                }
    }
}

// Heaviside cavity pressure p0: traction t = -p0 n with n the unit normal into the cavity.
inline std::vector<double> pressure_traction(const std::vector<double>& V, const std::vector<int>& F, double p0) {
    const size_t ne = F.size() / 3;
    std::vector<double> t(3 * ne);
    for (size_t e = 0; e < ne; ++e) {
        const double* a = &V[3 * F[3 * e]];
        const double* b = &V[3 * F[3 * e + 1]];
        const double* c = &V[3 * F[3 * e + 2]];
        const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        const double nn[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
        const double tw = std::sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
        for (int d = 0; d < 3; ++d) t[3 * e + d] = -p0 * (nn[d] / tw);
    }
    return t;
}

inline std::vector<double> random_traction(size_t ne, std::uint64_t seed) {
    XorShift64 g(seed);
    std::vector<double> t(3 * ne);
    for (auto& x : t) x = g.normal();
    return t;
}

}  // namespace fdsweep::cli
