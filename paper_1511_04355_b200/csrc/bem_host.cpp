// Host-side BEM preprocessing: per-element geometry records, the near-pair
// CSR list (subdivision levels), and the kernel-function constants.
// Same formulas and thresholds as the CPU oracle (oracle/bem_oracle.cpp) so
// both sides integrate every pair with the same rule.
#include <thread>
#include <algorithm>
#include <cmath>

#include "bem.cuh"

namespace fdsb {

int bem_subdivision_level(double d, double h) {
    if (d >= 2.0 * h) return 0;
    if (d >= 1.0 * h) return 1;
    if (d >= 0.5 * h) return 2;
    return 3;
}

void bem_build_geometry(const double* V, int nv, const int* F, int ne, std::vector<double>& geo,
                        std::vector<int>& pairs, std::vector<int>& near_ptr) {
    geo.assign(static_cast<size_t>(ne) * 16, 0.0);
    std::vector<double> h(ne);
    for (int e = 0; e < ne; ++e) {
        double v[3][3];
        for (int a = 0; a < 3; ++a) {
            const int id = F[3 * e + a];
            if (id < 0 || id >= nv) throw ValidationError("bem: triangle vertex index out of range");
            for (int d = 0; d < 3; ++d) v[a][d] = V[3 * id + d];
        }
        double c[3], u[3], w[3];
        for (int d = 0; d < 3; ++d) {
            c[d] = (v[0][d] + v[1][d] + v[2][d]) * (1.0 / 3.0);
            u[d] = v[1][d] - v[0][d];
            w[d] = v[2][d] - v[0][d];
        }
        const double nn[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
        const double tw = std::sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
        if (!(tw > 0.0)) throw ValidationError("bem: degenerate triangle");
        double* g = &geo[static_cast<size_t>(e) * 16];
        for (int a = 0; a < 3; ++a)
            for (int d = 0; d < 3; ++d) g[3 * a + d] = v[a][d];
        for (int d = 0; d < 3; ++d) {
            g[9 + d] = c[d];
            g[12 + d] = nn[d] / tw;
        }
        g[15] = 0.5 * tw;
        auto len = [](const double* a, const double* b) {
            const double x = a[0] - b[0], y = a[1] - b[1], z = a[2] - b[2];
            return std::sqrt(x * x + y * y + z * z);
        };
        h[e] = std::max({len(v[1], v[0]), len(v[2], v[1]), len(v[0], v[2])});
    }
    // near-pair lists (c-major, e ascending): rows are independent, so blocks of
    // collocation elements run on all host threads and are concatenated in
    // order; far pairs (d >= 2h, level 0) are rejected on d^2 without a sqrt
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const int nthreads = static_cast<int>(std::min<unsigned>(hw, static_cast<unsigned>(std::max(1, ne / 64))));
    std::vector<std::vector<int>> part(nthreads);
    std::vector<std::vector<int>> cnt(nthreads);
    auto work = [&](int t) {
        const int c0 = static_cast<int>(static_cast<long long>(ne) * t / nthreads);
        const int c1 = static_cast<int>(static_cast<long long>(ne) * (t + 1) / nthreads);
        std::vector<int>& out = part[t];
        cnt[t].assign(c1 - c0, 0);
        for (int c = c0; c < c1; ++c) {
            const double* gc = &geo[static_cast<size_t>(c) * 16];
            const size_t before = out.size();
            for (int e = 0; e < ne; ++e) {
                int level;
                if (e == c) {
                    level = -1;
                } else {
                    const double* ge = &geo[static_cast<size_t>(e) * 16];
                    const double x = gc[9] - ge[9], y = gc[10] - ge[10], z = gc[11] - ge[11];
                    const double d2 = x * x + y * y + z * z;
                    if (d2 >= 4.0 * h[e] * h[e] * (1.0 + 1e-12)) continue;  // certainly d >= 2h
                    level = bem_subdivision_level(std::sqrt(d2), h[e]);
                    if (level == 0) continue;
                }
                out.push_back(c);
                out.push_back(e);
                out.push_back(level);
            }
            cnt[t][c - c0] = static_cast<int>((out.size() - before) / 3);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    pairs.clear();
    near_ptr.assign(ne + 1, 0);
    size_t total = 0;
    for (const auto& p : part) total += p.size();
    pairs.reserve(total);
    int c = 0;
    for (int t = 0; t < nthreads; ++t) {
        pairs.insert(pairs.end(), part[t].begin(), part[t].end());
        for (int v : cnt[t]) {
            near_ptr[c + 1] = near_ptr[c] + v;
            ++c;
        }
    }
}

namespace {

void gauss_legendre01(int n, double* x, double* w) {
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < n; ++i) {
        double t = std::cos(pi * (i + 0.75) / (n + 0.5)), dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = t;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (t * p1 - p0) / (t * t - 1.0);
            const double dt = p1 / dp;
            t -= dt;
            if (std::abs(dt) < 1e-15) {
                p0 = 1.0;
                p1 = t;
                for (int k = 2; k <= n; ++k) {
                    const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
                    p0 = p1;
                    p1 = p2;
                }
                dp = n * (t * p1 - p0) / (t * t - 1.0);
                break;
            }
        }
        x[n - 1 - i] = 0.5 * (1.0 + t);
        w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

}  // namespace

BemParams make_bem_params(double mu, double nu, double rho) {
    if (!(mu > 0.0) || !(rho > 0.0) || !(nu > -1.0 && nu < 0.5))
        throw ValidationError("bem: material must satisfy mu > 0, rho > 0, -1 < nu < 0.5");
    BemParams P{};
    const double pi = 3.14159265358979323846;
    P.mu = mu;
    P.lambda = 2.0 * mu * nu / (1.0 - 2.0 * nu);
    P.lam_over_mu = P.lambda / mu;
    P.cs = std::sqrt(mu / rho);
    P.inv_cs = 1.0 / P.cs;
    const double cp = std::sqrt((P.lambda + 2.0 * mu) / rho);
    P.k = P.cs / cp;
    P.inv_k = cp / P.cs;
    P.inv_4pi_mu = 1.0 / (4.0 * pi * mu);
    double fact[BemParams::kTerms + 3];
    fact[0] = 1.0;
    for (int i = 1; i < BemParams::kTerms + 3; ++i) fact[i] = fact[i - 1] * i;
    for (int m = 0; m < BemParams::kTerms; ++m) {
        const double sg = (m % 2 == 0) ? 1.0 : -1.0;
        const double km2 = std::pow(P.k, m + 2);
        const double im1 = m >= 1 ? 1.0 / fact[m - 1] : 0.0;
        const double g = sg * (1.0 / fact[m] - 1.0 / fact[m + 1] + 1.0 / fact[m + 2]);
        const double h = sg * (-1.0 / fact[m + 1] + 1.0 / fact[m + 2]);
        const double q = sg * (1.0 / fact[m] - 3.0 / fact[m + 1] + 3.0 / fact[m + 2]);
        const double p = sg * (-im1 + 2.0 / fact[m] - 3.0 / fact[m + 1] + 3.0 / fact[m + 2]);
        const double w = sg * (-im1 + 4.0 / fact[m] - 9.0 / fact[m + 1] + 9.0 / fact[m + 2]);
        P.ta[m] = g - km2 * h;
        P.tb[m] = (1.0 - km2) * q;
        P.tc[m] = -p + km2 * q;
        P.td[m] = (km2 - 1.0) * w;
    }
    P.E10 = P.tc[0] - P.tb[0];
    P.E20 = P.lam_over_mu * (P.tc[0] - P.td[0] - 2.0 * P.tb[0]) - 2.0 * P.tb[0];
    const double s15 = std::sqrt(15.0);
    const double a = (6.0 - s15) / 21.0, b = (6.0 + s15) / 21.0;
    const double wa = (155.0 - s15) / 1200.0, wb = (155.0 + s15) / 1200.0;
    const double pts[7][3] = {{1.0 / 3, 1.0 / 3, 1.0 / 3}, {1 - 2 * a, a, a}, {a, 1 - 2 * a, a},
                              {a, a, 1 - 2 * a},         {1 - 2 * b, b, b}, {b, 1 - 2 * b, b},
                              {b, b, 1 - 2 * b}};
    const double ws[7] = {9.0 / 40, wa, wa, wa, wb, wb, wb};
    for (int q = 0; q < 7; ++q) {
        for (int d = 0; d < 3; ++d) P.r7l[q][d] = pts[q][d];
        P.r7w[q] = ws[q];
    }
    gauss_legendre01(BemParams::kSelfGauss, P.glx, P.glw);
    return P;
}

}  // namespace fdsb
