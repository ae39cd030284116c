// ORACLE — test infrastructure only (CPU checker for the B200 product path).
//
// NEW CPU oracle for the Laplace-domain 3D elastodynamic collocation BEM that
// sits behind FrequencySystem::evaluate (proj/include/fdsweep/systems.hpp:34-42).
// The reference has no BEM at all, so there is nothing to
// restate; this file implements SURVEY.md Appendix A and DESIGN.md §3 — the
// formulation the CUDA assembly kernel shares:
//   * U*_ij = (A δij − B r,i r,j) / (4πμ r),
//     4π r² T*_ij = (C−B)(δij r,n + r,j n_i) − 2B(r,i n_j − 2 r,i r,j r,n)
//                   − 2D r,i r,j r,n + (λ/μ)(C − D − 2B) r,i n_j,
//     A = rψ, B = rχ, C = r²ψ', D = r²χ' of z = s r / c_s, x1 = k z, k = c_s/c_p;
//     a 16-term Taylor branch for |z| < 0.3 (the P/S 1/z² terms cancel).
//   * constant flat triangles, collocation at centroids, 7-point Dunavant rule,
//     near-singular subdivision level L(d/h) = 0,1,2,3 for d/h ≥ 2, ≥ 1, ≥ 0.5, < 0.5;
//   * self element: polar quadrature about the centroid on 3 sub-triangles
//     (10x10 Gauss–Legendre), static antisymmetric T* part as an exact CPV
//     ∫ e(θ) ln R(θ) dθ, free term ½I.
//   * Unknown ordering element-major [e][x,y,z]; A = ½I + T̂, b = Û t p̂(s), p̂ = 1/s.
// Dense complex LU with partial pivoting on |re|+|im| (LAPACK izamax rule,
// first maximum wins), column-major, then forward/back substitution.
#include "bem_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>

namespace oracle {

namespace {

constexpr double kPi = std::numbers::pi;
using C = std::complex<double>;

struct V3 { double x, y, z; };
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 mul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

struct Elem { V3 v[3]; V3 c; V3 n; double area; double h; };

// 7-point degree-5 rule (Dunavant), barycentric + weights summing to 1.
struct Rule7 { double l[7][3]; double w[7]; };
Rule7 make_rule7() {
    Rule7 r{};
    const double s15 = std::sqrt(15.0);
    const double a = (6.0 - s15) / 21.0, b = (6.0 + s15) / 21.0;
    const double wa = (155.0 - s15) / 1200.0, wb = (155.0 + s15) / 1200.0;
    const double pts[7][3] = {{1.0 / 3, 1.0 / 3, 1.0 / 3},
                              {1 - 2 * a, a, a}, {a, 1 - 2 * a, a}, {a, a, 1 - 2 * a},
                              {1 - 2 * b, b, b}, {b, 1 - 2 * b, b}, {b, b, 1 - 2 * b}};
    const double ws[7] = {9.0 / 40, wa, wa, wa, wb, wb, wb};
    for (int q = 0; q < 7; ++q) {
        for (int d = 0; d < 3; ++d) r.l[q][d] = pts[q][d];
        r.w[q] = ws[q];
    }
    return r;
}

// Gauss–Legendre nodes/weights on [0,1] (Newton iteration on P_n), ascending.
void gauss_legendre01(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double t = std::cos(kPi * (i + 0.75) / (n + 0.5)), dp = 1.0;
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
                p0 = 1.0; p1 = t;
                for (int k = 2; k <= n; ++k) {
                    const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
                    p0 = p1;
                    p1 = p2;
                }
                dp = n * (t * p1 - p0) / (t * t - 1.0);
                break;
            }
        }
        // t descends with i; store ascending on [0,1]
        x[n - 1 - i] = 0.5 * (1.0 + t);
        w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Kernel functions A,B,C,D.
KernelCoeffs::KernelCoeffs(double mu, double nu, double rho) {
    this->mu = mu;
    lambda = 2.0 * mu * nu / (1.0 - 2.0 * nu);
    cs = std::sqrt(mu / rho);
    cp = std::sqrt((lambda + 2.0 * mu) / rho);
    k = cs / cp;
    lam_over_mu = lambda / mu;
    // Taylor coefficients in z = s r / c_s (x1 = k z).
    double fact[kTerms + 3];
    fact[0] = 1.0;
    for (int i = 1; i < kTerms + 3; ++i) fact[i] = fact[i - 1] * i;
    for (int m = 0; m < kTerms; ++m) {
        const double sg = (m % 2 == 0) ? 1.0 : -1.0;
        const double km2 = std::pow(k, m + 2);
        const double im1 = m >= 1 ? 1.0 / fact[m - 1] : 0.0;
        const double g = sg * (1.0 / fact[m] - 1.0 / fact[m + 1] + 1.0 / fact[m + 2]);
        const double h = sg * (-1.0 / fact[m + 1] + 1.0 / fact[m + 2]);
        const double q = sg * (1.0 / fact[m] - 3.0 / fact[m + 1] + 3.0 / fact[m + 2]);
        const double p = sg * (-im1 + 2.0 / fact[m] - 3.0 / fact[m + 1] + 3.0 / fact[m + 2]);
        const double w = sg * (-im1 + 4.0 / fact[m] - 9.0 / fact[m + 1] + 9.0 / fact[m + 2]);
        ta[m] = g - km2 * h;
        tb[m] = (1.0 - km2) * q;
        tc[m] = -p + km2 * q;
        td[m] = (km2 - 1.0) * w;
    }
}

void KernelCoeffs::abcd(C z, C& A, C& B, C& Cc, C& D) const {
    if (std::abs(z) < kSeriesRadius) {
        A = B = Cc = D = C(0.0, 0.0);
        for (int m = kTerms - 1; m >= 0; --m) {
            A = A * z + ta[m];
            B = B * z + tb[m];
            Cc = Cc * z + tc[m];
            D = D * z + td[m];
        }
        return;
    }
    const C x1 = k * z;
    const C e2 = std::exp(-z), e1 = std::exp(-x1);
    const C iz = 1.0 / z, iz2 = iz * iz, ix = 1.0 / x1, ix2 = ix * ix;
    const double k2 = k * k;
    A = (1.0 + iz + iz2) * e2 - k2 * (ix + ix2) * e1;
    B = (1.0 + 3.0 * iz + 3.0 * iz2) * e2 - k2 * (1.0 + 3.0 * ix + 3.0 * ix2) * e1;
    Cc = -(z + 2.0 + 3.0 * iz + 3.0 * iz2) * e2 + k2 * (1.0 + 3.0 * ix + 3.0 * ix2) * e1;
    D = -(z + 4.0 + 9.0 * iz + 9.0 * iz2) * e2 + k2 * (x1 + 4.0 + 9.0 * ix + 9.0 * ix2) * e1;
}

// Full U (3x3) and T (3x3) at field point y for source x: rv = y - x, n = n(y).
void KernelCoeffs::ut(const double rv[3], const double n[3], C s, C U[9], C T[9]) const {
    const double r = std::sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
    const double e[3] = {rv[0] / r, rv[1] / r, rv[2] / r};
    const double rn = e[0] * n[0] + e[1] * n[1] + e[2] * n[2];
    C A, B, Cc, D;
    abcd(s * (r / cs), A, B, Cc, D);
    const double fu = 1.0 / (4.0 * kPi * mu * r), ft = 1.0 / (4.0 * kPi * r * r);
    const C cb = Cc - B, e4 = lam_over_mu * (Cc - D - 2.0 * B);
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            const double dij = i == j ? 1.0 : 0.0;
            const double eij = e[i] * e[j];
            U[3 * i + j] = (A * dij - B * eij) * fu;
            T[3 * i + j] = (cb * (dij * rn + e[j] * n[i]) - 2.0 * B * (e[i] * n[j] - 2.0 * eij * rn) -
                            2.0 * D * eij * rn + e4 * e[i] * n[j]) * ft;
        }
    }
}

// ---------------------------------------------------------------------------

BemOracle::BemOracle(const std::vector<double>& vertices, const std::vector<int>& tris,
                     double mu, double nu, double rho, const std::vector<double>& traction)
    : kc_(mu, nu, rho), traction_(traction) {
    const int ne = static_cast<int>(tris.size() / 3);
    if (ne < 1) throw std::invalid_argument("bem: no elements");
    if (static_cast<int>(traction.size()) != 3 * ne) throw std::invalid_argument("bem: traction size");
    geo_.resize(static_cast<size_t>(ne) * 16);
    for (int e = 0; e < ne; ++e) {
        V3 v[3];
        for (int a = 0; a < 3; ++a) {
            const int id = tris[3 * e + a];
            v[a] = {vertices[3 * id], vertices[3 * id + 1], vertices[3 * id + 2]};
        }
        const V3 c = mul(add(add(v[0], v[1]), v[2]), 1.0 / 3.0);
        const V3 nn = cross(sub(v[1], v[0]), sub(v[2], v[0]));
        const double twice = norm(nn);
        const V3 n = mul(nn, 1.0 / twice);
        double* g = &geo_[static_cast<size_t>(e) * 16];
        for (int a = 0; a < 3; ++a) { g[3 * a] = v[a].x; g[3 * a + 1] = v[a].y; g[3 * a + 2] = v[a].z; }
        g[9] = c.x; g[10] = c.y; g[11] = c.z;
        g[12] = n.x; g[13] = n.y; g[14] = n.z;
        g[15] = 0.5 * twice;
    }
    ne_ = ne;
    gauss_legendre01(kSelfGauss, glx_, glw_);  // built once here: assemble() is OpenMP-parallel
}

namespace {

Elem elem_of(const double* g) {
    Elem el;
    for (int a = 0; a < 3; ++a) el.v[a] = {g[3 * a], g[3 * a + 1], g[3 * a + 2]};
    el.c = {g[9], g[10], g[11]};
    el.n = {g[12], g[13], g[14]};
    el.area = g[15];
    el.h = std::max({norm(sub(el.v[1], el.v[0])), norm(sub(el.v[2], el.v[1])), norm(sub(el.v[0], el.v[2]))});
    return el;
}

// Regular / near-singular integral over triangle (p0,p1,p2) with subdivision level L.
void integrate_tri(const KernelCoeffs& kc, const Rule7& rule, V3 x, V3 p0, V3 p1, V3 p2, V3 n,
                   int level, C s, C Ui[9], C Ti[9]) {
    if (level > 0) {
        const V3 m01 = mul(add(p0, p1), 0.5), m12 = mul(add(p1, p2), 0.5), m20 = mul(add(p2, p0), 0.5);
        integrate_tri(kc, rule, x, p0, m01, m20, n, level - 1, s, Ui, Ti);
        integrate_tri(kc, rule, x, m01, p1, m12, n, level - 1, s, Ui, Ti);
        integrate_tri(kc, rule, x, m20, m12, p2, n, level - 1, s, Ui, Ti);
        integrate_tri(kc, rule, x, m01, m12, m20, n, level - 1, s, Ui, Ti);
        return;
    }
    const double area = 0.5 * norm(cross(sub(p1, p0), sub(p2, p0)));
    const double nv[3] = {n.x, n.y, n.z};
    for (int q = 0; q < 7; ++q) {
        const V3 y = add(add(mul(p0, rule.l[q][0]), mul(p1, rule.l[q][1])), mul(p2, rule.l[q][2]));
        const double rv[3] = {y.x - x.x, y.y - x.y, y.z - x.z};
        C U[9], T[9];
        kc.ut(rv, nv, s, U, T);
        const double w = rule.w[q] * area;
        for (int i = 0; i < 9; ++i) { Ui[i] += w * U[i]; Ti[i] += w * T[i]; }
    }
}

}  // namespace

int subdivision_level(double d, double h) {
    if (d >= 2.0 * h) return 0;
    if (d >= 1.0 * h) return 1;
    if (d >= 0.5 * h) return 2;
    return 3;
}

// Self-element integrals (polar quadrature about the centroid).
void BemOracle::self_block(int e, C s, C Ui[9], C Ti[9]) const {
    const std::vector<double>& gx = glx_;
    const std::vector<double>& gw = glw_;
    const Elem el = elem_of(&geo_[static_cast<size_t>(e) * 16]);
    const double n[3] = {el.n.x, el.n.y, el.n.z};
    for (int i = 0; i < 9; ++i) Ui[i] = Ti[i] = C(0.0, 0.0);
    // E1(0) = C0 - B0 = -kappa ; E2(0) = +kappa  (static antisymmetric part)
    C A0, B0, C0, D0;
    kc_.abcd(C(0.0, 0.0), A0, B0, C0, D0);
    const C E10 = C0 - B0, E20 = kc_.lam_over_mu * (C0 - D0 - 2.0 * B0) - 2.0 * B0;
    for (int edge = 0; edge < 3; ++edge) {
        const V3 P = el.v[edge], Q = el.v[(edge + 1) % 3];
        const V3 PQ = sub(Q, P);
        const double L = norm(PQ);
        const double hperp = norm(cross(sub(P, el.c), PQ)) / L;
        for (int a = 0; a < kSelfGauss; ++a) {
            const V3 E = add(P, mul(PQ, gx[a]));
            const V3 d = sub(E, el.c);
            const double R = norm(d);
            const double ev[3] = {d.x / R, d.y / R, d.z / R};
            const double jt = hperp * L * gw[a];  // dθ = hperp L / R² dt
            // static antisymmetric CPV: ∫ (E(0)-terms)/(4π ρ²) dA → ln R(θ) dθ
            const double lnR = std::log(R) / (R * R) * jt;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    Ti[3 * i + j] += (E10 * ev[j] * n[i] + E20 * ev[i] * n[j]) * (lnR / (4.0 * kPi));
            for (int b = 0; b < kSelfGauss; ++b) {
                const double u = gx[b];
                const double rho = R * u;
                C A, B, Cc, D;
                kc_.abcd(s * (rho / kc_.cs), A, B, Cc, D);
                const double w = jt * gw[b];
                // U: ∫ f dA = hperp L ∫∫ f(R u) u du dt ; f = (A δ - B e e)/(4πμ ρ)
                const double fu = w * u / (4.0 * kPi * kc_.mu * rho);
                // T remainder (flat element: r,n = 0): [(E1-E10) e_j n_i + (E2-E20) e_i n_j]/(4π ρ²)
                const C dE1 = (Cc - B) - E10;
                const C dE2 = kc_.lam_over_mu * (Cc - D - 2.0 * B) - 2.0 * B - E20;
                const double ft = w * u / (4.0 * kPi * rho * rho);
                for (int i = 0; i < 3; ++i) {
                    for (int j = 0; j < 3; ++j) {
                        const double dij = i == j ? 1.0 : 0.0;
                        Ui[3 * i + j] += (A * dij - B * ev[i] * ev[j]) * fu;
                        Ti[3 * i + j] += (dE1 * ev[j] * n[i] + dE2 * ev[i] * n[j]) * ft;
                    }
                }
            }
        }
    }
}

// Integrals of U*, T* over source element e seen from the centroid of c (no ½I).
void BemOracle::block(int c, int e, C s, C Ui[9], C Ti[9]) const {
    for (int i = 0; i < 9; ++i) Ui[i] = Ti[i] = C(0.0, 0.0);
    if (e == c) {
        self_block(e, s, Ui, Ti);
        return;
    }
    const Rule7 rule = make_rule7();
    const Elem ec = elem_of(&geo_[static_cast<size_t>(c) * 16]);
    const Elem ee = elem_of(&geo_[static_cast<size_t>(e) * 16]);
    const int L = subdivision_level(norm(sub(ec.c, ee.c)), ee.h);
    integrate_tri(kc_, rule, ec.c, ee.v[0], ee.v[1], ee.v[2], ee.n, L, s, Ui, Ti);
}

C BemOracle::entry(int row, int col, C s) const {
    C Ui[9], Ti[9];
    const int c = row / 3, i = row % 3, e = col / 3, j = col % 3;
    block(c, e, s, Ui, Ti);
    C v = Ti[3 * i + j];
    if (c == e && i == j) v += 0.5;
    return v;
}

C BemOracle::rhs(int row, C s) const {
    const int c = row / 3, i = row % 3;
    C acc(0.0, 0.0);
    for (int e = 0; e < ne_; ++e) {
        C Ui[9], Ti[9];
        block(c, e, s, Ui, Ti);
        for (int j = 0; j < 3; ++j) acc += Ui[3 * i + j] * traction_[3 * e + j];
    }
    return acc * (1.0 / s);
}

void BemOracle::assemble(C s, std::vector<C>& A, std::vector<C>& b) const {
    const int ne = ne_, n = 3 * ne_;
    A.assign(static_cast<size_t>(n) * n, C(0.0, 0.0));
    b.assign(n, C(0.0, 0.0));
    const Rule7 rule = make_rule7();
    const C pload = 1.0 / s;  // Heaviside load factor p̂(s)
#pragma omp parallel for schedule(dynamic, 4)
    for (int c = 0; c < ne; ++c) {
        const Elem ec = elem_of(&geo_[static_cast<size_t>(c) * 16]);
        C bacc[3] = {C(0, 0), C(0, 0), C(0, 0)};
        for (int e = 0; e < ne; ++e) {
            C Ui[9], Ti[9];
            for (int i = 0; i < 9; ++i) Ui[i] = Ti[i] = C(0.0, 0.0);
            if (e == c) {
                self_block(e, s, Ui, Ti);
            } else {
                const Elem ee = elem_of(&geo_[static_cast<size_t>(e) * 16]);
                const int L = subdivision_level(norm(sub(ec.c, ee.c)), ee.h);
                integrate_tri(kc_, rule, ec.c, ee.v[0], ee.v[1], ee.v[2], ee.n, L, s, Ui, Ti);
            }
            for (int i = 0; i < 3; ++i) {
                for (int j = 0; j < 3; ++j) {
                    C v = Ti[3 * i + j];
                    if (e == c && i == j) v += 0.5;
                    A[static_cast<size_t>(3 * e + j) * n + 3 * c + i] = v;  // column-major
                    bacc[i] += Ui[3 * i + j] * traction_[3 * e + j];
                }
            }
        }
        for (int i = 0; i < 3; ++i) b[3 * c + i] = bacc[i] * pload;
    }
}

// Partial-pivot LU (LAPACK zgetf2 semantics: pivot = first max of |re|+|im|).
int lu_factor(int n, std::vector<C>& A, std::vector<int>& piv) {
    piv.assign(n, 0);
    int info = 0;
    for (int k = 0; k < n; ++k) {
        C* colk = &A[static_cast<size_t>(k) * n];
        int p = k;
        double best = -1.0;
        for (int i = k; i < n; ++i) {
            const double v = std::abs(colk[i].real()) + std::abs(colk[i].imag());
            if (v > best) { best = v; p = i; }
        }
        piv[k] = p;
        if (best == 0.0) { if (!info) info = k + 1; continue; }
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(A[static_cast<size_t>(j) * n + k], A[static_cast<size_t>(j) * n + p]);
        const C inv = 1.0 / colk[k];
        for (int i = k + 1; i < n; ++i) colk[i] *= inv;
#pragma omp parallel for schedule(static)
        for (int j = k + 1; j < n; ++j) {
            C* colj = &A[static_cast<size_t>(j) * n];
            const C u = colj[k];
            if (u == C(0.0, 0.0)) continue;
            for (int i = k + 1; i < n; ++i) colj[i] -= colk[i] * u;
        }
    }
    return info;
}

void lu_solve(int n, const std::vector<C>& A, const std::vector<int>& piv, std::vector<C>& b) {
    for (int k = 0; k < n; ++k) std::swap(b[k], b[piv[k]]);
    for (int k = 0; k < n; ++k) {
        const C* colk = &A[static_cast<size_t>(k) * n];
        const C v = b[k];
        for (int i = k + 1; i < n; ++i) b[i] -= colk[i] * v;
    }
    for (int k = n - 1; k >= 0; --k) {
        const C* colk = &A[static_cast<size_t>(k) * n];
        b[k] /= colk[k];
        const C v = b[k];
        for (int i = 0; i < k; ++i) b[i] -= colk[i] * v;
    }
}

std::vector<C> BemOracle::solve(C s) const {
    std::vector<C> A, b;
    assemble(s, A, b);
    std::vector<int> piv;
    if (lu_factor(3 * ne_, A, piv) != 0) throw std::runtime_error("bem oracle: singular system");
    lu_solve(3 * ne_, A, piv, b);
    return b;
}

}  // namespace oracle
