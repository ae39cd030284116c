// Eigenvalues of the M x M relocation matrix H = blockdiag(poles) - b c^T
// (vecfit.cpp:297-324; the reference calls Eigen::EigenSolver). M <= ~120, so
// this stays on the host: a few milliseconds at most of sequential bulge
// chasing that a GPU cannot shorten.
//
// Algorithm: Householder reduction to upper Hessenberg form followed by the
// small-bulge implicit double-shift QR iteration in the formulation of LAPACK's
// xLAHQR (eigenvalues only): the Ahues–Tisseur conservative deflation test,
// exceptional shifts every 10 iterations alternating between the bottom and
// the top of the active block, real Wilkinson-style shift selection, and the
// xLANV2 standardisation of each deflated 2 x 2 block (complex pairs come out
// exactly conjugate, real pairs exactly real). This is deliberately not the
// EISPACK-hqr formulation of the CPU oracle (oracle/linalg.hpp), so the product
// and the checker share no eigen code.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <complex>
#include <vector>

#include "eig_host.h"

namespace fdsb::eig {

namespace {

struct Hm {
    int n;
    std::vector<double> a;  // column-major
    double& operator()(int i, int j) { return a[static_cast<size_t>(j) * n + i]; }
};

double sgn(double mag, double s) { return std::copysign(std::fabs(mag), s); }

// Reflector (I - tau v v^T), v = (1, x), mapping (alpha, x) to (beta, 0).
void reflector(double& alpha, double* x, int nx, double& tau) {
    double xn = 0.0;
    for (int i = 0; i < nx; ++i) xn = std::hypot(xn, x[i]);
    if (xn == 0.0) {
        tau = 0.0;
        return;
    }
    const double beta = -sgn(std::hypot(alpha, xn), alpha);
    tau = (beta - alpha) / beta;
    const double sc = 1.0 / (alpha - beta);
    for (int i = 0; i < nx; ++i) x[i] *= sc;
    alpha = beta;
}

// Standardised Schur form of [a b; c d]; returns its two eigenvalues.
void schur2(double a, double b, double c, double d, std::complex<double>& e1, std::complex<double>& e2) {
    const double eps = DBL_EPSILON;
    if (c == 0.0) {
    } else if (b == 0.0) {
        std::swap(a, d);
        b = -c;
        c = 0.0;
    } else if (a - d == 0.0 && std::signbit(b) != std::signbit(c)) {
    } else {
        const double temp = a - d;
        double p = 0.5 * temp;
        const double bcmax = std::max(std::fabs(b), std::fabs(c));
        const double bcmis = std::min(std::fabs(b), std::fabs(c)) * sgn(1.0, b) * sgn(1.0, c);
        double scale = std::max(std::fabs(p), bcmax);
        double z = p / scale * p + bcmax / scale * bcmis;
        if (z >= 4.0 * eps) {  // real eigenvalues
            z = p + sgn(std::sqrt(scale) * std::sqrt(z), p);
            a = d + z;
            d = d - bcmax / z * bcmis;
            b = b - c;
            c = 0.0;
        } else {  // complex (or nearly equal real) eigenvalues: equalise the diagonal
            const double sigma = b + c;
            const double tau = std::hypot(sigma, temp);
            const double cs = std::sqrt(0.5 * (1.0 + std::fabs(sigma) / tau));
            const double sn = -(p / (tau * cs)) * sgn(1.0, sigma);
            const double aa = a * cs + b * sn, bb = -a * sn + b * cs;
            const double cc = c * cs + d * sn, dd = -c * sn + d * cs;
            a = aa * cs + cc * sn;
            b = bb * cs + dd * sn;
            c = -aa * sn + cc * cs;
            d = -bb * sn + dd * cs;
            const double mid = 0.5 * (a + d);
            a = d = mid;
            if (c != 0.0) {
                if (b != 0.0) {
                    if (std::signbit(b) == std::signbit(c)) {  // real pair
                        const double sab = std::sqrt(std::fabs(b)), sac = std::sqrt(std::fabs(c));
                        p = sgn(sab * sac, c);
                        a = mid + p;
                        d = mid - p;
                        b = b - c;
                        c = 0.0;
                    }
                } else {
                    b = -c;
                    c = 0.0;
                }
            }
        }
    }
    if (c == 0.0) {
        e1 = {a, 0.0};
        e2 = {d, 0.0};
    } else {
        const double im = std::sqrt(std::fabs(b)) * std::sqrt(std::fabs(c));
        e1 = {a, im};
        e2 = {d, -im};
    }
}

void to_hessenberg(Hm& h) {
    const int n = h.n;
    std::vector<double> v(n), w(n);
    for (int k = 0; k + 2 < n; ++k) {
        const int len = n - k - 1;  // rows k+1 .. n-1
        double alpha = h(k + 1, k);
        for (int i = 1; i < len; ++i) v[i] = h(k + 1 + i, k);
        double tau;
        reflector(alpha, v.data() + 1, len - 1, tau);
        h(k + 1, k) = alpha;
        for (int i = k + 2; i < n; ++i) h(i, k) = 0.0;
        if (tau == 0.0) continue;
        v[0] = 1.0;
        for (int j = k + 1; j < n; ++j) {  // left: (I - tau v v^T) H
            double d = 0.0;
            for (int i = 0; i < len; ++i) d += v[i] * h(k + 1 + i, j);
            d *= tau;
            for (int i = 0; i < len; ++i) h(k + 1 + i, j) -= d * v[i];
        }
        // right: H (I - tau v v^T), column-oriented (same per-row summation order)
        std::fill(w.begin(), w.end(), 0.0);
        for (int c = 0; c < len; ++c) {
            const double vc = v[c];
            const double* col = &h(0, k + 1 + c);
            for (int i = 0; i < n; ++i) w[i] += col[i] * vc;
        }
        for (int i = 0; i < n; ++i) w[i] *= tau;
        for (int c = 0; c < len; ++c) {
            const double vc = v[c];
            double* col = &h(0, k + 1 + c);
            for (int i = 0; i < n; ++i) col[i] -= w[i] * vc;
        }
    }
}

}  // namespace

bool eigenvalues(int n, const double* colmajor, std::vector<std::complex<double>>& ev) {
    ev.assign(n, {0.0, 0.0});
    if (n == 0) return true;
    Hm h{n, std::vector<double>(colmajor, colmajor + static_cast<size_t>(n) * n)};
    to_hessenberg(h);
    const double ulp = DBL_EPSILON;
    const double smlnum = DBL_MIN * (static_cast<double>(n) / ulp);
    const int itmax = 30 * std::max(10, n);
    constexpr int kExceptional = 10;
    int kdefl = 0;
    int i = n - 1;
    while (i >= 0) {
        int l = 0;
        bool done = false;
        for (int its = 0; its <= itmax; ++its) {
            int k;
            for (k = i; k > l; --k) {  // a negligible subdiagonal entry?
                const double sub = std::fabs(h(k, k - 1));
                if (sub <= smlnum) break;
                double tst = std::fabs(h(k - 1, k - 1)) + std::fabs(h(k, k));
                if (tst == 0.0) {
                    if (k - 2 >= 0) tst += std::fabs(h(k - 1, k - 2));
                    if (k + 1 <= n - 1) tst += std::fabs(h(k + 1, k));
                }
                if (sub <= ulp * tst) {
                    const double ab = std::max(sub, std::fabs(h(k - 1, k)));
                    const double ba = std::min(sub, std::fabs(h(k - 1, k)));
                    const double diff = std::fabs(h(k - 1, k - 1) - h(k, k));
                    const double aa = std::max(std::fabs(h(k, k)), diff);
                    const double bb = std::min(std::fabs(h(k, k)), diff);
                    const double s = aa + ab;
                    if (ba * (ab / s) <= std::max(smlnum, ulp * (bb * (aa / s)))) break;
                }
            }
            l = k;
            if (l > 0) h(l, l - 1) = 0.0;
            if (l >= i - 1) {
                done = true;
                break;
            }
            ++kdefl;
            double h11, h12, h21, h22;
            if (kdefl % (2 * kExceptional) == 0) {
                const double s = std::fabs(h(i, i - 1)) + std::fabs(h(i - 1, i - 2));
                h11 = 0.75 * s + h(i, i);
                h12 = -0.4375 * s;
                h21 = s;
                h22 = h11;
            } else if (kdefl % kExceptional == 0) {
                const double s = std::fabs(h(l + 1, l)) + std::fabs(h(l + 2, l + 1));
                h11 = 0.75 * s + h(l, l);
                h12 = -0.4375 * s;
                h21 = s;
                h22 = h11;
            } else {
                h11 = h(i - 1, i - 1);
                h21 = h(i, i - 1);
                h12 = h(i - 1, i);
                h22 = h(i, i);
            }
            double r1r = 0, r1i = 0, r2r = 0, r2i = 0;
            const double s = std::fabs(h11) + std::fabs(h12) + std::fabs(h21) + std::fabs(h22);
            if (s != 0.0) {
                h11 /= s; h21 /= s; h12 /= s; h22 /= s;
                const double tr = 0.5 * (h11 + h22);
                const double det = (h11 - tr) * (h22 - tr) - h12 * h21;
                const double rt = std::sqrt(std::fabs(det));
                if (det >= 0.0) {
                    r1r = r2r = tr * s;
                    r1i = rt * s;
                    r2i = -r1i;
                } else {  // two real shifts: use the one closer to h22 twice
                    r1r = tr + rt;
                    r2r = tr - rt;
                    if (std::fabs(r1r - h22) <= std::fabs(r2r - h22)) {
                        r1r *= s;
                        r2r = r1r;
                    } else {
                        r2r *= s;
                        r1r = r2r;
                    }
                    r1i = r2i = 0.0;
                }
            }
            // start of the bulge: two consecutive small subdiagonals
            int m;
            double v[3];
            for (m = i - 2; m >= l; --m) {
                double hs = h(m + 1, m);
                double sc = std::fabs(h(m, m) - r2r) + std::fabs(r2i) + std::fabs(hs);
                hs = h(m + 1, m) / sc;
                v[0] = hs * h(m, m + 1) + (h(m, m) - r1r) * ((h(m, m) - r2r) / sc) - r1i * (r2i / sc);
                v[1] = hs * (h(m, m) + h(m + 1, m + 1) - r1r - r2r);
                v[2] = hs * h(m + 2, m + 1);
                sc = std::fabs(v[0]) + std::fabs(v[1]) + std::fabs(v[2]);
                v[0] /= sc; v[1] /= sc; v[2] /= sc;
                if (m == l) break;
                const double h00 = std::fabs(h(m, m - 1)) * (std::fabs(v[1]) + std::fabs(v[2]));
                const double h01 = std::fabs(v[0]) * (std::fabs(h(m - 1, m - 1)) + std::fabs(h(m, m)) +
                                                      std::fabs(h(m + 1, m + 1)));
                if (h00 <= ulp * h01) break;
            }
            for (int kk = m; kk <= i - 1; ++kk) {  // chase the bulge
                const int nr = std::min(3, i - kk + 1);
                if (kk > m)
                    for (int q = 0; q < nr; ++q) v[q] = h(kk + q, kk - 1);
                double t1;
                reflector(v[0], v + 1, nr - 1, t1);
                if (kk > m) {
                    h(kk, kk - 1) = v[0];
                    h(kk + 1, kk - 1) = 0.0;
                    if (kk < i - 1) h(kk + 2, kk - 1) = 0.0;
                } else if (m > l) {
                    h(kk, kk - 1) *= (1.0 - t1);
                }
                const double v2 = v[1], t2 = t1 * v2;
                if (nr == 3) {
                    const double v3 = v[2], t3 = t1 * v3;
                    for (int j = kk; j <= i; ++j) {
                        const double sum = h(kk, j) + v2 * h(kk + 1, j) + v3 * h(kk + 2, j);
                        h(kk, j) -= sum * t1;
                        h(kk + 1, j) -= sum * t2;
                        h(kk + 2, j) -= sum * t3;
                    }
                    for (int j = l; j <= std::min(kk + 3, i); ++j) {
                        const double sum = h(j, kk) + v2 * h(j, kk + 1) + v3 * h(j, kk + 2);
                        h(j, kk) -= sum * t1;
                        h(j, kk + 1) -= sum * t2;
                        h(j, kk + 2) -= sum * t3;
                    }
                } else {
                    for (int j = kk; j <= i; ++j) {
                        const double sum = h(kk, j) + v2 * h(kk + 1, j);
                        h(kk, j) -= sum * t1;
                        h(kk + 1, j) -= sum * t2;
                    }
                    for (int j = l; j <= i; ++j) {
                        const double sum = h(j, kk) + v2 * h(j, kk + 1);
                        h(j, kk) -= sum * t1;
                        h(j, kk + 1) -= sum * t2;
                    }
                }
            }
        }
        if (!done) return false;
        if (l == i) {
            ev[i] = {h(i, i), 0.0};
        } else {  // l == i - 1
            schur2(h(i - 1, i - 1), h(i - 1, i), h(i, i - 1), h(i, i), ev[i - 1], ev[i]);
        }
        kdefl = 0;
        i = l - 1;
    }
    return true;
}

}  // namespace fdsb::eig
