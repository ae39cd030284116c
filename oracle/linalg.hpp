// ORACLE — test infrastructure only. Never linked into the product library.
//
// Dense real linear algebra used by the CPU restatement of the reference's
// vector fitting (proj/src/vecfit.cpp). The reference delegates these to
// Eigen3 (>= 3.3, unpinned; proj/CMakeLists.txt:13), which is absent from this
// image, so the published algorithms are restated here:
//   * HouseholderQR            — vecfit.cpp:265 (Eigen::HouseholderQR)
//   * ColPivHouseholderQR      — vecfit.cpp:281, :389 (Eigen::ColPivHouseholderQR,
//                                 norm-downdating pivoting, rank threshold
//                                 |R_ii| > min(m,n)*eps*max|R_kk|)
//   * real eigenvalues         — vecfit.cpp:324 (Eigen::EigenSolver): Householder
//                                 Hessenberg reduction + Francis double-shift QR
//                                 (SPEC.md:191), eigenvalues read off the real
//                                 Schur form in diagonal order.
// Matrices are column-major std::vector<double> with explicit row count.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <stdexcept>
#include <vector>

namespace oracle {

struct Mat {
    int rows = 0, cols = 0;
    std::vector<double> a;  // column-major
    Mat() = default;
    Mat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
    double& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
    double operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
    const double* ptr(int i, int j) const { return &a[static_cast<size_t>(j) * rows + i]; }
};

// Householder vector for x[0..n): H x = beta e0, H = I - tau v v^T, v[0] = 1.
// Sign convention beta = -sign(x0) ||x|| (the one Eigen's makeHouseholder uses).
inline void make_householder(double* x, int n, double& tau, double& beta) {
    double tail = 0.0;
    for (int i = 1; i < n; ++i) tail += x[i] * x[i];
    const double c0 = x[0];
    if (tail <= std::numeric_limits<double>::min()) {
        tau = 0.0;
        beta = c0;
        for (int i = 1; i < n; ++i) x[i] = 0.0;
        return;
    }
    beta = std::sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    const double inv = 1.0 / (c0 - beta);
    for (int i = 1; i < n; ++i) x[i] *= inv;
    tau = (beta - c0) / beta;
}

// Apply H = I - tau v v^T (v[0]=1, v[1..n) = ess) to vector y[0..n).
inline void apply_householder(const double* ess, int n, double tau, double* y) {
    if (tau == 0.0) return;
    double d = y[0];
    for (int i = 1; i < n; ++i) d += ess[i] * y[i];
    d *= tau;
    y[0] -= d;
    for (int i = 1; i < n; ++i) y[i] -= d * ess[i];
}

// Unpivoted Householder QR in place: R in the upper triangle, reflectors below.
struct HouseholderQR {
    Mat qr;
    std::vector<double> tau;
    explicit HouseholderQR(Mat a) : qr(std::move(a)) {
        const int m = qr.rows, n = qr.cols, size = std::min(m, n);
        tau.assign(size, 0.0);
        for (int k = 0; k < size; ++k) {
            double beta;
            double* col = &qr(k, k);
            make_householder(col, m - k, tau[k], beta);
            col[0] = beta;
            for (int j = k + 1; j < n; ++j) apply_householder(col, m - k, tau[k], &qr(k, j));
        }
    }
    // y <- Q^T y
    void apply_qt(std::vector<double>& y) const {
        const int m = qr.rows;
        for (int k = 0; k < static_cast<int>(tau.size()); ++k) {
            apply_householder(qr.ptr(k, k), m - k, tau[k], &y[k]);
        }
    }
};

// Column-pivoted Householder QR with Eigen's norm-downdating pivot rule and
// rank determination.
struct ColPivQR {
    Mat qr;
    std::vector<double> tau;
    std::vector<int> perm;  // perm[i] = original column at position i
    int nonzero_pivots = 0;
    double maxpivot = 0.0;

    explicit ColPivQR(Mat a) : qr(std::move(a)) {
        const int m = qr.rows, n = qr.cols, size = std::min(m, n);
        const double eps = std::numeric_limits<double>::epsilon();
        tau.assign(size, 0.0);
        perm.resize(n);
        for (int j = 0; j < n; ++j) perm[j] = j;
        std::vector<double> upd(n), dir(n);
        double maxcol = 0.0;
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = 0; i < m; ++i) s += qr(i, j) * qr(i, j);
            upd[j] = dir[j] = std::sqrt(s);
            maxcol = std::max(maxcol, dir[j]);
        }
        const double thr_helper = (maxcol * eps) * (maxcol * eps) / m;
        const double downdate_thr = std::sqrt(eps);
        nonzero_pivots = size;
        maxpivot = 0.0;
        for (int k = 0; k < size; ++k) {
            int big = k;
            for (int j = k + 1; j < n; ++j) if (upd[j] > upd[big]) big = j;
            const double big_sq = upd[big] * upd[big];
            if (nonzero_pivots == size && big_sq < thr_helper * (m - k)) nonzero_pivots = k;
            if (big != k) {
                for (int i = 0; i < m; ++i) std::swap(qr(i, k), qr(i, big));
                std::swap(upd[k], upd[big]);
                std::swap(dir[k], dir[big]);
                std::swap(perm[k], perm[big]);
            }
            double beta;
            double* col = &qr(k, k);
            make_householder(col, m - k, tau[k], beta);
            col[0] = beta;
            maxpivot = std::max(maxpivot, std::abs(beta));
            for (int j = k + 1; j < n; ++j) apply_householder(col, m - k, tau[k], &qr(k, j));
            for (int j = k + 1; j < n; ++j) {
                if (upd[j] != 0.0) {
                    double t = std::abs(qr(k, j)) / upd[j];
                    t = (1.0 + t) * (1.0 - t);
                    if (t < 0.0) t = 0.0;
                    const double r = upd[j] / dir[j];
                    const double t2 = t * r * r;
                    if (t2 <= downdate_thr) {
                        double s = 0.0;
                        for (int i = k + 1; i < m; ++i) s += qr(i, j) * qr(i, j);
                        dir[j] = upd[j] = std::sqrt(s);
                    } else {
                        upd[j] *= std::sqrt(t);
                    }
                }
            }
        }
    }
    int rank() const {
        const double thr = std::min(qr.rows, qr.cols) * std::numeric_limits<double>::epsilon();
        const double pre = std::abs(maxpivot) * thr;
        int r = 0;
        for (int i = 0; i < nonzero_pivots; ++i) r += std::abs(qr(i, i)) > pre;
        return r;
    }
    std::vector<double> solve(std::vector<double> b) const {
        const int n = qr.cols, np = nonzero_pivots, m = qr.rows;
        std::vector<double> x(n, 0.0);
        if (np == 0) return x;
        for (int k = 0; k < np; ++k) apply_householder(qr.ptr(k, k), m - k, tau[k], &b[k]);
        for (int i = np - 1; i >= 0; --i) {
            double s = b[i];
            for (int j = i + 1; j < np; ++j) s -= qr(i, j) * b[j];
            b[i] = s / qr(i, i);
        }
        for (int i = 0; i < np; ++i) x[perm[i]] = b[i];
        return x;
    }
};

// Eigenvalues of a real square matrix: Householder reduction to upper
// Hessenberg form, then the Francis implicit double-shift QR iteration with
// exceptional shifts at iterations 10 and 30 (EISPACK hqr). Returns false if
// an eigenvalue fails to converge in 30*n iterations. Eigenvalues are
// returned in diagonal order of the final quasi-triangular form; a complex
// pair occupies consecutive slots with the +imag member first.
inline bool real_eigenvalues(Mat h, std::vector<std::complex<double>>& ev) {
    const int n = h.rows;
    ev.assign(n, {0.0, 0.0});
    // Hessenberg reduction.
    std::vector<double> v(n);
    for (int k = 0; k + 2 < n; ++k) {
        const int len = n - k - 1;
        for (int i = 0; i < len; ++i) v[i] = h(k + 1 + i, k);
        double tau, beta;
        make_householder(v.data(), len, tau, beta);
        if (tau == 0.0) continue;
        // H <- P H P with P = I - tau u u^T acting on rows/cols k+1..n-1.
        for (int j = 0; j < n; ++j) {  // left: rows
            double d = h(k + 1, j);
            for (int i = 1; i < len; ++i) d += v[i] * h(k + 1 + i, j);
            d *= tau;
            h(k + 1, j) -= d;
            for (int i = 1; i < len; ++i) h(k + 1 + i, j) -= d * v[i];
        }
        for (int i = 0; i < n; ++i) {  // right: cols
            double d = h(i, k + 1);
            for (int c = 1; c < len; ++c) d += v[c] * h(i, k + 1 + c);
            d *= tau;
            h(i, k + 1) -= d;
            for (int c = 1; c < len; ++c) h(i, k + 1 + c) -= d * v[c];
        }
        for (int i = k + 2; i < n; ++i) h(i, k) = 0.0;
    }
    // Francis double-shift QR (EISPACK hqr, 0-based).
    double anorm = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::abs(h(i, j));
    int nn = n - 1;
    double t = 0.0;
    const double eps = std::numeric_limits<double>::epsilon();
    while (nn >= 0) {
        int its = 0, l;
        do {
            for (l = nn; l >= 1; --l) {
                const double s = std::abs(h(l - 1, l - 1)) + std::abs(h(l, l));
                const double ss = (s == 0.0) ? anorm : s;
                if (std::abs(h(l, l - 1)) <= eps * ss) {
                    h(l, l - 1) = 0.0;
                    break;
                }
            }
            const double x = h(nn, nn);
            if (l == nn) {
                ev[nn] = {x + t, 0.0};
                --nn;
            } else {
                const double y = h(nn - 1, nn - 1);
                const double w = h(nn, nn - 1) * h(nn - 1, nn);
                if (l == nn - 1) {
                    const double p = 0.5 * (y - x);
                    const double q = p * p + w;
                    const double z = std::sqrt(std::abs(q));
                    const double xx = x + t;
                    if (q >= 0.0) {
                        const double zz = p + (p >= 0.0 ? std::abs(z) : -std::abs(z));
                        double a1 = xx + zz, a2 = a1;
                        if (zz != 0.0) a2 = xx - w / zz;
                        // real pair: keep diagonal order (upper slot gets the
                        // root closer to h(nn-1,nn-1)-side as hqr does)
                        ev[nn - 1] = {a1, 0.0};
                        ev[nn] = {a2, 0.0};
                    } else {
                        ev[nn - 1] = {xx + p, z};
                        ev[nn] = {xx + p, -z};
                    }
                    nn -= 2;
                } else {
                    if (its == 30 * std::max(n, 1)) return false;
                    double xs = x, ys = y, ws = w;
                    if (its == 10 || its == 20) {
                        t += xs;
                        for (int i = 0; i <= nn; ++i) h(i, i) -= xs;
                        const double s = std::abs(h(nn, nn - 1)) + std::abs(h(nn - 1, nn - 2));
                        xs = ys = 0.75 * s;
                        ws = -0.4375 * s * s;
                    }
                    ++its;
                    int m;
                    double p = 0, q = 0, r = 0, z;
                    for (m = nn - 2; m >= l; --m) {
                        z = h(m, m);
                        r = xs - z;
                        const double s2 = ys - z;
                        p = (r * s2 - ws) / h(m + 1, m) + h(m, m + 1);
                        q = h(m + 1, m + 1) - z - r - s2;
                        r = h(m + 2, m + 1);
                        const double s = std::abs(p) + std::abs(q) + std::abs(r);
                        p /= s; q /= s; r /= s;
                        if (m == l) break;
                        const double u = std::abs(h(m, m - 1)) * (std::abs(q) + std::abs(r));
                        const double vv = std::abs(p) * (std::abs(h(m - 1, m - 1)) + std::abs(z) +
                                                         std::abs(h(m + 1, m + 1)));
                        if (u <= eps * vv) break;
                    }
                    for (int i = m + 2; i <= nn; ++i) {
                        h(i, i - 2) = 0.0;
                        if (i != m + 2) h(i, i - 3) = 0.0;
                    }
                    for (int k = m; k <= nn - 1; ++k) {
                        double xx = 0.0;
                        if (k != m) {
                            p = h(k, k - 1);
                            q = h(k + 1, k - 1);
                            r = (k != nn - 1) ? h(k + 2, k - 1) : 0.0;
                            xx = std::abs(p) + std::abs(q) + std::abs(r);
                            if (xx != 0.0) { p /= xx; q /= xx; r /= xx; }
                        }
                        const double s = std::copysign(std::sqrt(p * p + q * q + r * r), p);
                        if (s == 0.0) continue;
                        if (k == m) {
                            if (l != m) h(k, k - 1) = -h(k, k - 1);
                        } else {
                            h(k, k - 1) = -s * xx;
                        }
                        p += s;
                        const double xk = p / s, yk = q / s, zk = r / s;
                        q /= p;
                        r /= p;
                        for (int j = k; j <= nn; ++j) {
                            double pp = h(k, j) + q * h(k + 1, j);
                            if (k != nn - 1) { pp += r * h(k + 2, j); h(k + 2, j) -= pp * zk; }
                            h(k + 1, j) -= pp * yk;
                            h(k, j) -= pp * xk;
                        }
                        const int mmin = nn < k + 3 ? nn : k + 3;
                        for (int i = l; i <= mmin; ++i) {
                            double pp = xk * h(i, k) + yk * h(i, k + 1);
                            if (k != nn - 1) { pp += zk * h(i, k + 2); h(i, k + 2) -= pp * r; }
                            h(i, k + 1) -= pp * q;
                            h(i, k) -= pp;
                        }
                    }
                }
            }
        } while (nn >= 0 && l < nn - 1);
    }
    return true;
}

// Inputs of the last relocate_poles call's stacked sigma least squares and
// companion eigenproblem (test hook: lets tests/test_oracle_crosscheck.py run
// the same systems through LAPACK). Not thread-safe; tests call it serially.
struct RelocCapture {
    Mat stacked;               // K*red x M (vecfit.cpp:281)
    std::vector<double> rhs;   // K*red
    Mat h;                     // M x M (vecfit.cpp:324), valid when has_h
    bool has_h = false;
};
inline RelocCapture& reloc_capture() {
    static RelocCapture c;
    return c;
}

}  // namespace oracle
