// Host dense kernels for the VF driver (see host_linalg.h).
#include "host_linalg.h"

#include <algorithm>
#include <cmath>
#include <limits>

namespace fdsb::hla {

namespace {

constexpr double kEps = std::numeric_limits<double>::epsilon();

// Reflector H = I - tau v v^T (v0 = 1) with H x = beta e0, beta = -sign(x0)||x||.
void reflector(double* x, int len, double& tau, double& beta) {
    double sig = 0.0;
    for (int i = 1; i < len; ++i) sig += x[i] * x[i];
    const double x0 = x[0];
    if (sig <= std::numeric_limits<double>::min()) {
        tau = 0.0;
        beta = x0;
        for (int i = 1; i < len; ++i) x[i] = 0.0;
        return;
    }
    const double nrm = std::sqrt(x0 * x0 + sig);
    beta = x0 >= 0.0 ? -nrm : nrm;
    const double s = 1.0 / (x0 - beta);
    for (int i = 1; i < len; ++i) x[i] *= s;
    tau = (beta - x0) / beta;
}

void reflect(const double* v, int len, double tau, double* y) {
    if (tau == 0.0) return;
    double d = y[0];
    for (int i = 1; i < len; ++i) d += v[i] * y[i];
    d *= tau;
    y[0] -= d;
    for (int i = 1; i < len; ++i) y[i] -= d * v[i];
}

}  // namespace

PivotedQR::PivotedQR(Dense a) : qr(std::move(a)) {
    const int m = qr.m, n = qr.n, r = std::min(m, n);
    tau.assign(r, 0.0);
    perm.resize(n);
    std::vector<double> cur(n), ref(n);
    double big0 = 0.0;
    for (int j = 0; j < n; ++j) {
        perm[j] = j;
        double s = 0.0;
        for (int i = 0; i < m; ++i) s += qr.at(i, j) * qr.at(i, j);
        cur[j] = ref[j] = std::sqrt(s);
        big0 = std::max(big0, cur[j]);
    }
    const double floor_sq = (big0 * kEps) * (big0 * kEps) / m;
    const double refresh = std::sqrt(kEps);
    nonzero = r;
    for (int k = 0; k < r; ++k) {
        const int p = static_cast<int>(std::max_element(cur.begin() + k, cur.end()) - cur.begin());
        if (nonzero == r && cur[p] * cur[p] < floor_sq * (m - k)) nonzero = k;
        if (p != k) {
            std::swap_ranges(qr.col(k), qr.col(k) + m, qr.col(p));
            std::swap(cur[k], cur[p]);
            std::swap(ref[k], ref[p]);
            std::swap(perm[k], perm[p]);
        }
        double beta;
        reflector(qr.col(k) + k, m - k, tau[k], beta);
        qr.at(k, k) = beta;
        maxpivot = std::max(maxpivot, std::abs(beta));
        for (int j = k + 1; j < n; ++j) reflect(qr.col(k) + k, m - k, tau[k], qr.col(j) + k);
        for (int j = k + 1; j < n; ++j) {
            if (cur[j] == 0.0) continue;
            double t = std::abs(qr.at(k, j)) / cur[j];
            t = std::max(0.0, (1.0 + t) * (1.0 - t));
            const double q = cur[j] / ref[j];
            if (t * q * q <= refresh) {
                double s = 0.0;
                for (int i = k + 1; i < m; ++i) s += qr.at(i, j) * qr.at(i, j);
                cur[j] = ref[j] = std::sqrt(s);
            } else {
                cur[j] *= std::sqrt(t);
            }
        }
    }
}

int PivotedQR::rank() const {
    const double thr = std::abs(maxpivot) * std::min(qr.m, qr.n) * kEps;
    int rk = 0;
    for (int i = 0; i < nonzero; ++i) rk += std::abs(qr.at(i, i)) > thr;
    return rk;
}

std::vector<double> PivotedQR::solve(std::vector<double> b) const {
    const int m = qr.m, n = qr.n;
    std::vector<double> x(n, 0.0);
    for (int k = 0; k < nonzero; ++k) reflect(qr.col(k) + k, m - k, tau[k], b.data() + k);
    for (int i = nonzero - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < nonzero; ++j) s -= qr.at(i, j) * b[j];
        b[i] = s / qr.at(i, i);
    }
    for (int i = 0; i < nonzero; ++i) x[perm[i]] = b[i];
    return x;
}

Dense PivotedQR::solve_operator() const {
    Dense W(qr.n, qr.m);
    std::vector<double> e(qr.m);
    for (int c = 0; c < qr.m; ++c) {
        std::fill(e.begin(), e.end(), 0.0);
        e[c] = 1.0;
        const std::vector<double> x = solve(e);
        for (int i = 0; i < qr.n; ++i) W.at(i, c) = x[i];
    }
    return W;
}

bool eigenvalues(Dense h, std::vector<std::complex<double>>& out) {
    const int n = h.n;
    out.assign(n, {0.0, 0.0});
    // Hessenberg form by Householder similarity transforms.
    std::vector<double> v(n);
    for (int k = 0; k + 2 < n; ++k) {
        const int len = n - k - 1;
        for (int i = 0; i < len; ++i) v[i] = h.at(k + 1 + i, k);
        double tau, beta;
        reflector(v.data(), len, tau, beta);
        if (tau == 0.0) continue;
        for (int j = 0; j < n; ++j) {
            double d = h.at(k + 1, j);
            for (int i = 1; i < len; ++i) d += v[i] * h.at(k + 1 + i, j);
            d *= tau;
            h.at(k + 1, j) -= d;
            for (int i = 1; i < len; ++i) h.at(k + 1 + i, j) -= d * v[i];
        }
        for (int i = 0; i < n; ++i) {
            double d = h.at(i, k + 1);
            for (int c = 1; c < len; ++c) d += v[c] * h.at(i, k + 1 + c);
            d *= tau;
            h.at(i, k + 1) -= d;
            for (int c = 1; c < len; ++c) h.at(i, k + 1 + c) -= d * v[c];
        }
        for (int i = k + 2; i < n; ++i) h.at(i, k) = 0.0;
    }
    double norm1 = 0.0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i <= std::min(j + 1, n - 1); ++i) norm1 += std::abs(h.at(i, j));
    // Francis implicit double-shift QR on the active window [lo, hi].
    int hi = n - 1;
    double shift_acc = 0.0;
    int iter = 0;
    while (hi >= 0) {
        int lo = hi;
        while (lo > 0) {
            double s = std::abs(h.at(lo - 1, lo - 1)) + std::abs(h.at(lo, lo));
            if (s == 0.0) s = norm1;
            if (std::abs(h.at(lo, lo - 1)) <= kEps * s) {
                h.at(lo, lo - 1) = 0.0;
                break;
            }
            --lo;
        }
        if (lo == hi) {  // 1x1 block converged
            out[hi] = {h.at(hi, hi) + shift_acc, 0.0};
            --hi;
            iter = 0;
            continue;
        }
        const double a = h.at(hi - 1, hi - 1), b = h.at(hi - 1, hi), c = h.at(hi, hi - 1), d = h.at(hi, hi);
        if (lo == hi - 1) {  // 2x2 block converged
            const double p = 0.5 * (a - d);
            const double q = p * p + b * c;
            const double z = std::sqrt(std::abs(q));
            if (q >= 0.0) {
                const double zz = p + (p >= 0.0 ? z : -z);
                out[hi - 1] = {d + zz + shift_acc, 0.0};
                out[hi] = {zz != 0.0 ? d - b * c / zz + shift_acc : d + zz + shift_acc, 0.0};
            } else {
                out[hi - 1] = {d + p + shift_acc, z};
                out[hi] = {d + p + shift_acc, -z};
            }
            hi -= 2;
            iter = 0;
            continue;
        }
        if (++iter > 30 * n) return false;
        double x = d, y = a, w = b * c;
        if (iter == 11 || iter == 21) {  // exceptional shift
            shift_acc += x;
            for (int i = 0; i <= hi; ++i) h.at(i, i) -= x;
            const double s = std::abs(h.at(hi, hi - 1)) + std::abs(h.at(hi - 1, hi - 2));
            x = y = 0.75 * s;
            w = -0.4375 * s * s;
        }
        // first column of (H - s1)(H - s2) restricted to the bulge start
        int m = hi - 2;
        double p = 0, q = 0, r = 0;
        for (; m >= lo; --m) {
            const double zz = h.at(m, m);
            const double rr = x - zz, ss = y - zz;
            p = (rr * ss - w) / h.at(m + 1, m) + h.at(m, m + 1);
            q = h.at(m + 1, m + 1) - zz - rr - ss;
            r = h.at(m + 2, m + 1);
            const double sc = std::abs(p) + std::abs(q) + std::abs(r);
            p /= sc; q /= sc; r /= sc;
            if (m == lo) break;
            const double u = std::abs(h.at(m, m - 1)) * (std::abs(q) + std::abs(r));
            const double vv = std::abs(p) * (std::abs(h.at(m - 1, m - 1)) + std::abs(zz) + std::abs(h.at(m + 1, m + 1)));
            if (u <= kEps * vv) break;
        }
        for (int i = m + 2; i <= hi; ++i) {
            h.at(i, i - 2) = 0.0;
            if (i != m + 2) h.at(i, i - 3) = 0.0;
        }
        for (int k = m; k <= hi - 1; ++k) {
            double sc = 0.0;
            if (k != m) {
                p = h.at(k, k - 1);
                q = h.at(k + 1, k - 1);
                r = k != hi - 1 ? h.at(k + 2, k - 1) : 0.0;
                sc = std::abs(p) + std::abs(q) + std::abs(r);
                if (sc != 0.0) { p /= sc; q /= sc; r /= sc; }
            }
            const double s = std::copysign(std::sqrt(p * p + q * q + r * r), p);
            if (s == 0.0) continue;
            if (k == m) {
                if (lo != m) h.at(k, k - 1) = -h.at(k, k - 1);
            } else {
                h.at(k, k - 1) = -s * sc;
            }
            p += s;
            const double xk = p / s, yk = q / s, zk = r / s;
            q /= p;
            r /= p;
            for (int j = k; j <= hi; ++j) {
                double t = h.at(k, j) + q * h.at(k + 1, j);
                if (k != hi - 1) { t += r * h.at(k + 2, j); h.at(k + 2, j) -= t * zk; }
                h.at(k + 1, j) -= t * yk;
                h.at(k, j) -= t * xk;
            }
            const int top = std::min(hi, k + 3);
            for (int i = lo; i <= top; ++i) {
                double t = xk * h.at(i, k) + yk * h.at(i, k + 1);
                if (k != hi - 1) { t += zk * h.at(i, k + 2); h.at(i, k + 2) -= t * r; }
                h.at(i, k + 1) -= t * q;
                h.at(i, k) -= t;
            }
        }
    }
    return true;
}

}  // namespace fdsb::hla
