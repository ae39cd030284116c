// Small dense real factorizations executed on the host inside the VF driver:
// the per-fit shared least-squares matrix (<= 2J x M, J ~ 40-120) and the
// M x M relocation eigenproblem are latency-bound (microseconds) and are kept
// off the GPU by design. The per-channel /
// per-DOF work they feed runs in CUDA kernels (vf.cu).
//
// Semantics follow what the reference delegates to Eigen (vecfit.cpp:265,
// :281, :324, :389): Householder QR, column-pivoted QR with norm downdating
// and rank = #{|R_ii| > min(m,n) eps max|R_kk|}, real eigenvalues from a
// Hessenberg + Francis double-shift iteration.
#pragma once

#include <complex>
#include <vector>

namespace fdsb::hla {

// Column-major dense matrix.
struct Dense {
    int m = 0, n = 0;
    std::vector<double> v;
    Dense() = default;
    Dense(int rows, int cols) : m(rows), n(cols), v(static_cast<size_t>(rows) * cols, 0.0) {}
    double& at(int i, int j) { return v[static_cast<size_t>(j) * m + i]; }
    double at(int i, int j) const { return v[static_cast<size_t>(j) * m + i]; }
    double* col(int j) { return v.data() + static_cast<size_t>(j) * m; }
    const double* col(int j) const { return v.data() + static_cast<size_t>(j) * m; }
};

struct PivotedQR {
    Dense qr;                 // R above the diagonal, reflectors below
    std::vector<double> tau;
    std::vector<int> perm;    // column at position i
    int nonzero = 0;          // pivots before the remaining norm underflows
    double maxpivot = 0.0;
    explicit PivotedQR(Dense a);
    int rank() const;
    // least-squares solution of the factored system for rhs b (length m)
    std::vector<double> solve(std::vector<double> b) const;
    // W (n x m) with W b == solve(b): explicit pseudo-inverse of the full-rank system
    Dense solve_operator() const;
};

// Eigenvalues of a real square matrix (quasi-triangular diagonal order, a
// complex pair occupies consecutive slots with +imag first). false if the
// iteration did not converge.
bool eigenvalues(Dense a, std::vector<std::complex<double>>& out);

}  // namespace fdsb::hla
