// Host eigenvalue step of relocate_poles (vecfit.cpp:324, Eigen::EigenSolver in
// the reference). See eig_host.cpp.
#pragma once

#include <complex>
#include <vector>

namespace fdsb::eig {

// Eigenvalues of the real n x n matrix (column-major) in the diagonal order of
// its real Schur form; a complex pair occupies consecutive slots, +imag first,
// exactly conjugate; real eigenvalues have an exactly zero imaginary part.
// Returns false if the iteration does not converge.
bool eigenvalues(int n, const double* colmajor, std::vector<std::complex<double>>& ev);

}  // namespace fdsb::eig
