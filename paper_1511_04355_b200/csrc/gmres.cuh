// Restarted GMRES on a dense device-resident complex system (SURVEY.md §8f row
// f4: iterative solves for large N, where one O(N²) matrix–vector product per
// iteration costs far less than the O(N³) LU).
#pragma once

#include "common.cuh"

namespace fdsb {

struct GmresParams {
    double tol = 1e-12;  // stop at ||b - A x|| <= tol ||b||
    int restart = 60;    // Krylov dimension per cycle
    int max_iter = 1000;
};

struct GmresStats {
    int iterations = 0;
    double rel_residual = 0.0;  // true residual of the returned x
};

struct GmresWorkspace {
    double* V = nullptr;        // [restart+1][n] complex Krylov basis (interleaved)
    double* w = nullptr;        // [n] complex
    double* z = nullptr;        // [n] complex (preconditioned vector)
    double* pinv = nullptr;     // [n/3][3][3] complex block-Jacobi inverse
    double* partial = nullptr;  // reduction scratch
    double* h_dev = nullptr;    // [restart+2] complex
    double* bsave = nullptr;    // [n] complex right-hand side
    size_t n_cap = 0;
    int m_cap = 0;
    void ensure(int n, int m);
    void release();
    ~GmresWorkspace() { release(); }
};

// A: planar (re plane, im plane) column-major, leading dimension ld. b is
// overwritten with x (initial guess 0). Right block-Jacobi preconditioning with
// the 3x3 diagonal blocks (one per element, DOF-major u[3e+i]); n % 3 == 0.
// Deterministic: every reduction has a fixed order, so equal inputs give
// bit-identical x.
GmresStats gmres_solve(const double* Are, const double* Aim, int n, int ld, cplx* b, const GmresParams& p,
                       GmresWorkspace& ws, cudaStream_t st);

}  // namespace fdsb
