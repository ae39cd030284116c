// Restarted GMRES on a dense device-resident complex system (SURVEY.md §8f row
// f4: iterative solves for large N, where one O(N²) matrix–vector product per
// iteration costs far less than the O(N³) LU).
#pragma once

#include <vector>

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
    bool converged = false;
};

struct GmresWorkspace {
    double* V = nullptr;        // [B][restart+1][n] complex Krylov bases (interleaved)
    double* w = nullptr;        // [B][n] complex
    double* z = nullptr;        // [B][n] complex (preconditioned vector)
    double* pinv = nullptr;     // [B][n/3][3][3] complex block-Jacobi inverses
    double* partial = nullptr;  // reduction scratch
    double* h_dev = nullptr;    // [B][restart+2] complex
    double* bsave = nullptr;    // [B][n] complex right-hand sides
    double* scal = nullptr;     // [B] scale factors
    int* act = nullptr;         // [B] active system indices
    // pinned host staging for the per-step H2D copies (truly asynchronous):
    // active list, two coefficient slots, scale factors
    int* pin_act = nullptr;
    double* pin_coef[2] = {nullptr, nullptr};
    double* pin_scal = nullptr;
    size_t n_cap = 0;
    int m_cap = 0, b_cap = 0;
    void ensure(int n, int m, int B);
    void release();
    ~GmresWorkspace() { release(); }
};

// B systems A_b (planar: re plane at A + b*mstride, im plane at +plane,
// column-major, leading dimension ld); rhs_b at rhs + b*rstride is overwritten
// with x_b (initial guess 0). Right block-Jacobi preconditioning with the 3x3
// diagonal blocks (one per element, DOF-major u[3e+i]); n % 3 == 0. The systems
// iterate in lockstep, each leaving the Arnoldi loop at its own tolerance.
// Deterministic: every reduction has a fixed order, so equal inputs give
// bit-identical x. A system that misses tol within max_iter is reported with
// converged = false (its original right-hand side stays in ws.bsave).
std::vector<GmresStats> gmres_solve_batch(const double* A, size_t mstride, size_t plane, int n, int ld, int B,
                                          cplx* rhs, size_t rstride, const GmresParams& p, GmresWorkspace& ws,
                                          cudaStream_t st);
// One system: A's planes at Are / Aim (Aim = Are + plane).
GmresStats gmres_solve(const double* Are, const double* Aim, int n, int ld, cplx* b, const GmresParams& p,
                       GmresWorkspace& ws, cudaStream_t st);

}  // namespace fdsb
