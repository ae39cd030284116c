// BEM assembly data structures (device side) — see bem_assembly.cu.
#pragma once

#include <vector>

#include "common.cuh"

namespace fdsb {

constexpr int kFarThreads = 128;
constexpr int kFarChunk = 64;

// Kernel-function constants (passed by value as a kernel parameter).
struct BemParams {
    static constexpr int kTerms = 16;
    static constexpr double kSeriesR2 = 0.09;  // |z| < 0.3 -> Taylor branch
    static constexpr int kSelfGauss = 10;
    double mu, lambda, lam_over_mu, cs, inv_cs, k, inv_k, inv_4pi_mu;
    double E10, E20;  // static (z=0) values of C-B and (λ/μ)(C-D-2B)-2B
    double ta[kTerms], tb[kTerms], tc[kTerms], td[kTerms];
    double r7l[7][3], r7w[7];
    double glx[kSelfGauss], glw[kSelfGauss];
};

BemParams make_bem_params(double mu, double nu, double rho);

// Device-resident mesh + assembly workspace of one BEM handle.
struct BemDevice {
    int ne = 0;
    BemParams params;
    double* geo = nullptr;    // [ne][16]: v0 v1 v2 c n area
    double* trac = nullptr;   // [ne][3]
    int* pairs = nullptr;     // [npairs][3]: c, e, level (-1 = self)
    int* near_ptr = nullptr;  // [ne+1] CSR by c into pairs
    int* order = nullptr;     // [npairs] near-kernel processing order (costliest first)
    int npairs = 0;
    cplx* partial = nullptr;  // [B][nchunks][3ne]
    size_t pstride = 0;
    cplx* corr = nullptr;     // [B][npairs][3]
    size_t cstride = 0;
};

// Host-side geometry preprocessing (same formulas as oracle/bem_oracle.cpp).
void bem_build_geometry(const double* verts, int nv, const int* tris, int ne,
                        std::vector<double>& geo, std::vector<int>& pairs,
                        std::vector<int>& near_ptr);
int bem_subdivision_level(double d, double h);

void bem_assemble(const BemDevice& d, const cplx* svec_dev, int B, double* A, size_t mstride,
                  size_t plane, int ld, cplx* rhs, size_t rstride, cudaStream_t st);

}  // namespace fdsb
