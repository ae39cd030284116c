// ORACLE — test infrastructure only. See bem_oracle.cpp for the formulation.
#pragma once

#include <complex>
#include <vector>

namespace oracle {

struct KernelCoeffs {
    static constexpr int kTerms = 16;
    static constexpr double kSeriesRadius = 0.3;
    double mu, lambda, cs, cp, k, lam_over_mu;
    double ta[kTerms], tb[kTerms], tc[kTerms], td[kTerms];
    KernelCoeffs(double mu, double nu, double rho);
    void abcd(std::complex<double> z, std::complex<double>& A, std::complex<double>& B,
              std::complex<double>& C, std::complex<double>& D) const;
    void ut(const double rv[3], const double n[3], std::complex<double> s,
            std::complex<double> U[9], std::complex<double> T[9]) const;
};

int subdivision_level(double d, double h);
int lu_factor(int n, std::vector<std::complex<double>>& A, std::vector<int>& piv);
void lu_solve(int n, const std::vector<std::complex<double>>& A, const std::vector<int>& piv,
              std::vector<std::complex<double>>& b);

class BemOracle {
  public:
    static constexpr int kSelfGauss = 10;
    BemOracle(const std::vector<double>& vertices, const std::vector<int>& tris, double mu,
              double nu, double rho, const std::vector<double>& traction);
    int elements() const { return ne_; }
    void assemble(std::complex<double> s, std::vector<std::complex<double>>& A,
                  std::vector<std::complex<double>>& b) const;
    std::vector<std::complex<double>> solve(std::complex<double> s) const;
    void self_block(int e, std::complex<double> s, std::complex<double> U[9],
                    std::complex<double> T[9]) const;
    // Single entries at full-size configs (same arithmetic as assemble()).
    void block(int c, int e, std::complex<double> s, std::complex<double> U[9], std::complex<double> T[9]) const;
    std::complex<double> entry(int row, int col, std::complex<double> s) const;
    std::complex<double> rhs(int row, std::complex<double> s) const;
    const KernelCoeffs& coeffs() const { return kc_; }

  private:
    KernelCoeffs kc_;
    std::vector<double> traction_;
    std::vector<double> glx_, glw_;  // self-element Gauss–Legendre rule on [0,1]
    std::vector<double> geo_;  // per element: v0,v1,v2 (9), centroid (3), normal (3), area
    int ne_ = 0;
};

}  // namespace oracle
