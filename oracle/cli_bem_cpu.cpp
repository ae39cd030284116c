// ORACLE — test infrastructure only. The "bem" system of the CPU reference CLI
// (oracle/_ref/fdsweep_oracle_cli, same main as the product CLI,
// integration/fdsweep_cli.cpp): oracle assembly (OpenMP) and, when
// FDSWEEP_ORACLE_OPENBLAS names scipy's OpenBLAS, zgetrf/zgetrs; otherwise the
// oracle's own partial-pivot LU. Frequencies are solved one at a time.
#include <cstdlib>

#include "bem_oracle.hpp"
#include "cli_bem.hpp"

extern "C" int orc_bem_solve_openblas(void* h, const char* openblas_path, double sr, double si, double* u_out,
                                      double* t_out);
extern "C" const char* orc_last_error(void);

namespace fdsweep::cli {
namespace {

class OracleBemSystem : public FrequencySystem {
  public:
    explicit OracleBemSystem(const BemSpec& b)
        : bem_(b.vertices, b.triangles, b.shear_modulus, b.poisson_ratio, b.density, b.traction),
          channels_(b.channels) {
        const int n = 3 * bem_.elements();
        if (channels_.empty())
            for (int k = 0; k < n; ++k) channels_.push_back(k);
        for (int k : channels_) {
            if (k < 0 || k >= n) throw ValidationError("bem: channel index out of range");
            desc_.channel_labels.push_back("u" + std::to_string(k));
        }
        desc_.channel_count = static_cast<int>(channels_.size());
    }
    const SystemDescriptor& descriptor() const override { return desc_; }
    std::vector<Complex> evaluate(Complex s) const override {
        const int n = 3 * bem_.elements();
        std::vector<Complex> u;
        if (const char* ob = std::getenv("FDSWEEP_ORACLE_OPENBLAS")) {
            u.resize(n);
            if (orc_bem_solve_openblas(const_cast<oracle::BemOracle*>(&bem_), ob, s.real(), s.imag(),
                                       reinterpret_cast<double*>(u.data()), nullptr) != 0)
                throw NumericError(orc_last_error());
        } else {
            u = bem_.solve(s);
        }
        std::vector<Complex> out;
        out.reserve(channels_.size());
        for (int k : channels_) out.push_back(u[k]);
        return out;
    }

  private:
    oracle::BemOracle bem_;
    std::vector<int> channels_;
    SystemDescriptor desc_;
};

}  // namespace

std::unique_ptr<FrequencySystem> make_bem_system(const BemSpec& spec) {
    return std::make_unique<OracleBemSystem>(spec);
}

std::vector<std::vector<Complex>> evaluate_many(const FrequencySystem& system, std::span<const Complex> s) {
    std::vector<std::vector<Complex>> out;
    out.reserve(s.size());
    for (const Complex z : s) out.push_back(system.evaluate(z));
    return out;
}

const char* solver_name() { return "cpu-oracle"; }

std::optional<AfsResult> run_afs_native(const FrequencySystem&, const AfsConfig&) { return std::nullopt; }

}  // namespace fdsweep::cli
