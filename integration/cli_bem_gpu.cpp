// "bem" systems of the fdsweep_b200 CLI on the B200 library: one device
// handle per system (fds_bem_create), contour batches through
// fds_bem_evaluate_batch (batched assembly + LU + solve).
#include "cli_bem.hpp"
#include "fdsweep_b200_shim.hpp"

namespace fdsweep::cli {

std::unique_ptr<FrequencySystem> make_bem_system(const BemSpec& spec) {
    b200::BemMesh m;
    m.vertices = spec.vertices;
    m.triangles = spec.triangles;
    m.shear_modulus = spec.shear_modulus;
    m.poisson_ratio = spec.poisson_ratio;
    m.density = spec.density;
    m.traction = spec.traction;
    m.channels = spec.channels;
    auto sys = std::make_unique<b200::BemSystem>(m);
    if (spec.solver == "gmres") sys->set_solver(true, spec.tol, spec.restart, spec.max_iter);
    return sys;
}

std::vector<std::vector<Complex>> evaluate_many(const FrequencySystem& system, std::span<const Complex> s) {
    if (const auto* bem = dynamic_cast<const b200::BemSystem*>(&system)) return bem->evaluate_batch(s);
    std::vector<std::vector<Complex>> out;
    out.reserve(s.size());
    for (const Complex z : s) out.push_back(system.evaluate(z));
    return out;
}

const char* solver_name() { return "b200"; }

std::optional<AfsResult> run_afs_native(const FrequencySystem& system, const AfsConfig& cfg) {
    if (const auto* bem = dynamic_cast<const b200::BemSystem*>(&system)) return b200::run_afs_bem(*bem, cfg);
    return std::nullopt;
}

}  // namespace fdsweep::cli
