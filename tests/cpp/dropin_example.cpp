// A reference-shaped C++ caller of the B200 solve path through include/fracprec_b200.hpp:
// the same sequence the reference driver runs per Newton step (driver.cpp:229-255):
// build the preconditioner, wrap J and M^-1 as LinearOperators, solve with GMRES.
// Built by tests/test_cpp_dropin.py; run on a GPU it prints one "OK ..." line.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "fracprec_b200.hpp"
#include "fracprec_workload.h"

int main() {
  using namespace fracprec_b200;
  fp_fracture_spec frac{0, 0.5, 0.0, 1.0, 0.0, 1.0};
  fp_workload_spec spec{};
  spec.cells[0] = spec.cells[1] = spec.cells[2] = 6;
  spec.length[0] = spec.length[1] = spec.length[2] = 1.0;
  spec.n_fractures = 1;
  spec.fractures = &frac;
  spec.E_median = 10e9;
  spec.nu = 0.25;
  spec.frac_stick = 0.6;
  spec.frac_slip = 0.3;
  spec.aperture_median = 1e-4;
  spec.seed = 7;
  fp_workload* w = nullptr;
  check(fp_workload_preset(0, 0, &w) == FP_INVALID_ARGUMENT ? FP_OK : FP_INTERNAL_ERROR);  // ids are 1..5
  check(fp_workload_custom(&spec, &w));
  fp_block_system J{};
  check(fp_workload_system(w, &J));
  const double* xyz = nullptr;
  int32_t n_nodes = 0;
  check(fp_workload_coords(w, &xyz, &n_nodes));
  std::vector<std::array<double, 3>> coords(static_cast<size_t>(n_nodes));
  for (int v = 0; v < n_nodes; ++v) coords[v] = {xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]};
  if (std::getenv("FRACPREC_B200_COMPILE_ONLY")) {
    fp_workload_destroy(w);
    std::printf("OK compile-only n=%d\n", J.n_u + J.n_t + J.n_p);
    return 0;
  }
  GpuSystemOperator Jop(J);
  GpuPrecondOperator* M = build(Jop, J, FP_TUP, default_amg(), coords);
  std::mt19937 rng(42);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> b(static_cast<size_t>(Jop.dimension()));
  for (double& v : b) v = U(rng);
  M->reset_count();
  const std::vector<double> z = (*M)(b);
  const long calls = M->call_count();  // 2 inner V-cycles per t-u-p apply (test_precond.cpp:323-343)
  auto [x, st] = gmres(Jop, *M, b, 1e-10, 300, 50, true);
  // true residual of the unscaled system is not what GMRES minimized; check the scaled one via J
  double st_, sp_;
  check(fp_block_scaling(Jop.handle(), &st_, &sp_));
  std::printf("OK n=%d inner_calls=%ld iters=%d converged=%d final=%.3e ||z||=%.3e\n", Jop.dimension(), calls,
              st.iterations, int(st.converged), st.relative_residuals.empty() ? 0.0 : st.relative_residuals.back(),
              std::sqrt([&] { double s = 0; for (double v : z) s += v * v; return s; }()));
  delete M;
  fp_workload_destroy(w);
  return (calls == 2 && st.converged) ? 0 : 1;
}
