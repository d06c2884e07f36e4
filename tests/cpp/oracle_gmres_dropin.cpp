// Drop-in at the LinearOperator level (operator.hpp:17-28): the B200 operators are
// instantiated over the oracle's restatement of fracprec::LinearOperator (fpo::LinearOperator, a
// line-for-line image of the reference interface), and the oracle's restated reference gmres()
// (gmres.cpp:24-174) drives fp_system_apply / fp_precond_apply through the C ABI, exactly as the
// reference driver would once GpuSystemOperatorT<fracprec::LinearOperator> replaces its operators
// (driver.cpp:233-253).  TEST INFRASTRUCTURE: links the oracle as the driver, never the product path.
//
// Prints one line "OK iters_cpu_gmres=<k> iters_abi_gmres=<k'> ..." and exits 0 when the Krylov loop
// over the GPU applies converges and agrees with the C ABI's own fp_gmres (full GMRES, MGS).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../oracle/fpo.hpp"
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
  // J and M^-1 as subclasses of the (restated) reference interface
  GpuSystemOperatorT<fpo::LinearOperator> Jop(J);
  GpuPrecondOperatorT<fpo::LinearOperator>* M = build<fpo::LinearOperator>(Jop, J, FP_TUP, default_amg(), coords);
  const fpo::LinearOperator& Jbase = Jop;  // what the reference's gmres() sees
  const fpo::LinearOperator* Mbase = M;

  std::mt19937 rng(42);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> b(static_cast<size_t>(Jop.dimension()));
  for (double& v : b) v = U(rng);

  // the driver's scaled system (driver.cpp:229-255): D J D y = b with D^-1 M D^-1
  double st_ = 1.0, sp_ = 1.0;
  check(fp_block_scaling(Jop.handle(), &st_, &sp_));
  fpo::BlockScaling D{st_, sp_, J.n_u, J.n_t, J.n_p};
  fpo::ScaledOperator Js(Jbase, D, false), Ms(*Mbase, D, true);
  auto [y, st] = fpo::gmres(Js, &Ms, b, 1e-10, 300);

  // the same full GMRES through the C ABI (restart = max_iter, MGS: the reference's loop on the device)
  auto [y_abi, st_abi] = gmres(Jop, *M, b, 1e-10, 300, 300, true, FP_ORTH_MGS);
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < y.size(); ++i) {
    num += (y[i] - y_abi[i]) * (y[i] - y_abi[i]);
    den += y[i] * y[i];
  }
  const double rel = std::sqrt(num / den);
  // a wrong-length span is rejected like the reference's dimension checks
  bool threw = false;
  try {
    std::vector<double> shortv(3), out(3);
    Jop.apply(shortv, out);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  std::printf("OK iters_cpu_gmres=%d iters_abi_gmres=%d converged=%d/%d solution_rel=%.3e dim_check=%d\n",
              st.iterations, st_abi.iterations, int(st.converged), int(st_abi.converged), rel, int(threw));
  delete M;
  fp_workload_destroy(w);
  const bool ok = st.converged && st_abi.converged && std::abs(st.iterations - st_abi.iterations) <= 2 &&
                  rel <= 1e-8 && threw;
  return ok ? 0 : 1;
}
