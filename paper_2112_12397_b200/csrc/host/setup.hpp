// Host-side preconditioner setup of the B200 solve framework: the work the
// reference does in build_tpu/build_tup/amg_setup
// (/root/reference/proj/core/src/precond.cpp:119-202, amg.cpp:181-291) before the
// solve.  It runs multi-threaded on the host and its output is uploaded to HBM
// (device.cuh).  Per-row/per-aggregate arithmetic follows the reference order so
// the hierarchy is the one the reference algorithm builds.
#pragma once

#include <array>
#include <memory>
#include <vector>

#include "hcsr.hpp"

namespace fpb {

struct AmgOptions {
  double strength_threshold = 0.08;  // amg.hpp:20
  int max_coarse = 100;
  int pre_sweeps = 1, post_sweeps = 1;
  int smoother = 0;  // 0 weighted Jacobi (GPU path), 1 symmetric Gauss-Seidel (reference default),
                     // 2 Chebyshev, 3 multicolour symmetric Gauss-Seidel (extensions, SURVEY §8(f)
                     // item 4; restated in oracle/amg.cpp)
  int chebyshev_degree = 2;
  double chebyshev_ratio = 10.0;
  int power_iterations = 10;
  bool prolongation_smoothing = true;
  int cycles_per_apply = 1;
  double jacobi_omega = 2.0 / 3.0;
  double stall_ratio = 0.9;
  int max_levels = 25;
  int row_sum = 0;  // 0 ordered (reference order), 1 strided32 on A_l (l >= 1) and R_l
};

// A level operator built by the device setup (csrc/device/dsetup.cu) stays in HBM: DeviceMatrix is
// its device CSR (defined in engine.cuh, opaque here).  Such a level's host A / P hold only their
// shapes; A_nnz / P_nnz give the entry counts and fp_host_precond_matrix downloads on request.
struct DeviceMatrix;

struct HostLevel {
  Csr A;
  Csr P;  // prolongation from this level to the previous finer one (empty at level 0)
  std::shared_ptr<DeviceMatrix> dA, dP;  // device-resident A / P (device setup), else null
  int64_t A_nnz = -1, P_nnz = -1;        // entry counts of device-resident matrices
  int64_t a_nnz() const { return dA ? A_nnz : A.nnz(); }
  int64_t p_nnz() const { return dP ? P_nnz : P.nnz(); }
  std::vector<double> diag;
  double lambda_max = 0.0;     // chebyshev: 1.1 x power-iteration estimate of rho(D^-1 A)
  std::vector<int> aggregate;  // fine row -> aggregate id (coarse levels only)
  std::vector<int> aggregate_offsets;
  std::vector<int> color_rows, color_off;  // smoother 3: rows grouped by colour (ascending in a colour)
};

struct HostAmg {
  std::vector<HostLevel> levels;
  FullPivLU coarse;
  AmgOptions opt;
};

// SpGEMM of the setup (Galerkin products, Schur cores): a registered backend (the device
// SpGEMM, csrc/device/spgemm.cu, bitwise this routine) or the host spgemm.  The backend may
// decline a product (returns false) and the host routine runs instead.
using SpgemmBackend = bool (*)(const Csr&, const Csr&, std::span<const double>, Csr&);
void set_spgemm_backend(SpgemmBackend fn);
bool spgemm_backend_active();
Csr spgemm_setup(const Csr& A, const Csr& B, std::span<const double> row_scale = {});

// Chebyshev smoother (extension): the oracle's chebyshev_lambda_max / chebyshev_coefficients
// (oracle/amg.cpp), computed with the same operation order so the GPU matches it bit for bit.
double chebyshev_lambda_max(const Csr& A, const std::vector<double>& diag, int iterations);
struct ChebyshevCoefficients {
  double theta = 0.0;
  std::vector<double> c1, c2;
};
ChebyshevCoefficients chebyshev_coefficients(double lambda_max, double ratio, int degree);

// Multicolour smoother (extension): the greedy colouring in row order of the pattern of A + A^T (each
// row takes the smallest colour none of its earlier neighbours has), rows grouped by colour — the
// oracle's greedy_coloring (oracle/amg.cpp) rule
void color_rows(int n, const int64_t* rp, const int* ci, std::vector<int>& rows, std::vector<int>& off);

// A is taken by value and moved into level 0 (callers std::move the inner operator in)
HostAmg amg_setup(Csr A, const std::vector<std::vector<double>>& near_null, const AmgOptions& opt);
std::vector<std::vector<double>> rigid_body_modes(const std::vector<std::array<double, 3>>& coords);
int qr_colpiv(int m, int k, const std::vector<double>& B_colmajor, std::vector<double>& Q, std::vector<double>& Rp);

// HostSystem (block.hpp:36-45) is shared with the workload generator: wcsr.hpp

enum Variant { kTpu = 0, kTup = 1, kTupStar = 2 };

struct HostPrecond {
  int variant = kTup;
  std::vector<double> hblocks;  // regularized H~ = Bdiag(H,3), 9 per face
  std::vector<double> T_diag;   // t-p-u
  // the inner AMG operator S~ (t-p-u) or S1 (t-u-p) is amg.levels[0].A
  const Csr& S() const { return amg.levels.front().A; }
  HostAmg amg;
  std::vector<double> S_K;      // t-u-p fixed-stress diagonal
  Csr S2;                       // t-u-p S~2 = T - diag(S_K)
  BandFactor factor;            // T (t-p-u, LDL^T) or S~2 (t-u-p, LU)
  int factor_solve = 0;         // 0 auto, 1 sweeps, 2 explicit block inverse
};

HostPrecond build_precond(const HostSystem& J, int variant, const AmgOptions& opt,
                          const std::vector<std::array<double, 3>>& coords);
std::vector<double> fixed_stress_diag(const Csr& Q2, const Csr& S1, const Csr& Q1);

}  // namespace fpb
