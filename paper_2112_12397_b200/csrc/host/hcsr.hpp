// Host-side sparse containers and kernels of the B200 solve framework.
//
// These run on the host during preconditioner *setup* (not on the timed solve
// path).  Every row-local operation is parallelized over rows with OpenMP while
// keeping, inside each row, the exact accumulation order of the reference
// (/root/reference/proj/core/src/csr.cpp), so a setup built here is bitwise the
// one the reference algorithm produces.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "wcsr.hpp"

namespace fpb {

class numerical_error : public std::runtime_error {
 public:
  explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};

// Csr (csr.hpp:16-49 with 64-bit row offsets) is shared with the workload generator: wcsr.hpp

std::vector<double> spmv(const Csr& A, std::span<const double> x);
Csr transpose(const Csr& A);
// C = diag(row_scale) A B when row_scale is given (== spgemm(scale_rows(A, s), B) bitwise)
Csr spgemm(const Csr& A, const Csr& B, std::span<const double> row_scale = {});
Csr add_scaled(const Csr& A, const Csr& B, double alpha, double beta);
Csr scale_rows(const Csr& A, std::span<const double> s);
std::vector<double> diag_extract(const Csr& A);
std::vector<double> restrict_dense(const Csr& A, std::span<const int> idx);  // A(idx, idx), row-major

// 3x3 partial-pivot LU (csr.cpp:242-278)
bool lu3_factor(double m[9], int piv[3]);
void lu3_solve(const double m[9], const int piv[3], const double b[3], double x[3]);
// Block-diagonal surrogate H~ = Bdiag(H,3) with the 1e-10 shift (csr.cpp:216-237)
std::vector<double> bdiag3_extract(const Csr& H, double delta = 1e-10);
Csr bdiag3_inverse_csr(const std::vector<double>& blocks);

// Dense full-pivot LU: coarse AMG level and fixed-stress local solves.
struct FullPivLU {
  int n = 0, rank = 0;
  std::vector<double> lu;
  std::vector<int> prow, pcol;
  void compute(std::vector<double> a_rowmajor, int n);
  bool invertible() const { return rank == n; }
  std::vector<double> solve(std::span<const double> b) const;
};

// Banded exact factor (SparseFactor semantics), per independent diagonal block.
struct BandFactor {
  enum class Kind { spd, general };
  Kind kind = Kind::spd;
  int n = 0, kl = 0, ku = 0;
  std::vector<int> block_start;
  std::vector<double> Lc, diag, Lr, Uc;
  std::vector<int> piv;
  bool pivoted = false;  // general: any row swap (else the pivot path is skipped on the device)
  void factor(const Csr& A, Kind k);
  std::vector<double> solve(std::span<const double> b) const;  // host check path
  // Explicit inverse of every diagonal block (factor_solve = inverse), row-major,
  // block blk at off[blk]: column c = the sweep solve of e_c.  Zero pivots are
  // skipped, which changes at most the sign of zero entries (never a GEMV sum).
  void inverse_blocks(std::vector<double>& inv, std::vector<int64_t>& off) const;
};

}  // namespace fpb
