// CSR container and block system shared by the workload generator (this directory, an input-side
// host library: libfp_workload.so) and the B200 solve library, which builds on the same types.
// Layout is the reference's CsrMatrix (csr.hpp:16-49) with 64-bit row offsets; BlockSystem is
// block.hpp:36-45.
#pragma once

#include <cstdint>
#include <vector>

namespace fpb {

struct Csr {
  int n_rows = 0, n_cols = 0;
  std::vector<int64_t> rp{0};
  std::vector<int> ci;
  std::vector<double> v;

  Csr() = default;
  Csr(int r, int c) : n_rows(r), n_cols(c), rp(static_cast<size_t>(r) + 1, 0) {}
  int64_t nnz() const { return int64_t(ci.size()); }
  int row_len(int i) const { return int(rp[i + 1] - rp[i]); }

  struct Triplet { int row, col; double value; };
  static Csr identity(int n);
  static Csr from_triplets(int rows, int cols, std::vector<Triplet> t);  // stable (row,col) order
  std::vector<double> to_dense() const;  // row-major, small matrices only
};

// alpha A + beta B on the union pattern, explicit zeros kept (csr.cpp:181-206)
Csr csr_add(const Csr& A, const Csr& B, double alpha, double beta);

struct HostSystem {
  int n_u = 0, n_t = 0, n_p = 0;
  Csr A, C1, Q1, C2, H, Q2, T, F_u;
  void check_shapes() const;
};

}  // namespace fpb
