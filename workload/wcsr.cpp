// CSR container shared with the solve library (wcsr.hpp).
#include "wcsr.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace fpb {

namespace {
void need(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}
}  // namespace

Csr Csr::identity(int n) {
  Csr I(n, n);
  I.ci.resize(static_cast<size_t>(n));
  I.v.assign(static_cast<size_t>(n), 1.0);
  for (int i = 0; i < n; ++i) I.ci[i] = i, I.rp[i + 1] = i + 1;
  return I;
}

// from_triplets (csr.cpp:60-90): duplicates summed from 0.0; (row, col) order made stable (the
// reference's std::sort is not), so equal keys keep their insertion order.
Csr Csr::from_triplets(int rows, int cols, std::vector<Triplet> t) {
  for (const Triplet& e : t)
    need(e.row >= 0 && e.row < rows && e.col >= 0 && e.col < cols, "from_triplets: entry out of range");
  std::stable_sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  Csr A(rows, cols);
  A.ci.reserve(t.size());
  A.v.reserve(t.size());
  size_t i = 0;
  for (int r = 0; r < rows; ++r) {
    while (i < t.size() && t[i].row == r) {
      const int c = t[i].col;
      double s = 0.0;
      for (; i < t.size() && t[i].row == r && t[i].col == c; ++i) s += t[i].value;
      A.ci.push_back(c);
      A.v.push_back(s);
    }
    A.rp[r + 1] = int64_t(A.ci.size());
  }
  return A;
}

std::vector<double> Csr::to_dense() const {
  std::vector<double> D(static_cast<size_t>(n_rows) * n_cols, 0.0);
  for (int i = 0; i < n_rows; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) D[size_t(i) * n_cols + ci[k]] = v[k];
  return D;
}

Csr csr_add(const Csr& A, const Csr& B, double alpha, double beta) {
  need(A.n_rows == B.n_rows && A.n_cols == B.n_cols, "csr_add: shape mismatch");
  Csr C(A.n_rows, A.n_cols);
  C.ci.reserve(size_t(A.nnz() + B.nnz()));
  C.v.reserve(size_t(A.nnz() + B.nnz()));
  for (int i = 0; i < A.n_rows; ++i) {
    int64_t ka = A.rp[i], ea = A.rp[i + 1], kb = B.rp[i], eb = B.rp[i + 1];
    while (ka < ea || kb < eb) {
      const int ca = ka < ea ? A.ci[ka] : A.n_cols;
      const int cb = kb < eb ? B.ci[kb] : B.n_cols;
      if (ca < cb) {
        C.ci.push_back(ca);
        C.v.push_back(alpha * A.v[ka++]);
      } else if (cb < ca) {
        C.ci.push_back(cb);
        C.v.push_back(beta * B.v[kb++]);
      } else {
        C.ci.push_back(ca);
        const double va = alpha * A.v[ka++];
        const double vb = beta * B.v[kb++];
        C.v.push_back(va + vb);
      }
    }
    C.rp[i + 1] = int64_t(C.ci.size());
  }
  return C;
}

void HostSystem::check_shapes() const {
  auto expect = [](const Csr& M, int r, int c, const char* name) {
    if (M.n_rows != r || M.n_cols != c)
      throw std::invalid_argument(std::string("BlockSystem: bad shape for block ") + name);
  };
  expect(A, n_u, n_u, "A");
  expect(C1, n_u, n_t, "C1");
  expect(Q1, n_u, n_p, "Q1");
  expect(C2, n_t, n_u, "C2");
  expect(H, n_t, n_t, "H");
  expect(Q2, n_p, n_u, "Q2");
  expect(T, n_p, n_p, "T");
  if (F_u.n_rows > 0) expect(F_u, n_p, n_u, "F_u");
  if (n_t != 3 * n_p) throw std::invalid_argument("BlockSystem: n_t must equal 3*n_p");
}

}  // namespace fpb
