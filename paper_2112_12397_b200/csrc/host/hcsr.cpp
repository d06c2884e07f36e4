// Host sparse kernels (setup path).  Row-parallel with OpenMP; each row keeps the
// reference's left-to-right accumulation order (/root/reference/proj/core/src/csr.cpp).
#include "hcsr.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>

namespace fpb {

namespace {

void need(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

// Builds a CSR matrix row-parallel: fn(row, scratch, cols, vals) appends the
// entries of `row`.  Rows are processed in chunks; chunk results are stitched
// in row order, so the output does not depend on the thread schedule.
template <class Scratch, class MakeScratch, class RowFn>
Csr build_rows(int n_rows, int n_cols, MakeScratch make_scratch, RowFn fn) {
  constexpr int kChunk = 2048;
  const int n_chunks = (n_rows + kChunk - 1) / kChunk;
  struct Piece {
    std::vector<int> cols;
    std::vector<double> vals;
    std::vector<int64_t> counts;
  };
  std::vector<Piece> pieces(static_cast<size_t>(n_chunks));
  const int n_threads = omp_get_max_threads();
  std::vector<std::unique_ptr<Scratch>> scratch(static_cast<size_t>(n_threads));
#pragma omp parallel
  {
    const int tid = omp_get_thread_num();
    scratch[tid] = make_scratch();
#pragma omp for schedule(dynamic, 1)
    for (int c = 0; c < n_chunks; ++c) {
      Piece& p = pieces[c];
      const int r0 = c * kChunk, r1 = std::min(n_rows, r0 + kChunk);
      p.counts.resize(static_cast<size_t>(r1 - r0));
      for (int r = r0; r < r1; ++r) {
        const size_t before = p.cols.size();
        fn(r, *scratch[tid], p.cols, p.vals);
        p.counts[r - r0] = int64_t(p.cols.size() - before);
      }
    }
  }
  Csr C(n_rows, n_cols);
  std::vector<int64_t> chunk_off(static_cast<size_t>(n_chunks) + 1, 0);
  for (int c = 0; c < n_chunks; ++c) {
    chunk_off[c + 1] = chunk_off[c] + int64_t(pieces[c].cols.size());
    int64_t acc = chunk_off[c];
    for (size_t q = 0; q < pieces[c].counts.size(); ++q) {
      acc += pieces[c].counts[q];
      C.rp[size_t(c) * kChunk + q + 1] = acc;
    }
  }
  const size_t nnz = static_cast<size_t>(chunk_off[n_chunks]);
  if (nnz * (sizeof(int) + sizeof(double)) <= (size_t(8) << 30)) {
    // up to 8 GB of output: copy the pieces in parallel (transiently pieces + output)
    C.ci.resize(nnz);
    C.v.resize(nnz);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < n_chunks; ++c) {
      std::copy(pieces[c].cols.begin(), pieces[c].cols.end(), C.ci.begin() + chunk_off[c]);
      std::copy(pieces[c].vals.begin(), pieces[c].vals.end(), C.v.begin() + chunk_off[c]);
      std::vector<int>().swap(pieces[c].cols);
      std::vector<double>().swap(pieces[c].vals);
    }
    return C;
  }
  // larger (config 5): append chunk by chunk into reserved (untouched) storage, releasing
  // each piece right after, so the peak is one output plus one piece instead of two outputs
  C.ci.reserve(nnz);
  C.v.reserve(nnz);
  for (int c = 0; c < n_chunks; ++c) {
    C.ci.insert(C.ci.end(), pieces[c].cols.begin(), pieces[c].cols.end());
    C.v.insert(C.v.end(), pieces[c].vals.begin(), pieces[c].vals.end());
    std::vector<int>().swap(pieces[c].cols);
    std::vector<double>().swap(pieces[c].vals);
  }
  return C;
}

struct NoScratch {};

}  // namespace

std::vector<double> spmv(const Csr& A, std::span<const double> x) {
  need(int64_t(x.size()) == A.n_cols, "spmv: dimension mismatch");
  std::vector<double> y(static_cast<size_t>(A.n_rows));
#pragma omp parallel for schedule(static)
  for (int i = 0; i < A.n_rows; ++i) {
    double s = 0.0;
    for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) s += A.v[k] * x[A.ci[k]];
    y[i] = s;
  }
  return y;
}

// Counting transpose; row j of A^T lists the source rows in ascending order,
// which is the order the reference's scatter SpMV^T accumulates in.
Csr transpose(const Csr& A) {
  Csr T(A.n_cols, A.n_rows);
  const int nt = omp_get_max_threads();
  const int n = A.n_rows;
  std::vector<std::vector<int64_t>> cnt(static_cast<size_t>(nt));
  std::vector<int> r0(static_cast<size_t>(nt) + 1);
  for (int t = 0; t <= nt; ++t) r0[t] = int(int64_t(n) * t / nt);
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    cnt[t].assign(static_cast<size_t>(A.n_cols), 0);
    for (int i = r0[t]; i < r0[t + 1]; ++i)
      for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) ++cnt[t][A.ci[k]];
  }
  // T.rp and per-thread start offsets within each column
  std::vector<int64_t> col_total(static_cast<size_t>(A.n_cols), 0);
  for (int t = 0; t < nt; ++t)
    for (int j = 0; j < A.n_cols; ++j) col_total[j] += cnt[t][j];
  for (int j = 0; j < A.n_cols; ++j) T.rp[j + 1] = T.rp[j] + col_total[j];
  for (int j = 0; j < A.n_cols; ++j) {
    int64_t pos = T.rp[j];
    for (int t = 0; t < nt; ++t) {
      const int64_t c = cnt[t][j];
      cnt[t][j] = pos;
      pos += c;
    }
  }
  T.ci.resize(A.ci.size());
  T.v.resize(A.v.size());
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    std::vector<int64_t>& next = cnt[t];
    for (int i = r0[t]; i < r0[t + 1]; ++i)
      for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
        const int64_t p = next[A.ci[k]]++;
        T.ci[p] = i;
        T.v[p] = A.v[k];
      }
  }
  return T;
}

// Row-by-row Gustavson product with a dense accumulator (csr.cpp:149-179).
Csr spgemm(const Csr& A, const Csr& B, std::span<const double> row_scale) {
  need(A.n_cols == B.n_rows, "spgemm: dimension mismatch");
  need(row_scale.empty() || int64_t(row_scale.size()) == A.n_rows, "spgemm: row scale length mismatch");
  const bool scaled = !row_scale.empty();
  struct Acc {
    std::vector<double> acc;
    std::vector<char> seen;
    std::vector<int> touched;
  };
  const int nc = B.n_cols;
  return build_rows<Acc>(
      A.n_rows, B.n_cols,
      [nc] {
        auto s = std::make_unique<Acc>();
        s->acc.assign(static_cast<size_t>(nc), 0.0);
        s->seen.assign(static_cast<size_t>(nc), 0);
        return s;
      },
      [&](int i, Acc& s, std::vector<int>& cols, std::vector<double>& vals) {
        s.touched.clear();
        for (int64_t ka = A.rp[i]; ka < A.rp[i + 1]; ++ka) {
          const int k = A.ci[ka];
          // scaled: the entries of scale_rows(A, row_scale), rounded the same way, without the copy
          const double av = scaled ? A.v[ka] * row_scale[i] : A.v[ka];
          for (int64_t kb = B.rp[k]; kb < B.rp[k + 1]; ++kb) {
            const int j = B.ci[kb];
            if (!s.seen[j]) {
              s.seen[j] = 1;
              s.acc[j] = 0.0;
              s.touched.push_back(j);
            }
            s.acc[j] += av * B.v[kb];
          }
        }
        std::sort(s.touched.begin(), s.touched.end());
        for (int j : s.touched) {
          cols.push_back(j);
          vals.push_back(s.acc[j]);
          s.seen[j] = 0;
        }
      });
}

// Union pattern, explicit zeros kept (csr.cpp:181-206).
Csr add_scaled(const Csr& A, const Csr& B, double alpha, double beta) {
  need(A.n_rows == B.n_rows && A.n_cols == B.n_cols, "add_scaled: shape mismatch");
  return build_rows<NoScratch>(
      A.n_rows, A.n_cols, [] { return std::make_unique<NoScratch>(); },
      [&](int i, NoScratch&, std::vector<int>& cols, std::vector<double>& vals) {
        int64_t ka = A.rp[i], ea = A.rp[i + 1], kb = B.rp[i], eb = B.rp[i + 1];
        while (ka < ea || kb < eb) {
          const int ca = ka < ea ? A.ci[ka] : A.n_cols;
          const int cb = kb < eb ? B.ci[kb] : B.n_cols;
          if (ca < cb) {
            cols.push_back(ca);
            vals.push_back(alpha * A.v[ka++]);
          } else if (cb < ca) {
            cols.push_back(cb);
            vals.push_back(beta * B.v[kb++]);
          } else {
            cols.push_back(ca);
            const double va = alpha * A.v[ka++];
            const double vb = beta * B.v[kb++];
            vals.push_back(va + vb);
          }
        }
      });
}

Csr scale_rows(const Csr& A, std::span<const double> s) {
  need(int64_t(s.size()) == A.n_rows, "scale_rows: dimension mismatch");
  Csr C = A;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < A.n_rows; ++i)
    for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) C.v[k] *= s[i];
  return C;
}

std::vector<double> diag_extract(const Csr& A) {
  need(A.n_rows == A.n_cols, "diag_extract: matrix must be square");
  std::vector<double> d(static_cast<size_t>(A.n_rows), 0.0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < A.n_rows; ++i)
    for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
      if (A.ci[k] == i) d[i] = A.v[k];
  return d;
}

std::vector<double> restrict_dense(const Csr& A, std::span<const int> idx) {
  const size_t m = idx.size();
  std::vector<double> M(m * m, 0.0);
  for (size_t i = 0; i < m; ++i) {
    int64_t k = A.rp[idx[i]], e = A.rp[idx[i] + 1];
    for (size_t j = 0; j < m && k < e;) {
      if (A.ci[k] < idx[j]) ++k;
      else if (A.ci[k] > idx[j]) ++j;
      else M[i * m + j] = A.v[k++], ++j;
    }
  }
  return M;
}

bool lu3_factor(double m[9], int piv[3]) {
  piv[0] = 0, piv[1] = 1, piv[2] = 2;
  double scale = 0.0;
  for (int i = 0; i < 9; ++i) scale = std::max(scale, std::abs(m[i]));
  if (scale == 0.0) return false;
  for (int c = 0; c < 3; ++c) {
    int p = c;
    for (int r = c + 1; r < 3; ++r)
      if (std::abs(m[3 * r + c]) > std::abs(m[3 * p + c])) p = r;
    if (p != c) {
      for (int j = 0; j < 3; ++j) std::swap(m[3 * c + j], m[3 * p + j]);
      std::swap(piv[c], piv[p]);
    }
    if (std::abs(m[3 * c + c]) <= 1e-300 * scale || m[3 * c + c] == 0.0) return false;
    for (int r = c + 1; r < 3; ++r) {
      const double f = m[3 * r + c] / m[3 * c + c];
      m[3 * r + c] = f;
      for (int j = c + 1; j < 3; ++j) m[3 * r + j] -= f * m[3 * c + j];
    }
  }
  return true;
}

void lu3_solve(const double m[9], const int piv[3], const double b[3], double x[3]) {
  double y[3];
  for (int i = 0; i < 3; ++i) {
    y[i] = b[piv[i]];
    for (int j = 0; j < i; ++j) y[i] -= m[3 * i + j] * y[j];
  }
  for (int i = 2; i >= 0; --i) {
    x[i] = y[i];
    for (int j = i + 1; j < 3; ++j) x[i] -= m[3 * i + j] * x[j];
    x[i] /= m[3 * i + i];
  }
}

std::vector<double> bdiag3_extract(const Csr& H, double delta) {
  need(H.n_rows == H.n_cols && H.n_rows % 3 == 0, "bdiag3_extract: bad shape");
  const int nb = H.n_rows / 3;
  std::vector<double> B(9 * size_t(nb), 0.0);
#pragma omp parallel for schedule(static)
  for (int b = 0; b < nb; ++b) {
    double* blk = B.data() + 9 * size_t(b);
    for (int li = 0; li < 3; ++li) {
      const int i = 3 * b + li;
      for (int64_t k = H.rp[i]; k < H.rp[i + 1]; ++k)
        if (H.ci[k] / 3 == b) blk[3 * li + (H.ci[k] % 3)] = H.v[k];
    }
    const double dmax = std::max({std::abs(blk[0]), std::abs(blk[4]), std::abs(blk[8])});
    const double shift = delta * std::max(dmax, 1.0);
    for (int li = 0; li < 3; ++li)
      if (blk[4 * li] == 0.0) blk[4 * li] = shift;
  }
  return B;
}

Csr bdiag3_inverse_csr(const std::vector<double>& blocks) {
  const int nb = int(blocks.size() / 9);
  Csr A(3 * nb, 3 * nb);
  A.ci.resize(9 * size_t(nb));
  A.v.resize(9 * size_t(nb));
  for (int r = 0; r < 3 * nb; ++r) A.rp[r + 1] = 3 * int64_t(r + 1);
  bool bad = false;
  int bad_at = -1;
#pragma omp parallel for schedule(static)
  for (int b = 0; b < nb; ++b) {
    double lu[9];
    std::copy(blocks.begin() + 9 * size_t(b), blocks.begin() + 9 * size_t(b) + 9, lu);
    int piv[3];
    if (!lu3_factor(lu, piv)) {
#pragma omp critical
      {
        if (!bad || b < bad_at) bad_at = b;
        bad = true;
      }
      continue;
    }
    double inv[9];
    for (int c = 0; c < 3; ++c) {
      double e[3] = {0, 0, 0}, col[3];
      e[c] = 1.0;
      lu3_solve(lu, piv, e, col);
      for (int r = 0; r < 3; ++r) inv[3 * r + c] = col[r];
    }
    for (int li = 0; li < 3; ++li)
      for (int lj = 0; lj < 3; ++lj) {
        A.ci[9 * size_t(b) + 3 * li + lj] = 3 * b + lj;
        A.v[9 * size_t(b) + 3 * li + lj] = inv[3 * li + lj];
      }
  }
  if (bad) throw numerical_error("bdiag3_inverse_csr: singular 3x3 block at index " + std::to_string(bad_at));
  return A;
}

void FullPivLU::compute(std::vector<double> a, int nn) {
  n = nn;
  lu = std::move(a);
  prow.resize(static_cast<size_t>(n));
  pcol.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) prow[i] = pcol[i] = i;
  double maxpivot = 0.0;
  int nonzero = n;
  for (int k = 0; k < n; ++k) {
    int pi = k, pj = k;
    double best = -1.0;
    for (int i = k; i < n; ++i)
      for (int j = k; j < n; ++j) {
        const double v = std::abs(lu[size_t(i) * n + j]);
        if (v > best) best = v, pi = i, pj = j;
      }
    if (best == 0.0) {
      nonzero = k;
      break;
    }
    if (k == 0) maxpivot = best;
    if (pi != k) {
      for (int j = 0; j < n; ++j) std::swap(lu[size_t(k) * n + j], lu[size_t(pi) * n + j]);
      std::swap(prow[k], prow[pi]);
    }
    if (pj != k) {
      for (int i = 0; i < n; ++i) std::swap(lu[size_t(i) * n + k], lu[size_t(i) * n + pj]);
      std::swap(pcol[k], pcol[pj]);
    }
    const double piv = lu[size_t(k) * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double f = lu[size_t(i) * n + k] / piv;
      lu[size_t(i) * n + k] = f;
      for (int j = k + 1; j < n; ++j) lu[size_t(i) * n + j] -= f * lu[size_t(k) * n + j];
    }
  }
  const double thr = double(n) * std::numeric_limits<double>::epsilon() * maxpivot;
  rank = 0;
  for (int k = 0; k < nonzero; ++k)
    if (std::abs(lu[size_t(k) * n + k]) > thr) ++rank;
}

std::vector<double> FullPivLU::solve(std::span<const double> b) const {
  std::vector<double> c(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) c[i] = b[prow[i]];
  for (int j = 0; j < n; ++j) {
    const double cj = c[j];
    for (int i = j + 1; i < n; ++i) c[i] -= lu[size_t(i) * n + j] * cj;
  }
  for (int j = rank - 1; j >= 0; --j) {
    const double xj = c[j] / lu[size_t(j) * n + j];
    c[j] = xj;
    for (int i = 0; i < j; ++i) c[i] -= lu[size_t(i) * n + j] * xj;
  }
  std::vector<double> x(static_cast<size_t>(n), 0.0);
  for (int i = 0; i < rank; ++i) x[pcol[i]] = c[i];
  return x;
}

}  // namespace fpb
