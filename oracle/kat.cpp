// ORACLE known-answer tests (test infrastructure only).
// Re-expresses the reference's own unit tests for the solve path
// (/root/reference/proj/tests/unit/test_csr.cpp, test_gmres.cpp, test_amg.cpp,
// test_precond.cpp) and the SPEC.md examples against the restated oracle.
// Each case prints "PASS <name>" or "FAIL <name>: <detail>"; the process exits
// non-zero if any case failed.  Driven by tests/test_oracle_kat.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>

#include "fpo.hpp"

using namespace fpo;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;
bool g_case_failed = false;

void check(bool ok, const std::string& what) {
  ++g_checks;
  if (!ok && !g_case_failed) {
    std::printf("FAIL %s: %s\n", g_case.c_str(), what.c_str());
    g_case_failed = true;
  }
}
#define CHECK(c) check((c), #c)
template <class E, class F>
void check_throws(F&& f, const char* what) {
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
    check(false, std::string("wrong exception type: ") + what);
    return;
  }
  check(false, std::string("no exception: ") + what);
}
void run(const char* name, const std::function<void()>& body) {
  g_case = name;
  g_case_failed = false;
  try {
    body();
  } catch (const std::exception& e) {
    check(false, std::string("unexpected exception: ") + e.what());
  }
  if (g_case_failed)
    ++g_fail;
  else
    std::printf("PASS %s\n", name);
}
bool approx(double a, double b, double eps) {  // doctest::Approx semantics
  return std::abs(a - b) < eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

// ---------------------------------------------------------------- dense helpers
struct Dense {
  int r = 0, c = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int r_, int c_) : r(r_), c(c_), a(static_cast<size_t>(r_) * c_, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) * c + j]; }
  double operator()(int i, int j) const { return a[size_t(i) * c + j]; }
  static Dense of(const CsrMatrix& M) {
    Dense D(M.n_rows, M.n_cols);
    D.a = M.to_dense();
    return D;
  }
  static Dense eye(int n) {
    Dense D(n, n);
    for (int i = 0; i < n; ++i) D(i, i) = 1.0;
    return D;
  }
};
Dense operator*(const Dense& A, const Dense& B) {
  Dense C(A.r, B.c);
  for (int i = 0; i < A.r; ++i)
    for (int k = 0; k < A.c; ++k) {
      const double v = A(i, k);
      if (v == 0.0) continue;
      for (int j = 0; j < B.c; ++j) C(i, j) += v * B(k, j);
    }
  return C;
}
Dense operator+(Dense A, const Dense& B) {
  for (size_t i = 0; i < A.a.size(); ++i) A.a[i] += B.a[i];
  return A;
}
Dense operator-(Dense A, const Dense& B) {
  for (size_t i = 0; i < A.a.size(); ++i) A.a[i] -= B.a[i];
  return A;
}
Dense transpose(const Dense& A) {
  Dense T(A.c, A.r);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j) T(j, i) = A(i, j);
  return T;
}
double max_abs(const Dense& A) {
  double m = 0.0;
  for (double v : A.a) m = std::max(m, std::abs(v));
  return m;
}
double fro(const Dense& A) {
  double s = 0.0;
  for (double v : A.a) s += v * v;
  return std::sqrt(s);
}
// partial-pivot dense LU solve of A X = B (checker only)
Dense solve(Dense A, Dense B) {
  const int n = A.r;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(p, k))) p = i;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      for (int j = 0; j < B.c; ++j) std::swap(B(k, j), B(p, j));
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = A(i, k) / A(k, k);
      for (int j = k; j < n; ++j) A(i, j) -= f * A(k, j);
      for (int j = 0; j < B.c; ++j) B(i, j) -= f * B(k, j);
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < B.c; ++j) {
      double s = B(k, j);
      for (int q = k + 1; q < n; ++q) s -= A(k, q) * B(q, j);
      B(k, j) = s / A(k, k);
    }
  return B;
}
Dense inverse(const Dense& A) { return solve(A, Dense::eye(A.r)); }
Dense densify(const LinearOperator& op) {
  const int n = op.dimension();
  Dense M(n, n);
  std::vector<double> e(static_cast<size_t>(n), 0.0);
  for (int j = 0; j < n; ++j) {
    e[j] = 1.0;
    const auto col = op(e);
    e[j] = 0.0;
    for (int i = 0; i < n; ++i) M(i, j) = col[i];
  }
  return M;
}
Dense densify_fn(int n, const std::function<std::vector<double>(std::span<const double>)>& f) {
  return densify(FunctionOperator(n, f));
}
double col_norm_diff(const Dense& A, const Dense& B, int j, double* cn) {
  double d = 0.0, s = 0.0;
  for (int i = 0; i < A.r; ++i) {
    d += (A(i, j) - B(i, j)) * (A(i, j) - B(i, j));
    s += B(i, j) * B(i, j);
  }
  *cn = std::sqrt(s);
  return std::sqrt(d);
}
double vnorm(std::span<const double> v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

std::vector<double> random_vector(int n, std::mt19937& rng) {  // test_helpers.hpp:195-200
  std::uniform_real_distribution<double> val(-1.0, 1.0);
  std::vector<double> v(static_cast<size_t>(n));
  for (double& x : v) x = val(rng);
  return v;
}
CsrMatrix random_sparse(int rows, int cols, double density, std::mt19937& rng) {  // test_csr.cpp:16-24
  std::uniform_real_distribution<double> val(-1.0, 1.0), coin(0.0, 1.0);
  std::vector<CsrMatrix::Triplet> t;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j)
      if (coin(rng) < density) t.push_back({i, j, val(rng)});
  return CsrMatrix::from_triplets(rows, cols, std::move(t));
}
BlockVector random_block(const BlockSystem& J, std::mt19937& rng) {
  BlockVector w(J.n_u, J.n_t, J.n_p);
  w.u = random_vector(J.n_u, rng);
  w.t = random_vector(J.n_t, rng);
  w.p = random_vector(J.n_p, rng);
  return w;
}
Dense hs_dense(const HSurrogate& Hs, int n) {
  return densify_fn(n, [&](std::span<const double> v) { return Hs.solve(v); });
}

void csr_tests() {
  // test_csr.cpp:32-47
  run("spmv identity and zero", [] {
    const CsrMatrix I = CsrMatrix::identity(3);
    const std::vector<double> x{1, 2, 3};
    CHECK(spmv(I, x) == x);
    CHECK((spmv(CsrMatrix(2, 2), std::vector<double>{5, 7}) == std::vector<double>{0, 0}));
  });
  run("spmv dense row-by-row oracle", [] {
    const CsrMatrix A = CsrMatrix::from_triplets(2, 2, {{0, 0, 2.0}, {1, 0, 1.0}, {1, 1, 3.0}});
    CHECK((spmv(A, std::vector<double>{1, 1}) == std::vector<double>{2, 4}));
    check_throws<std::invalid_argument>([&] { spmv(A, std::vector<double>{1, 1, 1}); }, "spmv mismatch");
  });
  // test_csr.cpp:49-60
  run("spmv_transpose examples", [] {
    const std::vector<double> x{4, 5, 6};
    CHECK(spmv_transpose(CsrMatrix::identity(3), x) == x);
    const CsrMatrix A = CsrMatrix::from_triplets(2, 2, {{0, 0, 2.0}, {1, 0, 1.0}, {1, 1, 3.0}});
    CHECK((spmv_transpose(A, std::vector<double>{1, 1}) == std::vector<double>{3, 3}));
    const CsrMatrix col = CsrMatrix::from_triplets(2, 1, {{0, 0, 1.0}, {1, 0, 2.0}});
    CHECK((spmv_transpose(col, std::vector<double>{1, 1}) == std::vector<double>{3}));
    check_throws<std::invalid_argument>([&] { spmv_transpose(col, std::vector<double>{1}); }, "mismatch");
  });
  // test_csr.cpp:62-78
  run("spmv_transpose equals spmv of transpose", [] {
    std::mt19937 rng(42);
    for (int trial = 0; trial < 20; ++trial) {
      const int rows = 1 + int(rng() % 50), cols = 1 + int(rng() % 50);
      const CsrMatrix A = random_sparse(rows, cols, 0.2, rng);
      const CsrMatrix At = transpose(A);
      CHECK(max_abs(Dense::of(At) - transpose(Dense::of(A))) == 0.0);
      std::vector<double> x(static_cast<size_t>(rows));
      std::uniform_real_distribution<double> val(-1.0, 1.0);
      for (double& v : x) v = val(rng);
      const auto y1 = spmv_transpose(A, x), y2 = spmv(At, x);
      double d = 0.0;
      for (size_t i = 0; i < y1.size(); ++i) d += (y1[i] - y2[i]) * (y1[i] - y2[i]);
      CHECK(std::sqrt(d) <= 1e-14 * std::max(1.0, vnorm(y1)));
    }
  });
  // test_csr.cpp:80-115
  run("spgemm examples and dense oracle", [] {
    std::mt19937 rng(7);
    const CsrMatrix B = random_sparse(3, 3, 0.5, rng);
    CHECK(max_abs(Dense::of(spgemm(CsrMatrix::identity(3), B)) - Dense::of(B)) == 0.0);
    const CsrMatrix AZ = spgemm(B, CsrMatrix(3, 4));
    CHECK(AZ.nnz() == 0 && AZ.n_rows == 3 && AZ.n_cols == 4);
    const CsrMatrix A = random_sparse(3, 3, 0.5, rng);
    const Dense ref = Dense::of(A) * Dense::of(B);
    CHECK(max_abs(Dense::of(spgemm(A, B)) - ref) <= 1e-14 * std::max(1.0, max_abs(ref)));
    check_throws<std::invalid_argument>([&] { spgemm(A, CsrMatrix(4, 2)); }, "spgemm mismatch");
  });
  run("spgemm associativity", [] {
    std::mt19937 rng(2024);
    for (int trial = 0; trial < 10; ++trial) {
      const int n1 = 2 + int(rng() % 19), n2 = 2 + int(rng() % 19), n3 = 2 + int(rng() % 19), n4 = 2 + int(rng() % 19);
      const CsrMatrix A = random_sparse(n1, n2, 0.3, rng), B = random_sparse(n2, n3, 0.3, rng),
                      C = random_sparse(n3, n4, 0.3, rng);
      const Dense l = Dense::of(spgemm(spgemm(A, B), C)), r = Dense::of(spgemm(A, spgemm(B, C)));
      const double scale = fro(Dense::of(A)) * fro(Dense::of(B)) * fro(Dense::of(C));
      CHECK(fro(l - r) <= 1e-12 * std::max(1.0, scale));
    }
  });
  // test_csr.cpp:117-136
  run("add_scaled union pattern", [] {
    std::mt19937 rng(5);
    const CsrMatrix A = random_sparse(4, 4, 0.4, rng);
    const CsrMatrix AA = add_scaled(A, A, 1.0, -1.0);
    CHECK(AA.nnz() == A.nnz());
    for (double v : AA.values) CHECK(v == 0.0);
    const Dense two = Dense::of(add_scaled(A, CsrMatrix(4, 4), 2.0, 0.0));
    Dense ref = Dense::of(A);
    for (double& v : ref.a) v *= 2.0;
    CHECK(max_abs(two - ref) == 0.0);
    const CsrMatrix U = CsrMatrix::from_triplets(2, 2, {{0, 0, 1.0}}), V = CsrMatrix::from_triplets(2, 2, {{1, 1, 2.0}});
    const CsrMatrix W = add_scaled(U, V, 3.0, 4.0);
    CHECK(W.coeff(0, 0) == 3.0 && W.coeff(1, 1) == 8.0 && W.nnz() == 2);
    check_throws<std::invalid_argument>([&] { add_scaled(U, CsrMatrix(3, 2), 1.0, 1.0); }, "shape");
  });
  // test_csr.cpp:138-172
  run("bdiag3_extract slices diagonal blocks", [] {
    std::vector<CsrMatrix::Triplet> t;
    double v = 1.0;
    for (int b = 0; b < 2; ++b)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) t.push_back({3 * b + i, 3 * b + j, v += 1.0});
    const CsrMatrix H = CsrMatrix::from_triplets(6, 6, t);
    const BlockDiagonal3 D = bdiag3_extract(H);
    for (int b = 0; b < 2; ++b)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) CHECK(D.block(b)[3 * i + j] == H.coeff(3 * b + i, 3 * b + j));
    std::mt19937 rng(3);
    const CsrMatrix F = random_sparse(6, 6, 1.0, rng);
    const BlockDiagonal3 DF = bdiag3_extract(F);
    const Dense Fd = Dense::of(F);
    for (int b = 0; b < 2; ++b)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const double e = Fd(3 * b + i, 3 * b + j);
          if (i == j && e == 0.0) continue;
          CHECK(DF.block(b)[3 * i + j] == e);
        }
    check_throws<std::invalid_argument>([&] { bdiag3_extract(CsrMatrix(4, 4)); }, "not divisible");
    const BlockDiagonal3 DZ = bdiag3_extract(CsrMatrix(3, 3));
    CHECK(DZ.block(0)[0] == 1e-10 && DZ.block(0)[4] == 1e-10 && DZ.block(0)[8] == 1e-10);
  });
  // test_csr.cpp:174-210
  run("bdiag3_solve identity, scaling and dense oracle", [] {
    BlockDiagonal3 I;
    I.n_blocks = 2;
    I.blocks.assign(18, 0.0);
    for (int b = 0; b < 2; ++b)
      for (int i = 0; i < 3; ++i) I.block(b)[4 * i] = 1.0;
    const std::vector<double> w{1, 2, 3, 4, 5, 6};
    CHECK(bdiag3_solve(I, w) == w);
    BlockDiagonal3 two = I;
    for (double& v : two.blocks) v *= 2.0;
    const auto half = bdiag3_solve(two, w);
    for (size_t i = 0; i < w.size(); ++i) CHECK(approx(half[i], w[i] / 2, 1e-15));
    std::mt19937 rng(11);
    std::uniform_real_distribution<double> val(-1.0, 1.0);
    for (int trial = 0; trial < 1000; ++trial) {
      BlockDiagonal3 B;
      B.n_blocks = 1;
      B.blocks.resize(9);
      double det = 0.0;
      do {
        for (int i = 0; i < 9; ++i) B.blocks[i] = val(rng);
        const double* m = B.blocks.data();
        det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) + m[2] * (m[3] * m[7] - m[4] * m[6]);
      } while (std::abs(det) < 1e-2);
      const std::vector<double> rhs{val(rng), val(rng), val(rng)};
      const auto x = bdiag3_solve(B, rhs);
      double res = 0.0;
      for (int i = 0; i < 3; ++i) {
        double s = -rhs[i];
        for (int j = 0; j < 3; ++j) s += B.blocks[3 * i + j] * x[j];
        res += s * s;
      }
      CHECK(std::sqrt(res) <= 1e-12 * std::max(1.0, vnorm(rhs)));
    }
    BlockDiagonal3 S;
    S.n_blocks = 1;
    S.blocks.assign(9, 1.0);
    check_throws<numerical_error>([&] { bdiag3_solve(S, std::vector<double>{1, 1, 1}); }, "singular");
  });
  run("diag_extract", [] {  // test_csr.cpp:212-222
    CHECK((diag_extract(CsrMatrix::identity(4)) == std::vector<double>{1, 1, 1, 1}));
    const CsrMatrix off = CsrMatrix::from_triplets(3, 3, {{0, 1, 5.0}, {2, 0, 7.0}});
    CHECK((diag_extract(off) == std::vector<double>{0, 0, 0}));
    const CsrMatrix chain = CsrMatrix::from_triplets(
        3, 3, {{0, 0, 1.0}, {0, 1, -1.0}, {1, 0, -1.0}, {1, 1, 2.0}, {1, 2, -1.0}, {2, 1, -1.0}, {2, 2, 1.0}});
    CHECK((diag_extract(chain) == std::vector<double>{1, 2, 1}));
  });
  run("restrict_submatrix gathers dense blocks", [] {  // test_csr.cpp:224-242
    std::mt19937 rng(17);
    const CsrMatrix A = random_sparse(3, 3, 0.8, rng);
    const std::vector<int> all{0, 1, 2};
    const auto full = restrict_submatrix(A, all, all);
    CHECK(full == A.to_dense());
    CHECK(restrict_submatrix(A, std::vector<int>{}, std::vector<int>{}).empty());
    const std::vector<int> rows{0, 2}, cols{1};
    const auto g = restrict_submatrix(A, rows, cols);
    CHECK(g[0] == A.coeff(0, 1) && g[1] == A.coeff(2, 1));
    check_throws<std::invalid_argument>([&] { restrict_submatrix(A, std::vector<int>{2, 1}, cols); }, "unsorted");
    check_throws<std::invalid_argument>([&] { restrict_submatrix(A, std::vector<int>{0, 5}, cols); }, "oob");
  });
  run("csr invariants validated", [] {  // test_csr.cpp:261-266
    CsrMatrix A = CsrMatrix::identity(3);
    A.check_invariants();
    A.col_indices[1] = 9;
    check_throws<std::invalid_argument>([&] { A.check_invariants(); }, "invariant");
  });
}

void gmres_tests() {
  run("gmres on identity converges in one iteration", [] {  // test_gmres.cpp:15-23
    const CsrMatrix I = CsrMatrix::identity(5);
    CsrOperator op(I);
    const std::vector<double> b{1, -2, 3, -4, 5};
    auto [x, st] = gmres(op, nullptr, b, 1e-10);
    CHECK(st.converged && st.iterations == 1);
    for (int i = 0; i < 5; ++i) CHECK(approx(x[i], b[i], 1e-14));
  });
  run("gmres with exact inverse preconditioner: one iteration", [] {  // test_gmres.cpp:25-42
    const CsrMatrix A = spd_tridiagonal(20);
    BandFactor F;
    F.factor(A, BandFactor::Kind::spd);
    CsrOperator op(A);
    FunctionOperator pre(20, [&](std::span<const double> v) { return F.solve(v); });
    std::mt19937 rng(1);
    const auto b = random_vector(20, rng);
    auto [x, st] = gmres(op, &pre, b, 1e-12);
    CHECK(st.converged && st.iterations == 1);
    const auto Ax = spmv(A, x);
    double r = 0, nb = 0;
    for (int i = 0; i < 20; ++i) r += (b[i] - Ax[i]) * (b[i] - Ax[i]), nb += b[i] * b[i];
    CHECK(std::sqrt(r / nb) <= 1e-12);
  });
  run("gmres 2x2 direct-solve oracle", [] {  // test_gmres.cpp:44-51
    const CsrMatrix A = CsrMatrix::from_triplets(2, 2, {{0, 0, 4.0}, {0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 3.0}});
    CsrOperator op(A);
    auto [x, st] = gmres(op, nullptr, std::vector<double>{1, 2}, 1e-13);
    CHECK(st.converged && approx(x[0], 1.0 / 11.0, 1e-12) && approx(x[1], 7.0 / 11.0, 1e-12));
  });
  run("gmres monotone residuals and finite termination", [] {  // test_gmres.cpp:53-72
    std::mt19937 rng(77);
    for (int trial = 0; trial < 10; ++trial) {
      const int n = 5 + int(rng() % 46);
      std::vector<CsrMatrix::Triplet> t;
      for (int i = 0; i < n; ++i) {
        t.push_back({i, i, 4.0 + 0.1 * i});
        for (int r = 0; r < 3; ++r) {
          const int c = int(rng() % n);
          t.push_back({i, c, std::uniform_real_distribution<double>(-1, 1)(rng)});
        }
      }
      const CsrMatrix A = CsrMatrix::from_triplets(n, n, std::move(t));
      CsrOperator op(A);
      const auto b = random_vector(n, rng);
      auto [x, st] = gmres(op, nullptr, b, 1e-10, n + 5);
      CHECK(st.converged && st.iterations <= n);
      for (size_t i = 1; i < st.relative_residuals.size(); ++i)
        CHECK(st.relative_residuals[i] <= st.relative_residuals[i - 1] * (1 + 1e-12));
    }
  });
  run("right preconditioning: Arnoldi estimate equals true residual", [] {  // test_gmres.cpp:74-103
    std::mt19937 rng(31);
    for (int trial = 0; trial < 20; ++trial) {
      const int n = 8 + int(rng() % 25);
      CsrMatrix A = spd_tridiagonal(n, 3.0 + 0.05 * trial, -1.0);
      std::vector<CsrMatrix::Triplet> pert;
      for (int i = 0; i + 1 < n; ++i) pert.push_back({i, i + 1, 0.3});
      A = add_scaled(A, CsrMatrix::from_triplets(n, n, std::move(pert)), 1.0, 1.0);
      BandFactor F;
      F.factor(spd_tridiagonal(n, 3.5, -1.0), BandFactor::Kind::spd);
      CsrOperator op(A);
      FunctionOperator pre(n, [&](std::span<const double> v) { return F.solve(v); });
      const auto b = random_vector(n, rng);
      auto [xf, full] = gmres(op, &pre, b, 1e-12, n);
      const double nb = vnorm(b);
      for (int it = 1; it <= full.iterations; ++it) {
        auto [xi, si] = gmres(op, &pre, b, 1e-30, it);
        const auto Ax = spmv(A, xi);
        double r = 0;
        for (int i = 0; i < n; ++i) r += (b[i] - Ax[i]) * (b[i] - Ax[i]);
        const double tr = std::sqrt(r) / nb, est = full.relative_residuals[size_t(it) - 1];
        CHECK(std::abs(tr - est) <= 1e-6 * std::max(est, 1e-30) + 1e-12);
      }
    }
  });
  run("gmres basis orthogonality after reorthogonalization", [] {  // test_gmres.cpp:105-128
    std::mt19937 rng(13);
    const int n = 60;
    std::vector<CsrMatrix::Triplet> t;
    for (int i = 0; i < n; ++i) {
      t.push_back({i, i, std::pow(10.0, -6.0 + 12.0 * i / (n - 1.0))});
      if (i + 1 < n) t.push_back({i, i + 1, 1e-3});
    }
    const CsrMatrix A = CsrMatrix::from_triplets(n, n, std::move(t));
    CsrOperator op(A);
    const auto b = random_vector(n, rng);
    std::vector<std::vector<double>> V;
    auto [x, st] = gmres(op, nullptr, b, 1e-12, n, &V);
    CHECK(V.size() >= 2);
    double worst = 0;
    for (size_t i = 0; i < V.size(); ++i)
      for (size_t j = 0; j <= i; ++j) {
        double d = 0;
        for (int k = 0; k < n; ++k) d += V[i][k] * V[j][k];
        worst = std::max(worst, std::abs(d - (i == j ? 1.0 : 0.0)));
      }
    CHECK(worst <= 1e-8);
  });
  run("gmres reports non-convergence at max_iter", [] {  // test_gmres.cpp:130-138
    const CsrMatrix A = spd_tridiagonal(50, 2.0, -1.0);
    CsrOperator op(A);
    std::mt19937 rng(3);
    const auto b = random_vector(50, rng);
    auto [x, st] = gmres(op, nullptr, b, 1e-30, 5);
    CHECK(!st.converged && st.iterations == 5);
  });
  run("gmres happy breakdown yields exact solve", [] {  // test_gmres.cpp:140-150
    const CsrMatrix A = CsrMatrix::from_triplets(3, 3, {{0, 0, 2.0}, {1, 1, 3.0}, {2, 2, 4.0}});
    CsrOperator op(A);
    auto [x, st] = gmres(op, nullptr, std::vector<double>{0, 5, 0}, 1e-14, 10);
    CHECK(st.converged && st.breakdown && st.iterations == 1 && approx(x[1], 5.0 / 3.0, 1e-14));
  });
  run("gmres errors: mismatch, bad tol, zero rhs", [] {
    const CsrMatrix I = CsrMatrix::identity(3);
    CsrOperator op(I);
    check_throws<std::invalid_argument>([&] { gmres(op, nullptr, std::vector<double>{1, 2}, 1e-8); }, "rhs");
    check_throws<std::invalid_argument>([&] { gmres(op, nullptr, std::vector<double>{1, 2, 3}, 0.0); }, "tol");
    auto [x, st] = gmres(op, nullptr, std::vector<double>{0, 0, 0}, 1e-8);
    CHECK(st.converged && st.iterations == 0);
  });
  run("gmres(m) restart wrapper reaches the full-GMRES solution", [] {
    std::mt19937 rng(5);
    const int n = 120;
    CsrMatrix A = spd_tridiagonal(n, 2.2, -1.0);
    CsrOperator op(A);
    const auto b = random_vector(n, rng);
    auto [x, st] = gmres_restarted(op, nullptr, b, 1e-10, 10, 2000);
    CHECK(st.converged && st.restarts >= 1);
    const auto Ax = spmv(A, x);
    double r = 0;
    for (int i = 0; i < n; ++i) r += (b[i] - Ax[i]) * (b[i] - Ax[i]);
    CHECK(std::sqrt(r) <= 1e-10 * vnorm(b) * (1 + 1e-9));
  });
}

void amg_tests() {
  AmgConfig cfg;  // reference defaults (smoother = sgs)
  run("amg single level below max_coarse is a direct solve", [&] {  // test_amg.cpp:17-30
    const CsrMatrix A = spd_tridiagonal(40);
    const AmgHierarchy h = amg_setup(A, {}, cfg);
    CHECK(h.num_levels() == 1);
    std::mt19937 rng(4);
    const auto b = random_vector(40, rng);
    const auto x = amg_apply(h, b);
    const auto Ax = spmv(A, x);
    for (int i = 0; i < 40; ++i) CHECK(approx(Ax[i], b[i], 1e-11));
    const std::vector<double> zero(40, 0.0);
    CHECK(amg_apply(h, zero) == zero);
  });
  run("amg 1d poisson coarsening rate near one third", [&] {  // test_amg.cpp:32-41
    const AmgHierarchy h = amg_setup(poisson1d(1024), {}, cfg);
    CHECK(h.num_levels() >= 3);
    for (int l = 1; l < h.num_levels(); ++l) {
      const double ratio = double(h.levels[l].A.n_rows) / h.levels[l - 1].A.n_rows;
      CHECK(ratio < 0.45 && ratio > 0.2);
    }
  });
  run("amg galerkin identity on every level", [&] {  // test_amg.cpp:43-54
    const AmgHierarchy h = amg_setup(poisson3d(9), {}, cfg);
    CHECK(h.num_levels() >= 2);
    for (int l = 1; l < h.num_levels(); ++l) {
      const Dense Af = Dense::of(h.levels[l - 1].A), P = Dense::of(h.levels[l].P);
      const Dense ref = transpose(P) * Af * P;
      CHECK(fro(Dense::of(h.levels[l].A) - ref) <= 1e-13 * std::max(1.0, fro(ref)));
    }
  });
  for (int sm = 0; sm < 2; ++sm) {
    AmgConfig c = cfg;
    c.smoother = sm == 0 ? AmgConfig::Smoother::sgs : AmgConfig::Smoother::weighted_jacobi;
    run(sm == 0 ? "amg apply is linear (sgs)" : "amg apply is linear (jacobi)", [c] {  // test_amg.cpp:56-73
      const AmgHierarchy h = amg_setup(poisson1d(300), {}, c);
      std::mt19937 rng(8);
      const auto r1 = random_vector(300, rng), r2 = random_vector(300, rng);
      const double a = 1.7, b = -0.4;
      std::vector<double> mix(300);
      for (int i = 0; i < 300; ++i) mix[i] = a * r1[i] + b * r2[i];
      const auto y = amg_apply(h, mix), y1 = amg_apply(h, r1), y2 = amg_apply(h, r2);
      double err = 0, sc = 0;
      for (int i = 0; i < 300; ++i) {
        const double e = y[i] - (a * y1[i] + b * y2[i]);
        err += e * e;
        sc += y[i] * y[i];
      }
      CHECK(std::sqrt(err) <= 1e-12 * std::max(1.0, std::sqrt(sc)));
    });
  }
  run("amg v-cycle is symmetric for symmetric input with sgs", [&] {  // test_amg.cpp:75-82
    const CsrMatrix A = poisson1d(260);
    const AmgHierarchy h = amg_setup(A, {}, cfg);
    const Dense B = densify_fn(260, [&](std::span<const double> r) { return amg_apply(h, r); });
    CHECK(max_abs(B - transpose(B)) <= 1e-10 * max_abs(B));
  });
  run("amg 1d poisson error propagation spectral radius", [&] {  // test_amg.cpp:84-100
    const int n = 64;
    const CsrMatrix A = poisson1d(n);
    const AmgHierarchy h = amg_setup(A, {}, cfg);
    const Dense E = densify_fn(n, [&](std::span<const double> x) {
      const auto Ax = spmv(A, x);
      const auto BAx = amg_apply(h, Ax);
      std::vector<double> out(x.begin(), x.end());
      for (int i = 0; i < n; ++i) out[i] -= BAx[i];
      return out;
    });
    // rho(E) <= ||E^k||_F^(1/k) for every k; k = 2^8 (repeated squaring with renormalization)
    Dense Ek = E;
    double logscale = 0.0;
    for (int s = 0; s < 8; ++s) {
      Ek = Ek * Ek;
      logscale *= 2.0;
      const double f = fro(Ek);
      if (f > 0) {
        for (double& v : Ek.a) v /= f;
        logscale += std::log(f);
      }
    }
    const double bound = std::exp((logscale + std::log(std::max(fro(Ek), 1e-300))) / 256.0);
    CHECK(bound <= 0.35);
  });
  run("amg rigid body modes reproduced per aggregate", [] {  // test_amg.cpp:102-160
    const int m = 4, nn = m * m * m;
    std::vector<std::array<double, 3>> coords;
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) coords.push_back({double(i), double(j), double(k)});
    std::vector<CsrMatrix::Triplet> t;
    auto id = [m](int i, int j, int k) { return i + m * (j + m * k); };
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
          const int v = id(i, j, k);
          for (int d = 0; d < 3; ++d) t.push_back({3 * v + d, 3 * v + d, 6.0});
          auto couple = [&](int w) {
            for (int d = 0; d < 3; ++d) {
              t.push_back({3 * v + d, 3 * w + d, -1.0});
              t.push_back({3 * w + d, 3 * v + d, -1.0});
            }
          };
          if (i + 1 < m) couple(id(i + 1, j, k));
          if (j + 1 < m) couple(id(i, j + 1, k));
          if (k + 1 < m) couple(id(i, j, k + 1));
        }
    const CsrMatrix A = CsrMatrix::from_triplets(3 * nn, 3 * nn, std::move(t));
    AmgConfig c;
    c.prolongation_smoothing = false;
    c.max_coarse = 10;
    const auto modes = rigid_body_modes(coords);
    const AmgHierarchy h = amg_setup(A, modes, c);
    CHECK(h.num_levels() >= 2);
    const AmgLevel& L = h.levels[1];
    const Dense Pd = Dense::of(L.P);
    const int n_agg = int(L.aggregate_offsets.size()) - 1;
    int checked = 0;
    for (int a = 0; a < n_agg; ++a) {
      const int c0 = L.aggregate_offsets[a], c1 = L.aggregate_offsets[a + 1];
      if (c1 == c0) continue;
      ++checked;
      std::vector<int> rows;
      for (int i = 0; i < 3 * nn; ++i)
        if (L.fine_aggregate[i] == a) rows.push_back(i);
      Dense Pl(int(rows.size()), c1 - c0);
      for (size_t r = 0; r < rows.size(); ++r)
        for (int cc = c0; cc < c1; ++cc) Pl(int(r), cc - c0) = Pd(rows[r], cc);
      const Dense proj = Pl * inverse(transpose(Pl) * Pl) * transpose(Pl);
      for (const auto& mode : modes) {
        Dense v(int(rows.size()), 1);
        for (size_t r = 0; r < rows.size(); ++r) v(int(r), 0) = mode[rows[r]];
        CHECK(fro(proj * v - v) <= 1e-10 * std::max(1.0, fro(v)));
      }
    }
    CHECK(checked > 0);
  });
  for (int sm = 0; sm < 2; ++sm) {
    AmgConfig c = cfg;
    c.smoother = sm == 0 ? AmgConfig::Smoother::sgs : AmgConfig::Smoother::weighted_jacobi;
    run(sm == 0 ? "amg h-scalability on 3d poisson (sgs)" : "amg h-scalability on 3d poisson (jacobi)", [c] {
      std::vector<int> iters;  // test_amg.cpp:162-178
      for (int m : {8, 16, 24}) {
        const CsrMatrix A = poisson3d(m);
        const AmgHierarchy h = amg_setup(A, {}, c);
        CsrOperator op(A);
        FunctionOperator pre(A.n_rows, [&](std::span<const double> r) { return amg_apply(h, r); });
        std::mt19937 rng(55);
        const auto b = random_vector(A.n_rows, rng);
        auto [x, st] = gmres(op, &pre, b, 1e-8, 200);
        CHECK(st.converged);
        iters.push_back(st.iterations);
      }
      CHECK(*std::max_element(iters.begin(), iters.end()) - *std::min_element(iters.begin(), iters.end()) <= 2);
    });
  }
  run("amg rejects zero diagonal and non-square input", [&] {  // test_amg.cpp:180-184
    const CsrMatrix bad = CsrMatrix::from_triplets(2, 2, {{0, 0, 1.0}, {0, 1, 1.0}, {1, 0, 1.0}});
    check_throws<numerical_error>([&] { amg_setup(bad, {}, cfg); }, "zero diag");
    check_throws<std::invalid_argument>([&] { amg_setup(CsrMatrix(2, 3), {}, cfg); }, "non-square");
  });
}

void precond_tests() {
  PrecondConfig direct;
  direct.inner = PrecondConfig::Inner::direct;
  run("tpu decoupled: S == A, apply splits per physics", [&] {  // test_precond.cpp:34-52
    const BlockSystem J = toy_system(18, 2, ToyMode::decoupled);
    const TpuPreconditioner M = build_tpu(J, direct);
    CHECK(max_abs(Dense::of(M.S) - Dense::of(J.A)) == 0.0);
    std::mt19937 rng(2);
    const BlockVector w = random_block(J, rng);
    const BlockVector v = apply_tpu(M, J, w);
    Dense wu(J.n_u, 1);
    for (int i = 0; i < J.n_u; ++i) wu(i, 0) = w.u[i];
    const Dense vu = solve(Dense::of(J.A), wu);
    for (int i = 0; i < J.n_u; ++i) CHECK(approx(v.u[i], vu(i, 0), 1e-10));
    const auto ht = bdiag3_solve(M.Hs.block_diag, w.t);
    for (int i = 0; i < J.n_t; ++i) CHECK(approx(v.t[i], -ht[i], 1e-12));
    const auto tp = M.T_factor.solve(w.p);
    for (int i = 0; i < J.n_p; ++i) CHECK(approx(v.p[i], tp[i], 1e-12));
  });
  run("tpu all-stick schur complement is symmetric", [&] {  // test_precond.cpp:54-61
    const BlockSystem J = toy_system(30, 4, ToyMode::stick);
    const Dense S = Dense::of(build_tpu(J, direct).S);
    CHECK(max_abs(S - transpose(S)) <= 1e-12 * max_abs(S));
  });
  run("tpu mixed-state schur matches dense triple product", [&] {  // test_precond.cpp:63-80
    const BlockSystem J = toy_system(24, 2, ToyMode::mixed);
    const TpuPreconditioner M = build_tpu(J, direct);
    Dense Hb(J.n_t, J.n_t);
    const BlockDiagonal3 D = bdiag3_extract(J.H);
    for (int b = 0; b < D.n_blocks; ++b)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Hb(3 * b + i, 3 * b + j) = D.block(b)[3 * i + j];
    const auto td = diag_extract(J.T);
    Dense Tinv(J.n_p, J.n_p);
    for (int i = 0; i < J.n_p; ++i) Tinv(i, i) = 1.0 / td[i];
    const Dense ref = Dense::of(J.A) + Dense::of(J.C1) * solve(Hb, Dense::of(J.C2)) -
                      Dense::of(J.Q1) * Tinv * Dense::of(J.Q2);
    CHECK(max_abs(Dense::of(M.S) - ref) <= 1e-13 * std::max(1.0, max_abs(ref)));
  });
  run("tup build: stick -> S_K = 0, decoupled -> S1 == A, mixed -> dense S1", [&] {  // test_precond.cpp:82-102
    const BlockSystem Js = toy_system(30, 3, ToyMode::stick);
    const TupPreconditioner Ms = build_tup(Js, direct);
    for (double v : Ms.S_K) CHECK(v == 0.0);
    CHECK(max_abs(Dense::of(Ms.S2) - Dense::of(Js.T)) == 0.0);
    const BlockSystem Jd = toy_system(18, 2, ToyMode::decoupled);
    CHECK(max_abs(Dense::of(build_tup(Jd, direct).S1) - Dense::of(Jd.A)) == 0.0);
    const BlockSystem Jm = toy_system(24, 2, ToyMode::mixed);
    const TupPreconditioner Mm = build_tup(Jm, direct);
    const Dense S1ref = Dense::of(Jm.A) + Dense::of(Jm.C1) * hs_dense(Mm.Hs, Jm.n_t) * Dense::of(Jm.C2);
    CHECK(max_abs(Dense::of(Mm.S1) - S1ref) <= 1e-13 * std::max(1.0, max_abs(S1ref)));
    const Dense S2 = Dense::of(Mm.S2);
    CHECK(max_abs(S2 - transpose(S2)) <= 1e-12 * max_abs(S2));
  });
  run("fixed_stress_diag matches dense restriction oracle", [] {  // test_precond.cpp:104-154
    const CsrMatrix S1 = CsrMatrix::from_triplets(1, 1, {{0, 0, 2.0}});
    const CsrMatrix Q1 = CsrMatrix::from_triplets(1, 1, {{0, 0, 3.0}});
    const CsrMatrix Q2 = CsrMatrix::from_triplets(1, 1, {{0, 0, 5.0}});
    CHECK(approx(fixed_stress_diag(Q2, S1, Q1)[0], 7.5, 1e-14));
    CHECK(fixed_stress_diag(CsrMatrix(1, 1), S1, Q1)[0] == 0.0);
    std::mt19937 rng(10);
    std::uniform_real_distribution<double> val(-1.0, 1.0);
    for (int trial = 0; trial < 100; ++trial) {
      const int n_u = 12, n_p = 3;
      const CsrMatrix S = spd_tridiagonal(n_u, 5.0, -1.0);
      std::vector<CsrMatrix::Triplet> q1t, q2t;
      for (int k = 0; k < n_p; ++k) {
        const int base = int(rng() % (n_u - 6));
        for (int r = 0; r < 6; ++r) q1t.push_back({base + r, k, val(rng)});
        if (k != 1) {
          const int base2 = int(rng() % (n_u - 5));
          for (int r = 0; r < 5; ++r) q2t.push_back({k, base2 + r, val(rng)});
        }
      }
      const CsrMatrix Q1r = CsrMatrix::from_triplets(n_u, n_p, std::move(q1t));
      const CsrMatrix Q2r = CsrMatrix::from_triplets(n_p, n_u, std::move(q2t));
      const auto got = fixed_stress_diag(Q2r, S, Q1r);
      CHECK(got[1] == 0.0);
      const Dense Sd = Dense::of(S), Q1d = Dense::of(Q1r), Q2d = Dense::of(Q2r);
      for (int k = 0; k < n_p; ++k) {
        if (k == 1) continue;
        std::vector<int> idx;
        for (int i = 0; i < n_u; ++i)
          if (Q1d(i, k) != 0.0 || Q2d(k, i) != 0.0) idx.push_back(i);
        const int m = int(idx.size());
        Dense Sl(m, m), q1(m, 1);
        std::vector<double> q2(static_cast<size_t>(m));
        for (int a = 0; a < m; ++a) {
          q1(a, 0) = Q1d(idx[a], k);
          q2[a] = Q2d(k, idx[a]);
          for (int b = 0; b < m; ++b) Sl(a, b) = Sd(idx[a], idx[b]);
        }
        const Dense x = solve(Sl, q1);
        double ref = 0;
        for (int a = 0; a < m; ++a) ref += q2[a] * x(a, 0);
        CHECK(approx(got[k], ref, 1e-12));
      }
    }
  });
  run("tpu pressure unit vectors are fixed points", [&] {  // test_precond.cpp:197-203, bounds.cpp:185-206
    const BlockSystem J = toy_system(24, 2, ToyMode::mixed, 321);
    const TpuPreconditioner M = build_tpu(J, direct);
    BlockSystemOperator Jop(J);
    TpuOperator Mop(M, J);
    const int n = J.total_dimension();
    double dev = 0.0;
    for (int jp = 0; jp < J.n_p; ++jp) {
      std::vector<double> x(static_cast<size_t>(n), 0.0);
      x[size_t(J.n_u + J.n_t + jp)] = 1.0;
      const auto y = Mop(Jop(x));
      for (int i = 0; i < n; ++i) dev = std::max(dev, std::abs(y[i] - (i == J.n_u + J.n_t + jp ? 1.0 : 0.0)));
    }
    CHECK(dev <= 1e-10);
  });
  run("apply_tpu equals the dense block-LDU factor product", [&] {  // test_precond.cpp:205-248
    const BlockSystem J = toy_system(21, 2, ToyMode::mixed, 77);
    const TpuPreconditioner M = build_tpu(J, direct);
    const int nu = J.n_u, nt = J.n_t, np = J.n_p, n = nu + nt + np;
    const Dense Hinv = hs_dense(M.Hs, nt);
    const Dense Tinv = densify_fn(np, [&](std::span<const double> v) { return M.T_factor.solve(v); });
    const Dense Sinv = densify_fn(nu, [&](std::span<const double> v) { return M.S_solver.apply(v); });
    const Dense C1 = Dense::of(J.C1), C2 = Dense::of(J.C2), Q1 = Dense::of(J.Q1), Q2 = Dense::of(J.Q2);
    auto put = [](Dense& D, int r0, int c0, const Dense& B, double s) {
      for (int i = 0; i < B.r; ++i)
        for (int j = 0; j < B.c; ++j) D(r0 + i, c0 + j) = s * B(i, j);
    };
    Dense F1 = Dense::eye(n), Dm(n, n), F3 = Dense::eye(n);
    put(F1, 0, nt + np, Hinv * C2, 1.0);
    put(F1, nt, nt + np, Tinv * Q2, -1.0);
    put(Dm, 0, 0, Hinv, -1.0);
    put(Dm, nt, nt, Tinv, 1.0);
    put(Dm, nt + np, nt + np, Sinv, 1.0);
    put(F3, nt + np, 0, C1 * Hinv, 1.0);
    put(F3, nt + np, nt, Q1 * Tinv, -1.0);
    const Dense Mp = F1 * Dm * F3;
    std::vector<int> nat(static_cast<size_t>(n));
    for (int i = 0; i < nt; ++i) nat[i] = nu + i;
    for (int i = 0; i < np; ++i) nat[size_t(nt) + i] = nu + nt + i;
    for (int i = 0; i < nu; ++i) nat[size_t(nt) + np + i] = i;
    Dense Mn(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) Mn(nat[i], nat[j]) = Mp(i, j);
    const Dense Ma = densify(TpuOperator(M, J));
    for (int j = 0; j < n; ++j) {
      double cn;
      const double d = col_norm_diff(Ma, Mn, j, &cn);
      CHECK(d <= 1e-11 * std::max(1.0, cn));
    }
  });
  run("apply_tup and tup_star equal their dense factor forms", [&] {  // test_precond.cpp:250-303
    const BlockSystem J = toy_system(21, 2, ToyMode::mixed, 55);
    const TupPreconditioner M = build_tup(J, direct);
    const int nu = J.n_u, nt = J.n_t, np = J.n_p, n = nu + nt + np;
    const Dense Hinv = hs_dense(M.Hs, nt);
    const Dense S1inv = densify_fn(nu, [&](std::span<const double> v) { return M.S1_solver.apply(v); });
    const Dense S2inv = densify_fn(np, [&](std::span<const double> v) { return M.s2_solve(v); });
    const Dense C1 = Dense::of(J.C1), C2 = Dense::of(J.C2), Q1 = Dense::of(J.Q1), Q2 = Dense::of(J.Q2);
    auto put = [](Dense& D, int r0, int c0, const Dense& B, double s) {
      for (int i = 0; i < B.r; ++i)
        for (int j = 0; j < B.c; ++j) D(r0 + i, c0 + j) = s * B(i, j);
    };
    Dense U2 = Dense::eye(n), Di(n, n), L2 = Dense::eye(n);
    put(U2, 0, nt, Hinv * C2, 1.0);
    put(U2, 0, nt + nu, Hinv * C2 * S1inv * Q1, -1.0);
    put(U2, nt, nt + nu, S1inv * Q1, -1.0);
    put(Di, 0, 0, Hinv, -1.0);
    put(Di, nt, nt, S1inv, 1.0);
    put(Di, nt + nu, nt + nu, S2inv, 1.0);
    put(L2, nt, 0, C1 * Hinv, 1.0);
    put(L2, nt + nu, 0, Q2 * S1inv * C1 * Hinv, -1.0);
    put(L2, nt + nu, nt, Q2 * S1inv, -1.0);
    std::vector<int> nat(static_cast<size_t>(n));
    for (int i = 0; i < nt; ++i) nat[i] = nu + i;
    for (int i = 0; i < nu; ++i) nat[size_t(nt) + i] = i;
    for (int i = 0; i < np; ++i) nat[size_t(nt) + nu + i] = nu + nt + i;
    auto unperm = [&](const Dense& Mp) {
      Dense Mn(n, n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) Mn(nat[i], nat[j]) = Mp(i, j);
      return Mn;
    };
    const Dense Mfull = unperm(U2 * Di * L2), Ma = densify(TupOperator(M, J));
    const Dense Mstar = unperm(Di * L2), Msa = densify(TupOperator(M, J, true));
    for (int j = 0; j < n; ++j) {
      double cn;
      double d = col_norm_diff(Ma, Mfull, j, &cn);
      CHECK(d <= 1e-11 * std::max(1.0, cn));
      d = col_norm_diff(Msa, Mstar, j, &cn);
      CHECK(d <= 1e-11 * std::max(1.0, cn));
    }
  });
  run("tup_star equals tup on decoupled input and w = 0 maps to 0", [&] {  // test_precond.cpp:305-321
    const BlockSystem J = toy_system(18, 2, ToyMode::decoupled);
    const TupPreconditioner M = build_tup(J, direct);
    std::mt19937 rng(6);
    const BlockVector w = random_block(J, rng);
    const BlockVector a = apply_tup(M, J, w), b = apply_tup_star(M, J, w);
    for (int i = 0; i < J.n_u; ++i) CHECK(approx(a.u[i], b.u[i], 1e-13));
    for (int i = 0; i < J.n_t; ++i) CHECK(approx(a.t[i], b.t[i], 1e-13));
    for (int i = 0; i < J.n_p; ++i) CHECK(approx(a.p[i], b.p[i], 1e-13));
    CHECK(apply_tup(M, J, BlockVector(J.n_u, J.n_t, J.n_p)).norm2() == 0.0);
  });
  run("inner-solver cost contract: 1 tpu, 2 tup, 1 tup_star", [&] {  // test_precond.cpp:323-343
    const BlockSystem J = toy_system(24, 2, ToyMode::mixed, 11);
    const TpuPreconditioner M1 = build_tpu(J, direct);
    const TupPreconditioner M2 = build_tup(J, direct);
    std::mt19937 rng(12);
    const BlockVector w = random_block(J, rng);
    M1.S_solver.reset_count();
    apply_tpu(M1, J, w);
    CHECK(M1.S_solver.call_count() == 1);
    M2.S1_solver.reset_count();
    apply_tup(M2, J, w);
    CHECK(M2.S1_solver.call_count() == 2);
    M2.S1_solver.reset_count();
    apply_tup_star(M2, J, w);
    CHECK(M2.S1_solver.call_count() == 1);
  });
  for (int sm = 0; sm < 2; ++sm) {
    run(sm == 0 ? "preconditioner applications are linear (amg sgs)" : "preconditioner applications are linear (amg jacobi)",
        [sm] {  // test_precond.cpp:345-373
          const BlockSystem J = toy_system(24, 2, ToyMode::mixed, 44);
          PrecondConfig cfg;
          cfg.inner = PrecondConfig::Inner::amg;
          cfg.amg.max_coarse = 8;
          if (sm == 1) cfg.amg.smoother = AmgConfig::Smoother::weighted_jacobi;
          const TpuPreconditioner M1 = build_tpu(J, cfg);
          const TupPreconditioner M2 = build_tup(J, cfg);
          std::mt19937 rng(1);
          const auto x1 = random_vector(J.total_dimension(), rng), x2 = random_vector(J.total_dimension(), rng);
          const double a = 0.7, b = -1.3;
          TpuOperator o1(M1, J);
          TupOperator o2(M2, J);
          for (const LinearOperator* op : {static_cast<const LinearOperator*>(&o1), static_cast<const LinearOperator*>(&o2)}) {
            std::vector<double> mix(x1.size());
            for (size_t i = 0; i < mix.size(); ++i) mix[i] = a * x1[i] + b * x2[i];
            const auto y = (*op)(mix), y1 = (*op)(x1), y2 = (*op)(x2);
            double err = 0, sc = 0;
            for (size_t i = 0; i < y.size(); ++i) {
              const double e = y[i] - (a * y1[i] + b * y2[i]);
              err += e * e;
              sc += y[i] * y[i];
            }
            CHECK(std::sqrt(err) <= 1e-12 * std::max(1.0, std::sqrt(sc)));
          }
        });
  }
  run("band factors: spd and pivoted LU solve to the residual floor", [] {
    std::mt19937 rng(21);
    // two decoupled 2D grid blocks (5-point), like T per fracture
    std::vector<CsrMatrix::Triplet> t;
    int off = 0;
    for (int nb : {7, 5}) {
      for (int j = 0; j < nb; ++j)
        for (int i = 0; i < nb; ++i) {
          const int r = off + i + nb * j;
          t.push_back({r, r, 4.3});
          if (i + 1 < nb) t.push_back({r, r + 1, -1.0}), t.push_back({r + 1, r, -1.0});
          if (j + 1 < nb) t.push_back({r, r + nb, -1.0}), t.push_back({r + nb, r, -1.0});
        }
      off += nb * nb;
    }
    const int n = off;
    const CsrMatrix T = CsrMatrix::from_triplets(n, n, t);
    // indefinite shift for the general LU
    std::vector<CsrMatrix::Triplet> sh;
    for (int i = 0; i < n; i += 3) sh.push_back({i, i, -6.0});
    const CsrMatrix S2 = add_scaled(T, CsrMatrix::from_triplets(n, n, sh), 1.0, 1.0);
    BandFactor F1, F2;
    F1.factor(T, BandFactor::Kind::spd);
    F2.factor(S2, BandFactor::Kind::general);
    CHECK(F1.block_start.size() == 3 && F1.block_start[1] == 49);
    const auto b = random_vector(n, rng);
    for (int which = 0; which < 2; ++which) {
      const CsrMatrix& M = which == 0 ? T : S2;
      const auto x = (which == 0 ? F1 : F2).solve(b);
      const auto Mx = spmv(M, x);
      double r = 0;
      for (int i = 0; i < n; ++i) r += (Mx[i] - b[i]) * (Mx[i] - b[i]);
      CHECK(std::sqrt(r) <= 1e-13 * vnorm(b));
    }
  });
  run("scaled driver operators are similarity transforms", [] {  // driver.cpp:104-141,233-248
    const BlockSystem J = toy_system(24, 2, ToyMode::mixed, 7);
    const BlockScaling D = BlockScaling::from(J);
    CHECK(D.st > 0 && D.sp > 0);
    BlockSystemOperator Jop(J);
    ScaledOperator Js(Jop, D, false);
    std::mt19937 rng(3);
    auto v = random_vector(J.total_dimension(), rng);
    auto y = Js(v);
    auto w = v;
    D.scale(w, false);
    auto z = Jop(w);
    D.scale(z, false);
    CHECK(y == z);
  });
}

}  // namespace

int main() {
  csr_tests();
  gmres_tests();
  amg_tests();
  precond_tests();
  std::printf("SUMMARY failed=%d checks=%d\n", g_fail, g_checks);
  return g_fail == 0 ? 0 : 1;
}
