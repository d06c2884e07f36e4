// ============================================================================
// fracprec ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A CPU restatement (C++20, Eigen-free, single-threaded on the solve path) of
// the reference's solve phase: /root/reference/proj/core/src/{csr,block,gmres,
// amg,sparse_factor,precond}.cpp and the block scaling of driver.cpp:104-141,
// 229-255.  Every function cites the reference file:line it restates.
//
// Who may use it: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` legs, and only as the checker or the timed CPU baseline.
// The product (paper_2112_12397_b200/) never links, loads or calls it.
//
// Parity pinning.  The reference cannot be compiled here (it requires Eigen3,
// LAPACKE, doctest, CLI11; none are on disk), and it ships no golden vectors.
// The oracle is pinned against every known-answer test and property the
// reference's own suite holds for this path (SPEC.md examples,
// tests/unit/test_{csr,gmres,amg,precond}.cpp), re-expressed in
// tests/test_oracle_kat.py, on the reference's own toy_system fixture
// (test_helpers.hpp:54-193, reproduced bit-for-bit with std::mt19937 +
// std::uniform_real_distribution from the same libstdc++).
//
// Eigen numerics the reference relies on are restated with fixed, documented
// rules:
//   * ColPivHouseholderQR  -> qr_colpiv():   Householder, first-maximal column
//                             norm pivot with norms recomputed each step.
//   * FullPivLU            -> DenseFullPivLU: first-maximal |a_ij| pivot in
//                             row-major scan; rank threshold n*eps*|u_00|.
//   * SimplicialLDLT(AMD)  -> BandFactor (LDL^T, natural order, per diagonal block)
//   * SparseLU(COLAMD)     -> BandFactor (LU with partial pivoting, banded, per block)
// Triangular solves are column sweeps (each row receives its updates in
// ascending column order for forward solves, descending for backward solves);
// that order is part of the oracle's definition and the GPU reproduces it.
// Compile with -ffp-contract=off: no fused multiply-add anywhere.
// ============================================================================
#pragma once

#include <array>
#include <atomic>
#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace fpo {

// errors.hpp:15-18
class numerical_error : public std::runtime_error {
 public:
  explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------- csr.hpp:16-49
// int64 row offsets are an extension (the reference uses int); column indices
// stay 32-bit.
struct CsrMatrix {
  int n_rows = 0, n_cols = 0;
  std::vector<int64_t> row_offsets{0};
  std::vector<int> col_indices;
  std::vector<double> values;

  CsrMatrix() = default;
  CsrMatrix(int r, int c) : n_rows(r), n_cols(c), row_offsets(static_cast<size_t>(r) + 1, 0) {}
  int64_t nnz() const { return int64_t(col_indices.size()); }
  double coeff(int i, int j) const;
  void check_invariants() const;

  struct Triplet { int row, col; double value; };
  static CsrMatrix identity(int n);
  static CsrMatrix from_triplets(int rows, int cols, std::vector<Triplet> t);
  static CsrMatrix from_dense(const std::vector<double>& rowmajor, int rows, int cols,
                              double drop_tol = 0.0);
  std::vector<double> to_dense() const;  // row-major
};

// mmio.hpp (snapshot bundle blocks): oracle/mmio.cpp
CsrMatrix read_matrix_market(const std::string& path);
void write_matrix_market(const std::string& path, const CsrMatrix& A);

// csr.hpp:52-58
struct BlockDiagonal3 {
  int n_blocks = 0;
  std::vector<double> blocks;  // 9 per block, row-major
  double* block(int k) { return blocks.data() + 9 * size_t(k); }
  const double* block(int k) const { return blocks.data() + 9 * size_t(k); }
};

std::vector<double> spmv(const CsrMatrix& A, std::span<const double> x);
std::vector<double> spmv_transpose(const CsrMatrix& A, std::span<const double> x);
// EXTENSION (row_sum = strided32): y_i = xor-tree of 32 partials p_l = sum over the row's entries
// k = l, l + 32, ... (ascending, from +0.0) of a_k x_c(k); the tree is p_l <- p_l + p_(l^h) for
// h = 16, 8, 4, 2, 1 (one warp per row on the GPU, lane l owning p_l).
std::vector<double> spmv_strided32(const CsrMatrix& A, std::span<const double> x);
CsrMatrix transpose(const CsrMatrix& A);
CsrMatrix spgemm(const CsrMatrix& A, const CsrMatrix& B);
CsrMatrix add_scaled(const CsrMatrix& A, const CsrMatrix& B, double alpha, double beta);
CsrMatrix scale_rows(const CsrMatrix& A, std::span<const double> s);
BlockDiagonal3 bdiag3_extract(const CsrMatrix& H, double delta = 1e-10);
bool lu3_factor(double m[9], int piv[3]);
void lu3_solve(const double m[9], const int piv[3], const double b[3], double x[3]);
std::vector<double> bdiag3_solve(const BlockDiagonal3& H, std::span<const double> w);
CsrMatrix bdiag3_inverse_csr(const BlockDiagonal3& H);
std::vector<double> diag_extract(const CsrMatrix& T);
std::vector<double> restrict_submatrix(const CsrMatrix& A, std::span<const int> rows,
                                       std::span<const int> cols);  // row-major dense

// ------------------------------------------------------------- operator.hpp:17-56
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual int dimension() const = 0;
  virtual void apply(std::span<const double> x, std::span<double> y) const = 0;
  std::vector<double> operator()(std::span<const double> x) const {
    std::vector<double> y(static_cast<size_t>(dimension()));
    apply(x, y);
    return y;
  }
};

class CsrOperator : public LinearOperator {
 public:
  explicit CsrOperator(const CsrMatrix& A) : A_(&A) {}
  int dimension() const override { return A_->n_rows; }
  void apply(std::span<const double> x, std::span<double> y) const override;
 private:
  const CsrMatrix* A_;
};

class FunctionOperator : public LinearOperator {
 public:
  using Fn = std::function<std::vector<double>(std::span<const double>)>;
  FunctionOperator(int n, Fn f) : n_(n), f_(std::move(f)) {}
  int dimension() const override { return n_; }
  void apply(std::span<const double> x, std::span<double> y) const override;
 private:
  int n_;
  Fn f_;
};

// ---------------------------------------------------------------- block.hpp:16-57
struct BlockVector {
  std::vector<double> u, t, p;
  BlockVector() = default;
  BlockVector(int nu, int nt, int np) : u(static_cast<size_t>(nu), 0.0), t(static_cast<size_t>(nt), 0.0), p(static_cast<size_t>(np), 0.0) {}
  int dimension() const { return int(u.size() + t.size() + p.size()); }
  std::vector<double> flatten() const;
  static BlockVector split(std::span<const double> x, int nu, int nt, int np);
  double norm2() const;
};

struct BlockSystem {
  CsrMatrix A, C1, Q1, C2, H, Q2, T, F_u;
  int n_u = 0, n_t = 0, n_p = 0;
  int total_dimension() const { return n_u + n_t + n_p; }
  void check_shapes() const;
  BlockVector apply(const BlockVector& x) const;
};

class BlockSystemOperator : public LinearOperator {
 public:
  explicit BlockSystemOperator(const BlockSystem& J) : J_(&J) {}
  int dimension() const override { return J_->total_dimension(); }
  void apply(std::span<const double> x, std::span<double> y) const override;
 private:
  const BlockSystem* J_;
};

// ---------------------------------------------------------------- gmres.hpp:15-33
struct SolveStats {
  int iterations = 0;
  std::vector<double> relative_residuals;
  bool converged = false;
  bool breakdown = false;
  int restarts = 0;         // extension: GMRES(m) wrapper
  int precond_applies = 0;  // extension: bookkeeping
};

std::pair<std::vector<double>, SolveStats> gmres(
    const LinearOperator& op, const LinearOperator* precond, std::span<const double> b,
    double tol, int max_iter = 500, std::vector<std::vector<double>>* basis_out = nullptr);

// OPTION (off by default): GMRES dot products and norms as fixed 32768-entry chunk sums added in
// chunk order (deterministic, thread-count independent; not the reference's single left-to-right
// sum).  For the large-config tests and the timed CPU legs of bench.py (gmres.cpp).
void set_chunked_reductions(bool on);
bool chunked_reductions();

// GMRES(m): restart wrapper around the reference algorithm.
//   r = b - op(x); if ||r|| <= tol ||b|| stop; else run gmres() on r with
//   max_iter = min(m, remaining) and tol' = tol ||b|| / ||r||; x += dx.
std::pair<std::vector<double>, SolveStats> gmres_restarted(
    const LinearOperator& op, const LinearOperator* precond, std::span<const double> b,
    double tol, int restart, int max_iter);

// ------------------------------------------------------------- dense factors
// FullPivLU restatement (amg.hpp:49, amg.cpp:144-149,284-289, precond.cpp:273-278)
struct DenseFullPivLU {
  int n = 0, rank = 0;
  std::vector<double> lu;   // row-major n x n: unit-lower L below, U on/above diagonal
  std::vector<int> prow;    // c_i = b[prow[i]]
  std::vector<int> pcol;    // x[pcol[i]] = c_i
  void compute(const std::vector<double>& a_rowmajor, int n);
  bool is_invertible() const { return rank == n; }
  std::vector<double> solve(std::span<const double> b) const;
};

// Banded exact factor: restatement of SparseFactor (sparse_factor.cpp:30-67).
// The matrix is split into independent diagonal blocks (no entry couples two
// blocks); each block is factored in natural order inside its band.
//   kind spd     -> LDL^T (no pivoting)          [SimplicialLDLT semantics]
//   kind general -> LU with partial row pivoting [SparseLU semantics]
struct BandFactor {
  enum class Kind { spd, general };
  Kind kind = Kind::spd;
  int n = 0;
  int kl = 0;  // lower bandwidth of L (multipliers per column)
  int ku = 0;  // upper bandwidth of U (entries above the diagonal per column), 0 for spd
  std::vector<int> block_start;  // size n_blocks+1
  // L multipliers by column: Lc[j*kl + r] = L(j+1+r, j) (after pivoting for LU)
  std::vector<double> Lc;
  // spd:  D[j]                          general: U diagonal
  std::vector<double> diag;
  // spd: Lr[j*kl + r] = L(j, j-1-r)  (rows of L, for the backward sweep with L^T)
  // general: Uc[j*ku + r] = U(j-1-r, j)  (columns of U, for the backward sweep)
  std::vector<double> Lr, Uc;
  std::vector<int> piv;  // general: row swapped with j at step j (absolute index)
  // factor_solve = inverse: the explicit inverse of every
  // diagonal block, row-major, block blk at inv_off[blk]; column c is the sweep
  // solve of the unit vector e_c.  When present, solve() is the block GEMV
  // x_i = sum_c inv(i,c) b_c instead of the sweeps, summed as 32 partials over
  // c = j (mod 32) (c ascending, from 0.0) combined by an xor tree (factor.cpp).
  std::vector<double> inv;
  std::vector<size_t> inv_off;
  // factor_solve = panel (only without row interchanges): each block split into panels
  // of p_b rows, p_b = max(lower bandwidth of its L, upper bandwidth of its U) from the stored
  // nonzeros, so L and U are block bidiagonal.  Per panel q (s_q rows):
  //   H_q = L_qq^-1,  G_q = L_qq^-1 L_q,q-1      (forward:  y_q = H_q b_q - G_q y_q-1)
  //   K_q = U_qq^-1,  F_q = U_qq^-1 U_q,q+1      (backward: x_q = K_q z_q - F_q x_q+1)
  // (spd: U = L^T unit, z = y / D; general: z = y).  Each is built by the column sweeps of
  // solve_block applied to the columns of I or of the coupling block; each row product is summed as
  // 32 lane-strided partials (columns c = j mod 32 ascending, from 0.0) and the xor tree, the two
  // products of a row combined as (H b) - (G y).  Row-major dense s_q x s_q (H, K), s_q x s_q-1 (G),
  // s_q x s_q+1 (F) per panel, stacked per block at pan_off[blk].
  std::vector<int> pan_p;                 // per block: panel size
  std::vector<size_t> pan_off;            // per block: offset of its panel matrices in pan
  std::vector<double> pan;                // per block, per panel: H, G, K, F
  bool pivots() const;                    // general: any row interchange (panel mode unavailable)
  void build_panels();
  void factor(const CsrMatrix& A, Kind k);
  void build_inverse();
  void solve_block(int blk, double* x) const;  // sweeps on one block, in place
  std::vector<double> solve(std::span<const double> b) const;
};

// ---------------------------------------------------------------- amg.hpp:19-69
struct AmgConfig {
  double strength_threshold = 0.08;
  int max_coarse = 100;
  int pre_sweeps = 1, post_sweeps = 1;
  // chebyshev: EXTENSION (a non-goal of the reference), see amg.cpp
  // mcgs: EXTENSION — multicolour symmetric Gauss-Seidel: the reference's SGS
  // update (amg.cpp:115-134) with rows visited colour by colour (a greedy colouring in index order),
  // forward colours then backward colours; rows of one colour never reference each other, so each
  // colour is one parallel pass on the GPU.  A different operator from lexicographic SGS (amg.cpp).
  enum class Smoother { weighted_jacobi, sgs, chebyshev, mcgs };
  Smoother smoother = Smoother::sgs;
  int chebyshev_degree = 2;        // polynomial degree per sweep
  double chebyshev_ratio = 10.0;   // lambda_min = lambda_max / ratio
  int power_iterations = 10;       // lambda_max estimate of D^-1 A at setup
  bool prolongation_smoothing = true;
  int cycles_per_apply = 1;
  double jacobi_omega = 2.0 / 3.0;
  double stall_ratio = 0.9;
  int max_levels = 25;
  // EXTENSION: row-sum order of the coarse operators.  0 = ordered, the
  // reference's spmv / spmv_transpose order everywhere.  1 = strided32 for A_l (l >= 1) and the
  // restrictions R_l = P_l^T: spmv_strided32 (32 lane-strided partials + xor tree).
  int row_sum = 0;
};

struct AmgLevel {
  CsrMatrix A;
  CsrMatrix P;  // from this level to the previous finer one
  CsrMatrix R;  // P^T (counting transpose), present when config.row_sum = strided32
  std::vector<double> smoother_diag;
  double lambda_max = 0.0;  // chebyshev: 1.1 x power-iteration estimate of rho(D^-1 A)
  std::vector<int> fine_aggregate;
  std::vector<int> aggregate_offsets;
  // mcgs: rows grouped by colour (ascending inside a colour), colour c = color_rows[color_off[c] ..)
  std::vector<int> color_rows, color_off;
};
// EXTENSION (mcgs): greedy colouring in index order of the pattern of A + A^T — row i takes the
// smallest colour not used by its already coloured neighbours (j < i with an entry (i, j) or (j, i)), so
// rows of one colour never reference each other; returns the rows grouped by colour
void greedy_coloring(const CsrMatrix& A, std::vector<int>& rows, std::vector<int>& off);

struct AmgHierarchy {
  std::vector<AmgLevel> levels;
  DenseFullPivLU coarse_factor;
  std::vector<std::vector<double>> near_null;
  AmgConfig config;
  int fine_dimension() const { return levels.empty() ? 0 : levels.front().A.n_rows; }
  int num_levels() const { return int(levels.size()); }
};

// A is taken by value (amg.hpp:58 takes a const reference): callers that no longer need the
// operator move it in, so the hierarchy does not hold a second copy of a 25 GB config-5 operator
AmgHierarchy amg_setup(CsrMatrix A, const std::vector<std::vector<double>>& near_null,
                       const AmgConfig& cfg);
std::vector<double> amg_apply(const AmgHierarchy& h, std::span<const double> r);
// EXTENSION: switch the coarse operators' row-sum order (builds / drops the levels' R = P^T)
void amg_set_row_sum(AmgHierarchy& h, int row_sum);
std::vector<std::vector<double>> constant_near_null(int n);
// Chebyshev smoother support (extension): estimate and coefficients shared with the GPU path
double chebyshev_lambda_max(const CsrMatrix& A, std::span<const double> diag, int iterations);
struct ChebyshevCoefficients {
  double theta = 0.0;           // (lambda_max + lambda_min) / 2 ; step 0: d = (r / D) / theta
  std::vector<double> c1, c2;   // step k >= 1: d = c1[k] d + c2[k] (r / D)
};
ChebyshevCoefficients chebyshev_coefficients(double lambda_max, double ratio, int degree);
std::vector<std::vector<double>> rigid_body_modes(std::span<const std::array<double, 3>> coords);

// Column-pivoted Householder QR of a column-major m x k block (restates the
// Eigen::ColPivHouseholderQR use at amg.cpp:228-243).  Returns rank, Q (m x rank,
// column-major) and Rp = R(0:rank,:) * P^T (rank x k, row-major).
int qr_colpiv(int m, int k, const std::vector<double>& B_colmajor, std::vector<double>& Q,
              std::vector<double>& Rp);

// ------------------------------------------------------------- precond.hpp:19-116
struct PrecondConfig {
  enum class Variant { tpu, tup, tup_star };
  enum class Inner { amg, direct };
  Variant variant = Variant::tup;
  Inner inner = Inner::amg;
  AmgConfig amg;
};

struct InnerSolver {
  std::shared_ptr<AmgHierarchy> amg;
  std::shared_ptr<DenseFullPivLU> direct;  // restated SparseFactor(general) for small tests
  std::shared_ptr<std::atomic<long>> calls = std::make_shared<std::atomic<long>>(0);
  std::vector<double> apply(std::span<const double> r) const;
  long call_count() const { return calls->load(); }
  void reset_count() const { calls->store(0); }
};

struct HSurrogate {
  BlockDiagonal3 block_diag;
  std::vector<double> solve(std::span<const double> w) const { return bdiag3_solve(block_diag, w); }
};

struct TpuPreconditioner {
  HSurrogate Hs;
  BandFactor T_factor;
  std::vector<double> T_diag;
  CsrMatrix S;
  InnerSolver S_solver;
};

struct TupPreconditioner {
  HSurrogate Hs;
  CsrMatrix S1;
  InnerSolver S1_solver;
  std::vector<double> S_K;
  CsrMatrix S2;
  BandFactor S2_factor;
  std::vector<double> s2_solve(std::span<const double> w) const { return S2_factor.solve(w); }
};

TpuPreconditioner build_tpu(const BlockSystem& J, const PrecondConfig& cfg,
                            std::span<const std::array<double, 3>> coords = {});
BlockVector apply_tpu(const TpuPreconditioner& M, const BlockSystem& J, const BlockVector& w);
TupPreconditioner build_tup(const BlockSystem& J, const PrecondConfig& cfg,
                            std::span<const std::array<double, 3>> coords = {});
BlockVector apply_tup(const TupPreconditioner& M, const BlockSystem& J, const BlockVector& w);
BlockVector apply_tup_star(const TupPreconditioner& M, const BlockSystem& J, const BlockVector& w);
std::vector<double> fixed_stress_diag(const CsrMatrix& Q2, const CsrMatrix& S1, const CsrMatrix& Q1);

class TpuOperator : public LinearOperator {
 public:
  TpuOperator(const TpuPreconditioner& M, const BlockSystem& J) : M_(&M), J_(&J) {}
  int dimension() const override { return J_->total_dimension(); }
  void apply(std::span<const double> x, std::span<double> y) const override;
 private:
  const TpuPreconditioner* M_;
  const BlockSystem* J_;
};

class TupOperator : public LinearOperator {
 public:
  TupOperator(const TupPreconditioner& M, const BlockSystem& J, bool star = false)
      : M_(&M), J_(&J), star_(star) {}
  int dimension() const override { return J_->total_dimension(); }
  void apply(std::span<const double> x, std::span<double> y) const override;
 private:
  const TupPreconditioner* M_;
  const BlockSystem* J_;
  bool star_;
};

// --------------------------------------------------------- driver.cpp:104-141
struct BlockScaling {
  double st = 1.0, sp = 1.0;
  int n_u = 0, n_t = 0, n_p = 0;
  static BlockScaling from(const BlockSystem& J);
  void scale(std::vector<double>& v, bool inverse) const;
};

// The driver's scaled operators (driver.cpp:233-248): op = D J D, precond = D^-1 M D^-1.
class ScaledOperator : public LinearOperator {
 public:
  ScaledOperator(const LinearOperator& inner, const BlockScaling& D, bool inverse)
      : in_(&inner), D_(D), inv_(inverse) {}
  int dimension() const override { return in_->dimension(); }
  void apply(std::span<const double> x, std::span<double> y) const override;
 private:
  const LinearOperator* in_;
  BlockScaling D_;
  bool inv_;
};

// ------------------------------------------------ test_helpers.hpp:15-200 fixtures
CsrMatrix spd_tridiagonal(int n, double diag = 4.0, double off = -1.0);
CsrMatrix poisson1d(int n);
CsrMatrix poisson3d(int m);
enum class ToyMode { decoupled, stick, mixed, open_all };
BlockSystem toy_system(int n_u, int n_p, ToyMode mode, unsigned seed = 99);

}  // namespace fpo
