// fracprec_b200.hpp — header-only C++ adapter over the C ABI, shaped like the
// reference's solve-path API so reference C++ callers switch by changing types:
//
//   reference (proj/core/include/fracprec/)          this header (namespace fracprec_b200)
//   BlockSystemOperator(J)   block.hpp:48-57      -> GpuSystemOperator(view of J)
//   build_tup(J,cfg,coords)  precond.hpp:80-82    -> build_tup(system, view of J, cfg, coords)
//   TupOperator(M, J)        precond.hpp:105-116  -> GpuPrecondOperator (apply(span, span))
//   gmres(op, &M, b, tol)    gmres.hpp:29-33      -> gmres(system, precond, b, tol, max_iter, restart)
//   numerical_error          errors.hpp:15-18     -> fracprec_b200::numerical_error
//
// apply() takes host spans (as the reference's LinearOperator does); device
// pointers can be passed through apply_device().  No exceptions cross the C
// ABI; this header rethrows its status codes as the reference's exception types.
#ifndef FRACPREC_B200_HPP
#define FRACPREC_B200_HPP

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fracprec_b200.h"

namespace fracprec_b200 {

class numerical_error : public std::runtime_error {
 public:
  explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int status) {
  if (status == FP_OK) return;
  const std::string msg = fp_last_error();
  if (status == FP_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (status == FP_NUMERICAL_ERROR) throw numerical_error(msg);
  throw std::runtime_error(msg);
}

// CSR view in the reference's layout (CsrMatrix: int row offsets, csr.hpp:16-22).
inline fp_csr csr_view(int rows, int cols, const int* row_offsets, const int* col_indices, const double* values) {
  fp_csr v{};
  v.n_rows = rows, v.n_cols = cols;
  v.row_offsets32 = row_offsets;
  v.col_indices = col_indices;
  v.values = values;
  return v;
}

// Mirror of fracprec::LinearOperator (operator.hpp:17-28).  The GPU operators below are
// templates over their base class, so a reference build derives them from the reference's own
// interface instead: after #include "fracprec/operator.hpp",
//   using GpuSystemOperator = fracprec_b200::GpuSystemOperatorT<fracprec::LinearOperator>;
// and fracprec::gmres(op, &M, b, tol) drives the B200 applies unchanged (
// tests/cpp/oracle_gmres_dropin.cpp does exactly this with the oracle's restated gmres()).
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

// The reference's "spmv: dimension mismatch" / "gmres: rhs dimension mismatch" checks: the C ABI
// reads and writes n doubles through raw pointers, so a short span is rejected before the call.
inline void check_dims(const char* what, size_t n, std::span<const double> x, std::span<double> y) {
  if (x.size() != n || y.size() != n) throw std::invalid_argument(std::string(what) + ": dimension mismatch");
}

// Device-resident J (BlockSystemOperator, block.hpp:48-57).
template <class Base = LinearOperator>
class GpuSystemOperatorT : public Base {
 public:
  explicit GpuSystemOperatorT(const fp_block_system& J) {
    check(fp_system_create(&J, &h_));
    int32_t nu = 0, nt = 0, np = 0;
    check(fp_system_dims(h_, &nu, &nt, &np));
    n_ = nu + nt + np;
  }
  ~GpuSystemOperatorT() override { fp_system_destroy(h_); }
  GpuSystemOperatorT(const GpuSystemOperatorT&) = delete;
  GpuSystemOperatorT& operator=(const GpuSystemOperatorT&) = delete;
  int dimension() const override { return n_; }
  void apply(std::span<const double> x, std::span<double> y) const override {
    check_dims("BlockSystemOperator::apply", size_t(n_), x, y);
    check(fp_system_apply(h_, x.data(), y.data(), FP_MEM_HOST));
  }
  // x, y: device pointers to n = dimension() doubles whose producers have completed
  void apply_device(const double* x, double* y) const { check(fp_system_apply(h_, x, y, FP_MEM_DEVICE)); }
  fp_system* handle() const { return h_; }

 private:
  fp_system* h_ = nullptr;
  int n_ = 0;
};

// Device-resident M^-1 (TpuOperator / TupOperator, precond.hpp:94-116) with the
// inner-solver call counter of InnerSolver (precond.hpp:34-42).
template <class Base = LinearOperator>
class GpuPrecondOperatorT : public Base {
 public:
  template <class SysBase>
  GpuPrecondOperatorT(const GpuSystemOperatorT<SysBase>& sys, fp_precond* h) : h_(h), n_(sys.dimension()) {}
  ~GpuPrecondOperatorT() override { fp_precond_destroy(h_); }
  GpuPrecondOperatorT(const GpuPrecondOperatorT&) = delete;
  GpuPrecondOperatorT& operator=(const GpuPrecondOperatorT&) = delete;
  int dimension() const override { return n_; }
  void apply(std::span<const double> x, std::span<double> y) const override {
    check_dims("TupOperator::apply", size_t(n_), x, y);
    check(fp_precond_apply(h_, x.data(), y.data(), FP_MEM_HOST));
  }
  void apply_device(const double* x, double* y) const { check(fp_precond_apply(h_, x, y, FP_MEM_DEVICE)); }
  long call_count() const { return long(fp_precond_inner_calls(h_, 0)); }
  void reset_count() const { fp_precond_inner_calls(h_, 1); }
  fp_precond* handle() const { return h_; }

 private:
  fp_precond* h_;
  int n_;
};

using GpuSystemOperator = GpuSystemOperatorT<>;
using GpuPrecondOperator = GpuPrecondOperatorT<>;

inline fp_amg_config default_amg() {
  fp_amg_config c;
  fp_amg_config_default(&c);
  return c;
}

// build_tpu / build_tup / t-u-p* (precond.cpp:119-202): host setup, then upload.
template <class Base = LinearOperator, class SysBase>
inline GpuPrecondOperatorT<Base>* build(const GpuSystemOperatorT<SysBase>& sys, const fp_block_system& J,
                                        int variant, const fp_amg_config& amg,
                                        std::span<const std::array<double, 3>> coords = {}) {
  fp_precond_config cfg{variant, amg};
  fp_host_precond* hp = nullptr;
  check(fp_host_precond_build(&J, &cfg, coords.empty() ? nullptr : coords.data()->data(),
                              int32_t(coords.size()), &hp));
  fp_precond* p = nullptr;
  const int st = fp_precond_create(sys.handle(), hp, &p);
  fp_host_precond_destroy(hp);
  check(st);
  return new GpuPrecondOperatorT<Base>(sys, p);
}

struct SolveStats {  // gmres.hpp:15-22
  int iterations = 0;
  std::vector<double> relative_residuals;
  bool converged = false;
  bool breakdown = false;
  int restarts = 0;
  double device_seconds = 0.0;
};

// gmres(op, precond, b, tol, max_iter) (gmres.hpp:29-33); restart >= max_iter is
// the reference's full GMRES; scaled = the driver's D J D system (driver.cpp:229-255).
template <class SysBase, class PcBase>
inline std::pair<std::vector<double>, SolveStats> gmres(const GpuSystemOperatorT<SysBase>& op,
                                                        const GpuPrecondOperatorT<PcBase>& M,
                                                        std::span<const double> b, double tol, int max_iter = 500,
                                                        int restart = 0, bool scaled = false,
                                                        int orthogonalization = FP_ORTH_MGS) {
  if (int(b.size()) != op.dimension()) throw std::invalid_argument("gmres: rhs dimension mismatch");
  if (M.dimension() != op.dimension()) throw std::invalid_argument("gmres: preconditioner dimension mismatch");
  if (!(tol > 0.0)) throw std::invalid_argument("gmres: tol must be positive");
  std::vector<double> x(b.size());
  SolveStats st;
  st.relative_residuals.resize(static_cast<size_t>(std::max(1, max_iter)));
  fp_gmres_options o{tol, restart > 0 ? restart : max_iter, max_iter, scaled ? 1 : 0, orthogonalization};
  fp_solve_stats s{};
  s.residual_history = st.relative_residuals.data();
  s.history_capacity = int32_t(st.relative_residuals.size());
  check(fp_gmres(op.handle(), M.handle(), b.data(), x.data(), FP_MEM_HOST, &o, &s));
  st.iterations = s.iterations;
  st.relative_residuals.resize(static_cast<size_t>(s.history_len));
  st.converged = s.converged != 0;
  st.breakdown = s.breakdown != 0;
  st.restarts = s.restarts;
  st.device_seconds = s.device_seconds;
  return {std::move(x), std::move(st)};
}

}  // namespace fracprec_b200

#endif
