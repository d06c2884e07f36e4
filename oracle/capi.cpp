// ORACLE (test infrastructure only) — flat C entry points so the pytest suite and
// bench.py's CPU-baseline leg can drive the restated reference through ctypes.
// Object handles are heap C++ objects; every call catches exceptions and
// reports them through or_last_error().
#include <chrono>
#include <cstring>
#include <string>

#include "fpo.hpp"
#include "par.hpp"

using namespace fpo;

namespace {
thread_local std::string g_err;

struct Sys {
  BlockSystem J;
};
struct Pc {
  PrecondConfig cfg;
  const Sys* sys = nullptr;
  std::unique_ptr<TpuPreconditioner> tpu;
  std::unique_ptr<TupPreconditioner> tup;
  const InnerSolver& inner() const { return tpu ? tpu->S_solver : tup->S1_solver; }
  const AmgHierarchy& amg() const { return *inner().amg; }
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const numerical_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

CsrMatrix make_csr(int rows, int cols, const int64_t* rp, const int* ci, const double* v) {
  CsrMatrix M(rows, cols);
  if (rows > 0 && rp) M.row_offsets.assign(rp, rp + rows + 1);
  const int64_t nnz = M.row_offsets.back();
  M.col_indices.assign(ci, ci + nnz);
  M.values.assign(v, v + nnz);
  return M;
}

const CsrMatrix* block_of(const BlockSystem& J, int which) {
  switch (which) {
    case 0: return &J.A;
    case 1: return &J.C1;
    case 2: return &J.Q1;
    case 3: return &J.C2;
    case 4: return &J.H;
    case 5: return &J.Q2;
    case 6: return &J.T;
    case 7: return &J.F_u;
  }
  return nullptr;
}

AmgConfig amg_cfg(const double* d, const int* i) {
  AmgConfig c;
  if (d) {
    c.strength_threshold = d[0];
    c.jacobi_omega = d[1];
    c.stall_ratio = d[2];
  }
  if (i) {
    c.max_coarse = i[0];
    c.pre_sweeps = i[1];
    c.post_sweeps = i[2];
    c.smoother = i[3] == 0   ? AmgConfig::Smoother::weighted_jacobi
                 : i[3] == 2 ? AmgConfig::Smoother::chebyshev
                 : i[3] == 3 ? AmgConfig::Smoother::mcgs
                             : AmgConfig::Smoother::sgs;
    c.prolongation_smoothing = i[4] != 0;
    c.cycles_per_apply = i[5];
    c.max_levels = i[6];
    c.chebyshev_degree = i[7];
    c.power_iterations = i[8];
  }
  if (d) c.chebyshev_ratio = d[3];
  return c;
}
}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

// threads of the oracle's row / block / aggregate loops (par.hpp: results do not depend on it)
void or_set_threads(int n) { fpo::set_threads(n); }
int or_threads() { return fpo::threads(); }
// GMRES dots as fixed-chunk sums (fpo::set_chunked_reductions; off = the reference's single sum)
void or_set_chunked_reductions(int on) { fpo::set_chunked_reductions(on != 0); }

// ------------------------------------------------------------------ systems
// blocks: 8 CSR views in the order A, C1, Q1, C2, H, Q2, T, F_u (F_u may be empty)
int or_system_create(int nu, int nt, int np, const int64_t* const* rp, const int* const* ci,
                     const double* const* v, const int* rows, const int* cols, void** out) {
  return guard([&] {
    auto* s = new Sys;
    BlockSystem& J = s->J;
    J.n_u = nu, J.n_t = nt, J.n_p = np;
    CsrMatrix* dst[8] = {&J.A, &J.C1, &J.Q1, &J.C2, &J.H, &J.Q2, &J.T, &J.F_u};
    for (int b = 0; b < 8; ++b) *dst[b] = make_csr(rows[b], cols[b], rp[b], ci[b], v[b]);
    try {
      J.check_shapes();
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int or_system_toy(int nu, int np, int mode, unsigned seed, void** out) {
  return guard([&] {
    auto* s = new Sys;
    s->J = toy_system(nu, np, ToyMode(mode), seed);
    *out = s;
  });
}

void or_system_destroy(void* s) { delete static_cast<Sys*>(s); }

int or_system_dims(void* s, int* nu, int* nt, int* np) {
  const BlockSystem& J = static_cast<Sys*>(s)->J;
  *nu = J.n_u, *nt = J.n_t, *np = J.n_p;
  return 0;
}

const void* or_system_block(void* s, int which) { return block_of(static_cast<Sys*>(s)->J, which); }

int or_system_apply(void* s, const double* x, double* y) {
  return guard([&] {
    const BlockSystem& J = static_cast<Sys*>(s)->J;
    BlockSystemOperator op(J);
    op.apply({x, size_t(J.total_dimension())}, {y, size_t(J.total_dimension())});
  });
}

// -------------------------------------------------------------------- CSR
// Matrix Market (mmio.cpp:15-59): the CSR handle is owned by the caller (or_csr_destroy)
int or_mm_read(const char* path, void** out) {
  return guard([&] { *out = new CsrMatrix(read_matrix_market(path)); });
}
void or_csr_destroy(void* m) { delete static_cast<CsrMatrix*>(m); }
int or_mm_write(const char* path, int rows, int cols, const int64_t* rp, const int* ci, const double* v) {
  return guard([&] {
    CsrMatrix A(rows, cols);
    A.row_offsets.assign(rp, rp + rows + 1);
    A.col_indices.assign(ci, ci + rp[rows]);
    A.values.assign(v, v + rp[rows]);
    write_matrix_market(path, A);
  });
}

int or_csr_info(const void* m, int* rows, int* cols, int64_t* nnz) {
  const auto* M = static_cast<const CsrMatrix*>(m);
  if (!M) return 1;
  *rows = M->n_rows, *cols = M->n_cols, *nnz = M->nnz();
  return 0;
}
int or_csr_copy(const void* m, int64_t* rp, int* ci, double* v) {
  const auto* M = static_cast<const CsrMatrix*>(m);
  std::memcpy(rp, M->row_offsets.data(), sizeof(int64_t) * M->row_offsets.size());
  std::memcpy(ci, M->col_indices.data(), sizeof(int) * M->col_indices.size());
  std::memcpy(v, M->values.data(), sizeof(double) * M->values.size());
  return 0;
}

// --------------------------------------------------------------- precond
// variant 0 tpu, 1 tup, 2 tup_star; inner 0 amg, 1 direct.
// amg_d = {strength_threshold, jacobi_omega, stall_ratio, chebyshev_ratio}
// amg_i = {max_coarse, pre, post, smoother(0 jacobi,1 sgs,2 chebyshev,3 mcgs), prolongation_smoothing, cycles, max_levels,
//          chebyshev_degree, power_iterations}
int or_precond_build(void* s, int variant, int inner, const double* amg_d, const int* amg_i,
                     const double* coords, int n_nodes, void** out) {
  return guard([&] {
    auto* pc = new Pc;
    pc->sys = static_cast<Sys*>(s);
    pc->cfg.variant = PrecondConfig::Variant(variant);
    pc->cfg.inner = PrecondConfig::Inner(inner);
    pc->cfg.amg = amg_cfg(amg_d, amg_i);
    std::vector<std::array<double, 3>> xyz;
    for (int v = 0; coords && v < n_nodes; ++v) xyz.push_back({coords[3 * v], coords[3 * v + 1], coords[3 * v + 2]});
    try {
      if (variant == 0)
        pc->tpu = std::make_unique<TpuPreconditioner>(build_tpu(pc->sys->J, pc->cfg, xyz));
      else
        pc->tup = std::make_unique<TupPreconditioner>(build_tup(pc->sys->J, pc->cfg, xyz));
    } catch (...) {
      delete pc;
      throw;
    }
    *out = pc;
  });
}

void or_precond_destroy(void* p) { delete static_cast<Pc*>(p); }

// factor_solve: 0 = sweeps (SparseFactor::solve), 1 = explicit block inverse,
// 2 = panels (a factor without row interchanges)
int or_precond_set_factor_solve(void* p, int mode) {
  return guard([&] {
    Pc* pc = static_cast<Pc*>(p);
    BandFactor& F = pc->tpu ? pc->tpu->T_factor : pc->tup->S2_factor;
    if (mode == 1) {
      if (F.inv.empty()) F.build_inverse();
    } else {
      F.inv.clear(), F.inv_off.clear();
    }
    if (mode == 2) {
      if (F.pan.empty()) F.build_panels();
    } else {
      F.pan.clear(), F.pan_off.clear(), F.pan_p.clear();
    }
  });
}

// 1 when the factor took row interchanges (panel mode unavailable)
int or_precond_factor_pivots(void* p) {
  const Pc* pc = static_cast<Pc*>(p);
  const BandFactor& F = pc->tpu ? pc->tpu->T_factor : pc->tup->S2_factor;
  return F.pivots() ? 1 : 0;
}

// row_sum: 0 = ordered (reference), 1 = strided32 on the coarse operators
int or_precond_set_row_sum(void* p, int mode) {
  return guard([&] {
    Pc* pc = static_cast<Pc*>(p);
    InnerSolver& S = pc->tpu ? pc->tpu->S_solver : pc->tup->S1_solver;
    if (!S.amg) throw std::invalid_argument("or_precond_set_row_sum: no AMG inner solver");
    amg_set_row_sum(*S.amg, mode);
  });
}

int or_precond_apply(void* p, const double* x, double* y) {
  return guard([&] {
    const Pc* pc = static_cast<Pc*>(p);
    const BlockSystem& J = pc->sys->J;
    const size_t n = size_t(J.total_dimension());
    if (pc->tpu)
      TpuOperator(*pc->tpu, J).apply({x, n}, {y, n});
    else
      TupOperator(*pc->tup, J, pc->cfg.variant == PrecondConfig::Variant::tup_star).apply({x, n}, {y, n});
  });
}

long or_precond_inner_calls(void* p, int reset) {
  const Pc* pc = static_cast<Pc*>(p);
  const long c = pc->inner().call_count();
  if (reset) pc->inner().reset_count();
  return c;
}

// Exported pieces of the built preconditioner (the "reference-built" data the
// GPU uploads).  which: 0 = S (tpu) / S1 (tup), 1 = T (tpu) / S2 (tup)
const void* or_precond_matrix(void* p, int which) {
  const Pc* pc = static_cast<Pc*>(p);
  // the inner operator S~ / S1 lives in the AMG hierarchy's level 0 (the preconditioner drops its copy)
  if (pc->tpu)
    return which == 0 ? (pc->tpu->S_solver.amg ? &pc->tpu->S_solver.amg->levels[0].A : &pc->tpu->S) : &pc->sys->J.T;
  return which == 0 ? (pc->tup->S1_solver.amg ? &pc->tup->S1_solver.amg->levels[0].A : &pc->tup->S1) : &pc->tup->S2;
}
int or_precond_hblocks(void* p, double* out) {  // n_p * 9 raw (regularized) H~ blocks
  const Pc* pc = static_cast<Pc*>(p);
  const BlockDiagonal3& B = pc->tpu ? pc->tpu->Hs.block_diag : pc->tup->Hs.block_diag;
  std::memcpy(out, B.blocks.data(), sizeof(double) * B.blocks.size());
  return 0;
}
int or_precond_vec(void* p, int which, double* out) {  // 0: T_diag (tpu) / S_K (tup)
  const Pc* pc = static_cast<Pc*>(p);
  const std::vector<double>& v = pc->tpu ? pc->tpu->T_diag : pc->tup->S_K;
  (void)which;
  std::memcpy(out, v.data(), sizeof(double) * v.size());
  return int(v.size());
}
int or_amg_levels(void* p) { return static_cast<Pc*>(p)->amg().num_levels(); }
// which: 0 = A_l, 1 = P_l (l >= 1)
const void* or_amg_level_matrix(void* p, int l, int which) {
  const AmgLevel& L = static_cast<Pc*>(p)->amg().levels[size_t(l)];
  return which == 0 ? &L.A : &L.P;
}
double or_amg_level_lambda(void* p, int level) {
  const Pc* pc = static_cast<Pc*>(p);
  const auto& h = *pc->inner().amg;
  return level >= 0 && level < int(h.levels.size()) ? h.levels[level].lambda_max : -1.0;
}

int or_amg_level_diag(void* p, int l, double* out) {
  const AmgLevel& L = static_cast<Pc*>(p)->amg().levels[size_t(l)];
  std::memcpy(out, L.smoother_diag.data(), sizeof(double) * L.smoother_diag.size());
  return int(L.smoother_diag.size());
}
int or_amg_level_aggregates(void* p, int l, int* out) {
  const AmgLevel& L = static_cast<Pc*>(p)->amg().levels[size_t(l)];
  std::memcpy(out, L.fine_aggregate.data(), sizeof(int) * L.fine_aggregate.size());
  return int(L.fine_aggregate.size());
}
// mcgs (extension): colour count of a level, and its rows grouped by colour (color_rows / color_off)
int or_amg_level_colors(void* p, int l, int* rows, int* off) {
  const AmgLevel& L = static_cast<Pc*>(p)->amg().levels[l];
  if (rows) std::copy(L.color_rows.begin(), L.color_rows.end(), rows);
  if (off) std::copy(L.color_off.begin(), L.color_off.end(), off);
  return int(L.color_off.size()) - 1;
}

int or_amg_apply(void* p, const double* r, double* x) {
  return guard([&] {
    const AmgHierarchy& h = static_cast<Pc*>(p)->amg();
    const auto y = amg_apply(h, {r, size_t(h.fine_dimension())});
    std::memcpy(x, y.data(), sizeof(double) * y.size());
  });
}

// ------------------------------------------------------------------ solve
// Scaled solve as the driver does it (driver.cpp:229-255): op = D J D,
// precond = D^-1 M D^-1, b given for the scaled system, GMRES(restart).
// stats = {iterations, converged, breakdown, restarts, precond_applies}
int or_gmres(void* s, void* p, const double* b, double tol, int restart, int max_iter, int scaled,
             double* x, int* stats, double* hist, int hist_cap, double* seconds) {
  return guard([&] {
    const BlockSystem& J = static_cast<Sys*>(s)->J;
    const Pc* pc = static_cast<Pc*>(p);
    const int n = J.total_dimension();
    BlockSystemOperator Jop(J);
    std::unique_ptr<LinearOperator> M;
    if (pc) {
      if (pc->tpu)
        M = std::make_unique<TpuOperator>(*pc->tpu, J);
      else
        M = std::make_unique<TupOperator>(*pc->tup, J, pc->cfg.variant == PrecondConfig::Variant::tup_star);
    }
    BlockScaling D = BlockScaling::from(J);
    if (!scaled) D.st = D.sp = 1.0;
    ScaledOperator op(Jop, D, false);
    std::unique_ptr<ScaledOperator> pre;
    if (M) pre = std::make_unique<ScaledOperator>(*M, D, true);
    const auto t0 = std::chrono::steady_clock::now();
    auto [sol, st] = restart > 0 ? gmres_restarted(op, pre.get(), {b, size_t(n)}, tol, restart, max_iter)
                                 : gmres(op, pre.get(), {b, size_t(n)}, tol, max_iter);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(x, sol.data(), sizeof(double) * size_t(n));
    stats[0] = st.iterations;
    stats[1] = st.converged;
    stats[2] = st.breakdown;
    stats[3] = st.restarts;
    stats[4] = st.precond_applies;
    for (int i = 0; hist && i < hist_cap && i < int(st.relative_residuals.size()); ++i) hist[i] = st.relative_residuals[i];
  });
}

int or_block_scaling(void* s, double* st_sp) {
  const BlockScaling D = BlockScaling::from(static_cast<Sys*>(s)->J);
  st_sp[0] = D.st;
  st_sp[1] = D.sp;
  return 0;
}

}  // extern "C"
