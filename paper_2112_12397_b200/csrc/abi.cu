// C ABI of the B200 solve path (include/fracprec_b200.h).  No exception crosses
// the boundary: every entry point maps std::invalid_argument /
// numerical_error / CUDA failures to status codes (errors.hpp:15-24 of the
// reference; fracprec.cpp:453-465 maps them to CLI exit codes the same way).
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <span>
#include <string>

#include "../../include/fracprec_b200.h"
#include "device/engine.cuh"
#include "host/setup.hpp"
#include "../../include/fracprec_workload.h"
#include "workload.hpp"  // workload/ (libfp_workload.so): the fp_workload handle

namespace {

thread_local std::string g_err;

struct cuda_failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return FP_OK;
  } catch (const fpb::numerical_error& e) {
    g_err = e.what();
    return FP_NUMERICAL_ERROR;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FP_INVALID_ARGUMENT;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("allocation failure: ") + e.what();
    return FP_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return std::strstr(e.what(), "CUDA") ? FP_CUDA_ERROR : FP_INTERNAL_ERROR;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

fpb::Csr to_csr(const fp_csr& m, const char* name) {
  const std::string nm(name);
  need(m.n_rows >= 0 && m.n_cols >= 0, (nm + ": negative dimension").c_str());
  fpb::Csr A(m.n_rows, m.n_cols);
  if (m.n_rows == 0) return A;
  need((m.row_offsets32 != nullptr) != (m.row_offsets64 != nullptr),
       (nm + ": exactly one of row_offsets32 / row_offsets64 must be set").c_str());
  for (int i = 0; i <= m.n_rows; ++i) A.rp[i] = m.row_offsets32 ? int64_t(m.row_offsets32[i]) : m.row_offsets64[i];
  need(A.rp[0] == 0, (nm + ": row_offsets[0] != 0").c_str());
  const int64_t nnz = A.rp[m.n_rows];
  for (int i = 0; i < m.n_rows; ++i) need(A.rp[i] <= A.rp[i + 1], (nm + ": row_offsets not monotone").c_str());
  need(nnz == 0 || (m.col_indices && m.values), (nm + ": null column/value array").c_str());
  A.ci.assign(m.col_indices, m.col_indices + nnz);
  A.v.assign(m.values, m.values + nnz);
  for (int i = 0; i < m.n_rows; ++i)
    for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
      need(A.ci[k] >= 0 && A.ci[k] < m.n_cols, (nm + ": column out of range").c_str());
      if (k > A.rp[i]) need(A.ci[k - 1] < A.ci[k], (nm + ": columns not strictly increasing within a row").c_str());
    }
  return A;
}

fpb::HostSystem to_system(const fp_block_system& J) {
  fpb::HostSystem H;
  H.n_u = J.n_u, H.n_t = J.n_t, H.n_p = J.n_p;
  H.A = to_csr(J.A, "A");
  H.C1 = to_csr(J.C1, "C1");
  H.Q1 = to_csr(J.Q1, "Q1");
  H.C2 = to_csr(J.C2, "C2");
  H.H = to_csr(J.H, "H");
  H.Q2 = to_csr(J.Q2, "Q2");
  H.T = to_csr(J.T, "T");
  H.F_u = to_csr(J.F_u, "F_u");
  H.check_shapes();
  return H;
}

// The C ABI's CSR views validated in place (row-parallel) and borrowed for an upload: no copy of
// the entries (config 5's A alone is 25 GB).  32-bit row offsets are widened into `hold`.
struct ViewHold {
  std::vector<std::vector<int64_t>> widened;
};

fpd::HostCsrView checked_view(const fp_csr& m, const char* name, ViewHold& hold) {
  const std::string nm(name);
  need(m.n_rows >= 0 && m.n_cols >= 0, (nm + ": negative dimension").c_str());
  fpd::HostCsrView v;
  v.n_rows = m.n_rows, v.n_cols = m.n_cols;
  if (m.n_rows == 0) {
    hold.widened.emplace_back(1, 0);
    v.rp = hold.widened.back().data();
    return v;
  }
  need((m.row_offsets32 != nullptr) != (m.row_offsets64 != nullptr),
       (nm + ": exactly one of row_offsets32 / row_offsets64 must be set").c_str());
  if (m.row_offsets32) {
    hold.widened.emplace_back(m.row_offsets32, m.row_offsets32 + m.n_rows + 1);
    v.rp = hold.widened.back().data();
  } else {
    v.rp = m.row_offsets64;
  }
  need(v.rp[0] == 0, (nm + ": row_offsets[0] != 0").c_str());
  need(v.rp[m.n_rows] == 0 || (m.col_indices && m.values), (nm + ": null column/value array").c_str());
  v.ci = m.col_indices, v.v = m.values;
  int bad = 0;  // 1 monotone, 2 range, 3 order: the first failing row reports, like the sequential check
  long first = LONG_MAX;
#pragma omp parallel for schedule(static) reduction(min : first)
  for (long i = 0; i < m.n_rows; ++i) {
    int why = 0;
    if (v.rp[i] > v.rp[i + 1]) why = 1;
    for (int64_t k = v.rp[i]; k < v.rp[i + 1] && !why; ++k) {
      if (v.ci[k] < 0 || v.ci[k] >= m.n_cols) why = 2;
      else if (k > v.rp[i] && v.ci[k - 1] >= v.ci[k]) why = 3;
    }
    if (why && i < first) first = i;
  }
  if (first != LONG_MAX) {
    const long i = first;
    bad = v.rp[i] > v.rp[i + 1] ? 1 : 0;
    for (int64_t k = v.rp[i]; k < v.rp[i + 1] && !bad; ++k)
      bad = (v.ci[k] < 0 || v.ci[k] >= m.n_cols) ? 2 : (k > v.rp[i] && v.ci[k - 1] >= v.ci[k]) ? 3 : 0;
  }
  need(bad != 1, (nm + ": row_offsets not monotone").c_str());
  need(bad != 2, (nm + ": column out of range").c_str());
  need(bad != 3, (nm + ": columns not strictly increasing within a row").c_str());
  return v;
}

fpd::SystemView checked_system(const fp_block_system& J, ViewHold& hold) {
  hold.widened.reserve(8);
  fpd::SystemView S;
  S.n_u = J.n_u, S.n_t = J.n_t, S.n_p = J.n_p;
  S.A = checked_view(J.A, "A", hold);
  S.C1 = checked_view(J.C1, "C1", hold);
  S.Q1 = checked_view(J.Q1, "Q1", hold);
  S.C2 = checked_view(J.C2, "C2", hold);
  S.H = checked_view(J.H, "H", hold);
  S.Q2 = checked_view(J.Q2, "Q2", hold);
  S.T = checked_view(J.T, "T", hold);
  S.F_u = checked_view(J.F_u, "F_u", hold);
  auto expect = [](const fpd::HostCsrView& M, int r, int c, const char* name) {
    if (M.n_rows != r || M.n_cols != c)
      throw std::invalid_argument(std::string("BlockSystem: bad shape for block ") + name);
  };
  expect(S.A, S.n_u, S.n_u, "A");
  expect(S.C1, S.n_u, S.n_t, "C1");
  expect(S.Q1, S.n_u, S.n_p, "Q1");
  expect(S.C2, S.n_t, S.n_u, "C2");
  expect(S.H, S.n_t, S.n_t, "H");
  expect(S.Q2, S.n_p, S.n_u, "Q2");
  expect(S.T, S.n_p, S.n_p, "T");
  if (S.F_u.n_rows > 0) expect(S.F_u, S.n_p, S.n_u, "F_u");
  if (S.n_t != 3 * S.n_p) throw std::invalid_argument("BlockSystem: n_t must equal 3*n_p");
  return S;
}

fpb::AmgOptions to_amg(const fp_amg_config& c) {
  fpb::AmgOptions o;
  o.strength_threshold = c.strength_threshold;
  o.max_coarse = c.max_coarse;
  o.pre_sweeps = c.pre_sweeps;
  o.post_sweeps = c.post_sweeps;
  o.smoother = c.smoother;
  o.prolongation_smoothing = c.prolongation_smoothing != 0;
  o.cycles_per_apply = c.cycles_per_apply;
  o.jacobi_omega = c.jacobi_omega;
  o.stall_ratio = c.stall_ratio;
  o.max_levels = c.max_levels;
  o.chebyshev_degree = c.chebyshev_degree;
  o.chebyshev_ratio = c.chebyshev_ratio;
  o.power_iterations = c.power_iterations;
  o.row_sum = c.row_sum;
  need(o.row_sum == FP_ROW_SUM_ORDERED || o.row_sum == FP_ROW_SUM_STRIDED, "AmgConfig: unknown row_sum");
  need(o.smoother >= 0 && o.smoother <= 3, "AmgConfig: unknown smoother");
  need(o.smoother != 2 || (o.chebyshev_degree >= 1 && o.chebyshev_ratio > 1.0 && o.power_iterations >= 1),
       "AmgConfig: chebyshev needs degree >= 1, ratio > 1, power_iterations >= 1");
  return o;
}

fp_csr view_of(const fpb::Csr& A) {
  fp_csr v{};
  v.n_rows = A.n_rows, v.n_cols = A.n_cols;
  v.row_offsets64 = A.rp.data();
  v.col_indices = A.ci.data();
  v.values = A.v.data();
  return v;
}

}  // namespace

struct fp_system {
  std::unique_ptr<fpd::DeviceSystem> dev;
  cudaStream_t stream = nullptr;
  fpd::DevBuf<double> xin, yout;
  ~fp_system() {
    dev.reset();
    if (stream) cudaStreamDestroy(stream);
  }
};

struct fp_precond {
  fp_system* sys = nullptr;
  std::unique_ptr<fpd::DevicePrecond> dev;
  std::unique_ptr<fpd::GmresSolver> solver;
  int solver_restart = 0;
  fpd::DevBuf<double> xin, yout, bdev, xdev;
};

namespace fpd {
bool spgemm_device(const fpb::Csr& A, const fpb::Csr& B, std::span<const double> row_scale, fpb::Csr& C);
}

namespace {
// The setup's SpGEMMs can run on the device (bitwise the host routine).  With the
// hierarchy still built on the host that is transfer-bound, so the
// default is the host; FRACPREC_B200_DEVICE_SETUP=1 or fp_set_setup_backend(1) selects
// the device.  The environment is read on first use, not at load.
// Where build_tpu / build_tup run: 1 = the device-resident setup (dsetup.cu: fine-size products,
// strength graph and Galerkin products in HBM; the default when a CUDA device is present), 0 = the
// host setup (setup.cpp, OpenMP; the default without a device, or FRACPREC_B200_SETUP=host).
int g_setup_device = -1;
void ensure_setup_backend() {
  if (g_setup_device >= 0) return;
  int n = 0;
  const bool has = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
  cudaGetLastError();
  const char* e = std::getenv("FRACPREC_B200_SETUP");
  g_setup_device = has && !(e && std::strcmp(e, "host") == 0) ? 1 : 0;
}

// the generator library and this one share fp_workload's C++ layout (workload.hpp): refuse a stale build
void check_workload_layout() {
  if (fp_workload_layout() != workload_layout_fingerprint())
    throw std::runtime_error("libfp_workload.so and libfracprec_b200.so were built from different workload.hpp "
                             "versions; rebuild both (python -m paper_2112_12397_b200.build)");
}

fpb::HostPrecond build_any(const fpd::SystemView& V, const fpb::HostSystem* H, int variant, const fpb::AmgOptions& o,
                           const std::vector<std::array<double, 3>>& xyz) {
  ensure_setup_backend();
  if (g_setup_device) return fpd::build_precond_device(V, H, variant, o, xyz);
  if (H) return fpb::build_precond(*H, variant, o, xyz);
  ViewHold none;
  (void)none;
  fpb::HostSystem copy;  // the host setup works on owned CSR
  auto own = [](const fpd::HostCsrView& m) {
    fpb::Csr A(m.n_rows, m.n_cols);
    if (m.n_rows == 0) return A;
    A.rp.assign(m.rp, m.rp + m.n_rows + 1);
    A.ci.assign(m.ci, m.ci + m.nnz());
    A.v.assign(m.v, m.v + m.nnz());
    return A;
  };
  copy.n_u = V.n_u, copy.n_t = V.n_t, copy.n_p = V.n_p;
  copy.A = own(V.A), copy.C1 = own(V.C1), copy.Q1 = own(V.Q1), copy.C2 = own(V.C2);
  copy.H = own(V.H), copy.Q2 = own(V.Q2), copy.T = own(V.T), copy.F_u = own(V.F_u);
  return fpb::build_precond(copy, variant, o, xyz);
}
}  // namespace

struct fp_host_precond {
  fpb::HostPrecond hp;
};

struct fp_fracture_assembly {
  std::unique_ptr<fpd::DeviceFractureAssembly> dev;
};

extern "C" {

const char* fp_last_error(void) { return g_err.c_str(); }
const char* fp_version(void) { return "fracprec_b200 0.1 (sm_100a)"; }

void fp_amg_config_default(fp_amg_config* c) {
  const fpb::AmgOptions o;
  c->strength_threshold = o.strength_threshold;
  c->max_coarse = o.max_coarse;
  c->pre_sweeps = o.pre_sweeps;
  c->post_sweeps = o.post_sweeps;
  c->smoother = FP_SMOOTHER_JACOBI;
  c->prolongation_smoothing = 1;
  c->cycles_per_apply = o.cycles_per_apply;
  c->jacobi_omega = o.jacobi_omega;
  c->stall_ratio = o.stall_ratio;
  c->max_levels = o.max_levels;
  c->chebyshev_degree = o.chebyshev_degree;
  c->chebyshev_ratio = o.chebyshev_ratio;
  c->power_iterations = o.power_iterations;
  c->row_sum = FP_ROW_SUM_ORDERED;
}

// ------------------------------------------------------------------ system
int fp_system_create(const fp_block_system* J, fp_system** out) {
  return guard([&] {
    need(J && out, "fp_system_create: null argument");
    ViewHold hold;
    const fpd::SystemView V = checked_system(*J, hold);
    auto s = std::make_unique<fp_system>();
    fpd::cuda_check(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    s->dev = std::make_unique<fpd::DeviceSystem>(V);
    const int n = s->dev->n();
    s->xin.alloc(n), s->yout.alloc(n);
    *out = s.release();
  });
}

void fp_system_destroy(fp_system* s) { delete s; }

int fp_system_dims(const fp_system* s, int32_t* n_u, int32_t* n_t, int32_t* n_p) {
  return guard([&] {
    need(s, "fp_system_dims: null handle");
    if (n_u) *n_u = s->dev->n_u;
    if (n_t) *n_t = s->dev->n_t;
    if (n_p) *n_p = s->dev->n_p;
  });
}

int fp_block_scaling(const fp_system* s, double* st, double* sp) {
  return guard([&] {
    need(s, "fp_block_scaling: null handle");
    if (st) *st = s->dev->st;
    if (sp) *sp = s->dev->sp;
  });
}

int fp_system_apply(fp_system* s, const double* x, double* y, int32_t mem) {
  return guard([&] {
    need(s && x && y, "fp_system_apply: null argument");
    const size_t bytes = sizeof(double) * size_t(s->dev->n());
    const double* xd = x;
    double* yd = y;
    if (mem == FP_MEM_HOST) {
      fpd::cuda_check(cudaMemcpyAsync(s->xin.get(), x, bytes, cudaMemcpyHostToDevice, s->stream), "H2D");
      xd = s->xin.get(), yd = s->yout.get();
    }
    s->dev->enqueue_apply(xd, yd, 1.0, 1.0, s->stream);
    if (mem == FP_MEM_HOST)
      fpd::cuda_check(cudaMemcpyAsync(y, yd, bytes, cudaMemcpyDeviceToHost, s->stream), "D2H");
    fpd::cuda_check(cudaStreamSynchronize(s->stream), "fp_system_apply");
  });
}

// ------------------------------------------------------------- host build
int fp_host_precond_build(const fp_block_system* J, const fp_precond_config* cfg, const double* coords,
                          int32_t n_nodes, fp_host_precond** out) {
  return guard([&] {
    ensure_setup_backend();
    need(J && cfg && out, "fp_host_precond_build: null argument");
    need(cfg->factor_solve >= FP_FACTOR_AUTO && cfg->factor_solve <= FP_FACTOR_PANEL, "unknown factor_solve");
    ViewHold hold;
    const fpd::SystemView V = checked_system(*J, hold);
    std::vector<std::array<double, 3>> xyz;
    if (coords)
      for (int v = 0; v < n_nodes; ++v) xyz.push_back({coords[3 * v], coords[3 * v + 1], coords[3 * v + 2]});
    auto p = std::make_unique<fp_host_precond>();
    p->hp = build_any(V, nullptr, cfg->variant, to_amg(cfg->amg), xyz);
    p->hp.factor_solve = cfg->factor_solve;
    *out = p.release();
  });
}

void fp_host_precond_destroy(fp_host_precond* p) { delete p; }

int fp_host_precond_levels(const fp_host_precond* p, int32_t* n_levels, int32_t* rows) {
  return guard([&] {
    need(p, "null handle");
    const auto& L = p->hp.amg.levels;
    if (n_levels) *n_levels = int32_t(L.size());
    if (rows)
      for (size_t l = 0; l < L.size(); ++l) rows[l] = L[l].A.n_rows;
  });
}

int fp_host_precond_matrix(const fp_host_precond* p, int32_t what, int32_t level, int32_t* n_rows, int32_t* n_cols,
                           int64_t* nnz, int64_t* rp, int32_t* ci, double* v) {
  return guard([&] {
    need(p, "null handle");
    const auto& L = p->hp.amg.levels;
    const fpb::Csr* M = nullptr;
    const fpb::DeviceMatrix* dm = nullptr;  // a device-resident level (device setup)
    int64_t count = -1;
    if (what == 2)
      M = p->hp.variant == fpb::kTpu ? nullptr : &p->hp.S2;
    else {
      need(level >= 0 && level < int(L.size()), "level out of range");
      M = what == 0 ? &L[level].A : &L[level].P;
      dm = what == 0 ? L[level].dA.get() : L[level].dP.get();
      count = what == 0 ? L[level].a_nnz() : L[level].p_nnz();
    }
    need(M != nullptr, "matrix not available for this variant (T is part of the system)");
    if (n_rows) *n_rows = M->n_rows;
    if (n_cols) *n_cols = M->n_cols;
    if (nnz) *nnz = count >= 0 ? count : M->nnz();
    if (dm && (rp || ci || v)) {
      const fpb::Csr H = fpd::download_csr(dm->m);
      if (rp) std::memcpy(rp, H.rp.data(), sizeof(int64_t) * H.rp.size());
      if (ci) std::memcpy(ci, H.ci.data(), sizeof(int32_t) * H.ci.size());
      if (v) std::memcpy(v, H.v.data(), sizeof(double) * H.v.size());
      return;
    }
    if (rp) std::memcpy(rp, M->rp.data(), sizeof(int64_t) * M->rp.size());
    if (ci) std::memcpy(ci, M->ci.data(), sizeof(int32_t) * M->ci.size());
    if (v) std::memcpy(v, M->v.data(), sizeof(double) * M->v.size());
  });
}

int fp_host_precond_vector(const fp_host_precond* p, int32_t what, int32_t level, double* out, int64_t* len) {
  return guard([&] {
    need(p, "null handle");
    const std::vector<double>* v = nullptr;
    if (what == 0) v = &p->hp.hblocks;
    if (what == 1) v = p->hp.variant == fpb::kTpu ? &p->hp.T_diag : &p->hp.S_K;
    if (what == 2) {
      need(level >= 0 && level < int(p->hp.amg.levels.size()), "level out of range");
      v = &p->hp.amg.levels[level].diag;
    }
    std::vector<double> lam;
    if (what == 3) {  // Chebyshev lambda_max of the level (extension), a 1-vector
      need(level >= 0 && level < int(p->hp.amg.levels.size()), "level out of range");
      lam.assign(1, p->hp.amg.levels[level].lambda_max);
      v = &lam;
    }
    need(v != nullptr, "unknown vector");
    if (len) *len = int64_t(v->size());
    if (out) std::memcpy(out, v->data(), sizeof(double) * v->size());
  });
}

// ----------------------------------------------------------------- upload
int fp_host_precond_set_upload(fp_host_precond* p, int32_t row_sum, int32_t factor_solve) {
  return guard([&] {
    need(p != nullptr, "fp_host_precond_set_upload: null handle");
    need(row_sum == FP_ROW_SUM_ORDERED || row_sum == FP_ROW_SUM_STRIDED, "AmgConfig: unknown row_sum");
    need(factor_solve >= FP_FACTOR_AUTO && factor_solve <= FP_FACTOR_PANEL, "unknown factor_solve");
    p->hp.amg.opt.row_sum = row_sum;
    p->hp.factor_solve = factor_solve;
  });
}

int fp_precond_create(fp_system* s, const fp_host_precond* hp, fp_precond** out) {
  return guard([&] {
    need(s && hp && out, "fp_precond_create: null argument");
    auto p = std::make_unique<fp_precond>();
    p->sys = s;
    p->dev = std::make_unique<fpd::DevicePrecond>(*s->dev, hp->hp);
    const int n = s->dev->n();
    p->xin.alloc(n), p->yout.alloc(n), p->bdev.alloc(n), p->xdev.alloc(n);
    *out = p.release();
  });
}

int fp_precond_upload(fp_system* s, const fp_precond_desc* d, fp_precond** out) {
  return guard([&] {
    ensure_setup_backend();
    need(s && d && out && d->levels && d->n_levels >= 1 && d->h_blocks, "fp_precond_upload: null argument");
    need(d->variant >= FP_TPU && d->variant <= FP_TUP_STAR, "fp_precond_upload: unknown variant");
    fpb::HostPrecond hp;
    hp.variant = d->variant;
    hp.hblocks.assign(d->h_blocks, d->h_blocks + 9 * size_t(s->dev->n_p));
    const fpb::Csr F = to_csr(d->factor_matrix, "factor_matrix");
    hp.factor.factor(F, d->variant == FP_TPU ? fpb::BandFactor::Kind::spd : fpb::BandFactor::Kind::general);
    need(d->factor_solve >= FP_FACTOR_AUTO && d->factor_solve <= FP_FACTOR_PANEL, "unknown factor_solve");
    hp.factor_solve = d->factor_solve;
    hp.amg.opt = to_amg(d->amg);
    for (int l = 0; l < d->n_levels; ++l) {
      fpb::HostLevel L;
      L.A = to_csr(d->levels[l].A, "level A");
      if (l > 0) L.P = to_csr(d->levels[l].P, "level P");
      need(d->levels[l].smoother_diag != nullptr, "level smoother_diag is null");
      L.diag.assign(d->levels[l].smoother_diag, d->levels[l].smoother_diag + L.A.n_rows);
      hp.amg.levels.push_back(std::move(L));
    }
    const fpb::Csr& Ac = hp.amg.levels.back().A;
    hp.amg.coarse.compute(Ac.to_dense(), Ac.n_rows);
    if (hp.amg.opt.smoother == 3)  // multicolour GS (extension): the greedy colouring of the uploaded levels
      for (size_t l = 0; l + 1 < hp.amg.levels.size(); ++l) {
        fpb::HostLevel& L = hp.amg.levels[l];
        fpb::color_rows(L.A.n_rows, L.A.rp.data(), L.A.ci.data(), L.color_rows, L.color_off);
      }
    if (hp.amg.opt.smoother == 2)  // Chebyshev (extension): the oracle's lambda estimate on the uploaded levels
      for (size_t l = 0; l + 1 < hp.amg.levels.size(); ++l)
        hp.amg.levels[l].lambda_max =
            fpb::chebyshev_lambda_max(hp.amg.levels[l].A, hp.amg.levels[l].diag, hp.amg.opt.power_iterations);
    auto p = std::make_unique<fp_precond>();
    p->sys = s;
    p->dev = std::make_unique<fpd::DevicePrecond>(*s->dev, hp);
    const int n = s->dev->n();
    p->xin.alloc(n), p->yout.alloc(n), p->bdev.alloc(n), p->xdev.alloc(n);
    *out = p.release();
  });
}

void fp_precond_destroy(fp_precond* p) { delete p; }

int fp_precond_factor_solve(const fp_precond* p, int32_t* mode) {
  return guard([&] {
    need(p && mode, "null argument");
    *mode = p->dev->panel ? FP_FACTOR_PANEL : p->dev->inverse ? FP_FACTOR_INVERSE : FP_FACTOR_SWEEP;
  });
}

int fp_precond_apply(fp_precond* p, const double* x, double* y, int32_t mem) {
  return guard([&] {
    need(p && x && y, "fp_precond_apply: null argument");
    cudaStream_t st = p->sys->stream;
    const size_t bytes = sizeof(double) * size_t(p->sys->dev->n());
    const double* xd = x;
    double* yd = y;
    if (mem == FP_MEM_HOST) {
      fpd::cuda_check(cudaMemcpyAsync(p->xin.get(), x, bytes, cudaMemcpyHostToDevice, st), "H2D");
      xd = p->xin.get(), yd = p->yout.get();
    }
    p->dev->enqueue_apply(xd, yd, 1.0, 1.0, st);
    p->dev->inner_calls += p->dev->inner_per_apply();
    if (mem == FP_MEM_HOST) fpd::cuda_check(cudaMemcpyAsync(y, yd, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    fpd::cuda_check(cudaStreamSynchronize(st), "fp_precond_apply");
  });
}

int fp_amg_apply(fp_precond* p, const double* r, double* x, int32_t mem) {
  return guard([&] {
    need(p && r && x, "fp_amg_apply: null argument");
    cudaStream_t st = p->sys->stream;
    const size_t bytes = sizeof(double) * size_t(p->dev->amg->fine_n());
    const double* rd = r;
    double* xd = x;
    if (mem == FP_MEM_HOST) {
      fpd::cuda_check(cudaMemcpyAsync(p->xin.get(), r, bytes, cudaMemcpyHostToDevice, st), "H2D");
      rd = p->xin.get(), xd = p->yout.get();
    }
    p->dev->amg->enqueue_apply(rd, xd, nullptr, st);
    if (mem == FP_MEM_HOST) fpd::cuda_check(cudaMemcpyAsync(x, xd, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    fpd::cuda_check(cudaStreamSynchronize(st), "fp_amg_apply");
  });
}

int64_t fp_precond_inner_calls(fp_precond* p, int32_t reset) {
  if (!p) return -1;
  const int64_t c = p->dev->inner_calls;
  if (reset) p->dev->inner_calls = 0;
  return c;
}

int fp_precond_traffic(fp_precond* p, double* apply_bytes, int32_t* launches, double* japply_bytes) {
  return guard([&] {
    need(p, "null handle");
    fpd::Ledger a, j;
    cudaStream_t tmp;
    fpd::cuda_check(cudaStreamCreateWithFlags(&tmp, cudaStreamNonBlocking), "stream");
    cudaGraph_t g;
    fpd::cuda_check(cudaStreamBeginCapture(tmp, cudaStreamCaptureModeThreadLocal), "capture");
    p->dev->enqueue_apply(p->xin.get(), p->yout.get(), 1.0, 1.0, tmp, &a);
    p->sys->dev->enqueue_apply(p->xin.get(), p->yout.get(), 1.0, 1.0, tmp, &j);
    fpd::cuda_check(cudaStreamEndCapture(tmp, &g), "end capture");
    cudaGraphDestroy(g);
    cudaStreamDestroy(tmp);
    if (apply_bytes) *apply_bytes = a.bytes;
    if (launches) *launches = a.launches;
    if (japply_bytes) *japply_bytes = j.bytes;
  });
}

int fp_precond_profile(fp_precond* p, int32_t reps, fp_profile* out) {
  return guard([&] {
    need(p && out, "fp_precond_profile: null argument");
    const fpd::ProfileResult r = fpd::profile_precond(*p->sys->dev, *p->dev, reps, p->sys->stream);
    std::memset(out, 0, sizeof(*out));
    out->apply_ms = r.apply_ms, out->apply_bytes = r.apply_bytes, out->apply_launches = r.apply_launches;
    out->japply_ms = r.japply_ms, out->japply_bytes = r.japply_bytes;
    out->fine_resid_ms = r.fine_resid_ms, out->fine_resid_bytes = r.fine_resid_bytes;
    out->fine_post_ms = r.fine_post_ms, out->fine_post_bytes = r.fine_post_bytes;
    out->band_ms = r.band_ms, out->band_bytes = r.band_bytes, out->coarse_ms = r.coarse_ms;
    out->apply_wasted_bytes = r.apply_wasted_bytes;
    const auto& lv = p->dev->amg->lv;
    out->n_levels = int32_t(lv.size());
    for (size_t l = 0; l < lv.size() && l < 32; ++l) {
      out->level_rows[l] = lv[l].n;
      out->level_nnz[l] = lv[l].bsr3 ? 9 * lv[l].Ab.nblocks : lv[l].Am.nnz();
      out->vcycle_ms[l] = l < r.vcycle_ms.size() ? r.vcycle_ms[l] : 0.0;
    }
  });
}

int fp_gmres(fp_system* s, fp_precond* p, const double* b, double* x, int32_t mem, const fp_gmres_options* o,
             fp_solve_stats* stats) {
  return guard([&] {
    need(s && p && b && x && o, "fp_gmres: null argument");
    need(p->sys == s, "fp_gmres: preconditioner belongs to another system");
    need(o->max_iter >= 0, "fp_gmres: max_iter must be >= 0");
    const int restart = std::max(1, std::min(o->restart > 0 ? o->restart : o->max_iter, std::max(1, o->max_iter)));
    if (!p->solver || p->solver_restart != restart) {
      p->solver.reset();
      p->solver = std::make_unique<fpd::GmresSolver>(*s->dev, *p->dev, restart);
      p->solver_restart = restart;
    }
    cudaStream_t st = s->stream;
    const size_t bytes = sizeof(double) * size_t(s->dev->n());
    const double* bd = b;
    double* xd = x;
    if (mem == FP_MEM_HOST) {
      fpd::cuda_check(cudaMemcpyAsync(p->bdev.get(), b, bytes, cudaMemcpyHostToDevice, st), "H2D");
      bd = p->bdev.get(), xd = p->xdev.get();
    }
    fpd::SolveOptions so;
    need(o->orthogonalization == FP_ORTH_MGS || o->orthogonalization == FP_ORTH_CGS,
         "fp_gmres: orthogonalization must be FP_ORTH_MGS or FP_ORTH_CGS");
    so.tol = o->tol, so.restart = restart, so.max_iter = o->max_iter, so.scaled = o->scaled != 0;
    so.orth = o->orthogonalization == FP_ORTH_CGS ? fpd::kOrthCgs : fpd::kOrthMgs;
    so.probe = o->probe != 0;
    const fpd::SolveResult r = p->solver->solve(bd, xd, so, st);
    if (mem == FP_MEM_HOST) fpd::cuda_check(cudaMemcpyAsync(x, xd, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    fpd::cuda_check(cudaStreamSynchronize(st), "fp_gmres");
    if (stats) {
      stats->iterations = r.iterations;
      stats->converged = r.converged;
      stats->breakdown = r.breakdown;
      stats->restarts = r.restarts;
      stats->precond_applies = r.precond_applies;
      stats->final_rel_residual = r.final_rel_residual;
      stats->device_seconds = r.device_seconds;
      stats->kernel_launches = r.launches;
      stats->history_len = int32_t(r.history.size());
      stats->probe_ms = r.probe_ms;
      stats->probe_launches = r.probe_count;
      stats->reorth_steps = r.reorth_steps;
      if (stats->residual_history)
        for (int i = 0; i < stats->history_capacity && i < int(r.history.size()); ++i)
          stats->residual_history[i] = r.history[i];
    }
  });
}

// -------------------------------------------------------------- workload

int fp_workload_host_precond_build(const fp_workload* w, const fp_precond_config* cfg, fp_host_precond** out) {
  return guard([&] {
    ensure_setup_backend();
    need(w && cfg && out, "fp_workload_host_precond_build: null argument");
    check_workload_layout();
    need(cfg->factor_solve >= FP_FACTOR_AUTO && cfg->factor_solve <= FP_FACTOR_PANEL, "unknown factor_solve");
    auto p = std::make_unique<fp_host_precond>();
    p->hp = build_any(fpd::SystemView::of(w->w.J), &w->w.J, cfg->variant, to_amg(cfg->amg), w->w.coords);
    p->hp.factor_solve = cfg->factor_solve;
    *out = p.release();
  });
}

// -------------------------------------------------- fracture-block assembly (device)
int fp_fracture_assembly_create(const fp_workload* w, fp_fracture_assembly** out) {
  return guard([&] {
    need(w && out, "fp_fracture_assembly_create: null argument");
    check_workload_layout();
    auto a = std::make_unique<fp_fracture_assembly>();
    a->dev = std::make_unique<fpd::DeviceFractureAssembly>(w->w.model);
    *out = a.release();
  });
}

void fp_fracture_assembly_destroy(fp_fracture_assembly* a) { delete a; }

int fp_fracture_assembly_run(fp_fracture_assembly* a, const fp_fracture_state* st, fp_system* s) {
  return guard([&] {
    need(a && st, "fp_fracture_assembly_run: null argument");
    need(st->n_p == a->dev->n_p, "fp_fracture_assembly_run: state n_p does not match the model");
    need(st->n_p == 0 || (st->region && st->gap && st->traction_n && st->slip_dir && st->pressure),
         "fp_fracture_assembly_run: null state array");
    for (int f = 0; f < st->n_p; ++f)
      need(st->region[f] == 's' || st->region[f] == 'l' || st->region[f] == 'o',
           "fp_fracture_assembly_run: region must be s, l or o");
    a->dev->run(st->region, st->gap, st->traction_n, st->slip_dir, st->pressure);
    if (s) {
      need(s->dev->n_u == a->dev->n_u && s->dev->n_p == a->dev->n_p, "fp_fracture_assembly_run: system size mismatch");
      s->dev->set_fracture_blocks(a->dev->C2, a->dev->H, a->dev->T, a->dev->Q2);
    }
  });
}

int fp_fracture_assembly_matrix(const fp_fracture_assembly* a, int32_t what, int32_t* n_rows, int32_t* n_cols,
                                int64_t* nnz, int64_t* rp, int32_t* ci, double* v) {
  return guard([&] {
    need(a, "null handle");
    need(what >= 0 && what <= 4, "fp_fracture_assembly_matrix: what must be 0..4");
    const fpd::DCsr& M = what == 0 ? a->dev->C2 : what == 1 ? a->dev->H : what == 2 ? a->dev->T
                                                 : what == 3 ? a->dev->F_u : a->dev->Q2;
    if (n_rows) *n_rows = M.n_rows;
    if (n_cols) *n_cols = M.n_cols;
    if (nnz) *nnz = M.nnz;
    if (rp || ci || v) {
      const fpb::Csr H = fpd::download_csr(M);
      if (rp) std::memcpy(rp, H.rp.data(), sizeof(int64_t) * H.rp.size());
      if (ci) std::memcpy(ci, H.ci.data(), sizeof(int32_t) * H.ci.size());
      if (v) std::memcpy(v, H.v.data(), sizeof(double) * H.v.size());
    }
  });
}

int fp_set_setup_backend(int32_t device) {
  return guard([&] {
    ensure_setup_backend();
    if (!device) {
      g_setup_device = 0;
      return;
    }
    int n = 0;
    const bool has = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
    cudaGetLastError();
    need(has, "fp_set_setup_backend: no CUDA device");
    g_setup_device = 1;
  });
}

int fp_setup_backend(int32_t* device) {
  return guard([&] {
    need(device, "null argument");
    ensure_setup_backend();
    *device = g_setup_device;
  });
}

}  // extern "C"
