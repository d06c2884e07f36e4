// C ABI of the workload generator (include/fracprec_workload.h): synthetic BASELINE systems and the
// snapshot bundle reader/writer.  Input side only — this library has no solve code and no CUDA; the
// CPU oracle's callers (bench.py --impl reference) load it without the B200 solve library.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "../include/fracprec_workload.h"
#include "snapshot.hpp"
#include "workload.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return FP_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FP_INVALID_ARGUMENT;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("allocation failure: ") + e.what();
    return FP_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FP_INTERNAL_ERROR;
  }
}

void need(bool ok, const std::string& what) {
  if (!ok) throw std::invalid_argument(what);
}

fpb::Csr to_csr(const fp_csr& m, const char* name) {
  const std::string nm(name);
  need(m.n_rows >= 0 && m.n_cols >= 0, nm + ": negative dimension");
  fpb::Csr A(m.n_rows, m.n_cols);
  if (m.n_rows == 0) return A;
  need((m.row_offsets32 != nullptr) != (m.row_offsets64 != nullptr),
       nm + ": exactly one of row_offsets32 / row_offsets64 must be set");
  for (int i = 0; i <= m.n_rows; ++i) A.rp[i] = m.row_offsets32 ? int64_t(m.row_offsets32[i]) : m.row_offsets64[i];
  need(A.rp[0] == 0, nm + ": row_offsets[0] != 0");
  for (int i = 0; i < m.n_rows; ++i) need(A.rp[i] <= A.rp[i + 1], nm + ": row_offsets not monotone");
  const int64_t nnz = A.rp[m.n_rows];
  need(nnz == 0 || (m.col_indices && m.values), nm + ": null column/value array");
  A.ci.assign(m.col_indices, m.col_indices + nnz);
  A.v.assign(m.values, m.values + nnz);
  for (int64_t k = 0; k < nnz; ++k) need(A.ci[k] >= 0 && A.ci[k] < m.n_cols, nm + ": column out of range");
  return A;
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

extern "C" {

const char* fp_workload_last_error(void) { return g_err.c_str(); }

uint64_t fp_workload_layout(void) { return workload_layout_fingerprint(); }

int fp_workload_preset(int32_t id, uint64_t seed, fp_workload** out) {
  return guard([&] {
    need(out != nullptr, "fp_workload_preset: null out");
    auto w = std::make_unique<fp_workload>();
    w->w = fpb::generate_workload(fpb::preset_config(id, seed));
    *out = w.release();
  });
}

int fp_workload_custom(const fp_workload_spec* sp, fp_workload** out) {
  return guard([&] {
    need(sp && out, "fp_workload_custom: null argument");
    fpb::WorkloadSpec s;
    for (int d = 0; d < 3; ++d) s.cells[d] = sp->cells[d], s.length[d] = sp->length[d];
    for (int f = 0; f < sp->n_fractures; ++f) {
      const fp_fracture_spec& q = sp->fractures[f];
      s.fractures.push_back({q.normal_axis, q.coord, q.lo1, q.hi1, q.lo2, q.hi2});
    }
    s.E_median = sp->E_median, s.E_sigma_ln = sp->E_sigma_ln, s.E_layers = sp->E_layers;
    s.nu = sp->nu, s.nu_lo = sp->nu_lo, s.nu_hi = sp->nu_hi;
    s.frac_stick = sp->frac_stick, s.frac_slip = sp->frac_slip;
    s.aperture_median = sp->aperture_median, s.aperture_sigma_ln = sp->aperture_sigma_ln;
    s.seed = sp->seed;
    if (sp->stab_beta > 0.0) s.stab_beta = sp->stab_beta;
    if (sp->slip_factor > 0.0) s.slip_factor = sp->slip_factor;
    auto w = std::make_unique<fp_workload>();
    w->w = fpb::generate_workload(s);
    *out = w.release();
  });
}

void fp_workload_destroy(fp_workload* w) { delete w; }

int fp_workload_system(const fp_workload* w, fp_block_system* J) {
  return guard([&] {
    need(w && J, "null argument");
    const fpb::HostSystem& H = w->w.J;
    J->n_u = H.n_u, J->n_t = H.n_t, J->n_p = H.n_p;
    J->A = view_of(H.A), J->C1 = view_of(H.C1), J->Q1 = view_of(H.Q1), J->C2 = view_of(H.C2);
    J->H = view_of(H.H), J->Q2 = view_of(H.Q2), J->T = view_of(H.T), J->F_u = view_of(H.F_u);
  });
}

int fp_workload_coords(const fp_workload* w, const double** xyz, int32_t* n_nodes) {
  return guard([&] {
    need(w && xyz && n_nodes, "null argument");
    *xyz = w->w.coords.empty() ? nullptr : w->w.coords[0].data();
    *n_nodes = int32_t(w->w.coords.size());
  });
}

int fp_workload_region(const fp_workload* w, const char** region, double* dt) {
  return guard([&] {
    need(w && region && dt, "null argument");
    *region = w->w.region.c_str();
    *dt = w->w.dt;
  });
}

int fp_workload_info(const fp_workload* w, int32_t* c) {
  return guard([&] {
    need(w && c, "null argument");
    c[0] = w->w.n_stick, c[1] = w->w.n_slip, c[2] = w->w.n_open, c[3] = w->w.n_fractures;
  });
}

int fp_workload_state(const fp_workload* w, fp_fracture_state* out) {
  return guard([&] {
    need(w && out, "null argument");
    const fpb::FractureState& S = w->w.state;
    need(!S.region.empty() || w->w.J.n_p == 0, "fp_workload_state: this workload carries no fracture state");
    out->n_p = int32_t(S.region.size());
    out->region = S.region.c_str();
    out->gap = S.gap.empty() ? nullptr : S.gap[0].data();
    out->traction_n = S.trac_n.data();
    out->slip_dir = S.slip_dir.empty() ? nullptr : S.slip_dir[0].data();
    out->pressure = S.pressure.data();
  });
}

int fp_workload_set_state(fp_workload* w, const fp_fracture_state* st) {
  return guard([&] {
    need(w && st, "null argument");
    need(w->w.model.n_p == w->w.J.n_p && int(w->w.model.faces.size()) == w->w.J.n_p,
         "fp_workload_set_state: this workload carries no fracture model (imported bundle)");
    const int n_p = w->w.J.n_p;
    need(st->n_p == n_p, "fp_workload_set_state: n_p mismatch");
    need(n_p == 0 || (st->region && st->gap && st->traction_n && st->slip_dir && st->pressure),
         "fp_workload_set_state: null state array");
    fpb::FractureState S;
    S.region.assign(st->region, st->region + n_p);
    for (char c : S.region) need(c == 's' || c == 'l' || c == 'o', "fp_workload_set_state: region must be s, l or o");
    S.gap.resize(size_t(n_p)), S.slip_dir.resize(size_t(n_p));
    for (int f = 0; f < n_p; ++f) {
      S.gap[f] = {st->gap[3 * f], st->gap[3 * f + 1], st->gap[3 * f + 2]};
      S.slip_dir[f] = {st->slip_dir[2 * f], st->slip_dir[2 * f + 1]};
    }
    S.trac_n.assign(st->traction_n, st->traction_n + n_p);
    S.pressure.assign(st->pressure, st->pressure + n_p);
    fpb::assemble_fracture_blocks(w->w.model, S, w->w.J);
    w->w.state = std::move(S);
    w->w.region = w->w.state.region;
  });
}

int fp_snapshot_import(const char* dir, fp_workload** out) {
  return guard([&] {
    need(dir && out, "fp_snapshot_import: null argument");
    auto p = std::make_unique<fp_workload>();
    p->w = fpb::import_snapshot(dir);
    *out = p.release();
  });
}

int fp_snapshot_export(const char* dir, const fp_block_system* J, const char* region, double dt,
                       const double* node_coords, int32_t n_nodes) {
  return guard([&] {
    need(dir && J && region, "fp_snapshot_export: null argument");
    fpb::HostSystem H;
    H.n_u = J->n_u, H.n_t = J->n_t, H.n_p = J->n_p;
    H.A = to_csr(J->A, "A"), H.C1 = to_csr(J->C1, "C1"), H.Q1 = to_csr(J->Q1, "Q1");
    H.C2 = to_csr(J->C2, "C2"), H.H = to_csr(J->H, "H"), H.Q2 = to_csr(J->Q2, "Q2");
    H.T = to_csr(J->T, "T"), H.F_u = to_csr(J->F_u, "F_u");
    H.check_shapes();
    std::vector<std::array<double, 3>> xyz;
    for (int v = 0; node_coords && v < n_nodes; ++v)
      xyz.push_back({node_coords[3 * v], node_coords[3 * v + 1], node_coords[3 * v + 2]});
    fpb::export_snapshot(dir, H, std::string(region, strnlen(region, size_t(H.n_p) + 1)), dt, xyz);
  });
}

}  // extern "C"
