// Jacobian assembly of the state-dependent fracture blocks on the device:
// assemble_fracture_blocks (/root/reference/proj/core/src/assembly.cpp:229-406) — C2 (jump rows and the
// slip derivative), H (the slip / open diagonal and the traction stabilization), T (TPFA with the cubic
// law plus stabilization / dt), F_u (pressure-gap coupling) and Q2 = Q2gap + F_u — rebuilt every Newton
// step from the fracture state while A, C1, Q1 stay.
//
// Each block is a list of triplets emitted item by item (faces, then edges, then rim edges) in the
// reference's insertion order: a counting pass sizes every item, a scan places it, a filling pass writes
// it.  from_triplets (csr.cpp:60-90) follows as a stable radix sort of the (row, col) keys and one thread
// per distinct entry summing its duplicates from 0.0 in insertion order.  Every value is computed with
// the generator's expression order (workload/workload.cpp, no contraction), so the device blocks are
// bitwise the host assembly's (tests/test_gpu_parity.py::test_device_fracture_assembly_*).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "engine.cuh"
#include "workload.hpp"

namespace fpd {

namespace {

constexpr int kT = 256;
unsigned grid_for(long long n) { return unsigned(std::max(1LL, std::min((n + kT - 1) / kT, 1LL << 30))); }

struct ModelView {
  int n_u, n_p, n_e, n_b;
  const int *fminus, *fplus, *faxis;  // 4 n_p, 4 n_p, 3 n_p
  const double* farea;
  const int *ek, *el;
  const double *elen, *edk, *edl;
  const int* bk;
  const double *blen, *bd;
  const char* dir;
  double cohesion, tan_th, k_scale, stab_beta, E_ref, C_f0, mu_f, dt;
};
struct StateView {
  const char* region;
  const double *gap, *trac, *sdir, *pres;
  const double *cf, *dcf;
};

// counts (fill == false) or writes (fill == true) triplets from position pos
struct Sink {
  bool fill;
  long long pos;
  int *r, *c;
  double* v;
  __device__ void put(int row, int col, double val) {
    if (fill) r[pos] = row, c[pos] = col, v[pos] = val;
    ++pos;
  }
};

__device__ void jump_row(const ModelView& M, int f, int row, int comp, double scale, Sink& s) {
  const double w = M.farea[f] / 4.0;
  for (int v = 0; v < 4; ++v) {
    const int p = M.fplus[4 * f + v], m = M.fminus[4 * f + v];
    if (p == m) continue;
    for (int d = 0; d < 3; ++d) {
      const double val = scale * w * (M.faxis[3 * f + comp] == d ? 1.0 : 0.0);
      if (val == 0.0) continue;
      const int cp = 3 * p + d, cm = 3 * m + d;
      if (!M.dir[cp]) s.put(row, cp, val);
      if (!M.dir[cm]) s.put(row, cm, -val);
    }
  }
}

// the slip frame of face f: direction m and derivative D (assembly.cpp:269-283)
__device__ void slip_frame(const ModelView& M, const StateView& S, int f, double mm[2], double D[2][2]) {
  const double dg0 = S.gap[3 * f + 1], dg1 = S.gap[3 * f + 2];  // gap_prev = 0
  const double r = sqrt(dg0 * dg0 + dg1 * dg1);
  const double tau = M.cohesion - S.trac[f] * M.tan_th;
  const double thr = fmax(1e-12, 0.1 * fmax(tau, 0.0) / M.k_scale);
  D[0][0] = D[0][1] = D[1][0] = D[1][1] = 0.0;
  if (r >= thr) {
    mm[0] = dg0 / r, mm[1] = dg1 / r;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) D[a][b] = (tau / r) * ((a == b ? 1.0 : 0.0) - mm[a] * mm[b]);
  } else {
    mm[0] = S.sdir[2 * f], mm[1] = S.sdir[2 * f + 1];
  }
}

__device__ void c2_face(const ModelView& M, const StateView& S, int f, Sink& s) {
  const char reg = S.region[f];
  if (reg == 's') {
    for (int c = 0; c < 3; ++c) jump_row(M, f, 3 * f + c, c, 1.0, s);
  } else if (reg == 'l') {
    jump_row(M, f, 3 * f, 0, 1.0, s);
    double mm[2], D[2][2];
    slip_frame(M, S, f, mm, D);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b)
        if (D[a][b] != 0.0) jump_row(M, f, 3 * f + 1 + a, 1 + b, -D[a][b] / M.k_scale, s);
  }
}

__device__ double stab(const ModelView& M, int e) {  // beta (mean face area / E) |edge| (assembly.cpp:94-97)
  const double hh = 0.5 * (M.farea[M.ek[e]] + M.farea[M.el[e]]);
  return M.stab_beta * (hh / M.E_ref) * M.elen[e];
}

__device__ void h_item(const ModelView& M, const StateView& S, int it, Sink& s) {
  if (it < M.n_p) {  // the face's own rows
    const int f = it;
    const char reg = S.region[f];
    if (reg == 'l') {
      double mm[2], D[2][2];
      slip_frame(M, S, f, mm, D);
      for (int a = 0; a < 2; ++a) {
        s.put(3 * f + 1 + a, 3 * f + 1 + a, -M.farea[f] / M.k_scale);
        const double dtn = -M.tan_th * mm[a];
        if (dtn != 0.0) s.put(3 * f + 1 + a, 3 * f, (M.farea[f] / M.k_scale) * dtn);
      }
    } else if (reg == 'o') {
      for (int c = 0; c < 3; ++c) s.put(3 * f + c, 3 * f + c, -M.farea[f] / M.k_scale);
    }
    return;
  }
  const int e = it - M.n_p, k = M.ek[e], l = M.el[e];  // traction stabilization
  const bool ck = S.region[k] != 'o', cl = S.region[l] != 'o';
  if (!ck && !cl) return;
  const double sc = stab(M, e);
  for (int c = 0; c < 3; ++c) {
    if (ck && cl) {
      s.put(3 * k + c, 3 * k + c, sc);
      s.put(3 * l + c, 3 * l + c, sc);
      s.put(3 * k + c, 3 * l + c, -sc);
      s.put(3 * l + c, 3 * k + c, -sc);
    } else if (ck) {
      s.put(3 * k + c, 3 * k + c, sc);
    } else {
      s.put(3 * l + c, 3 * l + c, sc);
    }
  }
}

__device__ void fu_row(const ModelView& M, int row, int face, double coeff, Sink& s) {
  if (coeff == 0.0) return;
  for (int v = 0; v < 4; ++v) {
    const int p = M.fplus[4 * face + v], m = M.fminus[4 * face + v];
    if (p == m) continue;
    for (int d = 0; d < 3; ++d) {
      const double val = coeff * (M.faxis[3 * face] == d ? 1.0 : 0.0) / 4.0;
      if (val == 0.0) continue;
      const int cp = 3 * p + d, cm = 3 * m + d;
      if (!M.dir[cp]) s.put(row, cp, val);
      if (!M.dir[cm]) s.put(row, cm, -val);
    }
  }
}

// T (which == 0) or F_u (which == 1) items: the edges, then the rim edges
__device__ void tf_item(const ModelView& M, const StateView& S, int it, int which, Sink& s) {
  if (it < M.n_e) {
    const int e = it, k = M.ek[e], l = M.el[e];
    const double yk = (S.cf[k] / M.mu_f) * M.elen[e] / M.edk[e], yl = (S.cf[l] / M.mu_f) * M.elen[e] / M.edl[e];
    if (which == 0) {
      const double ykl = 2.0 * yk * yl / (yk + yl);
      s.put(k, k, ykl);
      s.put(l, l, ykl);
      s.put(k, l, -ykl);
      s.put(l, k, -ykl);
      const double sc = stab(M, e) / M.dt;
      s.put(k, k, sc);
      s.put(l, l, sc);
      s.put(k, l, -sc);
      s.put(l, k, -sc);
      return;
    }
    const double dp = S.pres[k] - S.pres[l];
    if (dp != 0.0) {
      const double dk = 2.0 * (yl / (yk + yl)) * (yl / (yk + yl)), dl = 2.0 * (yk / (yk + yl)) * (yk / (yk + yl));
      const double ck = dp * dk * (M.elen[e] / (M.mu_f * M.edk[e])) * S.dcf[k];
      const double cl = dp * dl * (M.elen[e] / (M.mu_f * M.edl[e])) * S.dcf[l];
      fu_row(M, k, k, ck, s);
      fu_row(M, k, l, cl, s);
      fu_row(M, l, k, -ck, s);
      fu_row(M, l, l, -cl, s);
    }
    return;
  }
  const int b = it - M.n_e, k = M.bk[b];
  if (which == 0) {
    s.put(k, k, (S.cf[k] / M.mu_f) * M.blen[b] / M.bd[b]);
    return;
  }
  const double pk = S.pres[k];
  if (pk != 0.0) fu_row(M, k, k, pk * (M.blen[b] / (M.mu_f * M.bd[b])) * S.dcf[k], s);
}

__device__ void q2gap_face(const ModelView& M, const StateView& S, int f, Sink& s) {
  if (S.region[f] != 'o') return;
  const double w = M.farea[f] / 4.0;
  for (int v = 0; v < 4; ++v) {
    const int p = M.fplus[4 * f + v], m = M.fminus[4 * f + v];
    if (p == m) continue;
    for (int d = 0; d < 3; ++d) {
      const double val = (w / M.dt) * (M.faxis[3 * f] == d ? 1.0 : 0.0);
      if (val == 0.0) continue;
      const int cp = 3 * p + d, cm = 3 * m + d;
      if (!M.dir[cp]) s.put(f, cp, val);
      if (!M.dir[cm]) s.put(f, cm, -val);
    }
  }
}

enum Block { kBlkC2 = 0, kBlkH = 1, kBlkT = 2, kBlkFu = 3, kBlkQ2gap = 4 };

template <bool fill>
__global__ void emit_kernel(ModelView M, StateView S, int block, int n_items, long long* cnt, const long long* off,
                            int* r, int* c, double* v) {
  const long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  Sink s{fill, fill ? off[it] : 0, r, c, v};
  switch (block) {
    case kBlkC2: c2_face(M, S, int(it), s); break;
    case kBlkH: h_item(M, S, int(it), s); break;
    case kBlkT: tf_item(M, S, int(it), 0, s); break;
    case kBlkFu: tf_item(M, S, int(it), 1, s); break;
    default: q2gap_face(M, S, int(it), s); break;
  }
  if (!fill) cnt[it] = s.pos;
}

__global__ void flow_kernel(ModelView M, const char* region, const double* gap, double* cf, double* dcf) {
  const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= M.n_p) return;
  const bool open = region[f] == 'o';
  const double g = open ? fmax(gap[3 * f], 0.0) : 0.0;
  cf[f] = M.C_f0 + g * g * g / 12.0;
  dcf[f] = open ? g * g / 4.0 : 0.0;
}

// ---- from_triplets on the device: a stable sort of the (row, col) keys, duplicates summed in order
__global__ void keys_kernel(long long n, const int* r, const int* c, unsigned long long* key, long long* idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    key[i] = ((unsigned long long)(unsigned)r[i] << 32) | (unsigned)c[i];
    idx[i] = i;
  }
}
__global__ void starts_kernel(long long n, const unsigned long long* key, long long* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n; i += (long long)gridDim.x * blockDim.x)
    flag[i] = i < n && (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}
__global__ void unique_kernel(long long n, const unsigned long long* key, const long long* flag, const long long* uid,
                              long long* start, int* ci, unsigned long long* rowcnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (flag[i]) {
      start[uid[i]] = i;
      ci[uid[i]] = int(key[i] & 0xffffffffull);
      atomicAdd(rowcnt + (key[i] >> 32), 1ull);
    }
}
__global__ void sum_kernel(long long n_unique, long long n, const long long* start, const long long* idx,
                           const double* val, double* out) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n_unique;
       u += (long long)gridDim.x * blockDim.x) {
    const long long e = u + 1 < n_unique ? start[u + 1] : n;
    double s = 0.0;
    for (long long i = start[u]; i < e; ++i) s += val[idx[i]];
    out[u] = s;
  }
}

long long scan_ll(DevBuf<long long>& in, long long n, DevBuf<long long>& out) {
  size_t tb = 0;
  cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tb, in.get(), out.get(), n + 1), "scan size");
  DevBuf<unsigned char> tmp(tb);
  cuda_check(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in.get(), out.get(), n + 1), "scan");
  long long total = 0;
  cuda_check(cudaMemcpy(&total, out.get() + n, sizeof(long long), cudaMemcpyDeviceToHost), "scan total");
  return total;
}

DCsr from_triplets_dev(int rows, int cols, long long n, const int* r, const int* c, const double* v) {
  DCsr A;
  A.n_rows = rows, A.n_cols = cols;
  DevBuf<unsigned long long> kin(static_cast<size_t>(std::max(1LL, n))), kout(static_cast<size_t>(std::max(1LL, n)));
  DevBuf<long long> iin(static_cast<size_t>(std::max(1LL, n))), iout(static_cast<size_t>(std::max(1LL, n)));
  if (n) {
    keys_kernel<<<1184, kT>>>(n, r, c, kin.get(), iin.get());
    size_t tb = 0;
    cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), iin.get(), iout.get(), n), "sort size");
    DevBuf<unsigned char> tmp(tb);
    cuda_check(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin.get(), kout.get(), iin.get(), iout.get(), n), "sort");
  }
  DevBuf<long long> flag(static_cast<size_t>(n) + 1), uid(static_cast<size_t>(n) + 1);
  starts_kernel<<<1184, kT>>>(n, kout.get(), flag.get());
  const long long nu = scan_ll(flag, n, uid);
  DevBuf<long long> start(static_cast<size_t>(std::max(1LL, nu)));
  DevBuf<unsigned long long> rowcnt(static_cast<size_t>(rows) + 1);
  rowcnt.zero();
  A.ci.alloc(size_t(nu));
  A.v.alloc(size_t(nu));
  A.nnz = nu;
  if (n) {
    unique_kernel<<<1184, kT>>>(n, kout.get(), flag.get(), uid.get(), start.get(), A.ci.get(), rowcnt.get());
    sum_kernel<<<1184, kT>>>(nu, n, start.get(), iout.get(), v, A.v.get());
  }
  A.rp.alloc(size_t(rows) + 1);
  size_t tb = 0;
  cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tb, reinterpret_cast<long long*>(rowcnt.get()), A.rp.get(), rows + 1),
             "scan size");
  DevBuf<unsigned char> tmp(tb);
  cuda_check(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, reinterpret_cast<long long*>(rowcnt.get()), A.rp.get(),
                                           rows + 1),
             "scan");
  cuda_check(cudaDeviceSynchronize(), "from_triplets_dev");
  return A;
}

template <class T>
void up(DevBuf<T>& d, const T* h, size_t n) {
  if (n) d.upload(h, n);
}

}  // namespace

struct DeviceFractureAssembly::Model {
  DevBuf<int> fminus, fplus, faxis, ek, el, bk;
  DevBuf<double> farea, elen, edk, edl, blen, bd;
  DevBuf<char> dir;
  ModelView view{};
};

DeviceFractureAssembly::DeviceFractureAssembly(const fpb::FractureModel& m) : model_(std::make_unique<Model>()) {
  Model& d = *model_;
  n_u = m.n_u, n_p = m.n_p;
  const size_t np = size_t(m.n_p), ne = m.edges.size(), nb = m.bc_edges.size();
  if (m.faces.size() != np || m.dir.size() != size_t(m.n_u))
    throw std::invalid_argument("fracture assembly: the workload carries no fracture model");
  std::vector<int> fminus(4 * np), fplus(4 * np), faxis(3 * np), ek(ne), el(ne), bk(nb);
  std::vector<double> farea(np), elen(ne), edk(ne), edl(ne), blen(nb), bd(nb);
  for (size_t f = 0; f < np; ++f) {
    for (int v = 0; v < 4; ++v) fminus[4 * f + v] = m.faces[f].minus[v], fplus[4 * f + v] = m.faces[f].plus[v];
    for (int a = 0; a < 3; ++a) faxis[3 * f + a] = m.faces[f].axis[a];
    farea[f] = m.faces[f].area;
  }
  for (size_t e = 0; e < ne; ++e)
    ek[e] = m.edges[e].k, el[e] = m.edges[e].l, elen[e] = m.edges[e].length, edk[e] = m.edges[e].dk,
    edl[e] = m.edges[e].dl;
  for (size_t b = 0; b < nb; ++b) bk[b] = m.bc_edges[b].k, blen[b] = m.bc_edges[b].length, bd[b] = m.bc_edges[b].d;
  up(d.fminus, fminus.data(), fminus.size()), up(d.fplus, fplus.data(), fplus.size());
  up(d.faxis, faxis.data(), faxis.size()), up(d.farea, farea.data(), np);
  up(d.ek, ek.data(), ne), up(d.el, el.data(), ne), up(d.elen, elen.data(), ne), up(d.edk, edk.data(), ne);
  up(d.edl, edl.data(), ne), up(d.bk, bk.data(), nb), up(d.blen, blen.data(), nb), up(d.bd, bd.data(), nb);
  up(d.dir, m.dir.data(), m.dir.size());
  d.view = ModelView{m.n_u, m.n_p, int(ne), int(nb), d.fminus.get(), d.fplus.get(), d.faxis.get(), d.farea.get(),
                     d.ek.get(), d.el.get(), d.elen.get(), d.edk.get(), d.edl.get(), d.bk.get(), d.blen.get(),
                     d.bd.get(), d.dir.get(), m.cohesion, m.tan_th, m.k_scale, m.stab_beta, m.E_ref, m.C_f0,
                     m.mu_f, m.dt};
}

DeviceFractureAssembly::~DeviceFractureAssembly() = default;

void DeviceFractureAssembly::run(const char* region, const double* gap, const double* trac, const double* sdir,
                                 const double* pres) {
  const ModelView& M = model_->view;
  const size_t np = size_t(n_p);
  DevBuf<char> dreg;
  DevBuf<double> dgap, dtrac, dsdir, dpres, cf(np), dcf(np);
  up(dreg, region, np), up(dgap, gap, 3 * np), up(dtrac, trac, np), up(dsdir, sdir, 2 * np), up(dpres, pres, np);
  if (np) flow_kernel<<<grid_for((long long)np), kT>>>(M, dreg.get(), dgap.get(), cf.get(), dcf.get());
  const StateView S{dreg.get(), dgap.get(), dtrac.get(), dsdir.get(), dpres.get(), cf.get(), dcf.get()};
  auto block = [&](int which, int n_items, int rows, int cols) {
    DevBuf<long long> cnt(size_t(n_items) + 1), off(size_t(n_items) + 1);
    cnt.zero();
    if (n_items)
      emit_kernel<false><<<grid_for(n_items), kT>>>(M, S, which, n_items, cnt.get(), nullptr, nullptr, nullptr, nullptr);
    const long long n = scan_ll(cnt, n_items, off);
    DevBuf<int> r(static_cast<size_t>(std::max(1LL, n))), c(static_cast<size_t>(std::max(1LL, n)));
    DevBuf<double> v(static_cast<size_t>(std::max(1LL, n)));
    if (n) emit_kernel<true><<<grid_for(n_items), kT>>>(M, S, which, n_items, nullptr, off.get(), r.get(), c.get(), v.get());
    return from_triplets_dev(rows, cols, n, r.get(), c.get(), v.get());
  };
  const int n_t = 3 * n_p, ne = M.n_e, nb = M.n_b;
  C2 = block(kBlkC2, n_p, n_t, n_u);
  H = block(kBlkH, n_p + ne, n_t, n_t);
  T = block(kBlkT, ne + nb, n_p, n_p);
  F_u = block(kBlkFu, ne + nb, n_p, n_u);
  const DCsr Q2gap = block(kBlkQ2gap, n_p, n_p, n_u);
  Q2 = add_dev(Q2gap, F_u, 1.0, 1.0);
}

}  // namespace fpd
