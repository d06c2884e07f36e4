// Preconditioner setup on the device: build_tpu / build_tup and amg_setup
// (/root/reference/proj/core/src/precond.cpp:18-36,119-202, amg.cpp:181-291) with every
// fine-size operator resident in HBM.
//
//   on the device: the Schur core A + C1 (H~^-1 C2) and t-p-u's Q1 (T_diag^-1 Q2) correction
//                  (device SpGEMM, spgemm.cu), the strength graph of B = (A + A^T)/2 (amg.cpp:27-54),
//                  Jacobi prolongation smoothing P - w D^-1 A P (amg.cpp:259-264), the Galerkin
//                  product P^T (A P) (amg.cpp:268), R = P^T, every diagonal;
//   on the host:   the BFS aggregation (amg.cpp:60-113: its visiting order defines the aggregates),
//                  the per-aggregate QR of the near-null space (amg.cpp:223-244, a few seconds even at
//                  config 5), the dense coarse LU, the fixed-stress local solves (on the S1 rows next to
//                  fractures, downloaded), and the banded T / S~2 factors (n_p rows).
//
// Every product keeps the reference's per-entry operation order (row-local, left to right, no
// contraction), so the hierarchy is bitwise the one the host setup and the CPU oracle build
// (tests/test_gpu_parity.py::test_device_setup_*).  The levels stay on the device and feed the
// upload (engine.cu) directly; the host copies in the returned HostPrecond hold only their shapes.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "engine.cuh"

namespace fpd {

namespace {

constexpr int kT = 256;
unsigned grid_for(long long n) { return unsigned(std::max(1LL, std::min((n + kT - 1) / kT, 1LL << 30))); }

struct Clock {
  bool on = std::getenv("FRACPREC_B200_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, long long a = -1) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dsetup] %-26s %8.3f s  %lld\n", what, std::chrono::duration<double>(now - t).count(), a);
    t = now;
  }
};

long long scan_counts(DevBuf<long long>& cnt, long long n, DevBuf<long long>& out) {
  // cnt[0..n) counts, cnt[n] = 0 -> out[0..n] exclusive offsets; returns the total
  size_t tmp_bytes = 0;
  cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.get(), out.get(), n + 1), "scan size");
  DevBuf<unsigned char> tmp(tmp_bytes);
  cuda_check(cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, cnt.get(), out.get(), n + 1), "scan");
  long long total = 0;
  cuda_check(cudaMemcpy(&total, out.get() + n, sizeof(long long), cudaMemcpyDeviceToHost), "scan total");
  return total;
}

// ---- alpha A + beta B on the union pattern (csr.cpp:181-206): row-local merge, explicit zeros kept
template <bool fill>
__global__ void add_rows_kernel(int n, const long long* arp, const int* aci, const double* av, const long long* brp,
                                const int* bci, const double* bv, double alpha, double beta, int n_cols,
                                long long* cnt, const long long* crp, int* cci, double* cv) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long ka = arp[i], ea = arp[i + 1], kb = brp[i], eb = brp[i + 1];
  long long o = fill ? crp[i] : 0, c = 0;
  while (ka < ea || kb < eb) {
    const int ca = ka < ea ? aci[ka] : n_cols;
    const int cb = kb < eb ? bci[kb] : n_cols;
    if (fill) {
      if (ca < cb) {
        cci[o] = ca, cv[o] = alpha * av[ka++];
      } else if (cb < ca) {
        cci[o] = cb, cv[o] = beta * bv[kb++];
      } else {
        const double va = alpha * av[ka++];
        const double vb = beta * bv[kb++];
        cci[o] = ca, cv[o] = va + vb;
      }
      ++o;
    } else {
      if (ca <= cb) ++ka;
      if (cb <= ca) ++kb;
      ++c;
    }
  }
  if (!fill) cnt[i] = c;
}

__global__ void scale_rows_kernel(int n, const long long* rp, const double* s, double* v) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (long long k = rp[i]; k < rp[i + 1]; ++k) v[k] *= s[i];
}

__global__ void diag_kernel(int n, const long long* rp, const int* ci, const double* v, double* d) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = 0.0;
  for (long long k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] == i) x = v[k];
  d[i] = x;
}

// ---- strength graph (amg.cpp:27-54) of B = 0.5 A + 0.5 A^T without forming B: row i of B is the
// merge of row i of A and row i of A^T with add_scaled's arithmetic
__device__ __forceinline__ double b_entry(bool in_a, bool in_t, double a, double t) {
  if (in_a && in_t) {
    const double va = 0.5 * a;
    const double vb = 0.5 * t;
    return va + vb;
  }
  return in_a ? 0.5 * a : 0.5 * t;
}

__global__ void bdiag_kernel(int n, const long long* arp, const int* aci, const double* av, const long long* trp,
                             const int* tci, const double* tv, double* d) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ia = false, it = false;
  double a = 0.0, t = 0.0;
  for (long long k = arp[i]; k < arp[i + 1]; ++k)
    if (aci[k] == i) ia = true, a = av[k];
  for (long long k = trp[i]; k < trp[i + 1]; ++k)
    if (tci[k] == i) it = true, t = tv[k];
  d[i] = (ia || it) ? b_entry(ia, it, a, t) : 0.0;
}

template <bool fill>
__global__ void strength_kernel(int n, const long long* arp, const int* aci, const double* av, const long long* trp,
                                const int* tci, const double* tv, const double* d, double theta, long long* cnt,
                                char* isolated, const long long* off, int* nbr, double* w) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long ka = arp[i], ea = arp[i + 1], kt = trp[i], et = trp[i + 1];
  long long o = fill ? off[i] : 0, strong = 0;
  int offdiag = 0;
  const double di = fabs(d[i]);
  while (ka < ea || kt < et) {
    const int ca = ka < ea ? aci[ka] : 0x7fffffff;
    const int ct = kt < et ? tci[kt] : 0x7fffffff;
    const int j = min(ca, ct);
    const bool in_a = ca == j, in_t = ct == j;
    const double b = b_entry(in_a, in_t, in_a ? av[ka] : 0.0, in_t ? tv[kt] : 0.0);
    if (in_a) ++ka;
    if (in_t) ++kt;
    if (j == i) continue;
    if (b != 0.0) ++offdiag;
    const double thr = theta * sqrt(di * fabs(d[j]));
    if (fabs(b) > thr) {
      if (fill) nbr[o] = j, w[o] = fabs(b), ++o;
      ++strong;
    }
  }
  if (!fill) {
    cnt[i] = strong;
    isolated[i] = offdiag == 0 ? 1 : 0;
  }
}

// With a structurally symmetric A (every level operator here: S1 / S~ and the Galerkin products
// P^T A P), row i of A^T has row i's columns and A^T(i, j) = A(j, i), found by binary search in row j,
// so B's rows need no transposed copy.  sym_check_kernel clears *ok on the first entry without a mirror.
__device__ __forceinline__ long long find_col(const long long* rp, const int* ci, int row, int col) {
  long long lo = rp[row], hi = rp[row + 1];
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (ci[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return (lo < rp[row + 1] && ci[lo] == col) ? lo : -1;
}

__global__ void sym_check_kernel(int n, const long long* rp, const int* ci, int* ok) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (long long k = rp[i]; k < rp[i + 1]; ++k)
    if (find_col(rp, ci, ci[k], int(i)) < 0) {
      *ok = 0;
      return;
    }
}

__global__ void bdiag_sym_kernel(int n, const long long* rp, const int* ci, const double* v, double* d) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = find_col(rp, ci, int(i), int(i));
  d[i] = k >= 0 ? b_entry(true, true, v[k], v[k]) : 0.0;
}

template <bool fill>
__global__ void strength_sym_kernel(int n, const long long* rp, const int* ci, const double* v, const double* d,
                                    double theta, long long* cnt, char* isolated, const long long* off, int* nbr,
                                    double* w) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long o = fill ? off[i] : 0, strong = 0;
  int offdiag = 0;
  const double di = fabs(d[i]);
  for (long long k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = ci[k];
    if (j == i) continue;
    const double b = b_entry(true, true, v[k], v[find_col(rp, ci, j, int(i))]);
    if (b != 0.0) ++offdiag;
    const double thr = theta * sqrt(di * fabs(d[j]));
    if (fabs(b) > thr) {
      if (fill) nbr[o] = j, w[o] = fabs(b), ++o;
      ++strong;
    }
  }
  if (!fill) {
    cnt[i] = strong;
    isolated[i] = offdiag == 0 ? 1 : 0;
  }
}

// weights of the leftover rows rows[0..m) (amg.cpp:98-111), packed
__global__ void gather_w_kernel(int m, const int* rows, const long long* off, const double* w, const long long* pos,
                                double* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const long long k0 = off[rows[t]], k1 = off[rows[t] + 1];
  for (long long k = k0; k < k1; ++k) out[pos[t] + (k - k0)] = w[k];
}

// ---- tentative prolongation (amg.cpp:214-257): one thread per aggregate runs the column-pivoted
// Householder QR of its near-null block B (m rows x k columns): pivot = first column of largest remaining
// norm (norms recomputed each step), reflectors in Eigen's makeHouseholder form, rank |R_jj| >
// 1e-12 max(1, |R_00|), Q = the first `rank` columns of H_0 ... H_mn-1 applied to unit vectors,
// Rp = R(0:rank, :) P^T.  W (m x k, column-major) and Q live in per-aggregate global scratch.
__device__ double householder_dev(double* x, int len) {
  double tail = 0.0;
  for (int i = 1; i < len; ++i) tail += x[i] * x[i];
  const double c0 = x[0];
  if (tail <= 2.2250738585072014e-308) {  // DBL_MIN
    for (int i = 1; i < len; ++i) x[i] = 0.0;
    return 0.0;
  }
  double beta = sqrt(c0 * c0 + tail);
  if (c0 >= 0.0) beta = -beta;
  const double denom = c0 - beta;
  for (int i = 1; i < len; ++i) x[i] = x[i] / denom;
  x[0] = beta;
  return (beta - c0) / beta;
}

constexpr int kQrMaxK = 8;

__global__ void qr_aggregates_kernel(int n_agg, int k, int n, const int* a_off, const int* a_rows, const double* nn,
                                     double* W, double* Q, int* rank_out, double* Rp) {
  const long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (a >= n_agg) return;
  const int r0 = a_off[a], m = a_off[a + 1] - r0;
  double* w = W + (long long)r0 * k;  // column c at w + c m
  for (int c = 0; c < k; ++c)
    for (int r = 0; r < m; ++r) w[c * m + r] = nn[(long long)c * n + a_rows[r0 + r]];
  int perm[kQrMaxK];
  double tau[kQrMaxK];
  for (int j = 0; j < k; ++j) perm[j] = j;
  const int mn = min(m, k);
  for (int j = 0; j < mn; ++j) {
    int p = j;
    double best = -1.0;
    for (int c = j; c < k; ++c) {
      double sq = 0.0;
      for (int i = j; i < m; ++i) sq += w[c * m + i] * w[c * m + i];
      if (sq > best) best = sq, p = c;
    }
    if (p != j) {
      for (int i = 0; i < m; ++i) {
        const double t = w[j * m + i];
        w[j * m + i] = w[p * m + i], w[p * m + i] = t;
      }
      const int t = perm[j];
      perm[j] = perm[p], perm[p] = t;
    }
    tau[j] = householder_dev(w + j * m + j, m - j);
    for (int c = j + 1; c < k; ++c) {
      double sv = w[c * m + j];
      for (int i = j + 1; i < m; ++i) sv += w[j * m + i] * w[c * m + i];
      sv *= tau[j];
      w[c * m + j] -= sv;
      for (int i = j + 1; i < m; ++i) w[c * m + i] -= sv * w[j * m + i];
    }
  }
  const double r00 = mn > 0 ? fabs(w[0]) : 0.0;
  const double tol = 1e-12 * fmax(1.0, r00);
  int rank = 0;
  for (int j = 0; j < mn; ++j)
    if (fabs(w[j * m + j]) > tol) ++rank;
  rank_out[a] = rank;
  double* q = Q + (long long)r0 * k;  // column c at q + c m
  for (int c = 0; c < rank; ++c) {
    double* qc = q + c * m;
    for (int i = 0; i < m; ++i) qc[i] = 0.0;
    qc[c] = 1.0;
    for (int j = min(c, mn - 1); j >= 0; --j) {
      double sv = qc[j];
      for (int i = j + 1; i < m; ++i) sv += w[j * m + i] * qc[i];
      sv *= tau[j];
      qc[j] -= sv;
      for (int i = j + 1; i < m; ++i) qc[i] -= sv * w[j * m + i];
    }
  }
  double* rp = Rp + a * (long long)k * k;
  for (int r = 0; r < rank; ++r) {
    for (int j = 0; j < k; ++j) rp[r * k + j] = 0.0;
    for (int j = r; j < k; ++j) rp[r * k + perm[j]] = w[j * m + r];
  }
}

// tentative P: row i (in aggregate a at local position r) holds the nonzero Q entries of a in
// ascending coarse column order; fill == false counts them
template <bool fill>
__global__ void ptent_kernel(int n, int k, const int* agg, const int* local, const int* a_off, const int* rank,
                             const int* coff, const double* Q, long long* cnt, const long long* rp, int* ci, double* v) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long c_out = 0, o = fill ? rp[i] : 0;
  const int a = agg[i];
  if (a >= 0) {
    const int m = a_off[a + 1] - a_off[a];
    const double* q = Q + (long long)a_off[a] * k;
    for (int c = 0; c < rank[a]; ++c) {
      const double val = q[c * m + local[i]];
      if (val != 0.0) {
        if (fill) ci[o] = coff[a] + c, v[o] = val, ++o;
        ++c_out;
      }
    }
  }
  if (!fill) cnt[i] = c_out;
}

// the next level's near-null space: nnc[c][coff[a] + r] = Rp_a(r, c) (amg.cpp:269-274)
__global__ void coarse_nn_kernel(int n_agg, int k, int nc, const int* rank, const int* coff, const double* Rp,
                                 double* nnc) {
  const long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (a >= n_agg) return;
  const double* rp = Rp + a * (long long)k * k;
  for (int r = 0; r < rank[a]; ++r)
    for (int c = 0; c < k; ++c) nnc[(long long)c * nc + coff[a] + r] = rp[r * k + c];
}

// rows rows[0..m) of A, packed (the fixed-stress neighbourhoods)
__global__ void gather_len_kernel(int m, const int* rows, const long long* rp, long long* cnt) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < m) cnt[t] = rp[rows[t] + 1] - rp[rows[t]];
  if (t == m) cnt[t] = 0;
}
__global__ void gather_rows_kernel(int m, const int* rows, const long long* rp, const int* ci, const double* v,
                                   const long long* off, int* oci, double* ov) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const long long r0 = rp[rows[t]], len = rp[rows[t] + 1] - r0;
  for (long long k = 0; k < len; ++k) oci[off[t] + k] = ci[r0 + k], ov[off[t] + k] = v[r0 + k];
}

DCsr clone(const DCsr& A) {
  DCsr C;
  C.n_rows = A.n_rows, C.n_cols = A.n_cols, C.nnz = A.nnz;
  C.rp.alloc(A.rp.size());
  C.ci.alloc(A.ci.size());
  C.v.alloc(A.v.size());
  if (A.rp.size()) cuda_check(cudaMemcpy(C.rp.get(), A.rp.get(), A.rp.bytes(), cudaMemcpyDeviceToDevice), "clone");
  if (A.ci.size()) cuda_check(cudaMemcpy(C.ci.get(), A.ci.get(), A.ci.bytes(), cudaMemcpyDeviceToDevice), "clone");
  if (A.v.size()) cuda_check(cudaMemcpy(C.v.get(), A.v.get(), A.v.bytes(), cudaMemcpyDeviceToDevice), "clone");
  return C;
}

// scale_rows (csr.cpp:208-214): a copy with v_ik * s_i
DCsr scale_rows_dev(const DCsr& A, const std::vector<double>& s) {
  DCsr C = clone(A);
  DevBuf<double> ds;
  ds.upload(s);
  if (A.n_rows) scale_rows_kernel<<<grid_for(A.n_rows), kT>>>(A.n_rows, C.rp.get(), ds.get(), C.v.get());
  cuda_check(cudaDeviceSynchronize(), "scale_rows_dev");
  return C;
}

std::vector<double> diag_dev(const DCsr& A) {
  if (A.n_rows != A.n_cols) throw std::invalid_argument("diag_extract: matrix must be square");
  DevBuf<double> d(static_cast<size_t>(A.n_rows));
  if (A.n_rows) diag_kernel<<<grid_for(A.n_rows), kT>>>(A.n_rows, A.rp.get(), A.ci.get(), A.v.get(), d.get());
  std::vector<double> h(static_cast<size_t>(A.n_rows));
  if (A.n_rows) cuda_check(cudaMemcpy(h.data(), d.get(), d.bytes(), cudaMemcpyDeviceToHost), "diag");
  return h;
}

// the host halves of the strength graph (the BFS runs on the host) plus the device weights
struct StrengthDev {
  std::vector<long long> off;
  std::vector<int> nbr;
  std::vector<char> isolated;
  DevBuf<double> w;
  DevBuf<long long> doff;
};

StrengthDev strength_dev(const DCsr& A, double theta) {
  const int n = A.n_rows;
  StrengthDev g;
  if (n == 0) {
    g.off.assign(1, 0);
    return g;
  }
  DevBuf<double> d(static_cast<size_t>(n));
  DevBuf<long long> cnt(size_t(n) + 1);
  g.doff.alloc(size_t(n) + 1);
  DevBuf<char> iso(static_cast<size_t>(n));
  cnt.zero();
  int sym = 1;
  {
    DevBuf<int> ok(1);
    cuda_check(cudaMemcpy(ok.get(), &sym, sizeof(int), cudaMemcpyHostToDevice), "flag");
    sym_check_kernel<<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), ok.get());
    cuda_check(cudaMemcpy(&sym, ok.get(), sizeof(int), cudaMemcpyDeviceToHost), "flag");
  }
  long long m = 0;
  DevBuf<int> nbr;
  if (sym) {
    bdiag_sym_kernel<<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), A.v.get(), d.get());
    strength_sym_kernel<false><<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), A.v.get(), d.get(), theta, cnt.get(),
                                                    iso.get(), nullptr, nullptr, nullptr);
    m = scan_counts(cnt, n, g.doff);
    nbr.alloc(size_t(m));
    g.w.alloc(size_t(m));
    if (m)
      strength_sym_kernel<true><<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), A.v.get(), d.get(), theta, nullptr,
                                                     nullptr, g.doff.get(), nbr.get(), g.w.get());
  } else {
    const DCsr At = transpose_dev(A, 0);
    bdiag_kernel<<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), A.v.get(), At.rp.get(), At.ci.get(), At.v.get(),
                                      d.get());
    strength_kernel<false><<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), A.v.get(), At.rp.get(), At.ci.get(),
                                                At.v.get(), d.get(), theta, cnt.get(), iso.get(), nullptr, nullptr,
                                                nullptr);
    m = scan_counts(cnt, n, g.doff);
    nbr.alloc(size_t(m));
    g.w.alloc(size_t(m));
    if (m)
      strength_kernel<true><<<grid_for(n), kT>>>(n, A.rp.get(), A.ci.get(), A.v.get(), At.rp.get(), At.ci.get(),
                                                 At.v.get(), d.get(), theta, nullptr, nullptr, g.doff.get(), nbr.get(),
                                                 g.w.get());
  }
  g.off.resize(size_t(n) + 1);
  g.nbr.resize(size_t(m));
  g.isolated.resize(size_t(n));
  cuda_check(cudaMemcpy(g.off.data(), g.doff.get(), g.doff.bytes(), cudaMemcpyDeviceToHost), "strength off");
  if (m) cuda_check(cudaMemcpy(g.nbr.data(), nbr.get(), nbr.bytes(), cudaMemcpyDeviceToHost), "strength nbr");
  cuda_check(cudaMemcpy(g.isolated.data(), iso.get(), iso.bytes(), cudaMemcpyDeviceToHost), "strength isolated");
  return g;
}

// amg.cpp:60-113 on the host graph; the weights of the leftover rows (the strongest-neighbour pass)
// are gathered on the device in one batch
std::pair<std::vector<int>, int> aggregate_host(const StrengthDev& g, int n) {
  std::vector<int> agg(static_cast<size_t>(n), -2);
  for (int i = 0; i < n; ++i)
    if (g.isolated[i]) agg[i] = -1;
  int n_agg = 0;
  std::vector<char> enq(static_cast<size_t>(n), 0);
  std::vector<int> queue;
  queue.reserve(static_cast<size_t>(n));
  for (int seed = 0; seed < n; ++seed) {
    if (agg[seed] != -2 || enq[seed]) continue;
    queue.clear();
    queue.push_back(seed);
    enq[seed] = 1;
    for (size_t head = 0; head < queue.size(); ++head) {
      const int i = queue[head];
      if (agg[i] == -2) {
        bool all_free = true;
        for (long long k = g.off[i]; k < g.off[i + 1]; ++k)
          if (agg[g.nbr[k]] >= 0) {
            all_free = false;
            break;
          }
        if (all_free) {
          const int id = n_agg++;
          agg[i] = id;
          for (long long k = g.off[i]; k < g.off[i + 1]; ++k)
            if (agg[g.nbr[k]] == -2) agg[g.nbr[k]] = id;
        }
      }
      for (long long k = g.off[i]; k < g.off[i + 1]; ++k) {
        const int j = g.nbr[k];
        if (!enq[j]) {
          enq[j] = 1;
          queue.push_back(j);
        }
      }
    }
  }
  std::vector<int> left;
  std::vector<long long> pos(1, 0);
  for (int i = 0; i < n; ++i)
    if (agg[i] == -2) left.push_back(i), pos.push_back(pos.back() + g.off[i + 1] - g.off[i]);
  std::vector<double> w(size_t(pos.back()));
  if (!left.empty() && pos.back() > 0) {
    DevBuf<int> drows;
    DevBuf<long long> dpos;
    drows.upload(left);
    dpos.upload(pos);
    DevBuf<double> dw(w.size());
    gather_w_kernel<<<grid_for((long long)left.size()), kT>>>(int(left.size()), drows.get(), g.doff.get(), g.w.get(),
                                                             dpos.get(), dw.get());
    cuda_check(cudaMemcpy(w.data(), dw.get(), dw.bytes(), cudaMemcpyDeviceToHost), "leftover weights");
  }
  for (size_t q = 0; q < left.size(); ++q) {  // in index order: a leftover may join one assigned before it
    const int i = left[q];
    int best = -1;
    double best_w = -1.0;
    for (long long k = g.off[i]; k < g.off[i + 1]; ++k) {
      const int j = g.nbr[k];
      const double wk = w[size_t(pos[q] + (k - g.off[i]))];
      if (agg[j] >= 0 && wk > best_w) best_w = wk, best = agg[j];
    }
    agg[i] = best >= 0 ? best : n_agg++;
  }
  return {agg, n_agg};
}

std::shared_ptr<fpb::DeviceMatrix> keep(DCsr&& m) {
  auto p = std::make_shared<fpb::DeviceMatrix>();
  p->m = std::move(m);
  return p;
}

fpb::Csr shape_only(int r, int c) {
  fpb::Csr A;
  A.n_rows = r, A.n_cols = c;
  A.rp.assign(1, 0);
  return A;
}

// amg_setup (amg.cpp:181-291) with the fine-size operators on the device
fpb::HostAmg amg_setup_dev(DCsr&& A0, const std::vector<std::vector<double>>& near_null, const fpb::AmgOptions& opt,
                           Clock& clk) {
  if (A0.n_rows != A0.n_cols) throw std::invalid_argument("amg_setup: matrix must be square");
  if (!(opt.strength_threshold >= 0.0 && opt.strength_threshold < 1.0))
    throw std::invalid_argument("amg_setup: strength_threshold must be in [0,1)");
  if (opt.pre_sweeps < 1 || opt.post_sweeps < 1) throw std::invalid_argument("amg_setup: sweeps must be >= 1");
  fpb::HostAmg h;
  h.opt = opt;
  std::vector<std::vector<double>> nn =
      near_null.empty() ? std::vector<std::vector<double>>{std::vector<double>(size_t(A0.n_rows), 1.0)} : near_null;
  for (const auto& v : nn)
    if (int(v.size()) != A0.n_rows) throw std::invalid_argument("amg_setup: near-null vector length mismatch");
  const int k = int(nn.size());
  DevBuf<double> nn_dev(size_t(k) * A0.n_rows);  // the near-null vectors, k columns of n
  for (int c = 0; c < k; ++c)
    if (A0.n_rows)
      cuda_check(cudaMemcpy(nn_dev.get() + size_t(c) * A0.n_rows, nn[c].data(), sizeof(double) * A0.n_rows,
                            cudaMemcpyHostToDevice), "near-null upload");
  nn.clear();
  {
    fpb::HostLevel f;
    f.diag = diag_dev(A0);
    f.A = shape_only(A0.n_rows, A0.n_cols);
    f.A_nnz = A0.nnz;
    f.dA = keep(std::move(A0));
    h.levels.push_back(std::move(f));
  }
  for (;;) {
    fpb::HostLevel& fine = h.levels.back();
    const DCsr& A = fine.dA->m;
    const int n = A.n_rows;
    for (int i = 0; i < n; ++i)
      if (fine.diag[i] == 0.0) throw fpb::numerical_error("amg_setup: zero diagonal entry at row " + std::to_string(i));
    if (n <= opt.max_coarse || int(h.levels.size()) >= opt.max_levels) break;
    clk.mark("level start", n);
    std::vector<int> agg;
    int n_agg = 0;
    {
      const StrengthDev g = strength_dev(A, opt.strength_threshold);
      clk.mark("strength (device)", (long long)g.nbr.size());
      std::tie(agg, n_agg) = aggregate_host(g, n);
    }
    clk.mark("aggregate (host BFS)", n_agg);
    if (n_agg == 0) break;
    std::vector<int> a_off(static_cast<size_t>(n_agg) + 1, 0), a_rows;
    for (int i = 0; i < n; ++i)
      if (agg[i] >= 0) ++a_off[size_t(agg[i]) + 1];
    for (int a = 0; a < n_agg; ++a) a_off[size_t(a) + 1] += a_off[a];
    a_rows.resize(static_cast<size_t>(a_off[n_agg]));
    {
      std::vector<int> next(a_off.begin(), a_off.end() - 1);
      for (int i = 0; i < n; ++i)
        if (agg[i] >= 0) a_rows[next[agg[i]]++] = i;
    }
    if (k > kQrMaxK) throw std::invalid_argument("amg_setup: more than 8 near-null vectors");
    // per-aggregate QR and the tentative P on the device (nn: k vectors of n, column-major in HBM)
    DevBuf<int> d_aoff, d_arows, d_agg, d_local, d_rank(static_cast<size_t>(n_agg)), d_coff;
    d_aoff.upload(a_off), d_arows.upload(a_rows), d_agg.upload(agg);
    std::vector<int> local(static_cast<size_t>(n), -1);
    for (int ag = 0; ag < n_agg; ++ag)
      for (int r = a_off[ag]; r < a_off[ag + 1]; ++r) local[a_rows[r]] = r - a_off[ag];
    d_local.upload(local);
    DevBuf<double> W(size_t(a_off[n_agg]) * k), Qd(size_t(a_off[n_agg]) * k), Rp(size_t(n_agg) * k * k);
    if (n_agg)
      qr_aggregates_kernel<<<grid_for(n_agg), kT>>>(n_agg, k, n, d_aoff.get(), d_arows.get(), nn_dev.get(), W.get(),
                                                     Qd.get(), d_rank.get(), Rp.get());
    std::vector<int> rank(static_cast<size_t>(n_agg));
    if (n_agg) cuda_check(cudaMemcpy(rank.data(), d_rank.get(), sizeof(int) * rank.size(), cudaMemcpyDeviceToHost), "ranks");
    W = DevBuf<double>();
    std::vector<int> coff(static_cast<size_t>(n_agg) + 1, 0);
    for (int ag = 0; ag < n_agg; ++ag) coff[size_t(ag) + 1] = coff[ag] + rank[ag];
    const int nc = coff[n_agg];
    if (nc == 0) break;
    d_coff.upload(coff);
    DCsr P;
    P.n_rows = n, P.n_cols = nc;
    {
      DevBuf<long long> cnt(size_t(n) + 1);
      cnt.zero();
      ptent_kernel<false><<<grid_for(n), kT>>>(n, k, d_agg.get(), d_local.get(), d_aoff.get(), d_rank.get(),
                                               d_coff.get(), Qd.get(), cnt.get(), nullptr, nullptr, nullptr);
      P.rp.alloc(size_t(n) + 1);
      P.nnz = scan_counts(cnt, n, P.rp);
      P.ci.alloc(size_t(P.nnz)), P.v.alloc(size_t(P.nnz));
      if (P.nnz)
        ptent_kernel<true><<<grid_for(n), kT>>>(n, k, d_agg.get(), d_local.get(), d_aoff.get(), d_rank.get(),
                                                d_coff.get(), Qd.get(), nullptr, P.rp.get(), P.ci.get(), P.v.get());
    }
    DevBuf<double> nnc(size_t(k) * nc);
    if (n_agg) coarse_nn_kernel<<<grid_for(n_agg), kT>>>(n_agg, k, nc, d_rank.get(), d_coff.get(), Rp.get(), nnc.get());
    cuda_check(cudaDeviceSynchronize(), "tentative P");
    clk.mark("tentative P (device QR)", P.nnz);
    if (opt.prolongation_smoothing) {  // P - w D^-1 A P
      std::vector<double> dinv(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) dinv[i] = 1.0 / fine.diag[i];
      DevBuf<double> ddinv;
      ddinv.upload(dinv);
      const DCsr DAP = spgemm_dev(A, P, ddinv.get());
      P = add_dev(P, DAP, 1.0, -opt.jacobi_omega);
    }
    clk.mark("smoothed P", P.nnz);
    if (nc > opt.stall_ratio * n) break;
    DCsr Ac;
    {
      const DCsr AP = spgemm_dev(A, P, nullptr);
      clk.mark("A P", AP.nnz);
      const DCsr Pt = transpose_dev(P, 0);
      Ac = spgemm_dev(Pt, AP, nullptr);
    }
    clk.mark("P^T (A P)", Ac.nnz);
    nn_dev = std::move(nnc);
    fpb::HostLevel next;
    next.diag = diag_dev(Ac);
    next.A = shape_only(Ac.n_rows, Ac.n_cols);
    next.A_nnz = Ac.nnz;
    next.P = shape_only(P.n_rows, P.n_cols);
    next.P_nnz = P.nnz;
    next.dA = keep(std::move(Ac));
    next.dP = keep(std::move(P));
    next.aggregate = std::move(agg);
    next.aggregate_offsets = std::move(coff);
    h.levels.push_back(std::move(next));
  }
  // coarse level: downloaded (at most max_levels / stall sized, typically <= 100 rows), dense LU
  {
    fpb::HostLevel& c = h.levels.back();
    c.A = download_csr(c.dA->m);
    h.coarse.compute(c.A.to_dense(), c.A.n_rows);
  }
  clk.mark("coarse LU", h.levels.back().A.n_rows);
  if (opt.smoother == 3)  // multicolour GS (extension): the colouring on the downloaded patterns
    for (size_t l = 0; l + 1 < h.levels.size(); ++l) {
      const fpb::Csr Al = download_csr(h.levels[l].dA->m);
      fpb::color_rows(Al.n_rows, Al.rp.data(), Al.ci.data(), h.levels[l].color_rows, h.levels[l].color_off);
    }
  if (opt.smoother == 2)  // Chebyshev (extension): the host estimate (index-order sums) on downloaded levels
    for (size_t l = 0; l + 1 < h.levels.size(); ++l) {
      const fpb::Csr Al = download_csr(h.levels[l].dA->m);
      h.levels[l].lambda_max = fpb::chebyshev_lambda_max(Al, h.levels[l].diag, opt.power_iterations);
    }
  return h;
}

}  // namespace

// alpha A + beta B on the union pattern (csr.cpp:181-206), row-parallel, explicit zeros kept
DCsr add_dev(const DCsr& A, const DCsr& B, double alpha, double beta) {
  if (A.n_rows != B.n_rows || A.n_cols != B.n_cols) throw std::invalid_argument("add_scaled: shape mismatch");
  DCsr C;
  C.n_rows = A.n_rows, C.n_cols = A.n_cols;
  DevBuf<long long> cnt(size_t(A.n_rows) + 1);
  cnt.zero();
  if (A.n_rows)
    add_rows_kernel<false><<<grid_for(A.n_rows), kT>>>(A.n_rows, A.rp.get(), A.ci.get(), A.v.get(), B.rp.get(), B.ci.get(),
                                                       B.v.get(), alpha, beta, A.n_cols, cnt.get(), nullptr, nullptr,
                                                       nullptr);
  C.rp.alloc(size_t(A.n_rows) + 1);
  C.nnz = scan_counts(cnt, A.n_rows, C.rp);
  C.ci.alloc(size_t(C.nnz));
  C.v.alloc(size_t(C.nnz));
  if (C.nnz)
    add_rows_kernel<true><<<grid_for(A.n_rows), kT>>>(A.n_rows, A.rp.get(), A.ci.get(), A.v.get(), B.rp.get(), B.ci.get(),
                                                      B.v.get(), alpha, beta, A.n_cols, nullptr, C.rp.get(), C.ci.get(),
                                                      C.v.get());
  cuda_check(cudaDeviceSynchronize(), "add_dev");
  return C;
}

// build_tpu / build_tup (precond.cpp:119-202) with the device-resident setup above
fpb::HostPrecond build_precond_device(const SystemView& J, const fpb::HostSystem* Jh, int variant,
                                      const fpb::AmgOptions& opt, const std::vector<std::array<double, 3>>& coords) {
  (void)Jh;
  if (variant < fpb::kTpu || variant > fpb::kTupStar) throw std::invalid_argument("build_precond: unknown variant");
  Clock clk;
  fpb::HostPrecond M;
  M.variant = variant;
  // the n_t / n_p-sized blocks are small: host copies for the host-side pieces
  const fpb::Csr H = host_copy(J.H), T = host_copy(J.T);
  M.hblocks = fpb::bdiag3_extract(H);
  DCsr core;
  {
    const DCsr dA = upload_csr(J.A), dC1 = upload_csr(J.C1), dC2 = upload_csr(J.C2);
    const DCsr Hinv = upload_csr(fpb::bdiag3_inverse_csr(M.hblocks));
    const DCsr HinvC2 = spgemm_dev(Hinv, dC2, nullptr);
    const DCsr C1HC2 = spgemm_dev(dC1, HinvC2, nullptr);
    core = add_dev(dA, C1HC2, 1.0, 1.0);
  }
  clk.mark("schur core", core.nnz);
  std::vector<std::vector<double>> nn;
  if (!coords.empty() && int(coords.size()) * 3 == J.n_u) nn = fpb::rigid_body_modes(coords);
  if (variant == fpb::kTpu) {
    M.T_diag = fpb::diag_extract(T);
    for (int i = 0; i < J.n_p; ++i)
      if (M.T_diag[i] == 0.0)
        throw fpb::numerical_error("build_tpu: singular diagonal entry of T at row " + std::to_string(i));
    M.factor.factor(T, fpb::BandFactor::Kind::spd);
    std::vector<double> tinv(M.T_diag.size());
    for (size_t i = 0; i < tinv.size(); ++i) tinv[i] = 1.0 / M.T_diag[i];
    DCsr S;
    {
      const DCsr dQ1 = upload_csr(J.Q1), dQ2s = scale_rows_dev(upload_csr(J.Q2), tinv);
      S = add_dev(core, spgemm_dev(dQ1, dQ2s, nullptr), 1.0, -1.0);
    }
    core = DCsr();
    M.amg = amg_setup_dev(std::move(S), nn, opt, clk);
  } else {
    M.amg = amg_setup_dev(std::move(core), nn, opt, clk);
    // fixed_stress_diag (precond.cpp:243-283) reads S1 only on the rows next to the fractures
    // (those of Q1^T and Q2): downloaded into a host matrix that is empty elsewhere
    const fpb::Csr Q1 = host_copy(J.Q1), Q2 = host_copy(J.Q2);
    std::vector<char> need(static_cast<size_t>(J.n_u), 0);
    for (int i = 0; i < Q1.n_rows; ++i)
      if (Q1.rp[i + 1] > Q1.rp[i]) need[i] = 1;
    for (int c : Q2.ci) need[c] = 1;
    std::vector<int> rows;
    for (int i = 0; i < J.n_u; ++i)
      if (need[i]) rows.push_back(i);
    const DCsr& S1 = M.amg.levels.front().dA->m;
    fpb::Csr S1n(J.n_u, J.n_u);  // rows `rows` filled, the others empty
    {
      DevBuf<int> drows;
      drows.upload(rows);
      const int m = int(rows.size());
      DevBuf<long long> cnt(size_t(m) + 1), off(size_t(m) + 1);
      if (m) gather_len_kernel<<<grid_for(m + 1), kT>>>(m, drows.get(), S1.rp.get(), cnt.get());
      else cnt.zero();
      const long long tot = scan_counts(cnt, m, off);
      DevBuf<int> oci(static_cast<size_t>(tot));
      DevBuf<double> ov(static_cast<size_t>(tot));
      if (m) gather_rows_kernel<<<grid_for(m), kT>>>(m, drows.get(), S1.rp.get(), S1.ci.get(), S1.v.get(), off.get(),
                                                     oci.get(), ov.get());
      std::vector<long long> hoff(size_t(m) + 1);
      cuda_check(cudaMemcpy(hoff.data(), off.get(), off.bytes(), cudaMemcpyDeviceToHost), "gather off");
      S1n.ci.resize(size_t(tot));
      S1n.v.resize(size_t(tot));
      if (tot) {
        cuda_check(cudaMemcpy(S1n.ci.data(), oci.get(), oci.bytes(), cudaMemcpyDeviceToHost), "gather ci");
        cuda_check(cudaMemcpy(S1n.v.data(), ov.get(), ov.bytes(), cudaMemcpyDeviceToHost), "gather v");
      }
      // row offsets: rows in `rows` take their packed ranges in order, the others are empty
      size_t q = 0;
      for (int i = 0; i < J.n_u; ++i) {
        const long long len = (q < rows.size() && rows[q] == i) ? hoff[q + 1] - hoff[q] : 0;
        if (q < rows.size() && rows[q] == i) ++q;
        S1n.rp[size_t(i) + 1] = S1n.rp[i] + len;
      }
    }
    M.S_K = fpb::fixed_stress_diag(Q2, S1n, Q1);
    clk.mark("fixed stress");
    std::vector<fpb::Csr::Triplet> sk;
    for (int k = 0; k < J.n_p; ++k)
      if (M.S_K[k] != 0.0) sk.push_back({k, k, M.S_K[k]});
    M.S2 = fpb::add_scaled(T, fpb::Csr::from_triplets(J.n_p, J.n_p, std::move(sk)), 1.0, -1.0);
    try {
      M.factor.factor(M.S2, fpb::BandFactor::Kind::general);
    } catch (const fpb::numerical_error&) {
      throw fpb::numerical_error("build_tup: singular S~2 factor (indefinite second-level Schur)");
    }
  }
  clk.mark("factor");
  return M;
}

}  // namespace fpd
