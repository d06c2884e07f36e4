// ORACLE (test infrastructure only) — exact direct factors used on the solve path.
//  * DenseFullPivLU restates Eigen::FullPivLU as used by the AMG coarse solve
//    (/root/reference/proj/core/src/amg.cpp:144-149,284-289) and the fixed-stress
//    local solves (precond.cpp:273-278).
//  * BandFactor restates SparseFactor (sparse_factor.cpp:30-67): LDL^T for
//    Kind::spd (T in t-p-u, precond.cpp:129), LU with partial pivoting for
//    Kind::general (S~2 in t-u-p, precond.cpp:182).  Bitwise parity with Eigen is
//    not pinned by any reference test; the reference only checks
//    residual-level properties (test_gmres.cpp:25-42), re-expressed in tests.
// Solve order (part of the oracle's definition, reproduced by the GPU):
// column sweeps — forward: for j ascending, finalize y_j, then subtract
// L(i,j)*y_j from each later row i; backward: for j descending, finalize x_j,
// then subtract U(i,j)*x_j from each earlier row i.
// factor_solve = inverse: the same operator as an explicit per-block inverse
// (columns = sweep solves of unit vectors) applied as a block GEMV whose row
// sums are 32 lane-strided partials combined by a fixed xor tree.
#include <algorithm>
#include <cmath>
#include <limits>

#include "fpo.hpp"
#include "par.hpp"

namespace fpo {

void DenseFullPivLU::compute(const std::vector<double>& a, int nn) {
  n = nn;
  lu = a;
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
    if (best == 0.0) {  // the remaining block is exactly zero
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
  // rank: pivots above n * eps * |largest pivot| (Eigen's default threshold rule)
  const double thr = double(n) * std::numeric_limits<double>::epsilon() * maxpivot;
  rank = 0;
  for (int k = 0; k < nonzero; ++k)
    if (std::abs(lu[size_t(k) * n + k]) > thr) ++rank;
}

std::vector<double> DenseFullPivLU::solve(std::span<const double> b) const {
  if (int(b.size()) != n) throw std::invalid_argument("DenseFullPivLU::solve: dimension mismatch");
  std::vector<double> c(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) c[i] = b[prow[i]];
  for (int j = 0; j < n; ++j) {  // unit lower, column sweep
    const double cj = c[j];
    for (int i = j + 1; i < n; ++i) c[i] -= lu[size_t(i) * n + j] * cj;
  }
  for (int j = rank - 1; j >= 0; --j) {  // upper on the leading rank x rank block
    const double xj = c[j] / lu[size_t(j) * n + j];
    c[j] = xj;
    for (int i = 0; i < j; ++i) c[i] -= lu[size_t(i) * n + j] * xj;
  }
  std::vector<double> x(static_cast<size_t>(n), 0.0);
  for (int i = 0; i < rank; ++i) x[pcol[i]] = c[i];
  return x;
}

// ---------------------------------------------------------------- BandFactor
namespace {

// Dense band working storage for one diagonal block [b0, b1): row-major with
// columns j in [i - lo, i + hi] mapped to slot (j - i + lo).
struct Band {
  int n, lo, hi, w;
  std::vector<double> a;
  Band(int n_, int lo_, int hi_) : n(n_), lo(lo_), hi(hi_), w(lo_ + hi_ + 1), a(static_cast<size_t>(n_) * (lo_ + hi_ + 1), 0.0) {}
  double& at(int i, int j) { return a[size_t(i) * w + (j - i + lo)]; }
  bool in(int i, int j) const { return j - i >= -lo && j - i <= hi; }
};

}  // namespace

void BandFactor::factor(const CsrMatrix& A, Kind k) {
  if (A.n_rows != A.n_cols) throw std::invalid_argument("SparseFactor: matrix must be square");
  kind = k;
  n = A.n_rows;
  // Independent diagonal blocks: a split at s is valid when no row < s has a
  // column >= s and no row >= s has a column < s.
  std::vector<int> maxcol(static_cast<size_t>(n), 0), mincol(static_cast<size_t>(n), 0);
  int lo = 0, hi = 0;
  for (int i = 0; i < n; ++i) {
    int mn = i, mx = i;
    for (int64_t q = A.row_offsets[i]; q < A.row_offsets[i + 1]; ++q) {
      mn = std::min(mn, A.col_indices[q]);
      mx = std::max(mx, A.col_indices[q]);
    }
    mincol[i] = mn;
    maxcol[i] = mx;
    lo = std::max(lo, i - mn);
    hi = std::max(hi, mx - i);
  }
  std::vector<int> suffix_min(static_cast<size_t>(n) + 1, n);
  for (int s = n - 1; s >= 0; --s) suffix_min[s] = std::min(suffix_min[size_t(s) + 1], mincol[s]);
  block_start.assign(1, 0);
  int prefix_max = -1;
  for (int s = 1; s < n; ++s) {
    prefix_max = std::max(prefix_max, maxcol[s - 1]);
    if (prefix_max < s && suffix_min[s] >= s) block_start.push_back(s);
  }
  block_start.push_back(n);
  if (n == 0) block_start.assign(1, 0);
  if (kind == Kind::spd) {
    kl = lo;
    ku = 0;
    Lc.assign(static_cast<size_t>(n) * std::max(kl, 1), 0.0);
    Lr.assign(static_cast<size_t>(n) * std::max(kl, 1), 0.0);
    diag.assign(static_cast<size_t>(n), 0.0);
    piv.clear();
    LoopError err;
    const long nblk = long(block_start.size()) - 1;
#pragma omp parallel for num_threads(threads()) schedule(dynamic)
    for (long blk = 0; blk < nblk; ++blk) {
     try {
      const int b0 = block_start[blk], b1 = block_start[blk + 1], nb = b1 - b0;
      Band L(nb, kl, 0);  // lower triangle of A (symmetric input: use the lower part)
      for (int i = b0; i < b1; ++i)
        for (int64_t q = A.row_offsets[i]; q < A.row_offsets[i + 1]; ++q) {
          const int j = A.col_indices[q];
          if (j <= i && j >= b0) L.at(i - b0, j - b0) = A.values[q];
        }
      // right-looking LDL^T inside the band: for each column j, D_j = pivot,
      // l_ij = a_ij / D_j, then a_ik -= l_ij * D_j * l_kj for j < k <= i.
      std::vector<double> D(static_cast<size_t>(nb));
      for (int j = 0; j < nb; ++j) {
        const double dj = L.at(j, j);
        if (!(std::abs(dj) > 0.0) || !std::isfinite(dj))
          throw numerical_error("SparseFactor: LDLT factorization failed (matrix not SPD?)");
        D[j] = dj;
        const int iend = std::min(nb, j + kl + 1);
        for (int i = j + 1; i < iend; ++i) L.at(i, j) = L.at(i, j) / dj;
        for (int i = j + 1; i < iend; ++i) {
          const double lij = L.at(i, j);
          if (lij == 0.0) continue;
          const double t = lij * dj;
          for (int kk = j + 1; kk <= i; ++kk) L.at(i, kk) -= t * L.at(kk, j);
        }
      }
      for (int j = 0; j < nb; ++j) {
        diag[b0 + j] = D[j];
        for (int r = 0; r < kl; ++r) {
          const int i = j + 1 + r;
          Lc[size_t(b0 + j) * kl + r] = i < nb ? L.at(i, j) : 0.0;
          const int c = j - 1 - r;
          Lr[size_t(b0 + j) * kl + r] = c >= 0 ? L.at(j, c) : 0.0;
        }
      }
     } catch (...) {
      err.capture(blk);
     }
    }
    err.rethrow();
    return;
  }
  // general: banded LU with partial pivoting (row interchanges within the band)
  kl = lo;
  ku = lo + hi;
  Lc.assign(static_cast<size_t>(n) * std::max(kl, 1), 0.0);
  Uc.assign(static_cast<size_t>(n) * std::max(ku, 1), 0.0);
  diag.assign(static_cast<size_t>(n), 0.0);
  piv.assign(static_cast<size_t>(n), 0);
  Lr.clear();
  LoopError err;
  const long nblk = long(block_start.size()) - 1;
#pragma omp parallel for num_threads(threads()) schedule(dynamic)
  for (long blk = 0; blk < nblk; ++blk) {
   try {
    const int b0 = block_start[blk], b1 = block_start[blk + 1], nb = b1 - b0;
    Band W(nb, kl, ku);
    for (int i = b0; i < b1; ++i)
      for (int64_t q = A.row_offsets[i]; q < A.row_offsets[i + 1]; ++q) {
        const int j = A.col_indices[q];
        if (j >= b0 && j < b1) W.at(i - b0, j - b0) = A.values[q];
      }
    for (int j = 0; j < nb; ++j) {
      const int iend = std::min(nb, j + kl + 1);
      int p = j;
      double best = std::abs(W.at(j, j));
      for (int i = j + 1; i < iend; ++i)
        if (std::abs(W.at(i, j)) > best) best = std::abs(W.at(i, j)), p = i;
      if (best == 0.0 || !std::isfinite(best))
        throw numerical_error("SparseFactor: sparse LU factorization failed (singular matrix?)");
      piv[b0 + j] = b0 + p;
      const int jend = std::min(nb, j + ku + 1);  // columns touched by row j after swaps
      if (p != j)
        for (int c = j; c < jend; ++c) std::swap(W.at(j, c), W.at(p, c));
      const double ujj = W.at(j, j);
      for (int i = j + 1; i < iend; ++i) {
        const double f = W.at(i, j) / ujj;
        W.at(i, j) = f;
        if (f == 0.0) continue;
        for (int c = j + 1; c < jend; ++c) W.at(i, c) -= f * W.at(j, c);
      }
    }
    for (int j = 0; j < nb; ++j) {
      diag[b0 + j] = W.at(j, j);
      for (int r = 0; r < kl; ++r) {
        const int i = j + 1 + r;
        Lc[size_t(b0 + j) * kl + r] = i < nb ? W.at(i, j) : 0.0;
      }
      for (int r = 0; r < ku; ++r) {
        const int i = j - 1 - r;
        Uc[size_t(b0 + j) * ku + r] = (i >= 0 && W.in(i, j)) ? W.at(i, j) : 0.0;
      }
    }
   } catch (...) {
    err.capture(blk);
   }
  }
  err.rethrow();
}

void BandFactor::solve_block(int blk, double* x) const {
  const int b0 = block_start[blk], b1 = block_start[blk + 1];
  // forward sweep: (pivot) + unit-lower L
  for (int j = b0; j < b1; ++j) {
    if (kind == Kind::general && piv[j] != j) std::swap(x[j], x[piv[j]]);
    const double yj = x[j];
    for (int r = 0; r < kl; ++r) {
      const int i = j + 1 + r;
      if (i >= b1) break;
      x[i] -= Lc[size_t(j) * kl + r] * yj;
    }
  }
  if (kind == Kind::spd) {
    for (int j = b0; j < b1; ++j) x[j] = x[j] / diag[j];
    // backward sweep with L^T: x_j final, then x_i -= L(j,i) x_j for i < j
    for (int j = b1 - 1; j >= b0; --j) {
      const double xj = x[j];
      for (int r = 0; r < kl; ++r) {
        const int i = j - 1 - r;
        if (i < b0) break;
        x[i] -= Lr[size_t(j) * kl + r] * xj;
      }
    }
  } else {
    for (int j = b1 - 1; j >= b0; --j) {
      const double xj = x[j] / diag[j];
      x[j] = xj;
      for (int r = 0; r < ku; ++r) {
        const int i = j - 1 - r;
        if (i < b0) break;
        x[i] -= Uc[size_t(j) * ku + r] * xj;
      }
    }
  }
}

void BandFactor::build_inverse() {
  const int nblk = int(block_start.size()) - 1;
  inv_off.assign(size_t(nblk) + 1, 0);
  for (int blk = 0; blk < nblk; ++blk) {
    const size_t nb = size_t(block_start[blk + 1] - block_start[blk]);
    inv_off[blk + 1] = inv_off[blk] + nb * nb;
  }
  inv.assign(inv_off.back(), 0.0);
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = block_start[blk], nb = block_start[blk + 1] - b0;
#pragma omp parallel num_threads(threads())
    {
      std::vector<double> e(static_cast<size_t>(n), 0.0);  // solve_block indexes absolute rows
#pragma omp for schedule(dynamic, 16)
      for (int c = 0; c < nb; ++c) {
        std::fill(e.begin() + b0, e.begin() + b0 + nb, 0.0);
        e[b0 + c] = 1.0;
        solve_block(blk, e.data());
        for (int i = 0; i < nb; ++i) inv[inv_off[blk] + size_t(i) * nb + c] = e[b0 + i];
      }
    }
  }
}

// ------------------------------------------------- factor_solve = panel (fpo.hpp)
bool BandFactor::pivots() const {
  if (kind == Kind::spd) return false;
  for (int j = 0; j < n; ++j)
    if (piv[j] != j) return true;
  return false;
}

namespace {
// 32 lane-strided partials over c ascending from 0.0, then the xor tree h = 16..1 (the warp order)
double strided_dot(const double* row, const double* x, int len) {
  double v[32];
  for (int j = 0; j < 32; ++j) {
    double s = 0.0;
    for (int c = j; c < len; c += 32) s = s + row[c] * x[c];
    v[j] = s;
  }
  for (int h = 16; h >= 1; h >>= 1) {
    double w[32];
    for (int j = 0; j < 32; ++j) w[j] = v[j] + v[j ^ h];
    std::copy(w, w + 32, v);
  }
  return v[0];
}
}  // namespace

void BandFactor::build_panels() {
  if (pivots()) throw std::invalid_argument("factor_solve = panel needs a factor without row interchanges");
  const int nblk = int(block_start.size()) - 1;
  pan_p.assign(size_t(nblk), 1);
  pan_off.assign(size_t(nblk) + 1, 0);
  const int ub = kind == Kind::spd ? kl : ku;  // stored upper band of U (spd: L^T)
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = block_start[blk], b1 = block_start[blk + 1];
    int p = 1;
    for (int j = b0; j < b1; ++j) {
      for (int r = 0; r < kl; ++r)
        if (Lc[size_t(j) * kl + r] != 0.0) p = std::max(p, r + 1);
      for (int r = 0; r < ub; ++r)
        if ((kind == Kind::spd ? Lr[size_t(j) * kl + r] : Uc[size_t(j) * ku + r]) != 0.0) p = std::max(p, r + 1);
    }
    pan_p[blk] = p;
    const int m = b1 - b0, P = (m + p - 1) / p;
    size_t sz = 0;
    for (int q = 0; q < P; ++q) {
      const size_t s = size_t(std::min(p, m - q * p));
      const size_t sp = q > 0 ? size_t(p) : 0, sn = q + 1 < P ? size_t(std::min(p, m - (q + 1) * p)) : 0;
      sz += s * s + s * sp + s * s + s * sn;
    }
    pan_off[blk + 1] = pan_off[blk] + sz;
  }
  pan.assign(pan_off.back(), 0.0);
  // L(gi, gj) / U(gi, gj) from the band storage (0 outside the band)
  auto Lv = [&](int gi, int gj) { return gi > gj && gi - gj <= kl ? Lc[size_t(gj) * kl + (gi - gj - 1)] : 0.0; };
  auto Uv = [&](int gi, int gj) {  // strictly upper part (spd: L(gj, gi))
    if (!(gj > gi)) return 0.0;
    if (kind == Kind::spd) return gj - gi <= kl ? Lr[size_t(gj) * kl + (gj - gi - 1)] : 0.0;
    return gj - gi <= ku ? Uc[size_t(gj) * ku + (gj - gi - 1)] : 0.0;
  };
#pragma omp parallel for num_threads(threads()) schedule(dynamic)
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = block_start[blk], m = block_start[blk + 1] - b0, p = pan_p[blk], P = (m + p - 1) / p;
    double* out = pan.data() + pan_off[blk];
    std::vector<double> z(static_cast<size_t>(p));
    for (int q = 0; q < P; ++q) {
      const int r0 = b0 + q * p, s = std::min(p, m - q * p);
      const int sp = q > 0 ? p : 0, sn = q + 1 < P ? std::min(p, m - (q + 1) * p) : 0;
      auto fwd = [&]() {  // z <- L_qq^-1 z (unit lower, column sweeps)
        for (int j = 0; j < s; ++j) {
          const double zj = z[j];
          for (int i = j + 1; i < s; ++i) z[i] -= Lv(r0 + i, r0 + j) * zj;
        }
      };
      auto bwd = [&]() {  // z <- U_qq^-1 z (general: divide by the diagonal; spd: unit)
        for (int j = s - 1; j >= 0; --j) {
          double zj = z[j];
          if (kind == Kind::general) {
            zj = zj / diag[r0 + j];
            z[j] = zj;
          }
          for (int i = j - 1; i >= 0; --i) z[i] -= Uv(r0 + i, r0 + j) * zj;
        }
      };
      double* H = out;
      double* G = H + size_t(s) * s;
      double* K = G + size_t(s) * sp;
      double* F = K + size_t(s) * s;
      for (int c = 0; c < s; ++c) {
        std::fill(z.begin(), z.begin() + s, 0.0);
        z[c] = 1.0;
        fwd();
        for (int i = 0; i < s; ++i) H[size_t(i) * s + c] = z[i];
        std::fill(z.begin(), z.begin() + s, 0.0);
        z[c] = 1.0;
        bwd();
        for (int i = 0; i < s; ++i) K[size_t(i) * s + c] = z[i];
      }
      for (int c = 0; c < sp; ++c) {  // G column c: L(panel q rows, panel q-1 column c)
        for (int i = 0; i < s; ++i) z[i] = Lv(r0 + i, r0 - sp + c);
        fwd();
        for (int i = 0; i < s; ++i) G[size_t(i) * sp + c] = z[i];
      }
      for (int c = 0; c < sn; ++c) {  // F column c: U(panel q rows, panel q+1 column c)
        for (int i = 0; i < s; ++i) z[i] = Uv(r0 + i, r0 + s + c);
        bwd();
        for (int i = 0; i < s; ++i) F[size_t(i) * sn + c] = z[i];
      }
      out = F + size_t(s) * sn;
    }
  }
}

std::vector<double> BandFactor::solve(std::span<const double> b) const {
  if (int(b.size()) != n) throw std::invalid_argument("SparseFactor::solve: dimension mismatch");
  std::vector<double> x(b.begin(), b.end());
  const int nblk = int(block_start.size()) - 1;
#pragma omp parallel for num_threads(threads()) schedule(dynamic)
  for (int blk = 0; blk < nblk; ++blk) {
    if (!pan.empty()) {  // factor_solve = panel
      const int b0 = block_start[blk], m = block_start[blk + 1] - b0, p = pan_p[blk], P = (m + p - 1) / p;
      std::vector<double> y(static_cast<size_t>(m));
      const double* base = pan.data() + pan_off[blk];
      std::vector<const double*> Kq(static_cast<size_t>(P)), Fq(static_cast<size_t>(P));
      for (int q = 0; q < P; ++q) {  // forward: y_q = H_q b_q - G_q y_q-1
        const int s = std::min(p, m - q * p), sp = q > 0 ? p : 0, sn = q + 1 < P ? std::min(p, m - (q + 1) * p) : 0;
        const double* H = base;
        const double* G = H + size_t(s) * s;
        Kq[q] = G + size_t(s) * sp;
        Fq[q] = Kq[q] + size_t(s) * s;
        base = Fq[q] + size_t(s) * sn;
        for (int i = 0; i < s; ++i) {
          const double sh = strided_dot(H + size_t(i) * s, b.data() + b0 + q * p, s);
          const double sg = sp ? strided_dot(G + size_t(i) * sp, y.data() + (q - 1) * p, sp) : 0.0;
          y[size_t(q) * p + i] = sp ? sh - sg : sh;
        }
      }
      if (kind == Kind::spd)
        for (int i = 0; i < m; ++i) y[i] = y[i] / diag[b0 + i];
      for (int q = P - 1; q >= 0; --q) {  // backward: x_q = K_q z_q - F_q x_q+1
        const int s = std::min(p, m - q * p), sn = q + 1 < P ? std::min(p, m - (q + 1) * p) : 0;
        for (int i = 0; i < s; ++i) {
          const double sk = strided_dot(Kq[q] + size_t(i) * s, y.data() + q * p, s);
          const double sf = sn ? strided_dot(Fq[q] + size_t(i) * sn, x.data() + b0 + (q + 1) * p, sn) : 0.0;
          x[b0 + q * p + i] = sn ? sk - sf : sk;
        }
      }
      continue;
    }
    if (inv.empty()) {
      solve_block(blk, x.data());
      continue;
    }
    // row i: 32 strided partial sums v[j] = sum_{c = j mod 32} inv(i,c) b_c (c
    // ascending, from 0.0), combined by the xor tree v[j] += v[j ^ h], h = 16..1;
    // x_i = v[0]  (a warp per row, lane j owning columns j, j+32, ...)
    const int b0 = block_start[blk], nb = block_start[blk + 1] - b0;
    for (int i = 0; i < nb; ++i) {
      const double* row = inv.data() + inv_off[blk] + size_t(i) * nb;
      double v[32];
      for (int j = 0; j < 32; ++j) {
        double s = 0.0;
        for (int c = j; c < nb; c += 32) s = s + row[c] * b[b0 + c];
        v[j] = s;
      }
      for (int h = 16; h >= 1; h >>= 1) {
        double w[32];
        for (int j = 0; j < 32; ++j) w[j] = v[j] + v[j ^ h];
        std::copy(w, w + 32, v);
      }
      x[b0 + i] = v[0];
    }
  }
  return x;
}

}  // namespace fpo
