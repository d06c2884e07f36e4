// Banded exact factors for T (t-p-u, LDL^T) and S~2 (t-u-p, LU with partial
// pivoting): the framework's restatement of SparseFactor
// (/root/reference/proj/core/src/sparse_factor.cpp:30-67).  T and S~2 have no
// entries coupling two fractures (TPFA/stabilization edges are per patch,
// mesh.cpp:157-178), and faces are numbered first_face + i1 + nb*i2
// (mesh.cpp:128-130), so every fracture is an independent diagonal block with
// bandwidth nb in natural order.  Blocks are factored in parallel; the device
// solves them one warp per block (band_solve_kernel in kernels.cu).
#include <omp.h>

#include <algorithm>
#include <cmath>

#include "hcsr.hpp"

namespace fpb {

namespace {
struct Band {
  int n, lo, hi, w;
  std::vector<double> a;
  Band(int n_, int lo_, int hi_) : n(n_), lo(lo_), hi(hi_), w(lo_ + hi_ + 1), a(size_t(n_) * size_t(lo_ + hi_ + 1), 0.0) {}
  double& at(int i, int j) { return a[size_t(i) * w + size_t(j - i + lo)]; }
  bool in(int i, int j) const { return j - i >= -lo && j - i <= hi; }
};
}  // namespace

void BandFactor::factor(const Csr& A, Kind k) {
  if (A.n_rows != A.n_cols) throw std::invalid_argument("SparseFactor: matrix must be square");
  kind = k;
  n = A.n_rows;
  std::vector<int> maxcol(static_cast<size_t>(n)), mincol(static_cast<size_t>(n));
  int lo = 0, hi = 0;
  for (int i = 0; i < n; ++i) {
    int mn = i, mx = i;
    for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q) mn = std::min(mn, A.ci[q]), mx = std::max(mx, A.ci[q]);
    mincol[i] = mn, maxcol[i] = mx;
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
  const int nblk = int(block_start.size()) - 1;
  bool failed = false;

  if (kind == Kind::spd) {
    kl = lo;
    ku = 0;
    Lc.assign(size_t(n) * std::max(kl, 1), 0.0);
    Lr.assign(size_t(n) * std::max(kl, 1), 0.0);
    diag.assign(static_cast<size_t>(n), 0.0);
    piv.clear();
#pragma omp parallel for schedule(dynamic, 1)
    for (int blk = 0; blk < nblk; ++blk) {
      const int b0 = block_start[blk], b1 = block_start[blk + 1], nb = b1 - b0;
      Band L(nb, kl, 0);
      for (int i = b0; i < b1; ++i)
        for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q) {
          const int j = A.ci[q];
          if (j <= i && j >= b0) L.at(i - b0, j - b0) = A.v[q];
        }
      bool ok = true;
      for (int j = 0; j < nb && ok; ++j) {
        const double dj = L.at(j, j);
        if (!(std::abs(dj) > 0.0) || !std::isfinite(dj)) {
          ok = false;
          break;
        }
        diag[b0 + j] = dj;
        const int iend = std::min(nb, j + kl + 1);
        for (int i = j + 1; i < iend; ++i) L.at(i, j) = L.at(i, j) / dj;
        for (int i = j + 1; i < iend; ++i) {
          const double lij = L.at(i, j);
          if (lij == 0.0) continue;
          const double t = lij * dj;
          for (int kk = j + 1; kk <= i; ++kk) L.at(i, kk) -= t * L.at(kk, j);
        }
      }
      if (!ok) {
#pragma omp atomic write
        failed = true;
        continue;
      }
      for (int j = 0; j < nb; ++j)
        for (int r = 0; r < kl; ++r) {
          const int i = j + 1 + r, c = j - 1 - r;
          Lc[size_t(b0 + j) * kl + r] = i < nb ? L.at(i, j) : 0.0;
          Lr[size_t(b0 + j) * kl + r] = c >= 0 ? L.at(j, c) : 0.0;
        }
    }
    if (failed) throw numerical_error("SparseFactor: LDLT factorization failed (matrix not SPD?)");
    return;
  }
  kl = lo;
  ku = lo + hi;
  Lc.assign(size_t(n) * std::max(kl, 1), 0.0);
  Uc.assign(size_t(n) * std::max(ku, 1), 0.0);
  diag.assign(static_cast<size_t>(n), 0.0);
  piv.assign(static_cast<size_t>(n), 0);
  Lr.clear();
#pragma omp parallel for schedule(dynamic, 1)
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = block_start[blk], b1 = block_start[blk + 1], nb = b1 - b0;
    Band W(nb, kl, ku);
    for (int i = b0; i < b1; ++i)
      for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q) {
        const int j = A.ci[q];
        if (j >= b0 && j < b1) W.at(i - b0, j - b0) = A.v[q];
      }
    bool ok = true;
    for (int j = 0; j < nb; ++j) {
      const int iend = std::min(nb, j + kl + 1);
      int p = j;
      double best = std::abs(W.at(j, j));
      for (int i = j + 1; i < iend; ++i)
        if (std::abs(W.at(i, j)) > best) best = std::abs(W.at(i, j)), p = i;
      if (best == 0.0 || !std::isfinite(best)) {
        ok = false;
        break;
      }
      piv[b0 + j] = b0 + p;
      const int jend = std::min(nb, j + ku + 1);
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
    if (!ok) {
#pragma omp atomic write
      failed = true;
      continue;
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
  }
  if (failed) throw numerical_error("SparseFactor: sparse LU factorization failed (singular matrix?)");
  // Trim U to its effective bandwidth and record whether any row swap happened.
  // Dropped entries are exact zeros (x_i - 0 * x_j == x_i), so the solve is
  // unchanged bit for bit; without swaps the device skips the pivot path.
  pivoted = false;
  for (int j = 0; j < n; ++j) pivoted = pivoted || piv[j] != j;
  int ku_eff = 0;
  for (int j = 0; j < n; ++j)
    for (int r = ku - 1; r >= ku_eff; --r)
      if (Uc[size_t(j) * ku + r] != 0.0) {
        ku_eff = r + 1;
        break;
      }
  if (ku_eff < ku) {
    std::vector<double> U2(size_t(n) * std::max(ku_eff, 1), 0.0);
    for (int j = 0; j < n; ++j)
      for (int r = 0; r < ku_eff; ++r) U2[size_t(j) * ku_eff + r] = Uc[size_t(j) * ku + r];
    Uc.swap(U2);
    ku = ku_eff;
  }
}

std::vector<double> BandFactor::solve(std::span<const double> b) const {
  std::vector<double> x(b.begin(), b.end());
  const int nblk = int(block_start.size()) - 1;
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = block_start[blk], b1 = block_start[blk + 1];
    for (int j = b0; j < b1; ++j) {
      if (kind == Kind::general && piv[j] != j) std::swap(x[j], x[piv[j]]);
      const double yj = x[j];
      for (int r = 0; r < kl && j + 1 + r < b1; ++r) x[j + 1 + r] -= Lc[size_t(j) * kl + r] * yj;
    }
    if (kind == Kind::spd) {
      for (int j = b0; j < b1; ++j) x[j] = x[j] / diag[j];
      for (int j = b1 - 1; j >= b0; --j) {
        const double xj = x[j];
        for (int r = 0; r < kl && j - 1 - r >= b0; ++r) x[j - 1 - r] -= Lr[size_t(j) * kl + r] * xj;
      }
    } else {
      for (int j = b1 - 1; j >= b0; --j) {
        const double xj = x[j] / diag[j];
        x[j] = xj;
        for (int r = 0; r < ku && j - 1 - r >= b0; ++r) x[j - 1 - r] -= Uc[size_t(j) * ku + r] * xj;
      }
    }
  }
  return x;
}

void BandFactor::inverse_blocks(std::vector<double>& inv, std::vector<int64_t>& off) const {
  const int nblk = int(block_start.size()) - 1;
  off.assign(size_t(nblk) + 1, 0);
  for (int blk = 0; blk < nblk; ++blk) {
    const int64_t nb = block_start[blk + 1] - block_start[blk];
    off[blk + 1] = off[blk] + nb * nb;
  }
  inv.assign(size_t(off.back()), 0.0);
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = block_start[blk], nb = block_start[blk + 1] - b0;
    double* out = inv.data() + off[blk];
#pragma omp parallel
    {
      std::vector<double> xv(static_cast<size_t>(nb));
      double* x = xv.data() - b0;  // absolute indexing inside the block
#pragma omp for schedule(dynamic, 16)
      for (int c = 0; c < nb; ++c) {
        std::fill(xv.begin(), xv.end(), 0.0);
        x[b0 + c] = 1.0;
        for (int j = b0; j < b0 + nb; ++j) {
          if (kind == Kind::general && piv[j] != j) std::swap(x[j], x[piv[j]]);
          const double yj = x[j];
          if (yj == 0.0) continue;
          const int e = std::min(kl, b0 + nb - 1 - j);
          const double* l = Lc.data() + size_t(j) * kl;
          for (int r = 0; r < e; ++r) x[j + 1 + r] -= l[r] * yj;
        }
        if (kind == Kind::spd) {
          for (int j = b0; j < b0 + nb; ++j) x[j] = x[j] / diag[j];
          for (int j = b0 + nb - 1; j >= b0; --j) {
            const double xj = x[j];
            if (xj == 0.0) continue;
            const int e = std::min(kl, j - b0);
            const double* l = Lr.data() + size_t(j) * kl;
            for (int r = 0; r < e; ++r) x[j - 1 - r] -= l[r] * xj;
          }
        } else {
          for (int j = b0 + nb - 1; j >= b0; --j) {
            const double xj = x[j] / diag[j];
            x[j] = xj;
            if (xj == 0.0) continue;
            const int e = std::min(ku, j - b0);
            const double* u = Uc.data() + size_t(j) * ku;
            for (int r = 0; r < e; ++r) x[j - 1 - r] -= u[r] * xj;
          }
        }
        for (int i = 0; i < nb; ++i) out[size_t(i) * nb + c] = xv[size_t(i)];
      }
    }
  }
}

}  // namespace fpb
