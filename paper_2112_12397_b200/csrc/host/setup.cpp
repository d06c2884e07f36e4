// Host preconditioner setup (see setup.hpp).  Reference algorithm:
// strength (amg.cpp:27-54), BFS aggregation (:60-113), per-aggregate QR of the
// near-null space (:214-257), damped-Jacobi prolongation smoothing (:259-264),
// stall test (:266), Galerkin RAP (:268), coarse full-pivot LU (:284-289);
// schur_core (precond.cpp:18-36), fixed_stress_diag (:243-283), build_tpu
// (:119-151), build_tup (:168-202).
#include "setup.hpp"

#include <omp.h>

#include <algorithm>
#include <tuple>
#include <cmath>
#include <cstdio>
#include <deque>
#include <chrono>
#include <cstdlib>
#include <limits>

namespace fpb {

namespace {

// FRACPREC_B200_VERBOSE=1 prints per-phase setup times to stderr
struct PhaseLog {
  bool on = std::getenv("FRACPREC_B200_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, long a = -1, long b = -1) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    long pages = 0, rss = 0;
    if (FILE* f = std::fopen("/proc/self/statm", "r")) {
      if (std::fscanf(f, "%ld %ld", &pages, &rss) != 2) rss = 0;
      std::fclose(f);
    }
    std::fprintf(stderr, "[setup] %-28s %8.3f s  %ld %ld  rss %.1f GB\n", what,
                 std::chrono::duration<double>(now - t).count(), a, b, double(rss) * 4096.0 / 1e9);
    t = now;
  }
};

struct Strength {
  std::vector<int64_t> off;
  std::vector<int> nbr;
  std::vector<double> w;
  std::vector<char> isolated;
};

Strength build_strength(const Csr& A, double theta) {
  const Csr B = add_scaled(A, transpose(A), 0.5, 0.5);
  const std::vector<double> d = diag_extract(B);
  const int n = A.n_rows;
  Strength g;
  g.isolated.assign(static_cast<size_t>(n), 0);
  // count, then fill (row-parallel; row contents follow B's column order)
  std::vector<int64_t> cnt(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    int offdiag = 0, strong = 0;
    for (int64_t k = B.rp[i]; k < B.rp[i + 1]; ++k) {
      const int j = B.ci[k];
      if (j == i) continue;
      if (B.v[k] != 0.0) ++offdiag;
      const double thr = theta * std::sqrt(std::abs(d[i]) * std::abs(d[j]));
      if (std::abs(B.v[k]) > thr) ++strong;
    }
    cnt[size_t(i) + 1] = strong;
    if (offdiag == 0) g.isolated[i] = 1;
  }
  for (int i = 0; i < n; ++i) cnt[size_t(i) + 1] += cnt[i];
  g.off = cnt;
  g.nbr.resize(static_cast<size_t>(cnt[n]));
  g.w.resize(static_cast<size_t>(cnt[n]));
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    int64_t p = g.off[i];
    for (int64_t k = B.rp[i]; k < B.rp[i + 1]; ++k) {
      const int j = B.ci[k];
      if (j == i) continue;
      const double thr = theta * std::sqrt(std::abs(d[i]) * std::abs(d[j]));
      if (std::abs(B.v[k]) > thr) {
        g.nbr[p] = j;
        g.w[p] = std::abs(B.v[k]);
        ++p;
      }
    }
  }
  return g;
}

// Sequential BFS aggregation: the visiting order defines the aggregates, so it
// is kept exactly as the reference's.
std::pair<std::vector<int>, int> aggregate(const Strength& g, int n) {
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
        for (int64_t k = g.off[i]; k < g.off[i + 1]; ++k)
          if (agg[g.nbr[k]] >= 0) {
            all_free = false;
            break;
          }
        if (all_free) {
          const int id = n_agg++;
          agg[i] = id;
          for (int64_t k = g.off[i]; k < g.off[i + 1]; ++k)
            if (agg[g.nbr[k]] == -2) agg[g.nbr[k]] = id;
        }
      }
      for (int64_t k = g.off[i]; k < g.off[i + 1]; ++k) {
        const int j = g.nbr[k];
        if (!enq[j]) {
          enq[j] = 1;
          queue.push_back(j);
        }
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    if (agg[i] != -2) continue;
    int best = -1;
    double best_w = -1.0;
    for (int64_t k = g.off[i]; k < g.off[i + 1]; ++k) {
      const int j = g.nbr[k];
      if (agg[j] >= 0 && g.w[k] > best_w) best_w = g.w[k], best = agg[j];
    }
    agg[i] = best >= 0 ? best : n_agg++;
  }
  return {agg, n_agg};
}

double householder(double* x, int len) {
  double tail = 0.0;
  for (int i = 1; i < len; ++i) tail += x[i] * x[i];
  const double c0 = x[0];
  if (tail <= std::numeric_limits<double>::min()) {
    for (int i = 1; i < len; ++i) x[i] = 0.0;
    return 0.0;
  }
  double beta = std::sqrt(c0 * c0 + tail);
  if (c0 >= 0.0) beta = -beta;
  const double denom = c0 - beta;
  for (int i = 1; i < len; ++i) x[i] = x[i] / denom;
  x[0] = beta;
  return (beta - c0) / beta;
}

}  // namespace

int qr_colpiv(int m, int k, const std::vector<double>& B, std::vector<double>& Q, std::vector<double>& Rp) {
  std::vector<double> W = B;
  std::vector<int> perm(static_cast<size_t>(k));
  for (int j = 0; j < k; ++j) perm[j] = j;
  const int mn = std::min(m, k);
  std::vector<double> tau(static_cast<size_t>(mn), 0.0);
  auto col = [&](int j) { return W.data() + size_t(j) * m; };
  for (int j = 0; j < mn; ++j) {
    int p = j;
    double best = -1.0;
    for (int c = j; c < k; ++c) {
      double s = 0.0;
      for (int i = j; i < m; ++i) s += col(c)[i] * col(c)[i];
      if (s > best) best = s, p = c;
    }
    if (p != j) {
      for (int i = 0; i < m; ++i) std::swap(col(j)[i], col(p)[i]);
      std::swap(perm[j], perm[p]);
    }
    tau[j] = householder(col(j) + j, m - j);
    for (int c = j + 1; c < k; ++c) {
      double s = col(c)[j];
      for (int i = j + 1; i < m; ++i) s += col(j)[i] * col(c)[i];
      s *= tau[j];
      col(c)[j] -= s;
      for (int i = j + 1; i < m; ++i) col(c)[i] -= s * col(j)[i];
    }
  }
  const double r00 = mn > 0 ? std::abs(col(0)[0]) : 0.0;
  const double tol = 1e-12 * std::max(1.0, r00);
  int rank = 0;
  for (int j = 0; j < mn; ++j)
    if (std::abs(col(j)[j]) > tol) ++rank;
  Q.assign(size_t(m) * rank, 0.0);
  for (int c = 0; c < rank; ++c) {
    double* q = Q.data() + size_t(c) * m;
    q[c] = 1.0;
    for (int j = std::min(c, mn - 1); j >= 0; --j) {
      double s = q[j];
      for (int i = j + 1; i < m; ++i) s += col(j)[i] * q[i];
      s *= tau[j];
      q[j] -= s;
      for (int i = j + 1; i < m; ++i) q[i] -= s * col(j)[i];
    }
  }
  Rp.assign(size_t(rank) * k, 0.0);
  for (int r = 0; r < rank; ++r)
    for (int j = r; j < k; ++j) Rp[size_t(r) * k + perm[j]] = col(j)[r];
  return rank;
}

HostAmg amg_setup(Csr A, const std::vector<std::vector<double>>& near_null, const AmgOptions& opt) {
  if (A.n_rows != A.n_cols) throw std::invalid_argument("amg_setup: matrix must be square");
  if (!(opt.strength_threshold >= 0.0 && opt.strength_threshold < 1.0))
    throw std::invalid_argument("amg_setup: strength_threshold must be in [0,1)");
  if (opt.pre_sweeps < 1 || opt.post_sweeps < 1) throw std::invalid_argument("amg_setup: sweeps must be >= 1");
  HostAmg h;
  h.opt = opt;
  std::vector<std::vector<double>> nn =
      near_null.empty() ? std::vector<std::vector<double>>{std::vector<double>(size_t(A.n_rows), 1.0)} : near_null;
  for (const auto& v : nn)
    if (int(v.size()) != A.n_rows) throw std::invalid_argument("amg_setup: near-null vector length mismatch");
  {
    HostLevel f;
    f.diag = diag_extract(A);
    f.A = std::move(A);
    h.levels.push_back(std::move(f));
  }
  PhaseLog plog;
  for (;;) {
    HostLevel& fine = h.levels.back();
    const int n = fine.A.n_rows;
    for (int i = 0; i < n; ++i)
      if (fine.diag[i] == 0.0) throw numerical_error("amg_setup: zero diagonal entry at row " + std::to_string(i));
    if (n <= opt.max_coarse || int(h.levels.size()) >= opt.max_levels) break;
    plog.mark("level start", n, long(fine.A.nnz()));
    std::vector<int> agg;
    int n_agg = 0;
    {  // the strength graph lives only for the aggregation
      const Strength g = build_strength(fine.A, opt.strength_threshold);
      plog.mark("strength", long(g.nbr.size()));
      std::tie(agg, n_agg) = aggregate(g, n);
    }
    plog.mark("aggregate", n_agg);
    if (n_agg == 0) break;
    const int k = int(nn.size());
    // rows of each aggregate in ascending order (counting sort)
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
    std::vector<std::vector<double>> qs(static_cast<size_t>(n_agg)), rps(static_cast<size_t>(n_agg));
    std::vector<int> rank(static_cast<size_t>(n_agg));
#pragma omp parallel for schedule(dynamic, 64)
    for (int a = 0; a < n_agg; ++a) {
      const int m = a_off[a + 1] - a_off[a];
      std::vector<double> B(size_t(m) * k);
      for (int c = 0; c < k; ++c)
        for (int r = 0; r < m; ++r) B[size_t(c) * m + r] = nn[c][a_rows[a_off[a] + r]];
      rank[a] = qr_colpiv(m, k, B, qs[a], rps[a]);
    }
    std::vector<int> coff(static_cast<size_t>(n_agg) + 1, 0);
    for (int a = 0; a < n_agg; ++a) coff[size_t(a) + 1] = coff[a] + rank[a];
    const int nc = coff[n_agg];
    if (nc == 0) break;
    // tentative P: each fine row lies in one aggregate, so its entries are the
    // nonzero Q entries of that aggregate in ascending coarse column order
    Csr P(n, nc);
    {
      std::vector<int> local(static_cast<size_t>(n), -1);
      for (int a = 0; a < n_agg; ++a)
        for (int r = a_off[a]; r < a_off[a + 1]; ++r) local[a_rows[r]] = r - a_off[a];
      for (int i = 0; i < n; ++i) {
        int cnt = 0;
        if (agg[i] >= 0) {
          const int a = agg[i], m = a_off[a + 1] - a_off[a];
          for (int c = 0; c < rank[a]; ++c) cnt += qs[a][size_t(c) * m + local[i]] != 0.0;
        }
        P.rp[size_t(i) + 1] = P.rp[i] + cnt;
      }
      P.ci.resize(static_cast<size_t>(P.rp[n]));
      P.v.resize(static_cast<size_t>(P.rp[n]));
#pragma omp parallel for schedule(static)
      for (int i = 0; i < n; ++i) {
        if (agg[i] < 0) continue;
        const int a = agg[i], m = a_off[a + 1] - a_off[a];
        int64_t p = P.rp[i];
        for (int c = 0; c < rank[a]; ++c) {
          const double v = qs[a][size_t(c) * m + local[i]];
          if (v != 0.0) P.ci[p] = coff[a] + c, P.v[p] = v, ++p;
        }
      }
    }
    plog.mark("tentative P", nc, long(P.nnz()));
    if (opt.prolongation_smoothing) {
      std::vector<double> dinv(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) dinv[i] = 1.0 / fine.diag[i];
      P = add_scaled(P, spgemm_setup(fine.A, P, dinv), 1.0, -opt.jacobi_omega);  // P - w D^-1 A P
    }
    plog.mark("smoothed P", long(P.nnz()));
    if (nc > opt.stall_ratio * n) break;
    const Csr AP = spgemm_setup(fine.A, P);
    plog.mark("A P", long(AP.nnz()));
    const Csr Pt = transpose(P);
    plog.mark("P^T");
    Csr Ac = spgemm_setup(Pt, AP);
    plog.mark("P^T (A P)", long(Ac.nnz()));
    std::vector<std::vector<double>> nnc(static_cast<size_t>(k), std::vector<double>(static_cast<size_t>(nc), 0.0));
    for (int a = 0; a < n_agg; ++a)
      for (int r = 0; r < rank[a]; ++r)
        for (int c = 0; c < k; ++c) nnc[c][coff[a] + r] = rps[a][size_t(r) * k + c];
    nn = std::move(nnc);
    HostLevel next;
    next.A = std::move(Ac);
    next.P = std::move(P);
    next.diag = diag_extract(next.A);
    next.aggregate = std::move(agg);
    next.aggregate_offsets = std::move(coff);
    h.levels.push_back(std::move(next));
  }
  const Csr& Ac = h.levels.back().A;
  h.coarse.compute(Ac.to_dense(), Ac.n_rows);
  plog.mark("coarse LU", Ac.n_rows);
  if (opt.smoother == 2) {
    for (size_t l = 0; l + 1 < h.levels.size(); ++l)
      h.levels[l].lambda_max = chebyshev_lambda_max(h.levels[l].A, h.levels[l].diag, opt.power_iterations);
    plog.mark("chebyshev lambda_max");
  }
  if (opt.smoother == 3)
    for (size_t l = 0; l + 1 < h.levels.size(); ++l) {
      const Csr& A = h.levels[l].A;
      color_rows(A.n_rows, A.rp.data(), A.ci.data(), h.levels[l].color_rows, h.levels[l].color_off);
    }
  return h;
}

void color_rows(int n, const int64_t* rp, const int* ci, std::vector<int>& rows, std::vector<int>& off) {
  // earlier neighbours in either direction: j < i in row i, and the rows j < i holding an entry (j, i)
  std::vector<int64_t> tp(static_cast<size_t>(n) + 1, 0);
  for (int64_t k = 0; k < rp[n]; ++k) ++tp[size_t(ci[k]) + 1];
  for (int i = 0; i < n; ++i) tp[size_t(i) + 1] += tp[i];
  std::vector<int> trow(static_cast<size_t>(rp[n]));
  {
    std::vector<int64_t> next(tp.begin(), tp.end() - 1);
    for (int i = 0; i < n; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) trow[size_t(next[size_t(ci[k])]++)] = i;
  }
  std::vector<int> color(static_cast<size_t>(n), -1);
  std::vector<int> seen;  // seen[c] == i: colour c is taken by a neighbour of row i
  int n_colors = 0;
  for (int i = 0; i < n; ++i) {
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] < i) seen[size_t(color[ci[k]])] = i;
    for (int64_t k = tp[i]; k < tp[i + 1]; ++k)
      if (trow[k] < i) seen[size_t(color[trow[k]])] = i;
    int c = 0;
    while (c < n_colors && seen[size_t(c)] == i) ++c;
    color[i] = c;
    if (c == n_colors) ++n_colors, seen.push_back(-1);
  }
  off.assign(static_cast<size_t>(n_colors) + 1, 0);
  for (int i = 0; i < n; ++i) ++off[size_t(color[i]) + 1];
  for (int c = 0; c < n_colors; ++c) off[size_t(c) + 1] += off[c];
  rows.resize(static_cast<size_t>(n));
  std::vector<int> next(off.begin(), off.end() - 1);
  for (int i = 0; i < n; ++i) rows[size_t(next[size_t(color[i])]++)] = i;
}

double chebyshev_lambda_max(const Csr& A, const std::vector<double>& diag, int iterations) {
  const int n = A.n_rows;
  if (n == 0) return 1.0;
  std::vector<double> v(static_cast<size_t>(n), 1.0 / std::sqrt(double(n))), w(static_cast<size_t>(n));
  double lam = 0.0;
  for (int it = 0; it < std::max(1, iterations); ++it) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {  // each row summed left to right from 0.0 (csr.cpp:112-117)
      double s = 0.0;
      for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) s += A.v[k] * v[A.ci[k]];
      w[i] = s / diag[i];
    }
    double s = 0.0;  // index order, one thread: the oracle's sum
    for (int i = 0; i < n; ++i) s += w[i] * w[i];
    const double nrm = std::sqrt(s);
    if (!(nrm > 0.0) || !std::isfinite(nrm)) throw numerical_error("chebyshev: power iteration broke down");
    lam = nrm;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) v[i] = w[i] / nrm;
  }
  return 1.1 * lam;
}

ChebyshevCoefficients chebyshev_coefficients(double lambda_max, double ratio, int degree) {
  if (!(lambda_max > 0.0) || !(ratio > 1.0) || degree < 1)
    throw std::invalid_argument("chebyshev: need lambda_max > 0, ratio > 1, degree >= 1");
  ChebyshevCoefficients c;
  const double lmin = lambda_max / ratio;
  c.theta = (lambda_max + lmin) / 2.0;
  const double delta = (lambda_max - lmin) / 2.0;
  const double sigma = c.theta / delta;
  double rho = 1.0 / sigma;
  for (int k = 1; k < degree; ++k) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    c.c1.push_back(rho_new * rho);
    c.c2.push_back(2.0 * rho_new / delta);
    rho = rho_new;
  }
  return c;
}

std::vector<std::vector<double>> rigid_body_modes(const std::vector<std::array<double, 3>>& c) {
  const size_t n = c.size();
  std::vector<std::vector<double>> m(6, std::vector<double>(3 * n, 0.0));
  for (size_t v = 0; v < n; ++v) {
    const double x = c[v][0], y = c[v][1], z = c[v][2];
    m[0][3 * v] = 1.0;
    m[1][3 * v + 1] = 1.0;
    m[2][3 * v + 2] = 1.0;
    m[3][3 * v + 1] = -z;
    m[3][3 * v + 2] = y;
    m[4][3 * v] = z;
    m[4][3 * v + 2] = -x;
    m[5][3 * v] = -y;
    m[5][3 * v + 1] = x;
  }
  return m;
}

std::vector<double> fixed_stress_diag(const Csr& Q2, const Csr& S1, const Csr& Q1) {
  if (Q1.n_cols != Q2.n_rows || Q1.n_rows != Q2.n_cols || S1.n_rows != Q1.n_rows || S1.n_rows != S1.n_cols)
    throw std::invalid_argument("fixed_stress_diag: inconsistent shapes");
  const int n_p = Q1.n_cols;
  const Csr Q1t = transpose(Q1);
  std::vector<double> sk(static_cast<size_t>(n_p), 0.0);
  int warned = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : warned)
  for (int k = 0; k < n_p; ++k) {
    const int64_t q2b = Q2.rp[k], q2e = Q2.rp[k + 1];
    if (q2b == q2e) continue;
    const int64_t q1b = Q1t.rp[k], q1e = Q1t.rp[k + 1];
    std::vector<int> idx(Q1t.ci.begin() + q1b, Q1t.ci.begin() + q1e);
    idx.insert(idx.end(), Q2.ci.begin() + q2b, Q2.ci.begin() + q2e);
    std::sort(idx.begin(), idx.end());
    idx.erase(std::unique(idx.begin(), idx.end()), idx.end());
    const int m = int(idx.size());
    std::vector<double> q1(static_cast<size_t>(m), 0.0), q2(static_cast<size_t>(m), 0.0);
    for (int64_t e = q1b; e < q1e; ++e)
      q1[size_t(std::lower_bound(idx.begin(), idx.end(), Q1t.ci[e]) - idx.begin())] = Q1t.v[e];
    for (int64_t e = q2b; e < q2e; ++e)
      q2[size_t(std::lower_bound(idx.begin(), idx.end(), Q2.ci[e]) - idx.begin())] = Q2.v[e];
    FullPivLU lu;
    lu.compute(restrict_dense(S1, idx), m);
    if (!lu.invertible()) {
      warned = 1;
      continue;
    }
    const std::vector<double> x = lu.solve(q1);
    double d = 0.0;
    for (int i = 0; i < m; ++i) d += q2[i] * x[i];
    sk[k] = d;
  }
  if (warned) std::fprintf(stderr, "fixed_stress_diag: singular local block(s), entries set to 0\n");
  return sk;
}

namespace {
SpgemmBackend g_spgemm_backend = nullptr;
}
void set_spgemm_backend(SpgemmBackend fn) { g_spgemm_backend = fn; }
bool spgemm_backend_active() { return g_spgemm_backend != nullptr; }
Csr spgemm_setup(const Csr& A, const Csr& B, std::span<const double> row_scale) {
  Csr C;
  if (g_spgemm_backend && g_spgemm_backend(A, B, row_scale, C)) return C;
  return spgemm(A, B, row_scale);
}

HostPrecond build_precond(const HostSystem& J, int variant, const AmgOptions& opt,
                          const std::vector<std::array<double, 3>>& coords) {
  J.check_shapes();
  if (variant < kTpu || variant > kTupStar) throw std::invalid_argument("build_precond: unknown variant");
  HostPrecond M;
  PhaseLog plog;
  M.variant = variant;
  M.hblocks = bdiag3_extract(J.H);
  const Csr HinvC2 = spgemm_setup(bdiag3_inverse_csr(M.hblocks), J.C2);
  Csr core = add_scaled(J.A, spgemm_setup(J.C1, HinvC2), 1.0, 1.0);
  plog.mark("schur core", long(core.nnz()));
  std::vector<std::vector<double>> nn;
  if (!coords.empty() && int(coords.size()) * 3 == J.n_u) nn = rigid_body_modes(coords);
  if (variant == kTpu) {
    M.T_diag = diag_extract(J.T);
    for (int i = 0; i < J.n_p; ++i)
      if (M.T_diag[i] == 0.0) throw numerical_error("build_tpu: singular diagonal entry of T at row " + std::to_string(i));
    M.factor.factor(J.T, BandFactor::Kind::spd);
    std::vector<double> tinv(M.T_diag.size());
    for (size_t i = 0; i < tinv.size(); ++i) tinv[i] = 1.0 / M.T_diag[i];
    Csr S = add_scaled(core, spgemm_setup(J.Q1, scale_rows(J.Q2, tinv)), 1.0, -1.0);
    core = Csr();  // free the fine-size temporary before the hierarchy is built
    M.amg = amg_setup(std::move(S), nn, opt);
  } else {
    M.amg = amg_setup(std::move(core), nn, opt);
    plog.mark("amg setup (all levels)");
    M.S_K = fixed_stress_diag(J.Q2, M.S(), J.Q1);
    plog.mark("fixed stress");
    std::vector<Csr::Triplet> sk;
    for (int k = 0; k < J.n_p; ++k)
      if (M.S_K[k] != 0.0) sk.push_back({k, k, M.S_K[k]});
    M.S2 = add_scaled(J.T, Csr::from_triplets(J.n_p, J.n_p, std::move(sk)), 1.0, -1.0);
    try {
      M.factor.factor(M.S2, BandFactor::Kind::general);
    } catch (const numerical_error&) {
      throw numerical_error("build_tup: singular S~2 factor (indefinite second-level Schur)");
    }
  }
  return M;
}

}  // namespace fpb
