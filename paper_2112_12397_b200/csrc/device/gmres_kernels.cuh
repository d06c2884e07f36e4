// Device-resident Arnoldi for right-preconditioned GMRES
// (/root/reference/proj/core/src/gmres.cpp:81-167).  One cooperative kernel
// per iteration performs modified Gram-Schmidt with the reference's selective
// reorthogonalization (gmres.cpp:96-102), the happy-breakdown test (:107),
// normalization (:145-149) and the Givens update of the least-squares problem
// (:151-171).  Each MGS step is one fused pass "w -= h_i V_i ; partial(V_{i+1}.w)"
// followed by a grid barrier; reductions are fixed-order (per-block tree, then
// every block sums the block partials in index order), so runs are bitwise
// reproducible.
#pragma once

#include <cooperative_groups.h>

#include "device.cuh"

namespace fpd {

struct MgsArgs {
  long long n, ldv;
  int m;        // V_0..V_m exist; the new column index is m
  int ldr;      // leading dimension of R (restart + 1)
  double* V;    // basis, V_i = V + i*ldv; V_{m+1} receives the new vector
  const double* w_in;  // J z
  double* stage;       // preconditioner input staging (receives V_{m+1})
  double* partial;     // 2 * 2 * gridDim doubles (double-buffered)
  double* h;           // ldr + 1
  double* cs;          // rotations
  double* sn;
  double* g;           // ldr + 1
  double* R;           // ldr * ldr, column j at R + j*ldr
  double beta;         // ||r|| of the cycle
  GmresStatus* status;
};

constexpr int kMgsThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* sm) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sm[i];
  return s;  // valid in thread 0
}

// All blocks reduce the same partials with the same fixed tree (coalesced
// load, warp shuffles, then the warp sums in index order) -> identical totals
// in every block, bitwise reproducible run to run.
__device__ __forceinline__ double grid_total(const double* part, int nb, double* sm) {
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += __ldcg(part + b);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sm[i];
    sm[32] = s;
  }
  __syncthreads();
  return sm[32];
}

// status + Givens update of the least-squares problem (gmres.cpp:114-131), one thread
__device__ __forceinline__ void mgs_finish(const MgsArgs& a, double hnext, double wnorm_pre, int reorth, bool finite,
                                           bool happy) {
  GmresStatus st;
  st.hnext = hnext;
  st.wnorm_pre = wnorm_pre;
  st.happy = happy;
  st.nonfinite = !finite;
  st.reorth = reorth;
  st.m = a.m;
  st.est = 0.0;
  if (finite) {
    double* h = a.h;
    const int m = a.m;
    h[m + 1] = hnext;
    for (int i = 0; i < m; ++i) {  // accumulated Givens rotations
      const double t0 = a.cs[i] * h[i] + a.sn[i] * h[i + 1];
      const double t1 = -a.sn[i] * h[i] + a.cs[i] * h[i + 1];
      h[i] = t0;
      h[i + 1] = t1;
    }
    const double denom = hypot(h[m], h[m + 1]);
    const double c = denom == 0.0 ? 1.0 : h[m] / denom;
    const double s = denom == 0.0 ? 0.0 : h[m + 1] / denom;
    a.cs[m] = c;
    a.sn[m] = s;
    h[m] = denom;
    h[m + 1] = 0.0;
    for (int i = 0; i <= m; ++i) a.R[(long long)m * a.ldr + i] = h[i];
    const double gm = a.g[m];
    a.g[m] = c * gm;
    a.g[m + 1] = -s * gm;
    st.est = fabs(a.g[m + 1]) / a.beta;
  }
  *a.status = st;
}

__global__ void __launch_bounds__(kMgsThreads) mgs_kernel(MgsArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sm[40];
  const int nb = gridDim.x;
  const long long chunk = ((a.n + nb - 1) / nb + 31) / 32 * 32;
  const long long lo = blockIdx.x * chunk, hi = lo + chunk < a.n ? lo + chunk : a.n;
  double* w = a.V + (long long)(a.m + 1) * a.ldv;
  int buf = 0;
  auto publish = [&](double v) {
    const double s = block_sum(v, sm);
    if (threadIdx.x == 0) a.partial[buf * nb + blockIdx.x] = s;
    grid.sync();
    const double t = grid_total(a.partial + buf * nb, nb, sm);
    buf ^= 1;
    return t;
  };
  // pass 0: copy J z into the new column, ||w||^2 and V_0 . w
  double n2 = 0.0, d0 = 0.0;
  const double* V0 = a.V;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = a.w_in[i];
    w[i] = v;
    n2 += v * v;
    d0 += V0[i] * v;
  }
  {
    const double s = block_sum(n2, sm);
    const double t = block_sum(d0, sm);
    if (threadIdx.x == 0) {
      a.partial[2 * nb + blockIdx.x] = s;  // second half of the buffer as a scratch pair
      a.partial[3 * nb + blockIdx.x] = t;
    }
    grid.sync();
  }
  const double wnorm_pre = sqrt(grid_total(a.partial + 2 * nb, nb, sm));
  __syncthreads();
  double hcur = grid_total(a.partial + 3 * nb, nb, sm);
  __syncthreads();
  buf = 0;
  if (!isfinite(wnorm_pre)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.status->nonfinite = 1;
      a.status->wnorm_pre = wnorm_pre;
    }
    return;  // uniform across the grid
  }
  double hloc[2] = {0, 0};
  (void)hloc;
  double nrm2 = 0.0;
  for (int i = 0; i <= a.m; ++i) {
    if (blockIdx.x == 0 && threadIdx.x == 0) a.h[i] = hcur;
    const double* Vi = a.V + (long long)i * a.ldv;
    const double* Vn = i < a.m ? a.V + (long long)(i + 1) * a.ldv : nullptr;
    double acc = 0.0;
    for (long long k = lo + threadIdx.x; k < hi; k += blockDim.x) {
      const double wv = w[k] - hcur * Vi[k];
      w[k] = wv;
      acc += Vn ? Vn[k] * wv : wv * wv;
    }
    const double t = publish(acc);
    __syncthreads();
    if (i < a.m)
      hcur = t;
    else
      nrm2 = t;
  }
  double hnext = sqrt(nrm2);
  int reorth = 0;
  if (hnext < 0.70710678118654752 * wnorm_pre) {  // gmres.cpp:96
    reorth = 1;
    double acc = 0.0;
    for (long long k = lo + threadIdx.x; k < hi; k += blockDim.x) acc += V0[k] * w[k];
    double c = publish(acc);
    __syncthreads();
    for (int i = 0; i <= a.m; ++i) {
      if (blockIdx.x == 0 && threadIdx.x == 0) a.h[i] += c;
      const double* Vi = a.V + (long long)i * a.ldv;
      const double* Vn = i < a.m ? a.V + (long long)(i + 1) * a.ldv : nullptr;
      double acc2 = 0.0;
      for (long long k = lo + threadIdx.x; k < hi; k += blockDim.x) {
        const double wv = w[k] - c * Vi[k];
        w[k] = wv;
        acc2 += Vn ? Vn[k] * wv : wv * wv;
      }
      const double t = publish(acc2);
      __syncthreads();
      if (i < a.m)
        c = t;
      else
        nrm2 = t;
    }
    hnext = sqrt(nrm2);
  }
  const bool finite = isfinite(hnext);
  const bool happy = hnext <= 1e-14 * fmax(1.0, wnorm_pre);
  if (finite && !happy)
    for (long long k = lo + threadIdx.x; k < hi; k += blockDim.x) {
      const double v = w[k] / hnext;
      w[k] = v;
      a.stage[k] = v;
    }
  if (blockIdx.x == 0 && threadIdx.x == 0) mgs_finish(a, hnext, wnorm_pre, reorth, finite, happy);
}

// The grid MGS with this block's slice of w in shared memory and its slices
// of the basis columns in registers (E per thread): step i loads V_{i+1} (and,
// for E <= 8, already V_{i+2} before the barrier, hiding the load behind it),
// so the only exposed latency per projection is the barrier + fixed-order sum.
// Leaner fixed-order reductions for mgs_fast_kernel: warp shuffles, then warp 0
// combines the warp sums (one block barrier); after the grid barrier warp 0 alone
// reads the nb partials and broadcasts through shared memory (one more barrier).
// Same order in every block and every run: deterministic.
__device__ __forceinline__ double block_sum_w0(double v, double* sm) {  // valid in warp 0
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = l < int(blockDim.x >> 5) ? sm[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;
}
__device__ __forceinline__ double grid_total_w0(const double* part, int nb, double* sm) {
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) v += __ldcg(part + b);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) sm[36] = v;
  }
  __syncthreads();
  return sm[36];
}

template <int E>
__global__ void __launch_bounds__(kMgsThreads) mgs_fast_kernel(MgsArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr bool kAhead = E <= 8;
  extern __shared__ double mgs_ws[];
  __shared__ double sm[40];
  const int nb = gridDim.x;
  const long long chunk = ((a.n + nb - 1) / nb + 31) / 32 * 32;
  const long long lo = blockIdx.x * chunk;
  const int len = lo < a.n ? int(min(chunk, a.n - lo)) : 0;
  int buf = 0;
  auto publish = [&](double v) {
    const double s = block_sum_w0(v, sm);
    if (threadIdx.x == 0) a.partial[buf * nb + blockIdx.x] = s;
    grid.sync();
    const double t = grid_total_w0(a.partial + buf * nb, nb, sm);
    buf ^= 1;
    return t;
  };
  auto load = [&](const double* V, double (&r)[E]) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int k = threadIdx.x + j * kMgsThreads;
      r[j] = k < len ? __ldcg(V + lo + k) : 0.0;
    }
  };
  double vc[E], vn[E];
  // pass 0: w = J z, ||w||^2 and V_0 . w (two partial sets, one barrier)
  {
    double n2 = 0.0, d0 = 0.0;
    load(a.V, vc);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int k = threadIdx.x + j * kMgsThreads;
      const double v = k < len ? a.w_in[lo + k] : 0.0;
      if (k < len) mgs_ws[k] = v;
      n2 += v * v;
      d0 += vc[j] * v;
    }
    const double s = block_sum_w0(n2, sm);
    const double t = block_sum_w0(d0, sm + 16);
    if (threadIdx.x == 0) {
      a.partial[2 * nb + blockIdx.x] = s;
      a.partial[3 * nb + blockIdx.x] = t;
    }
    if (kAhead && a.m >= 1) load(a.V + a.ldv, vn);
    grid.sync();
  }
  const double wnorm_pre = sqrt(grid_total_w0(a.partial + 2 * nb, nb, sm));
  __syncthreads();
  const double h0 = grid_total_w0(a.partial + 3 * nb, nb, sm);
  if (!isfinite(wnorm_pre)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.status->nonfinite = 1;
      a.status->wnorm_pre = wnorm_pre;
    }
    return;  // uniform across the grid
  }
  // one MGS sweep; on entry vc = V_0 slice and (kAhead) vn = V_1 slice
  auto sweep = [&](double c, bool accumulate) {
    double nrm2 = 0.0;
    for (int i = 0; i <= a.m; ++i) {
      if (blockIdx.x == 0 && threadIdx.x == 0) a.h[i] = accumulate ? a.h[i] + c : c;
      const bool last = i == a.m;
      if (!kAhead && !last) load(a.V + (long long)(i + 1) * a.ldv, vn);
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const int k = threadIdx.x + j * kMgsThreads;
        if (k < len) {
          const double wv = mgs_ws[k] - c * vc[j];
          mgs_ws[k] = wv;
          acc += last ? wv * wv : vn[j] * wv;
        }
      }
      if (!last) {
#pragma unroll
        for (int j = 0; j < E; ++j) vc[j] = vn[j];
        if (kAhead && i + 2 <= a.m) load(a.V + (long long)(i + 2) * a.ldv, vn);  // behind the barrier
      }
      const double t = publish(acc);
      if (!last)
        c = t;
      else
        nrm2 = t;
    }
    return nrm2;
  };
  double hnext = sqrt(sweep(h0, false));
  int reorth = 0;
  if (hnext < 0.70710678118654752 * wnorm_pre) {  // gmres.cpp:96
    reorth = 1;
    load(a.V, vc);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int k = threadIdx.x + j * kMgsThreads;
      if (k < len) acc += vc[j] * mgs_ws[k];
    }
    if (kAhead && a.m >= 1) load(a.V + a.ldv, vn);
    const double c = publish(acc);
    hnext = sqrt(sweep(c, true));
  }
  const bool finite = isfinite(hnext);
  const bool happy = hnext <= 1e-14 * fmax(1.0, wnorm_pre);
  double* wg = a.V + (long long)(a.m + 1) * a.ldv + lo;
  for (int k = threadIdx.x; k < len; k += blockDim.x) {
    const double v = (finite && !happy) ? mgs_ws[k] / hnext : mgs_ws[k];
    wg[k] = v;
    if (finite && !happy) a.stage[lo + k] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) mgs_finish(a, hnext, wnorm_pre, reorth, finite, happy);
}

// Classical Gram-Schmidt Arnoldi step with the same DGKS test as the reference
// (gmres.cpp:96-102: a second pass when ||w|| < ||w_pre|| / sqrt 2), selectable
// instead of MGS (orthogonalization = cgs).  Every projection coefficient of a
// pass comes from ONE grid reduction (all m + 1 dot products at once), so a step
// costs 2 grid barriers (4 with the second pass) instead of 2 (m + 1), at the
// price of reading the basis twice per pass.  In exact arithmetic the basis,
// H and the iterates are the MGS ones; classical GS twice ("twice is enough",
// Kahan-Parlett / DGKS) keeps the basis orthogonal to working precision, and
// tests/test_gpu_parity.py holds it to the reference bars against the oracle's
// MGS (+-2 iterations, solution 1e-8).
// E > 0: this block's slice of w is held in registers (E values per thread,
// k = threadIdx + j * kMgsThreads); E == 0: w lives in its final column V_{m+1}.
// Basis columns are read in batches so ~16 loads per thread are in flight.
constexpr int kCgsGroup = 32;     // coefficients reduced per block-level pass
constexpr int kCgsMaxCols = 511;  // restart length limit of the classical kernel
constexpr int kCgsBatch = 8;

template <int E>
__global__ void __launch_bounds__(kMgsThreads) cgs_kernel(MgsArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int kWarps = kMgsThreads / 32;
  constexpr int EW = E > 0 ? E : 1;
  constexpr int kB = E > 0 ? (16 / E > 1 ? 16 / E : 1) : kCgsBatch;  // columns per batch (<= 16 loads in flight)
  __shared__ double red[kCgsGroup][kWarps];
  __shared__ double hs[kCgsMaxCols + 1];  // coefficients of the current pass
  __shared__ double sc[4];
  const int nb = gridDim.x, m = a.m, ncol = m + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long chunk = ((a.n + nb - 1) / nb + 31) / 32 * 32;
  const long long lo = blockIdx.x * chunk;
  const long long len = lo < a.n ? (chunk < a.n - lo ? chunk : a.n - lo) : 0;
  double* wg = a.V + (long long)(m + 1) * a.ldv + lo;  // final column (and w itself when E == 0)
  const double* Vb = a.V + lo;
  double* partA = a.partial;                                 // ncol sets: <V_i, w>
  double* partB = a.partial + (long long)ncol * nb;          // ||w||^2 after a pass
  double* partC = a.partial + (long long)(ncol + 1) * nb;    // ||w_pre||^2
  double* partD = a.partial + (long long)(ncol + 2) * nb;    // ncol sets: second-pass <V_i, w'>
  double* partE = a.partial + (long long)(2 * ncol + 2) * nb;  // ||w''||^2
  double wr[EW];
  // fixed-order totals of `cnt` partial sets: warp q sums sets q, q + 16, ... (lanes
  // strided over blocks, then an xor tree): identical in every block and run
  auto totals = [&](const double* part, int cnt, double* out) {
    for (int i = warp; i < cnt; i += kWarps) {
      double v = 0.0;
      for (int b = lane; b < nb; b += 32) v += __ldcg(part + (long long)i * nb + b);
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) out[i] = v;
    }
    __syncthreads();
  };
  // block sum of one value per thread -> part[blockIdx.x]
  auto block_partial = [&](double v, double* part) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[0][warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kWarps; ++q) t += red[0][q];
      part[blockIdx.x] = t;
    }
  };
  // block partials of <V_i, w>, i < ncol -> partA
  auto dots = [&](double* dst) {
    for (int i0 = 0; i0 < ncol; i0 += kB) {
      double acc[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) acc[u] = 0.0;
      if constexpr (E > 0) {
        double v[kB][EW];
#pragma unroll
        for (int u = 0; u < kB; ++u)
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const int k = threadIdx.x + j * kMgsThreads;
            v[u][j] = (i0 + u < ncol && k < len) ? __ldcg(Vb + (long long)(i0 + u) * a.ldv + k) : 0.0;
          }
#pragma unroll
        for (int u = 0; u < kB; ++u)
#pragma unroll
          for (int j = 0; j < E; ++j) acc[u] += v[u][j] * wr[j];
      } else {
        for (long long k = threadIdx.x; k < len; k += kMgsThreads) {
          const double wk = wg[k];
#pragma unroll
          for (int u = 0; u < kB; ++u)
            if (i0 + u < ncol) acc[u] += __ldcg(Vb + (long long)(i0 + u) * a.ldv + k) * wk;
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        double t = acc[u];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[(i0 + u) % kCgsGroup][warp] = t;
      }
      const int done = i0 + kB;
      if (done % kCgsGroup == 0 || done >= ncol) {  // flush this group of coefficients
        const int g0 = (done - 1) / kCgsGroup * kCgsGroup;
        const int cnt = (ncol < g0 + kCgsGroup ? ncol : g0 + kCgsGroup) - g0;
        __syncthreads();
        if (threadIdx.x < cnt) {
          double t = 0.0;
          for (int q = 0; q < kWarps; ++q) t += red[threadIdx.x][q];
          dst[(long long)(g0 + threadIdx.x) * nb + blockIdx.x] = t;
        }
        __syncthreads();
      }
    }
  };
  // w -= sum_i c_i V_i (i ascending for every entry); returns this thread's ||w||^2 share
  auto project = [&](const double* c) {
    double n2 = 0.0;
    if constexpr (E > 0) {
      for (int i0 = 0; i0 < ncol; i0 += kB) {
        double v[kB][EW];
#pragma unroll
        for (int u = 0; u < kB; ++u)
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const int k = threadIdx.x + j * kMgsThreads;
            v[u][j] = (i0 + u < ncol && k < len) ? __ldcg(Vb + (long long)(i0 + u) * a.ldv + k) : 0.0;
          }
#pragma unroll
        for (int u = 0; u < kB; ++u)
          if (i0 + u < ncol) {
            const double cu = c[i0 + u];
#pragma unroll
            for (int j = 0; j < E; ++j) wr[j] = wr[j] - cu * v[u][j];
          }
      }
#pragma unroll
      for (int j = 0; j < E; ++j) n2 += wr[j] * wr[j];  // out-of-range slots hold 0
    } else {
      for (long long k = threadIdx.x; k < len; k += kMgsThreads) {
        double wv = wg[k];
        for (int i0 = 0; i0 < ncol; i0 += kB) {
          double v[kB];
#pragma unroll
          for (int u = 0; u < kB; ++u)
            v[u] = i0 + u < ncol ? __ldcg(Vb + (long long)(i0 + u) * a.ldv + k) : 0.0;
#pragma unroll
          for (int u = 0; u < kB; ++u)
            if (i0 + u < ncol) wv = wv - c[i0 + u] * v[u];
        }
        wg[k] = wv;
        n2 += wv * wv;
      }
    }
    return n2;
  };
  // w = J z and ||w_pre||^2
  double n2 = 0.0;
  if constexpr (E > 0) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int k = threadIdx.x + j * kMgsThreads;
      wr[j] = k < len ? a.w_in[lo + k] : 0.0;
      n2 += wr[j] * wr[j];
    }
  } else {
    for (long long k = threadIdx.x; k < len; k += kMgsThreads) {
      const double v = a.w_in[lo + k];
      wg[k] = v;
      n2 += v * v;
    }
  }
  dots(partA);
  block_partial(n2, partC);
  grid.sync();
  totals(partA, ncol, hs);
  totals(partC, 1, sc);
  const double wnorm_pre = sqrt(sc[0]);
  if (!isfinite(wnorm_pre)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.status->nonfinite = 1;
      a.status->wnorm_pre = wnorm_pre;
    }
    return;  // uniform across the grid
  }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < ncol; i += kMgsThreads) a.h[i] = hs[i];
  // E > 0: the second pass's dot products are formed right after the first projection from the
  // same registers (speculatively: the DGKS test, true in ~97% of the bench's steps, decides after
  // the barrier whether they are used), saving one grid barrier; same sums, same order
  const double n2p = project(hs);
  if constexpr (E > 0) dots(partD);
  block_partial(n2p, partB);
  grid.sync();
  totals(partB, 1, sc + 1);
  double hnext = sqrt(sc[1]);
  int reorth = 0;
  if (hnext < 0.70710678118654752 * wnorm_pre) {  // gmres.cpp:96
    reorth = 1;
    if constexpr (E == 0) {
      dots(partD);
      grid.sync();
    }
    totals(partD, ncol, hs);
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < ncol; i += kMgsThreads) a.h[i] += hs[i];
    block_partial(project(hs), partE);
    grid.sync();
    totals(partE, 1, sc + 2);
    hnext = sqrt(sc[2]);
  }
  const bool finite = isfinite(hnext);
  const bool happy = hnext <= 1e-14 * fmax(1.0, wnorm_pre);
  if constexpr (E > 0) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int k = threadIdx.x + j * kMgsThreads;
      if (k < len) {
        const double v = (finite && !happy) ? wr[j] / hnext : wr[j];
        wg[k] = v;
        if (finite && !happy) a.stage[lo + k] = v;
      }
    }
  } else {
    for (long long k = threadIdx.x; k < len; k += kMgsThreads) {
      const double v = (finite && !happy) ? wg[k] / hnext : wg[k];
      wg[k] = v;
      if (finite && !happy) a.stage[lo + k] = v;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) mgs_finish(a, hnext, wnorm_pre, reorth, finite, happy);
}

// ---- classical Gram-Schmidt for large n (the basis slice of a block no longer fits
// registers): the same pass structure as cgs_kernel as a chain of ordinary kernels over
// a wide grid (tiles of kBigTile entries, 8 per thread in registers), partial sums per
// tile reduced in a fixed order by one warp per coefficient.  The DGKS decision and the
// non-finite checks live in a device-side state, so the chain runs without the host.
constexpr int kBigT = 512, kBigE = 8, kBigTile = kBigT * kBigE, kBigB = 2;  // kBigB columns per load round
struct CgsState {
  double wnorm_pre, hnext;
  int reorth, abort;
};
struct CgsBigArgs {
  MgsArgs a;
  int nblk;            // tiles
  double* part;        // (ncol + 1) * nblk tile partials
  double* coef;        // ncol + 1: this pass's coefficients (+ ||w||^2)
  CgsState* st;
  int pass;            // 0: first pass, 1: the DGKS second pass
};

__device__ __forceinline__ double big_block_sum(double v, double* red) {  // valid in thread 0
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < kBigT / 32; ++q) t += red[q];
  __syncthreads();
  return t;
}

// tile partials of <V_i, w> (i <= m) and, in the first pass, ||w||^2 (w = J z is copied to V_{m+1}).
// Each warp leaves its sum of a column in shared memory; after one barrier a thread per column adds
// the 16 warp sums in warp order (big_block_sum's order, without its two barriers per column).
__global__ void __launch_bounds__(kBigT) cgs_big_dots(CgsBigArgs b) {
  if (b.st->abort || (b.pass == 1 && !b.st->reorth)) return;
  extern __shared__ double wsum[];  // (m + 2) x 16 warp sums (dynamic: cgs_dots_smem_bytes)
  constexpr int kW = kBigT / 32;
  const MgsArgs& a = b.a;
  const int ncol = a.m + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lo = (long long)blockIdx.x * kBigTile;
  double* wg = a.V + (long long)(a.m + 1) * a.ldv;
  double wr[kBigE];
  double n2 = 0.0;
#pragma unroll
  for (int j = 0; j < kBigE; ++j) {
    const long long k = lo + threadIdx.x + (long long)j * kBigT;
    wr[j] = k < a.n ? (b.pass == 0 ? a.w_in[k] : wg[k]) : 0.0;
    if (b.pass == 0 && k < a.n) wg[k] = wr[j];
    n2 += wr[j] * wr[j];
  }
  auto warp_sum = [](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  for (int i0 = 0; i0 < ncol; i0 += kBigB) {
    double acc[kBigB] = {};
    double v[kBigB][kBigE];
#pragma unroll
    for (int u = 0; u < kBigB; ++u)
#pragma unroll
      for (int j = 0; j < kBigE; ++j) {
        const long long k = lo + threadIdx.x + (long long)j * kBigT;
        v[u][j] = (i0 + u < ncol && k < a.n) ? __ldcs(a.V + (long long)(i0 + u) * a.ldv + k) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < kBigB; ++u)
#pragma unroll
      for (int j = 0; j < kBigE; ++j) acc[u] += v[u][j] * wr[j];
#pragma unroll
    for (int u = 0; u < kBigB; ++u) {
      const double t = warp_sum(acc[u]);
      if (lane == 0 && i0 + u < ncol) wsum[(i0 + u) * kW + warp] = t;
    }
  }
  if (b.pass == 0) {
    const double t = warp_sum(n2);
    if (lane == 0) wsum[ncol * kW + warp] = t;
  }
  __syncthreads();
  const int nsets = ncol + (b.pass == 0 ? 1 : 0);
  for (int i = threadIdx.x; i < nsets; i += kBigT) {
    double t = 0.0;
    for (int q = 0; q < kW; ++q) t += wsum[i * kW + q];
    b.part[(long long)i * b.nblk + blockIdx.x] = t;
  }
}

inline size_t cgs_dots_smem_bytes(int restart) { return sizeof(double) * size_t(restart + 2) * (kBigT / 32); }

// coefficients: block i sums the tile partials of set i (thread-strided, then the fixed-order block
// sum); the first pass also sets h and ||w_pre||, the second adds to h (gmres.cpp:96-102).
// Grid: m + 1 blocks, + 1 in the first pass (||w||^2).
__global__ void __launch_bounds__(kBigT) cgs_big_reduce(CgsBigArgs b) {
  if (b.st->abort || (b.pass == 1 && !b.st->reorth)) return;
  __shared__ double red[kBigT / 32];
  const MgsArgs& a = b.a;
  const int ncol = a.m + 1, i = blockIdx.x;
  double v = 0.0;
  for (int t = threadIdx.x; t < b.nblk; t += kBigT) v += b.part[(long long)i * b.nblk + t];
  const double tot = big_block_sum(v, red);
  if (threadIdx.x != 0) return;
  if (i < ncol) {
    b.coef[i] = tot;
    a.h[i] = b.pass == 0 ? tot : a.h[i] + tot;
  } else {
    const double wn = sqrt(tot);
    b.st->wnorm_pre = wn;
    if (!isfinite(wn)) {
      b.st->abort = 1;
      a.status->nonfinite = 1;
      a.status->wnorm_pre = wn;
    }
  }
}

// w -= sum_i coef_i V_i (i ascending per entry); tile partials of ||w||^2 into set 0
__global__ void __launch_bounds__(kBigT) cgs_big_project(CgsBigArgs b) {
  if (b.st->abort || (b.pass == 1 && !b.st->reorth)) return;
  __shared__ double red[kBigT / 32];
  __shared__ double c[kCgsMaxCols + 1];
  const MgsArgs& a = b.a;
  const int ncol = a.m + 1;
  for (int i = threadIdx.x; i < ncol; i += kBigT) c[i] = b.coef[i];
  __syncthreads();
  const long long lo = (long long)blockIdx.x * kBigTile;
  double* wg = a.V + (long long)(a.m + 1) * a.ldv;
  double wr[kBigE];
#pragma unroll
  for (int j = 0; j < kBigE; ++j) {
    const long long k = lo + threadIdx.x + (long long)j * kBigT;
    wr[j] = k < a.n ? wg[k] : 0.0;
  }
  for (int i0 = 0; i0 < ncol; i0 += kBigB) {
    double v[kBigB][kBigE];
#pragma unroll
    for (int u = 0; u < kBigB; ++u)
#pragma unroll
      for (int j = 0; j < kBigE; ++j) {
        const long long k = lo + threadIdx.x + (long long)j * kBigT;
        v[u][j] = (i0 + u < ncol && k < a.n) ? __ldcs(a.V + (long long)(i0 + u) * a.ldv + k) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < kBigB; ++u)
      if (i0 + u < ncol)
#pragma unroll
        for (int j = 0; j < kBigE; ++j) wr[j] = wr[j] - c[i0 + u] * v[u][j];
  }
  double n2 = 0.0;
#pragma unroll
  for (int j = 0; j < kBigE; ++j) {
    const long long k = lo + threadIdx.x + (long long)j * kBigT;
    if (k < a.n) wg[k] = wr[j];
    n2 += wr[j] * wr[j];
  }
  const double t = big_block_sum(n2, red);
  if (threadIdx.x == 0) b.part[blockIdx.x] = t;
}

// ||w|| after a pass (fixed order), the DGKS test after the first, and after the last
// pass the status, h[m+1] and the Givens update (mgs_finish); one block
__global__ void __launch_bounds__(kBigT) cgs_big_norm(CgsBigArgs b, int last) {
  if (b.st->abort || (b.pass == 1 && !b.st->reorth && !last)) return;
  const MgsArgs& a = b.a;
  __shared__ double sm[40];
  if (!(b.pass == 1 && !b.st->reorth)) {  // the pass ran: its norm
    double v = 0.0;
    for (int t = threadIdx.x; t < b.nblk; t += kBigT) v += b.part[t];
    const double tot = big_block_sum(v, sm);
    if (threadIdx.x == 0) b.st->hnext = sqrt(tot);
  }
  if (threadIdx.x != 0) return;
  if (b.pass == 0 && !last) {
    b.st->reorth = b.st->hnext < 0.70710678118654752 * b.st->wnorm_pre;  // gmres.cpp:96
    return;
  }
  const double hnext = b.st->hnext, wnorm_pre = b.st->wnorm_pre;
  const bool finite = isfinite(hnext);
  const bool happy = hnext <= 1e-14 * fmax(1.0, wnorm_pre);
  mgs_finish(a, hnext, wnorm_pre, b.st->reorth, finite, happy);
}

// V_{m+1} = w / ||w|| (and the preconditioner's staging copy) unless happy / non-finite
__global__ void __launch_bounds__(kBigT) cgs_big_normalize(CgsBigArgs b) {
  if (b.st->abort) return;
  const MgsArgs& a = b.a;
  const double hnext = b.st->hnext;
  if (!isfinite(hnext) || hnext <= 1e-14 * fmax(1.0, b.st->wnorm_pre)) return;
  double* wg = a.V + (long long)(a.m + 1) * a.ldv;
  const long long lo = (long long)blockIdx.x * kBigTile;
#pragma unroll
  for (int j = 0; j < kBigE; ++j) {
    const long long k = lo + threadIdx.x + (long long)j * kBigT;
    if (k < a.n) {
      const double v = wg[k] / hnext;
      wg[k] = v;
      a.stage[k] = v;
    }
  }
}

// y = R(0:m,0:m)^-1 g(0:m)  (gmres.cpp:55-61), one thread; flags a zero pivot
__global__ void backsub_kernel(int m, int ldr, const double* R, const double* g, double* y, int* singular) {
  pdl_entry();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *singular = 0;
  for (int i = m - 1; i >= 0; --i) {
    double s = g[i];
    for (int j = i + 1; j < m; ++j) s -= R[(long long)j * ldr + i] * y[j];
    const double rii = R[(long long)i * ldr + i];
    if (rii == 0.0) {
      *singular = 1;
      return;
    }
    y[i] = s / rii;
  }
}

// u_i = sum_{j<m} V_j[i] y_j, j ascending from 0 (gmres.cpp:62-64)
__global__ void basis_combine_kernel(long long n, long long ldv, int m, const double* V, const double* y, double* u) {
  pdl_entry();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < m; ++j) s += V[(long long)j * ldv + i] * __ldg(y + j);
  u[i] = s;
}

// deterministic sum of squares: per-block partials, then one block sums them in order
constexpr int kRedThreads = 512;
__global__ void __launch_bounds__(kRedThreads) sumsq_partial_kernel(long long n, const double* a, const double* b,
                                                                    double* diff_out, double* partial) {
  pdl_entry();
  // v = a - b (b may be null); optionally stores v; partial[block] = sum v^2
  __shared__ double sm[40];
  const long long chunk = ((n + gridDim.x - 1) / gridDim.x + 31) / 32 * 32;
  const long long lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  double acc = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = b ? a[i] - b[i] : a[i];
    if (diff_out) diff_out[i] = v;
    acc += v * v;
  }
  const double s = block_sum(acc, sm);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void __launch_bounds__(kRedThreads) finish_sum_kernel(int nb, const double* partial, double* out_dev,
                                                                 double* out_host, int take_sqrt) {
  pdl_entry();
  __shared__ double sm[40];
  double s = grid_total(partial, nb, sm);
  if (threadIdx.x != 0) return;
  if (take_sqrt) s = sqrt(s);
  if (out_dev) *out_dev = s;
  if (out_host) *out_host = s;
}
// V_0 = r / beta, also into the preconditioner staging buffer; g = [beta, 0...]
__global__ void start_cycle_kernel(long long n, const double* r, const double* beta_dev, double* v0, double* stage) {
  pdl_entry();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = r[i] / *beta_dev;
  v0[i] = v;
  stage[i] = v;
}

}  // namespace fpd
