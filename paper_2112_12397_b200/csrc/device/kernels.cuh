// sm_100a kernels of the solve path.  Compiled with -fmad=false: every
// multiply-add is a separately rounded DMUL + DADD, matching the CPU oracle
// (built with -ffp-contract=off) bit for bit.  All kernels are HBM-bound
// (SpMV ~0.24 flop/B): the levers are coalesced 256-byte warp loads (SELL-32
// layout), read-only cache for matrix streams, enough loads in flight per
// thread (unrolled row loops) and fusing the elementwise work of the reference
// (Jacobi updates, residuals, axpys, block scaling) into the SpMV that produces
// its operand.
#pragma once

#include <cooperative_groups.h>

#include "device.cuh"

namespace fpd {

// ------------------------------------------------------------------ gathers
struct GPlain {  // x_j
  const double* x;
  __device__ __forceinline__ double operator()(int j) const { return __ldg(x + j); }
};
struct GScaled {  // x_j * s  (driver block scaling D, driver.cpp:127-132)
  const double* x;
  double s;
  __device__ __forceinline__ double operator()(int j) const { return __ldg(x + j) * s; }
};
struct GPresmooth {  // first Jacobi sweep from x = 0: (omega * b_j) / d_j  (amg.cpp:136-140)
  const double* b;
  const double* d;
  double w;
  __device__ __forceinline__ double operator()(int j) const { return (w * __ldg(b + j)) / __ldg(d + j); }
};

// One SELL-32 row, left to right (csr.cpp:109-119).  U entries per batch: all U column and
// value loads (then all U gathers) are issued before the U ordered adds.
template <class G, int U = 4>
__device__ __forceinline__ double sell_row_at(const SellView& A, int slot, int len, const G& g) {
  const long long base = A.slice_off[slot >> 5] + (slot & 31);
  const int* __restrict__ C = A.cols + base;
  const double* __restrict__ V = A.vals + base;
  double s = 0.0;
  int k = 0;
  for (; k + U <= len; k += U) {
    int c[U];
    double v[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldg(C + 32 * (k + u)), v[u] = __ldg(V + 32 * (k + u));
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = g(c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s = s + v[u] * x[u];
  }
  for (; k < len; ++k) s = s + __ldg(V + 32 * k) * g(__ldg(C + 32 * k));
  return s;
}
template <class G, int U = 4>
__device__ __forceinline__ double sell_row(const SellView& A, int row, const G& g) {  // slot = row
  return sell_row_at<G, U>(A, row, A.row_len[row], g);
}

// ---------------------------------------------------------------- epilogues
// Two-phase epilogues: load(i) fetches the row's operands (b_i, d_i, x_i, ...)
// before the row loop so their latency overlaps the matrix stream; apply
// (operator()) then combines them with the row sum s.  Each formula is the
// reference's expression order.
struct NoPre {};
struct EStore {
  double* y;
  using P = NoPre;
  __device__ __forceinline__ P load(int) const { return {}; }
  __device__ __forceinline__ void operator()(int i, double s, const P&) const { y[i] = s; }
};
struct EAddTo {  // y_i = a_i + s   (x += P e_c, amg.cpp:168-169; t_u = w_u + C1 t_t, precond.cpp:217)
  const double* a;
  double* y;
  struct P { double a; };
  __device__ __forceinline__ P load(int i) const { return {a[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const { y[i] = p.a + s; }
};
// Producers of an AMG right-hand side b also emit the first Jacobi sweep from
// zero, xh = (omega b_i) / d_i (amg.cpp:136-140 with x = 0), so the V-cycle's
// first residual is a plain SpMV instead of a divide per gathered entry.
struct EStorePre {  // y_i = s ; xh_i = (w s) / d_i   (restriction r_c = P^T r)
  double* y;
  const double* d;
  double w;
  double* xh;
  struct P { double d; };
  __device__ __forceinline__ P load(int i) const { return {d[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const {
    y[i] = s;
    xh[i] = (w * s) / p.d;
  }
};
struct EAddToPre {  // y_i = a_i + s ; xh_i = (w y_i) / d_i   (t_u = w_u + C1 t_t)
  const double* a;
  double* y;
  const double* d;
  double w;
  double* xh;
  struct P { double a, d; };
  __device__ __forceinline__ P load(int i) const { return {a[i], d[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const {
    const double v = p.a + s;
    y[i] = v;
    xh[i] = (w * v) / p.d;
  }
};
struct ESubFromScaled {  // y_i = a_i * sa - s   (t_p = w_p - Q2 s_u with w_p = D^-1 v_p)
  const double* a;
  double sa;
  double* y;
  struct P { double a; };
  __device__ __forceinline__ P load(int i) const { return {a[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const { y[i] = p.a * sa - s; }
};
struct EResid {  // r_i = b_i - s   (amg.cpp:162-164)
  const double* b;
  double* r;
  struct P { double b; };
  __device__ __forceinline__ P load(int i) const { return {b[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const { r[i] = p.b - s; }
};
struct EJacobi {  // x'_i = x_i + (omega (b_i - s)) / d_i   (amg.cpp:139)
  const double* b;
  const double* d;
  double w;
  const double* x;
  double* xo;
  struct P { double b, d, x; };
  __device__ __forceinline__ P load(int i) const { return {b[i], d[i], x[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const {
    xo[i] = p.x + (w * (p.b - s)) / p.d;
  }
};
struct EJacobiSubFrom {  // out_i = c_i - (Jacobi update)   (v_u = s_u - v_u2, precond.cpp:224)
  const double* b;
  const double* d;
  double w;
  const double* x;
  const double* c;
  double* out;
  struct P { double b, d, x, c; };
  __device__ __forceinline__ P load(int i) const { return {b[i], d[i], x[i], c[i]}; }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const {
    const double xn = p.x + (w * (p.b - s)) / p.d;
    out[i] = p.c - xn;
  }
};
// EXTENSION — Chebyshev smoother step (oracle/amg.cpp chebyshev_sweep), s = (A x)_i:
//   first (step 0, x != 0): d_i = ((b_i - s) / D_i) / theta
//   else  (step k >= 1):    d_i = c1 d_i + c2 ((b_i - s) / D_i)
//   x'_i = x_i + d_i, or out_i = c_i - x'_i on the last post-smoothing step of v_u = s_u - AMG(t_u2)
struct ECheb {
  const double* b;
  const double* D;
  double* dv;
  const double* x;
  double* xo;
  const double* c;
  double theta, c1, c2;
  int first;
  struct P { double b, D, d, x, c; };
  __device__ __forceinline__ P load(int i) const {
    return {b[i], D[i], first ? 0.0 : dv[i], x[i], c ? c[i] : 0.0};
  }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const {
    const double r = p.b - s;
    const double dn = first ? (r / p.D) / theta : c1 * p.d + c2 * (r / p.D);
    dv[i] = dn;
    const double xn = p.x + dn;
    xo[i] = c ? p.c - xn : xn;
  }
};
// J apply, displacement rows: y_u = (A u + C1 (st v_t)) + Q1 (sp v_p)   (block.cpp:55-60);
// the short C1 / Q1 row sums are formed before the A row loop.
struct EJu {
  SellView C1, Q1;
  const double* vt;
  const double* vp;
  double st, sp;
  double* y;
  struct P { double b, c; };
  __device__ __forceinline__ P load(int i) const {
    return {sell_row(C1, i, GScaled{vt, st}), sell_row(Q1, i, GScaled{vp, sp})};
  }
  __device__ __forceinline__ void operator()(int i, double s, const P& p) const { y[i] = s + p.b + p.c; }
};

// ------------------------------------------------------------- SELL kernels
// U entries per row per round: 8 for long rows (fewer dependent index -> gather rounds)
template <class G, class E, int U = 4>
__global__ void __launch_bounds__(256) sell_kernel(SellView A, G g, E epi) {
  pdl_entry();
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  int row = slot;
  if (A.rows) {  // length-sorted slices
    if (slot >= A.n_slots) return;
    row = A.rows[slot];
    if (row < 0) return;
  } else if (row >= A.n_rows) {
    return;
  }
  const auto pre = epi.load(row);
  epi(row, sell_row_at<G, U>(A, slot, A.row_len[row], g), pre);
}

// Node-blocked rows (Bp3View): one thread per node, its three scalar rows summed left to
// right in three independent chains (each exactly the CSR row sum of csr.cpp:112-117);
// one column load and one gather serve all three rows.
template <class G, class E, int U = 4>
__global__ void __launch_bounds__(256) bp3_kernel(Bp3View A, G g, E epi) {
  pdl_entry();
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= A.n_slots) return;
  const int node = A.node[slot];  // nodes sorted by length inside windows (less padding per slice)
  if (node < 0) return;
  const auto p0 = epi.load(3 * node), p1 = epi.load(3 * node + 1), p2 = epi.load(3 * node + 2);
  const long long s0 = A.slice_off[slot >> 5];
  const int lane = slot & 31, len = A.node_len[node];
  const int* __restrict__ C = A.cols + s0 + lane;
  const double* __restrict__ V = A.vals + 3 * s0 + lane;
  double a = 0.0, b = 0.0, c = 0.0;
  int k = 0;
  for (; k + U <= len; k += U) {
    int col[U];
    double x[U], v[U][3];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      col[u] = __ldg(C + 32 * (k + u));
#pragma unroll
      for (int d = 0; d < 3; ++d) v[u][d] = __ldg(V + 96 * (k + u) + 32 * d);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = g(col[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a = a + v[u][0] * x[u];
      b = b + v[u][1] * x[u];
      c = c + v[u][2] * x[u];
    }
  }
  for (; k < len; ++k) {
    const double x = g(__ldg(C + 32 * k));
    a = a + __ldg(V + 96 * k) * x;
    b = b + __ldg(V + 96 * k + 32) * x;
    c = c + __ldg(V + 96 * k + 64) * x;
  }
  epi(3 * node, a, p0);
  epi(3 * node + 1, b, p1);
  epi(3 * node + 2, c, p2);
}

// ------------------------------------------------------- warp-row CSR kernel
// Slice kernel for few / long rows: one CTA per 32 consecutive rows.  In each
// window of kSliceWin entries per row, the 8 warps load their rows' entries
// (contiguous in CSR, so coalesced) and store the products a_ik x_k to shared
// memory; then lane r of warp 0 adds row r's window strictly left to right.
// The ordered sum costs two instructions per 32 entries (one per lane) instead
// of per entry, and the loads of a window are all in flight together.
// Geometry: R rows per CTA, windows of W entries per row (dynamic shared memory
// 2 R (W+1) doubles).  Many rows: R = 32, W = 64; few long rows: R = 8, W = 512
// so that each CTA keeps 16 loads per lane in flight.
template <int R, int W>
constexpr size_t slice_smem_bytes() {
  return sizeof(double) * 2 * R * (W + 1);
}
template <int R, int W, class G, class E>
__global__ void __launch_bounds__(256) csr_slice_kernel(CsrView A, G g, E epi) {
  pdl_entry();
  __shared__ double prod[2 * R * (W + 1)];  // [2][R][W + 1]
  __shared__ long long rb[R + 1];
  const int row0 = blockIdx.x * R;
  const int nrows = A.n_rows - row0 < R ? A.n_rows - row0 : R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x <= nrows) rb[threadIdx.x] = A.rp[row0 + threadIdx.x];
  __syncthreads();
  long long maxlen = 0;
  for (int r = 0; r < nrows; ++r) maxlen = max(maxlen, rb[r + 1] - rb[r]);
  typename E::P pre{};
  if (warp == 0 && lane < nrows) pre = epi.load(row0 + lane);
  double s = 0.0;
  int buf = 0;
  for (long long w0 = 0; w0 < maxlen; w0 += W) {
    // produce: element t of the R x W window goes to thread t % 256 (consecutive
    // threads read consecutive entries of one row: coalesced)
#pragma unroll
    for (int h = 0; h < R * W / 256; ++h) {
      const int t = threadIdx.x + 256 * h, r = t / W, c = t - r * W;
      if (r < nrows) {
        const long long k = rb[r] + w0 + c;
        prod[(size_t(buf) * R + r) * (W + 1) + c] = k < rb[r + 1] ? __ldg(A.v + k) * g(__ldg(A.ci + k)) : 0.0;
      }
    }
    __syncthreads();
    if (warp == 0 && lane < nrows) {
      const long long len = rb[lane + 1] - rb[lane] - w0;
      const int cnt = len < W ? int(len) : W;
      const double* src = prod + (size_t(buf) * R + lane) * (W + 1);
      int k = 0;
      for (; k + 8 <= cnt; k += 8) {  // loads batched ahead of the (in-order) add chain
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = src[k + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + t[u];
      }
      for (; k < cnt; ++k) s = s + src[k];
    }
    buf ^= 1;  // the next window fills the other buffer while warp 0 sums this one
  }
  if (warp == 0 && lane < nrows) epi(row0 + lane, s, pre);
}

// ------------------------------------- strided32 row sums (AmgConfig row_sum = strided)
// EXTENSION, the coarse operators A_l (l >= 1) and R_l = P_l^T only:
// a row's sum is the xor tree (h = 16..1) of 32 partials, partial l accumulating the
// row's entries l, l + 32, l + 64, ... in order from +0.0 — restated by the oracle's
// spmv_strided32, so the result is still bitwise the oracle's in this mode.  The
// dependent add chain of a row drops from len to len / 32 + 5.
__device__ __forceinline__ double xor_tree32(double s) {
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, h);
  return s;
}

// many rows: one warp per row, lane l owning partial l (coalesced 256-byte loads);
// U entries per lane per batch (predicated): U = 8 for long rows (fewer dependent
// rounds of index loads + gathers), 4 otherwise (fewer idle slots)
template <int U, class G, class E>
__global__ void __launch_bounds__(256) csr_warp_kernel(CsrView A, G g, E epi) {
  pdl_entry();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= A.n_rows) return;
  const int grow = A.row_map ? A.row_map[row] : row;  // row subset: sum global row grow
  typename E::P pre{};
  if (lane == 0) pre = epi.load(grow);
  const long long k0 = A.rp[grow], k1 = A.rp[grow + 1];
  // column of entry k at ci[k] (shared column lists: the group's list, offset by the row's start)
  const int* __restrict__ ci = A.cp ? A.ci + (A.cp[grow] - k0) : A.ci;
  double s = 0.0;
  long long k = k0 + lane;
  for (; k + 32 * (U - 1) < k1; k += 32 * U) {
    int c[U];
    double v[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldg(ci + k + 32 * u), v[u] = __ldg(A.v + k + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = g(c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s = s + v[u] * x[u];
  }
  if (k < k1) {  // tail: up to U - 1 entries, predicated in one round
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = k + 32 * u < k1;
      c[u] = in ? __ldg(ci + k + 32 * u) : 0;
      v[u] = in ? __ldg(A.v + k + 32 * u) : 0.0;
    }
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = k + 32 * u < k1 ? g(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + 32 * u < k1) s = s + v[u] * x[u];
  }
  s = xor_tree32(s);
  if (lane == 0) epi(grow, s, pre);
}

// many rows (>= 65,536): four lanes per row over sorted slices of 8 rows (SrtView), still the strided32
// sum.  Lane (rl, q) keeps the partials 8 q .. 8 q + 7 of row rl (entry k -> partial k mod 32, each in
// order from +0.0); the xor tree's levels h = 16 and 8 are shuffles between the row's four lanes
// (partial l ^ 16 lives in lane q ^ 2, l ^ 8 in q ^ 1), the levels 4, 2, 1 add inside the lane, every
// addition "own + partner" as in xor_tree32 — lane q = 0's partial 0 ends as that tree's lane-0
// result bit for bit.  All 8 loads of a lane's round are issued together; the warp's u-th value load
// is one 256-byte line, the column lists (shared by the rows of an aggregate) come through L1.
template <class G, class E>
__global__ void __launch_bounds__(256, 3) srt_kernel(SrtView A, G g, E epi) {
  pdl_entry();
  const int slice = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (slice >= A.n_slices) return;  // warp-uniform
  const int lane = threadIdx.x & 31, rl = lane >> 2, q = lane & 3;
  const int row = A.row[slice * kSrtRows + rl];
  // a padding lane (row < 0, last slice only) runs the unpredicated rounds on the slice's first row's
  // column list and its own zero values; its sums are never stored
  const int rowv = row >= 0 ? row : A.row[slice * kSrtRows];
  const int lenv = A.row_len[rowv], len = row >= 0 ? lenv : 0;
  const int orow = row >= 0 && A.out_row ? A.out_row[row] : row;  // a row-subset copy computes row out_row[row]
  typename E::P pre{};
  if (q == 0 && row >= 0) pre = epi.load(orow);
  const long long o0 = A.slice_off[slice];
  const int rounds = int((A.slice_off[slice + 1] - o0) >> 8);  // 256 values per round
  const int full = __reduce_min_sync(0xffffffffu, lenv) >> 5;  // rounds in which every row has 32 entries
  const int* __restrict__ C = A.ci + A.cp[rowv] + 8 * q;
  const double* __restrict__ V = A.vals + o0 + lane;
  double s[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) s[u] = 0.0;
  int t = 0;
  for (; t < full; ++t, C += 32, V += 256) {  // the rows of a sorted slice have nearly one length: most rounds
    int c[8];
    double v[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = __ldg(C + u), v[u] = __ldg(V + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = g(c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] = s[u] + v[u] * x[u];
  }
  for (; t < rounds; ++t, C += 32, V += 256) {  // ragged end: entry k0 + u exists for k0 + u < len
    const int k0 = 32 * t + 8 * q;
    int c[8];
    double v[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool in = k0 + u < len;
      c[u] = in ? __ldg(C + u) : 0;
      v[u] = in ? __ldg(V + 32 * u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = k0 + u < len ? g(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < len) s[u] = s[u] + v[u] * x[u];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) s[u] = s[u] + __shfl_xor_sync(0xffffffffu, s[u], 2);  // h = 16
#pragma unroll
  for (int u = 0; u < 8; ++u) s[u] = s[u] + __shfl_xor_sync(0xffffffffu, s[u], 1);  // h = 8
#pragma unroll
  for (int h = 4; h > 0; h >>= 1)
#pragma unroll
    for (int u = 0; u < h; ++u) s[u] = s[u] + s[u + h];
  if (q == 0 && row >= 0) epi(orow, s[0], pre);
}

// few long rows: R rows per CTA of 512 threads; in each window of W = 4096 / R
// entries per row every thread loads 8 entries (one round of loads for the whole
// window) and stores their products in shared memory; warp r then adds row r's
// window into its 32 partials (window entry c -> lane c mod 32; W % 32 == 0
// keeps entry k -> lane k mod 32 across windows).  R is chosen at upload from
// the operator's average row length (most rows fit one window).
constexpr int kStridedThreads = 512, kStridedWin = 4096;
template <int R, class G, class E>
__global__ void __launch_bounds__(kStridedThreads) csr_slice_strided_kernel(CsrView A, G g, E epi) {
  pdl_entry();
  constexpr int W = kStridedWin / R;
  extern __shared__ double prod[];  // [R][W + 1]
  __shared__ long long rb[R + 1];
  const int row0 = blockIdx.x * R;
  const int nrows = A.n_rows - row0 < R ? A.n_rows - row0 : R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x <= nrows) rb[threadIdx.x] = A.rp[row0 + threadIdx.x];
  __syncthreads();
  long long maxlen = 0;
  for (int r = 0; r < nrows; ++r) maxlen = max(maxlen, rb[r + 1] - rb[r]);
  typename E::P pre{};
  if (warp < nrows && lane == 0) pre = epi.load(row0 + warp);
  double s = 0.0;
  for (long long w0 = 0; w0 < maxlen; w0 += W) {
    constexpr int kPer = R * W / kStridedThreads;
    int c[kPer];
    double v[kPer];
    bool in[kPer];
#pragma unroll
    for (int h = 0; h < kPer; ++h) {
      const int t = threadIdx.x + kStridedThreads * h, r = t / W, cc = t - r * W;
      const long long k = r < nrows ? rb[r] + w0 + cc : 0;
      in[h] = r < nrows && k < rb[r + 1];
      c[h] = in[h] ? __ldg(A.ci + k) : 0;
      v[h] = in[h] ? __ldg(A.v + k) : 0.0;
    }
    if (w0 > 0) __syncthreads();  // the previous window has been summed
#pragma unroll
    for (int h = 0; h < kPer; ++h) {
      const int t = threadIdx.x + kStridedThreads * h, r = t / W, cc = t - r * W;
      if (r < nrows) prod[r * (W + 1) + cc] = in[h] ? v[h] * g(c[h]) : 0.0;
    }
    __syncthreads();
    if (warp < nrows) {
      const long long len = rb[warp + 1] - rb[warp] - w0;
      const int cnt = len < W ? int(len) : W;
      const double* src = prod + warp * (W + 1);
      for (int cc = lane; cc < cnt; cc += 32) s = s + src[cc];
    }
  }
  if (warp < nrows) {
    s = xor_tree32(s);
    if (lane == 0) epi(row0 + warp, s, pre);
  }
}
inline size_t strided_smem_bytes(int R) { return sizeof(double) * size_t(R) * (kStridedWin / R + 1); }

// ------------------------------------------------ ordered long-row CSR pipeline
// Rows of tens to thousands of entries (AMG levels >= 1, R = P^T) whose sums
// must stay in column order.  One CTA owns kPipeRows rows: warp 0 is the
// consumer (lane r sums row r, in order), warps 1..kPipeStages are producers,
// producer q filling stage q of a shared ring with the windows w = q (mod
// kPipeStages) — kPipeW columns of every row, lane = column (coalesced) —
// so up to kPipeStages windows of loads and gathers are in flight while the
// consumer sums.  Stage q is handed over with named barriers: FULL = 1 + q
// (producer arrives, consumer waits), EMPTY = 1 + kPipeStages + q (reverse).
constexpr int kPipeStages = 7, kPipeThreads = 32 * (kPipeStages + 1);
constexpr size_t kPipeSmem = sizeof(double) * kPipeStages * kPipeRows * (kPipeW + 1);  // dynamic (> 48 KB)

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <class G, class E>
__global__ void __launch_bounds__(kPipeThreads, kPipeCtasPerSm) csr_pipe_kernel(PipeView A, G g, E epi) {
  pdl_entry();
  extern __shared__ double pipe_smem[];
  double(*ring)[kPipeRows][kPipeW + 1] = reinterpret_cast<double(*)[kPipeRows][kPipeW + 1]>(pipe_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = A.cta_slice[blockIdx.x], s1 = A.cta_slice[blockIdx.x + 1];
  if (s0 >= s1) return;
  // this CTA's windows are contiguous: [woff[s0], woff[s1])
  const long long w_first = A.woff[s0];
  const long long nwin = A.woff[s1] - w_first;
  if (warp == 0) {  // consumer: lane r sums row r of the current slice in column order
    int sl = s0;
    long long s_begin = A.woff[sl], s_end = A.woff[sl + 1];
    int row = A.row[sl * kPipeRows + lane], len = A.len[sl * kPipeRows + lane];
    typename E::P pre{};
    if (row >= 0) pre = epi.load(row);
    double s = 0.0;
    for (long long w = 0; w < nwin; ++w) {
      const long long wg = w_first + w;
      while (wg >= s_end) {  // slice done (also skips empty slices)
        if (row >= 0) epi(row, s, pre);
        ++sl;
        s_begin = s_end, s_end = A.woff[sl + 1];
        row = A.row[sl * kPipeRows + lane], len = A.len[sl * kPipeRows + lane];
        if (row >= 0) pre = epi.load(row);
        s = 0.0;
      }
      const int q = int(w % kPipeStages);
      named_sync(1 + q, 64);
      const int rem = len - int(wg - s_begin) * kPipeW;
      const double* src = &ring[q][lane][0];
      if (rem >= kPipeW) {
#pragma unroll
        for (int k = 0; k < kPipeW; ++k) s = s + src[k];
      } else {
        for (int k = 0; k < rem; ++k) s = s + src[k];
      }
      if (w + kPipeStages < nwin) named_arrive(1 + kPipeStages + q, 64);
    }
    for (;;) {  // the last slice and any empty slices after it
      if (row >= 0) epi(row, s, pre);
      if (++sl >= s1) break;
      row = A.row[sl * kPipeRows + lane];
      if (row >= 0) pre = epi.load(row);
      s = 0.0;
    }
    return;
  }
  const int q = warp - 1;  // producer q: windows q, q + kPipeStages, ... into stage q
  for (long long w = q; w < nwin; w += kPipeStages) {
    if (w >= kPipeStages) named_sync(1 + kPipeStages + q, 64);
    const long long base = (w_first + w) * (kPipeRows * kPipeW) + lane;
    const double* __restrict__ vp = A.v + base;
    const int* __restrict__ cp = A.ci + base;
    double v[kPipeRows];
    int c[kPipeRows];
#pragma unroll
    for (int r = 0; r < kPipeRows; ++r) v[r] = __ldcs(vp + r * kPipeW), c[r] = __ldcs(cp + r * kPipeW);
#pragma unroll
    for (int r = 0; r < kPipeRows; ++r) ring[q][r][lane] = v[r] * g(c[r]);
    named_arrive(1 + q, 64);
  }
}

// ------------------------------------------------------------- BSR3 kernel
// 96 threads per slice: warp li (0..2) computes scalar row 3*brow+li of the 32
// block rows of the slice.  Sum order = block columns ascending, then j = 0,1,2:
// the CSR column order.
#ifndef FP_BSR_THREADS
#define FP_BSR_THREADS 96
#endif
constexpr int kBsrThreads = FP_BSR_THREADS;  // one 96-thread slice per CTA: finest tail balance (measured +6% at config 2)
// matrix stream loads of the BSR3 kernel: evict-first (the 3x3 blocks are read once per
// sweep and exceed L2; keeping them out leaves L2 to the gathered vector)
#ifndef FP_BSR_LD
#define FP_BSR_LD __ldcs
#endif

// kKeep: the finest AMG operator, streamed four times per t-u-p apply — a fraction
// A.l2_keep of its lines is loaded evict-last (createpolicy.fractional), the rest
// evict-first, so that fraction stays L2-resident from one sweep to the next.
__device__ __forceinline__ unsigned long long l2_keep_policy(float fraction) {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(fraction));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_hint(const int* a, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}

template <class G, class E, bool kKeep = false, bool kPv = false>
__global__ void __launch_bounds__(kBsrThreads) bsr3_kernel(Bsr3View A, G g, E epi) {
  pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int slice = t / 96, r = t - slice * 96, li = r >> 5, lane = r & 31;
  const int brow = slice * kSlice + lane;
  if (brow >= A.n_brows) return;
  unsigned long long pol = 0;
  if constexpr (kKeep) pol = l2_keep_policy(A.l2_keep);
  auto LD = [&](auto* p) {
    if constexpr (kKeep)
      return ld_hint(p, pol);
    else
      return FP_BSR_LD(p);
  };
  const long long base = A.slice_off[slice];
  const int len = A.brow_len[brow];
  const int grow = A.brow_map ? A.brow_map[brow] : brow;  // row-subset matrix: global block row
  const auto pre = epi.load(3 * grow + li);
  const int* __restrict__ C = A.bcols + base + lane;
  const double* __restrict__ V = A.vals + base * 9 + li * 96 + lane;
  double s = 0.0;
  int k = 0;
  // the next pair's block columns (kPv: and values) are loaded one iteration ahead, so a
  // pair's gathers do not wait for an index load issued in the same iteration.  kPv costs
  // registers (56 vs 48: fewer resident CTAs), so it is used for grids of several waves.
  // A/B, same session: index prefetch: config 2 apply 0.387 -> 0.366 ms, config 3 2.013 ->
  // 1.986 ms; + values (kPv): config 3 1.986 -> 1.874 ms, config 2 0.366 -> 0.379 ms.
  int n0 = len >= 2 ? LD(C) : 0, n1 = len >= 2 ? LD(C + 32) : 0;
  double b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0;
  if (kPv && len >= 2) b0 = LD(V), b1 = LD(V + 32), b2 = LD(V + 64), b3 = LD(V + 288), b4 = LD(V + 320), b5 = LD(V + 352);
  for (; k + 2 <= len; k += 2) {
    const int c0 = 3 * n0, c1 = 3 * n1;
    if (k + 4 <= len) n0 = LD(C + 32 * (k + 2)), n1 = LD(C + 32 * (k + 3));
    double a00, a01, a02, a10, a11, a12;
    if constexpr (kPv) {
      a00 = b0, a01 = b1, a02 = b2, a10 = b3, a11 = b4, a12 = b5;
      if (k + 4 <= len) {
        const double* V1 = V + 288 * (k + 2);
        b0 = LD(V1), b1 = LD(V1 + 32), b2 = LD(V1 + 64), b3 = LD(V1 + 288), b4 = LD(V1 + 320), b5 = LD(V1 + 352);
      }
    } else {
      const double* V0 = V + 288 * k;
      a00 = LD(V0), a01 = LD(V0 + 32), a02 = LD(V0 + 64);
      a10 = LD(V0 + 288), a11 = LD(V0 + 320), a12 = LD(V0 + 352);
    }
    const double x00 = g(c0), x01 = g(c0 + 1), x02 = g(c0 + 2);
    const double x10 = g(c1), x11 = g(c1 + 1), x12 = g(c1 + 2);
    s = s + a00 * x00;
    s = s + a01 * x01;
    s = s + a02 * x02;
    s = s + a10 * x10;
    s = s + a11 * x11;
    s = s + a12 * x12;
  }
  if (k < len) {
    const int c0 = 3 * LD(C + 32 * k);
    const double* V0 = V + 288 * k;
    s = s + LD(V0) * g(c0);
    s = s + LD(V0 + 32) * g(c0 + 1);
    s = s + LD(V0 + 64) * g(c0 + 2);
  }
  epi(3 * grow + li, s, pre);
}

// ------------------------------------------------ t/p rows of the J apply
// y_t = st (C2 u - H (st v_t)),  y_p = sp (Q2 u + T (sp v_p))   (block.cpp:61-67)
__global__ void __launch_bounds__(256) jtp_kernel(SellView C2, SellView H, SellView Q2, SellView T, const double* u,
                                                  const double* vt, const double* vp, double st, double sp, double* yt,
                                                  double* yp) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < C2.n_rows) {
    const double d = sell_row(C2, i, GPlain{u});
    const double e = sell_row(H, i, GScaled{vt, st});
    yt[i] = (d - e) * st;
  } else if (i < C2.n_rows + Q2.n_rows) {
    const int k = i - C2.n_rows;
    const double f = sell_row(Q2, k, GPlain{u});
    const double g = sell_row(T, k, GScaled{vp, sp});
    yp[k] = (f + g) * sp;
  }
}

// t_u = (w_u + C1 t_t) - Q1 t_p   (precond.cpp:159, t-p-u)
__global__ void __launch_bounds__(256) tpu_tu_kernel(SellView C1, SellView Q1, const double* wu, const double* tt,
                                                     const double* tp, double* tu, const double* d, double w,
                                                     double* xh) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C1.n_rows) return;
  const double b = sell_row(C1, i, GPlain{tt});
  const double c = sell_row(Q1, i, GPlain{tp});
  const double v = (wu[i] + b) - c;
  tu[i] = v;
  xh[i] = (w * v) / d[i];
}

// --------------------------------------------------------- 3x3 block solves
// lu3_solve of csr.cpp:267-278 on blocks pre-factored at upload with the same
// lu3_factor (factoring is deterministic, so this equals refactoring per call).
__device__ __forceinline__ void lu3_solve_dev(const double* m, int pv, const double b[3], double x[3]) {
  const int p0 = pv & 3, p1 = (pv >> 2) & 3, p2 = (pv >> 4) & 3;
  double y0 = b[p0];
  double y1 = b[p1];
  y1 -= m[3] * y0;
  double y2 = b[p2];
  y2 -= m[6] * y0;
  y2 -= m[7] * y1;
  double x2 = y2;
  x2 /= m[8];
  double x1 = y1;
  x1 -= m[5] * x2;
  x1 /= m[4];
  double x0 = y0;
  x0 -= m[1] * x1;
  x0 -= m[2] * x2;
  x0 /= m[0];
  x[0] = x0, x[1] = x1, x[2] = x2;
}

// t_t = H~^-1 (at * v_t); optionally y_t = (-t_t) * at  (t-u-p*: v_t = -t_t, precond.cpp:239)
__global__ void __launch_bounds__(256) hsolve_in_kernel(int n_faces, const double* hlu, const int* hpiv, const double* vt,
                                                        double at, double* tt, double* yt_neg) {
  pdl_entry();
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_faces) return;
  const double w[3] = {vt[3 * f] * at, vt[3 * f + 1] * at, vt[3 * f + 2] * at};
  double x[3];
  lu3_solve_dev(hlu + 9 * size_t(f), hpiv[f], w, x);
  for (int c = 0; c < 3; ++c) {
    tt[3 * f + c] = x[c];
    if (yt_neg) yt_neg[3 * f + c] = (-x[c]) * at;
  }
}

// y_t = at * (H~^-1 (C2 v_u) - t_t)   (precond.cpp:163-164 / 226-227)
// 32 faces per 96-thread CTA: thread r sums C2 row r (16-wide load batches, in order), then
// thread f of the first warp solves face f's 3x3 system from the three row sums.
constexpr int kHoutFaces = 32;
__global__ void __launch_bounds__(3 * kHoutFaces) hsolve_out_kernel(int n_faces, SellView C2, const double* vu,
                                                                   const double* hlu, const int* hpiv,
                                                                   const double* tt, double at, double* yt) {
  pdl_entry();
  __shared__ double srow[3 * kHoutFaces];
  const int f0 = blockIdx.x * kHoutFaces;
  const int row = 3 * f0 + threadIdx.x;
  if (row < 3 * n_faces) srow[threadIdx.x] = sell_row<GPlain, 16>(C2, row, GPlain{vu});
  __syncthreads();
  const int f = f0 + threadIdx.x;
  if (threadIdx.x >= kHoutFaces || f >= n_faces) return;
  const double s[3] = {srow[3 * threadIdx.x], srow[3 * threadIdx.x + 1], srow[3 * threadIdx.x + 2]};
  double x[3];
  lu3_solve_dev(hlu + 9 * size_t(f), hpiv[f], s, x);
  for (int c = 0; c < 3; ++c) yt[3 * f + c] = (x[c] - tt[3 * f + c]) * at;
}

// ------------------------------------------------------- banded solves
// One warp per independent diagonal block (one fracture).  The block's
// right-hand side lives in shared memory; each step finalizes one unknown and
// the warp applies its column of L (forward) or U / L^T (backward) to the
// following rows in parallel — the column-sweep order of the oracle.
// The columns of L / U needed D steps ahead are prefetched into a register ring
// (lane l holds entries l, l+32, ... of a column), so a step costs one shared-
// memory round trip instead of a global-memory latency.
// Modes: out_mode 0: out = x;  1: out = (sub - x) * os;  2: out = x, out2 = x * os.

// Bulk prefetch of [p, p + bytes) into L2 (sm_90+ TMA-engine prefetch), so the
// register ring below streams the block's factor from L2, not HBM.
__device__ __forceinline__ void l2_prefetch_range(const void* p, size_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  while (a < e) {
    const uint32_t chunk = uint32_t((e - a) > (1u << 20) ? (1u << 20) : (e - a));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(chunk) : "memory");
    a += chunk;
  }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Prefetch ring: cp.async copies the factor column for step j + D into a
// per-lane shared-memory slot while step j computes (async groups, not register
// scoreboards, track completion; each lane reads back only what it copied).
constexpr int kBandDepth = 16;
constexpr int kBandMaxQ = 12;  // band widths up to 32*12 - 1 = 383 (fracture patches up to 191 faces wide)
__host__ __device__ constexpr int band_ring_doubles(int q) { return kBandDepth * 32 * (q + 1); }

// Register window.  At step j, lane l / slot q holds the current value of row
// j + l + 32q (forward) or j - l - 32q (backward); the window spans 32Q > band
// rows, so every row a step updates is in registers.  After the step the window
// shifts by one row (shuffle down), the next pivot comes from lane 0 by
// shuffle, and the row entering at the far end is read from shared memory.  The
// dependent chain per step is DMUL, DADD and two shuffles; shared memory and
// barriers stay off it.  Factor columns arrive through the cp.async ring.
template <int Q>
__device__ __forceinline__ double window_select(const double (&v)[Q], int sq) {
  double s = v[0];
#pragma unroll
  for (int q = 1; q < Q; ++q)
    if (sq == q) s = v[q];
  return s;
}

template <int Q>
__device__ __forceinline__ void window_shift(double (&v)[Q], int lane, double entering) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double down = __shfl_down_sync(0xffffffffu, v[q], 1);
    const double wrap = q + 1 < Q ? __shfl_sync(0xffffffffu, v[q + 1 < Q ? q + 1 : q], 0) : entering;
    v[q] = lane == 31 ? wrap : down;
  }
}

// Forward sweep with (optional) partial-pivot row swaps: for j ascending,
// y_j = x[piv_j] (swapped with x_j), then x_i -= L(i,j) y_j for i in (j, j+kl].
template <int Q, bool PIV>
__device__ __forceinline__ void band_forward(double* xs, double* ring, int nb, int b0, int kl,
                                             const double* __restrict__ Lc, const int* __restrict__ piv, int lane) {
  constexpr int D = kBandDepth;
  double* R = ring + lane;                                     // slot (u,q): R[(u*Q+q)*32] = L(., lane+32q-1)
  int* PR = reinterpret_cast<int*>(ring + D * Q * 32) + lane;  // slot u: PR[u*32]
  auto issue = [&](int u, int jj) {
    if (jj < nb) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int r = lane + 32 * q - 1;
        if (r >= 0 && r < kl) cp_async8(R + (u * Q + q) * 32, Lc + size_t(b0 + jj) * kl + r);
      }
      if (PIV) cp_async4(PR + u * 32, piv + b0 + jj);
    }
    cp_commit();
  };
#pragma unroll
  for (int u = 0; u < D; ++u) issue(u, u);
  double v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) v[q] = lane + 32 * q < nb ? xs[lane + 32 * q] : 0.0;
  for (int j0 = 0; j0 < nb; j0 += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int j = j0 + u;
      if (j < nb) {
        cp_wait<D - 1>();
        const double a = __shfl_sync(0xffffffffu, v[0], 0);
        double yj = a;
        if (PIV) {
          const int d = PR[u * 32] - b0 - j;  // pivot row offset in the window, 0..kl
          const int sq = d >> 5, ls = d & 31;
          yj = __shfl_sync(0xffffffffu, window_select<Q>(v, sq), ls);
          if (d > 0 && lane == ls) {  // the pivot row now holds the old x_j
#pragma unroll
            for (int q = 0; q < Q; ++q)
              if (q == sq) v[q] = a;
          }
        }
        if (lane == 0) xs[j] = yj;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int r = lane + 32 * q - 1;
          if (r >= 0 && r < kl) v[q] = v[q] - R[(u * Q + q) * 32] * yj;
        }
        const int ent = j + 32 * Q;
        window_shift<Q>(v, lane, ent < nb ? xs[ent] : 0.0);
        issue(u, j + D);
      }
    }
  }
  cp_wait<0>();
  __syncwarp();
}

// Backward sweep: for j descending, x_j = x_j / diag_j (DIV) then
// x_i -= C(j, r) x_j for i = j-1-r, r < kb (C = U columns, or rows of L for L^T).
template <int Q, bool DIV>
__device__ __forceinline__ void band_backward(double* xs, double* ring, int nb, int b0, int kb,
                                              const double* __restrict__ C, const double* __restrict__ diag,
                                              int lane) {
  constexpr int D = kBandDepth;
  double* R = ring + lane;
  double* DR = ring + D * Q * 32 + lane;  // slot u: DR[u*32] (lane 0's copy is used)
  auto issue = [&](int u, int j) {
    if (j >= 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int r = lane + 32 * q - 1;
        if (r >= 0 && r < kb) cp_async8(R + (u * Q + q) * 32, C + size_t(b0 + j) * kb + r);
      }
      if (DIV && lane == 0) cp_async8(DR + u * 32, diag + b0 + j);
    }
    cp_commit();
  };
#pragma unroll
  for (int u = 0; u < D; ++u) issue(u, nb - 1 - u);
  double v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = nb - 1 - lane - 32 * q;
    v[q] = i >= 0 ? xs[i] : 0.0;
  }
  for (int j0 = nb - 1; j0 >= 0; j0 -= D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int j = j0 - u;
      if (j >= 0) {
        cp_wait<D - 1>();
        const double c0 = DIV && lane == 0 ? v[0] / DR[u * 32] : v[0];
        const double xj = __shfl_sync(0xffffffffu, c0, 0);
        if (lane == 0) xs[j] = xj;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int r = lane + 32 * q - 1;
          if (r >= 0 && r < kb) v[q] = v[q] - R[(u * Q + q) * 32] * xj;
        }
        const int ent = j - 32 * Q;
        window_shift<Q>(v, lane, ent >= 0 ? xs[ent] : 0.0);
        issue(u, j - D);
      }
    }
  }
  cp_wait<0>();
  __syncwarp();
}

template <int Q>
__device__ __forceinline__ void band_forward_any(double* xs, double* ring, int nb, int b0, const BandView& F,
                                                 int lane) {
  if (F.spd)
    band_forward<Q, false>(xs, ring, nb, b0, F.kl, F.Lc, F.piv, lane);
  else
    if (F.pivoted)
      band_forward<Q, true>(xs, ring, nb, b0, F.kl, F.Lc, F.piv, lane);
    else
      band_forward<Q, false>(xs, ring, nb, b0, F.kl, F.Lc, F.piv, lane);
}
template <int Q>
__device__ __forceinline__ void band_backward_any(double* xs, double* ring, int nb, int b0, const BandView& F,
                                                  int lane) {
  if (F.spd)
    band_backward<Q, false>(xs, ring, nb, b0, F.kl, F.Lr, F.diag, lane);
  else
    band_backward<Q, true>(xs, ring, nb, b0, F.ku, F.Uc, F.diag, lane);
}

__global__ void __launch_bounds__(32) band_solve_kernel(BandView F, const double* rhs, double rs, double* out,
                                                        double* out2, const double* sub, double os, int out_mode) {
  pdl_entry();
  extern __shared__ double band_smem[];
  double* ring = band_smem;                                    // band_ring_doubles(kBandMaxQ) doubles
  double* xs = band_smem + band_ring_doubles(kBandMaxQ);       // the block's right-hand side / solution
  const int blk = blockIdx.x, lane = threadIdx.x;
  const int b0 = F.block_start[blk], b1 = F.block_start[blk + 1], nb = b1 - b0;
  if (lane == 0) {
    l2_prefetch_range(F.Lc + size_t(b0) * F.kl, sizeof(double) * size_t(nb) * F.kl);
    if (F.spd)
      l2_prefetch_range(F.Lr + size_t(b0) * F.kl, sizeof(double) * size_t(nb) * F.kl);
    else {
      l2_prefetch_range(F.Uc + size_t(b0) * F.ku, sizeof(double) * size_t(nb) * F.ku);
      l2_prefetch_range(F.piv + b0, sizeof(int) * size_t(nb));
    }
    l2_prefetch_range(F.diag + b0, sizeof(double) * size_t(nb));
  }
  for (int i = lane; i < nb; i += 32) xs[i] = rhs[b0 + i] * rs;
  __syncwarp();
  const int qf = (F.kl + 32) / 32;  // window of 32 Q rows must exceed the band (rows j+1 .. j+kl)
  if (qf <= 1)
    band_forward_any<1>(xs, ring, nb, b0, F, lane);
  else if (qf <= 2)
    band_forward_any<2>(xs, ring, nb, b0, F, lane);
  else if (qf <= 3)
    band_forward_any<3>(xs, ring, nb, b0, F, lane);
  else if (qf <= 4)
    band_forward_any<4>(xs, ring, nb, b0, F, lane);
  else if (qf <= 8)
    band_forward_any<8>(xs, ring, nb, b0, F, lane);
  else
    band_forward_any<12>(xs, ring, nb, b0, F, lane);
  if (F.spd) {
    for (int i = lane; i < nb; i += 32) xs[i] = xs[i] / F.diag[b0 + i];
    __syncwarp();
  }
  const int qb = ((F.spd ? F.kl : F.ku) + 32) / 32;
  if (qb <= 1)
    band_backward_any<1>(xs, ring, nb, b0, F, lane);
  else if (qb <= 2)
    band_backward_any<2>(xs, ring, nb, b0, F, lane);
  else if (qb <= 3)
    band_backward_any<3>(xs, ring, nb, b0, F, lane);
  else if (qb <= 4)
    band_backward_any<4>(xs, ring, nb, b0, F, lane);
  else if (qb <= 8)
    band_backward_any<8>(xs, ring, nb, b0, F, lane);
  else
    band_backward_any<12>(xs, ring, nb, b0, F, lane);
  for (int i = lane; i < nb; i += 32) {
    const double x = xs[i];
    if (out_mode == 1)
      out[b0 + i] = (sub[b0 + i] - x) * os;
    else
      out[b0 + i] = x;
    if (out_mode == 2) out2[b0 + i] = x * os;
  }
}

// ------------------------------------------- explicit block inverse apply
// factor_solve = inverse: one warp per row of the stacked block
// inverses, streaming the row once with coalesced 256-byte loads; lane j keeps
// the partial sum over columns c = j (mod 32) in ascending c and the partials
// meet in the xor tree h = 16..1 — the order the oracle's BandFactor::solve
// (factor.cpp) defines for this mode.  8 loads per lane in flight per step.
constexpr int kDinvThreads = 256;
__global__ void __launch_bounds__(kDinvThreads) dinv_kernel(DinvView D, int n, int n_blocks, const double* rhs,
                                                            double rs, double* out, double* out2, const double* sub,
                                                            double os, int out_mode) {
  pdl_entry();
  const int row = (blockIdx.x * kDinvThreads + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;  // warp-uniform
  int lo = 0, hi = n_blocks - 1;  // block of this row: block_start[blk] <= row < block_start[blk + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (D.block_start[mid] <= row) lo = mid; else hi = mid - 1;
  }
  const int b0 = D.block_start[lo], nb = D.block_start[lo + 1] - b0;
  const double* M = D.v + D.off[lo] + (long long)(row - b0) * nb;
  const double* g = rhs + b0;
  double s = 0.0;
  int c = lane;
  // 16 entries per lane per round, the tail predicated into one round (A/B: config 2 S~2 solve 12.3 -> 7.5 us,
  // config 3 165 -> 151 us = 6.5 TB/s); every lane still sums its columns c = lane (mod 32) in ascending order
  constexpr int U = 16;
  for (; c < nb; c += U * 32) {
    double m[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = c + 32 * u < nb;
      m[u] = in ? __ldcs(M + c + 32 * u) : 0.0;
      x[u] = in ? __ldg(g + c + 32 * u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c + 32 * u < nb) s = s + m[u] * (x[u] * rs);
  }
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, h);
  if (lane == 0) {
    if (out_mode == 1)
      out[row] = (sub[row] - s) * os;
    else
      out[row] = s;
    if (out_mode == 2) out2[row] = s * os;
  }
}

// ------------------------------------- multicolour Gauss-Seidel (extension)
// One colour of the multicolour symmetric Gauss-Seidel smoother: rows of a colour never reference
// each other, so each row of the colour is updated by one thread exactly as the reference's SGS row
// update (amg.cpp:118-122): s = b_i - sum_{j != i} a_ij x_j (left to right), x_i = s / d_i.
__global__ void mcgs_color_kernel(CsrView A, const int* rows, int n_rows, const double* b, const double* d,
                                  double* x) {
  pdl_entry();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n_rows) return;
  const int i = rows[t];
  double s = b[i];
  for (long long k = A.rp[i]; k < A.rp[i + 1]; ++k) {
    const int j = A.ci[k];
    if (j != i) s -= A.v[k] * x[j];
  }
  x[i] = s / d[i];
}

// ----------------------------------------------- panel (block-bidiagonal) solve
// factor_solve = panel: one thread-block cluster of kPanelCluster CTAs per fracture
// block.  The forward chain runs over the block's panels q = 0..P-1:
//     y_q = H_q (rs b_q) - G_q y_q-1,
// the backward chain over q = P-1..0:
//     x_q = K_q z_q - F_q x_q+1      (z = y / D for LDL^T, else y),
// one warp per row (rows of a panel dealt round-robin over the cluster's warps), each product summed
// as 32 lane-strided partials + xor tree (the oracle's BandFactor::solve in this mode).  The new panel
// (y_q or x_q) is written into every CTA's shared memory through distributed shared memory, then one
// cluster barrier; the matrices stream from HBM once per apply (H, G forward; K, F backward) and
// their loads do not depend on the chain, so they issue ahead of the barrier.
constexpr int kPanelCluster = 8, kPanelThreads = 512, kPanelWarps = kPanelCluster * kPanelThreads / 32;
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ double warp_tree(double s) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, h);
  return s;
}

// one chain (forward: D = H, C = G, x = rs b; backward: D = K, C = F, x = z) over the block's panels;
// before each cluster barrier a warp already loads the next panel's coupling rows into registers and
// forms its local product, so a step's critical path is the barrier plus a shared-memory dot.  A step
// broadcasts the new panel into every CTA's chain buffer; the forward chain also stores z = y / D (the
// backward chain's input) to global memory, the backward chain keeps the rows its warps own (own) and
// writes them out after the last barrier.
// R rows of a panel per warp and E entries of a row per lane (templated so a step issues only the
// instructions the block's panel size needs: p <= 128 * R, p <= 32 * E).
template <bool fwd, int R, int E>
__device__ __forceinline__ void panel_chain(const PanelView& V, int blk, int gw, int lane, double (*chain)[kPanelMax],
                                            double* zs, double* own, const double* xin, double xs,
                                            cooperative_groups::cluster_group& cluster) {
  const int b0 = V.block_start[blk], m = V.block_start[blk + 1] - b0, p = V.p[blk], P = (m + p - 1) / p;
  const double* base = V.m + V.off[blk];
  auto rows_of = [&](int q) { return min(p, m - q * p); };
  auto panel_size = [&](int q) {
    const int s = rows_of(q), sp = q > 0 ? p : 0, sn = q + 1 < P ? rows_of(q + 1) : 0;
    return s * s + s * sp + s * s + s * sn;
  };
  double dl[R], cr[R][E], dg[R];
  // panel q's local product D_q x_q and coupling rows C_q (and the forward's D), for this warp's rows
  auto prefetch = [&](int q, int o) {
    const int s = rows_of(q), sc = fwd ? (q > 0 ? p : 0) : (q + 1 < P ? rows_of(q + 1) : 0);
    const double* Dm = base + o + (fwd ? 0 : s * s + s * (q > 0 ? p : 0));
    const double* Cm = Dm + s * s;
    const double* xq = fwd ? xin + b0 + q * p : zs + b0 + q * p;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = gw + r * kPanelWarps;
      if (i >= s) break;  // warp-uniform
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int c = lane + 32 * e;
        if (c < s) acc = acc + Dm[i * s + c] * ((fwd ? xq[c] : __ldcg(xq + c)) * xs);  // z: written by other SMs
        cr[r][e] = c < sc ? Cm[i * sc + c] : 0.0;
      }
      dl[r] = warp_tree(acc);
      if (fwd) dg[r] = V.diag ? V.diag[b0 + q * p + i] : 1.0;
    }
  };
  int o = 0;
  int q = fwd ? 0 : P - 1;
  if (!fwd)
    for (int t = 0; t < P - 1; ++t) o += panel_size(t);
  prefetch(q, o);
  for (int step = 0; step < P; ++step, q += fwd ? 1 : -1) {
    const int s = rows_of(q), sc = fwd ? (q > 0 ? p : 0) : (q + 1 < P ? rows_of(q + 1) : 0);
    const double* prev = chain[(q + (fwd ? -1 : 1)) & 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = gw + r * kPanelWarps;
      if (i >= s) break;  // warp-uniform
      double acc = 0.0;
      if (sc) {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (lane + 32 * e < sc) acc = acc + cr[r][e] * prev[lane + 32 * e];
        acc = warp_tree(acc);
      }
      const double v = sc ? dl[r] - acc : dl[r];
      if (lane < kPanelCluster) *cluster.map_shared_rank(&chain[q & 1][i], lane) = v;
      if (fwd) {
        if (lane == 8) zs[b0 + q * p + i] = V.diag ? v / dg[r] : v;  // z = y / D (LDL^T), else y
      } else if (lane == 0) {
        own[q * R + r] = v;
      }
    }
    cluster_arrive();
    const int qn = q + (fwd ? 1 : -1);
    if (fwd ? qn < P : qn >= 0) {
      o += fwd ? panel_size(q) : -panel_size(qn);
      prefetch(qn, o);
    }
    cluster_wait();
  }
}

template <int R, int E>
__global__ void __cluster_dims__(kPanelCluster, 1, 1) __launch_bounds__(kPanelThreads)
    panel_solve_kernel(PanelView V, const double* rhs, double rs, double* out, double* out2, const double* sub,
                       double os, int out_mode) {
  pdl_entry();
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  __shared__ double chain[2][kPanelMax];  // the previous panel of the running chain (y or x)
  extern __shared__ double pan_dyn[];     // each warp's own x rows
  const int rank = int(cluster.block_rank());
  const int blk = V.order[blockIdx.x / kPanelCluster];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = rank * (kPanelThreads / 32) + warp;
  const int b0 = V.block_start[blk], m = V.block_start[blk + 1] - b0, p = V.p[blk], P = (m + p - 1) / p;
  // z stays in global memory (L2): written once by the forward chain, read once by the backward chain a
  // panel ahead of its use; the cluster barriers between the chains order the accesses.  Shared memory
  // per CTA is then a few KB, two CTAs fit an SM, and all of config 5's 40 clusters are resident at once.
  double* zs = V.z;
  double* own = pan_dyn + warp * (V.p_max_panels * R);
  panel_chain<true, R, E>(V, blk, gw, lane, chain, zs, own, rhs, rs, cluster);
  panel_chain<false, R, E>(V, blk, gw, lane, chain, zs, own, zs, 1.0, cluster);
  if (lane == 0)
    for (int q = 0; q < P; ++q)
      for (int r = 0; r < R; ++r) {
        const int i = gw + r * kPanelWarps;
        if (i >= min(p, m - q * p)) break;
        const long long row = b0 + (long long)q * p + i;
        const double x = own[q * R + r];
        if (out_mode == 1) {
          out[row] = (sub[row] - x) * os;
        } else {
          out[row] = x;
          if (out_mode == 2) out2[row] = x * os;
        }
      }
}

// Builds the panel matrices from the band factor (upload): one thread per (panel, column, matrix),
// the column sweeps of the oracle's BandFactor::build_panels in the same order.
__global__ void panel_build_kernel(BandView F, PanelView V, const int* task_blk, const int* task_q, int n_tasks,
                                   double* pan) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long task = t / (4 * kPanelMax);
  if (task >= n_tasks) return;
  const int which = int((t / kPanelMax) % 4), c = int(t % kPanelMax);
  const int blk = task_blk[task], q = task_q[task];
  const int b0 = V.block_start[blk], m = V.block_start[blk + 1] - b0, p = V.p[blk], P = (m + p - 1) / p;
  const int r0 = b0 + q * p, s = min(p, m - q * p), sp = q > 0 ? p : 0, sn = q + 1 < P ? min(p, m - (q + 1) * p) : 0;
  const int cols = which == 1 ? sp : which == 3 ? sn : s;
  if (c >= cols) return;
  long long o = V.off[blk];
  for (int u = 0; u < q; ++u) {
    const long long su = min(p, m - u * p), sup = u > 0 ? p : 0, sun = u + 1 < P ? min(p, m - (u + 1) * p) : 0;
    o += su * su + su * sup + su * su + su * sun;
  }
  double* M = pan + o + (which >= 1 ? (long long)s * s : 0) + (which >= 2 ? (long long)s * sp : 0) +
              (which >= 3 ? (long long)s * s : 0);
  auto Lv = [&](int gi, int gj) {
    return gi > gj && gi - gj <= F.kl ? F.Lc[(long long)gj * F.kl + (gi - gj - 1)] : 0.0;
  };
  auto Uv = [&](int gi, int gj) {
    if (!(gj > gi)) return 0.0;
    if (F.spd) return gj - gi <= F.kl ? F.Lr[(long long)gj * F.kl + (gj - gi - 1)] : 0.0;
    return gj - gi <= F.ku ? F.Uc[(long long)gj * F.ku + (gj - gi - 1)] : 0.0;
  };
  double z[kPanelMax];
  for (int i = 0; i < s; ++i) z[i] = 0.0;
  if (which == 0 || which == 2) z[c] = 1.0;
  if (which == 1)
    for (int i = 0; i < s; ++i) z[i] = Lv(r0 + i, r0 - sp + c);
  if (which == 3)
    for (int i = 0; i < s; ++i) z[i] = Uv(r0 + i, r0 + s + c);
  if (which <= 1) {
    for (int j = 0; j < s; ++j) {
      const double zj = z[j];
      for (int i = j + 1; i < s; ++i) z[i] -= Lv(r0 + i, r0 + j) * zj;
    }
  } else {
    for (int j = s - 1; j >= 0; --j) {
      double zj = z[j];
      if (!F.spd) {
        zj = zj / F.diag[r0 + j];
        z[j] = zj;
      }
      for (int i = j - 1; i >= 0; --i) z[i] -= Uv(r0 + i, r0 + j) * zj;
    }
  }
  for (int i = 0; i < s; ++i) M[(long long)i * cols + c] = z[i];
}

// ---------------------------------------------------- coarse dense solve
// x = Q U^-1 L^-1 P b on the full-pivot LU (restated FullPivLU::solve), one CTA,
// column sweeps.  LU is column-major so each step reads one contiguous column.
constexpr int kCoarseThreads = 256;
// When the factor fits (n <= kCoarseSmemN) it is staged in shared memory first,
// so the 2n dependent steps cost shared-memory latency, not L2/HBM latency.
constexpr int kCoarseSmemN = 160;
__global__ void __launch_bounds__(kCoarseThreads) coarse_solve_kernel(DenseLUView F, const double* b, double* x) {
  pdl_entry();
  extern __shared__ double c[];
  const int n = F.n, tid = threadIdx.x;
  const double* lu = F.lu;
  if (n <= kCoarseSmemN) {
    double* s_lu = c + n;
    for (int i = tid; i < n * n; i += blockDim.x) s_lu[i] = F.lu[i];
    lu = s_lu;
  }
  for (int i = tid; i < n; i += blockDim.x) c[i] = b[F.prow[i]];
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double cj = c[j];
    const double* col = lu + size_t(j) * n;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) c[i] -= col[i] * cj;
    __syncthreads();
  }
  for (int j = F.rank - 1; j >= 0; --j) {
    const double xj = c[j] / lu[size_t(j) * n + j];
    __syncthreads();
    if (tid == 0) c[j] = xj;
    const double* col = lu + size_t(j) * n;
    for (int i = tid; i < j; i += blockDim.x) c[i] -= col[i] * xj;
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) x[F.pcol[i]] = i < F.rank ? c[i] : 0.0;
}
// n <= 64: one warp, no block barriers — rows lane and lane + 32 live in
// registers, the pivot value travels by shuffle; same operation order as above.
constexpr int kCoarseWarpN = 64;
__global__ void __launch_bounds__(32) coarse_warp_kernel(DenseLUView F, const double* b, double* x) {
  pdl_entry();
  __shared__ double s_lu[kCoarseWarpN * kCoarseWarpN];
  const int n = F.n, lane = threadIdx.x;
#pragma unroll 8
  for (int i = lane; i < n * n; i += 32) s_lu[i] = F.lu[i];
  double c0 = lane < n ? b[F.prow[lane]] : 0.0;
  double c1 = lane + 32 < n ? b[F.prow[lane + 32]] : 0.0;
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    const double cj = __shfl_sync(0xffffffffu, j < 32 ? c0 : c1, j & 31);
    const double* col = s_lu + j * n;
    if (lane > j && lane < n) c0 -= col[lane] * cj;
    if (lane + 32 > j && lane + 32 < n) c1 -= col[lane + 32] * cj;
  }
  for (int j = F.rank - 1; j >= 0; --j) {
    const double xj = __shfl_sync(0xffffffffu, j < 32 ? c0 : c1, j & 31) / s_lu[j * n + j];
    if (lane == j) c0 = xj;
    if (lane + 32 == j) c1 = xj;
    const double* col = s_lu + j * n;
    if (lane < j) c0 -= col[lane] * xj;
    if (lane + 32 < j) c1 -= col[lane + 32] * xj;
  }
  if (lane < n) x[F.pcol[lane]] = lane < F.rank ? c0 : 0.0;
  if (lane + 32 < n) x[F.pcol[lane + 32]] = lane + 32 < F.rank ? c1 : 0.0;
}

inline int coarse_threads(int n) {  // small coarse systems: fewer threads, cheaper barriers
  const int t = (n + 31) / 32 * 32;
  return t < 32 ? 32 : (t > kCoarseThreads ? kCoarseThreads : t);
}
inline size_t coarse_smem_bytes(int n) {
  return sizeof(double) * (size_t(n > 0 ? n : 1) + (n <= kCoarseSmemN ? size_t(n) * n : 0));
}

// ---------------------------------------------------------- elementwise
// EXTENSION — Chebyshev step 0 from x = 0: r = b exactly (A 0 = +0), d = (b / D) / theta, x = 0 + d
__global__ void cheb_first_kernel(int n, const double* b, const double* D, double theta, double* dv, double* x) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dn = (b[i] / D[i]) / theta;
  dv[i] = dn;
  x[i] = 0.0 + dn;
}
__global__ void presmooth_kernel(int n, const double* b, const double* d, double w, double* x) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (w * b[i]) / d[i];
}
__global__ void scale_copy_kernel(int n_u, int n_t, int n_p, const double* x, double st, double sp, double* y) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = n_u + n_t + n_p;
  if (i >= n) return;
  const double v = x[i];
  y[i] = i < n_u ? v : (i < n_u + n_t ? v * st : v * sp);
}
__global__ void axpy_kernel(long long n, const double* a, const double* b, double beta, double* y) {  // y = a + beta b
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] + beta * b[i];
}
__global__ void add_inplace_kernel(long long n, double* x, const double* dx) {
  pdl_entry();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] + dx[i];
}

}  // namespace fpd
