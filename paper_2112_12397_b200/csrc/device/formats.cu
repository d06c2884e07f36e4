// Device-side construction of the solve path's sparse layouts (device.cuh) from CSR resident in
// HBM.  The CSR arrives either from the host (upload_csr: one raw copy of row offsets, columns and
// values) or from the device setup (dsetup.cu), and every layout — BSR3-SELL, SELL-32, node-blocked
// SELL, the windowed pipeline, R = P^T — is built by kernels over it, so the host never loops over
// the entries of an operator.  Each builder produces exactly the layout the host builders of round 1
// produced (same slot order, same zero padding); the solve kernels are unchanged.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "engine.cuh"

namespace fpd {

namespace {

constexpr int kT = 256;

unsigned grid_for(long long n, int t = kT) { return unsigned(std::max(1LL, std::min((n + t - 1) / t, 1LL << 30))); }

// exclusive prefix sum of n values into out[0..n] (out[n] = total); returns the total
long long exclusive_scan(const long long* in, long long* out, long long n, cudaStream_t s) {
  size_t tmp_bytes = 0;
  cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, n + 1, s), "scan size");
  DevBuf<unsigned char> tmp(tmp_bytes);
  cuda_check(cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, in, out, n + 1, s), "scan");
  long long total = 0;
  cuda_check(cudaMemcpyAsync(&total, out + n, sizeof(long long), cudaMemcpyDeviceToHost, s), "scan total");
  cuda_check(cudaStreamSynchronize(s), "scan sync");
  return total;
}

__global__ void row_len_kernel(int n, const long long* rp, int* len) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) len[i] = int(rp[i + 1] - rp[i]);
}

// per slice of 32 rows: 32 * (longest row); in[n_slices] = 0 (scan input of n_slices + 1)
__global__ void slice_slots_kernel(int n_rows, int n_slices, const int* len, long long* out) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s > n_slices) return;
  if (s == n_slices) {
    out[s] = 0;
    return;
  }
  int mx = 0;
  for (int r = 0; r < kSlice; ++r) {
    const long long i = s * kSlice + r;
    if (i < n_rows) mx = max(mx, len[i]);
  }
  out[s] = (long long)mx * kSlice;
}

__global__ void sell_fill_kernel(int n, const long long* rp, const int* ci, const double* v, const long long* off,
                                 int* cols, double* vals) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long base = off[i / kSlice] + (i % kSlice);
  const long long r0 = rp[i], m = rp[i + 1] - r0;
  for (long long k = 0; k < m; ++k) {
    cols[base + k * kSlice] = ci[r0 + k];
    vals[base + k * kSlice] = v[r0 + k];
  }
}

// node n: rows 3n..3n+2 share one column pattern (else *ok = 0)
__global__ void bp3_check_kernel(int nn, const long long* rp, const int* ci, int* ok) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= nn) return;
  const long long r0 = rp[3 * n], len = rp[3 * n + 1] - r0;
  for (int d = 1; d < 3; ++d) {
    const long long rd = rp[3 * n + d];
    if (rp[3 * n + d + 1] - rd != len) {
      *ok = 0;
      return;
    }
    for (long long k = 0; k < len; ++k)
      if (ci[r0 + k] != ci[rd + k]) {
        *ok = 0;
        return;
      }
  }
}

__global__ void bp3_len_kernel(int nn, const long long* rp, int* len) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n < nn) len[n] = int(rp[3 * n + 1] - rp[3 * n]);
}

// sort key of node n: its window in the high bits, then longest first inside the window
__global__ void bp3_key_kernel(int nn, const int* len, unsigned long long* key, int* val) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= nn) return;
  key[n] = ((unsigned long long)(n / kBp3Window) << 32) | (unsigned)(0x7fffffff - len[n]);
  val[n] = int(n);
}
// slot -> node (sorted order, -1 past the end) and the slots of each slice
__global__ void bp3_slots_kernel(int nn, int ns, const int* sorted, const int* len, int* node, long long* out) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s > ns) return;
  if (s == ns) {
    out[s] = 0;
    return;
  }
  int mx = 0;
  for (int r = 0; r < kSlice; ++r) {
    const long long q = s * kSlice + r;
    const int n = q < nn ? sorted[q] : -1;
    node[q] = n;
    if (n >= 0) mx = max(mx, len[n]);
  }
  out[s] = (long long)mx * kSlice;
}
__global__ void bp3_fill_kernel(int n_slots, const int* node, const long long* rp, const int* ci, const double* v,
                                const long long* off, int* cols, double* vals) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= n_slots) return;
  const long long n = node[q];
  if (n < 0) return;
  const long long s0 = off[q / kSlice];
  const int lane = int(q % kSlice);
  const long long len = rp[3 * n + 1] - rp[3 * n];
  for (long long k = 0; k < len; ++k) {
    cols[s0 + k * kSlice + lane] = ci[rp[3 * n] + k];
    for (int d = 0; d < 3; ++d) vals[3 * (s0 + k * kSlice) + 32 * d + lane] = v[rp[3 * n + d] + k];
  }
}

// Block columns of block row b (global block row g): the union of c / 3 over its three scalar rows,
// each sorted, so a three-way merge.  fill == false: count; fill == true: write slots.
template <bool fill>
__global__ void bsr3_rows_kernel(int nb, const int* brows, const long long* rp, const int* ci, const double* v,
                                 int* len, const long long* off, int* bcols, double* vals) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const long long g = brows ? brows[b] : b;
  long long p[3], e[3];
  for (int li = 0; li < 3; ++li) p[li] = rp[3 * g + li], e[li] = rp[3 * g + li + 1];
  const long long s = b / kSlice;
  const int lane = int(b % kSlice);
  int k = 0;
  for (;;) {
    int cb = 0x7fffffff;
    for (int li = 0; li < 3; ++li)
      if (p[li] < e[li]) cb = min(cb, ci[p[li]] / 3);
    if (cb == 0x7fffffff) break;
    if (fill) {
      const long long slot = off[s] + (long long)k * kSlice;
      bcols[slot + lane] = cb;
      for (int li = 0; li < 3; ++li)
        for (; p[li] < e[li] && ci[p[li]] / 3 == cb; ++p[li])
          vals[slot * 9 + (li * 3 + ci[p[li]] % 3) * kSlice + lane] = v[p[li]];
    } else {
      for (int li = 0; li < 3; ++li)
        while (p[li] < e[li] && ci[p[li]] / 3 == cb) ++p[li];
    }
    ++k;
  }
  if (!fill) len[b] = k;
}

__global__ void pipe_fill_kernel(int n_slices, const int* perm, const long long* woff, const long long* rp,
                                 const int* ci, const double* v, double* pv, int* pci) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n_slices * kPipeRows) return;
  const long long s = t / kPipeRows;
  const int r = int(t % kPipeRows);
  const int i = perm[t];
  if (i < 0) return;
  constexpr long long kWin = (long long)kPipeRows * kPipeW;
  const long long r0 = rp[i], m = rp[i + 1] - r0;
  for (long long k = 0; k < m; ++k) {
    const long long idx = (woff[s] + k / kPipeW) * kWin + (long long)r * kPipeW + k % kPipeW;
    pv[idx] = v[r0 + k];
    pci[idx] = ci[r0 + k];
  }
}

// ---- transpose (rows of A^T list the source rows ascending, like the counting transpose): a STABLE
// radix sort of the entries by column, taken in row-major order, so equal columns keep ascending rows
__global__ void col_count_kernel(long long nnz, const int* ci, unsigned long long* cnt) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz; k += (long long)gridDim.x * blockDim.x)
    atomicAdd(cnt + ci[k], 1ull);
}

template <class Idx>
__global__ void iota_kernel(long long n, Idx* out) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    out[k] = Idx(k);
}

// entry k of A (row-major) lands at position pos: its row by binary search of the row offsets
template <class Idx>
__global__ void gather_t_kernel(long long nnz, int n_rows, const long long* rp, const double* v, const Idx* src,
                                int* tci, double* tv) {
  for (long long pos = blockIdx.x * (long long)blockDim.x + threadIdx.x; pos < nnz;
       pos += (long long)gridDim.x * blockDim.x) {
    const long long k = (long long)src[pos];
    int lo = 0, hi = n_rows;  // largest row r with rp[r] <= k
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rp[mid] <= k) lo = mid;
      else hi = mid;
    }
    tci[pos] = lo;
    tv[pos] = v[k];
  }
}

template <class Idx>
void transpose_fill(const DCsr& A, DCsr& T, cudaStream_t s) {
  int bits = 1;
  while ((1LL << bits) < (long long)A.n_cols) ++bits;
  DevBuf<int> kin(size_t(A.nnz)), kout(size_t(A.nnz));
  DevBuf<Idx> vin(size_t(A.nnz)), vout(size_t(A.nnz));
  cuda_check(cudaMemcpyAsync(kin.get(), A.ci.get(), kin.bytes(), cudaMemcpyDeviceToDevice, s), "keys");
  iota_kernel<Idx><<<1184, kT, 0, s>>>(A.nnz, vin.get());
  size_t tb = 0;
  cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), vin.get(), vout.get(), A.nnz, 0, bits, s),
             "radix size");
  {
    DevBuf<unsigned char> tmp(tb);
    cuda_check(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin.get(), kout.get(), vin.get(), vout.get(), A.nnz, 0,
                                               bits, s),
               "radix sort");
  }
  kin = DevBuf<int>(), kout = DevBuf<int>(), vin = DevBuf<Idx>();
  gather_t_kernel<Idx><<<1184, kT, 0, s>>>(A.nnz, A.n_rows, A.rp.get(), A.v.get(), vout.get(), T.ci.get(), T.v.get());
}

}  // namespace

// ------------------------------------------------------------------ host <-> device CSR
DCsr upload_csr(const HostCsrView& A) {
  DCsr D;
  D.n_rows = A.n_rows, D.n_cols = A.n_cols, D.nnz = A.nnz();
  static_assert(sizeof(long long) == sizeof(int64_t), "row offsets");
  if (A.n_rows > 0) D.rp.upload(reinterpret_cast<const long long*>(A.rp), size_t(A.n_rows) + 1);
  else D.rp.alloc(1), D.rp.zero();
  D.ci.upload(A.ci, size_t(D.nnz));
  D.v.upload(A.v, size_t(D.nnz));
  return D;
}

fpb::Csr host_copy(const HostCsrView& A) {
  fpb::Csr C(A.n_rows, A.n_cols);
  if (A.n_rows == 0) return C;
  C.rp.assign(A.rp, A.rp + A.n_rows + 1);
  C.ci.assign(A.ci, A.ci + A.nnz());
  C.v.assign(A.v, A.v + A.nnz());
  return C;
}

fpb::Csr download_csr(const DCsr& D) {
  fpb::Csr A(D.n_rows, D.n_cols);
  if (D.n_rows > 0)
    cuda_check(cudaMemcpy(A.rp.data(), D.rp.get(), sizeof(long long) * (size_t(D.n_rows) + 1), cudaMemcpyDeviceToHost),
               "download rp");
  A.ci.resize(size_t(D.nnz));
  A.v.resize(size_t(D.nnz));
  if (D.nnz) {
    cuda_check(cudaMemcpy(A.ci.data(), D.ci.get(), sizeof(int) * size_t(D.nnz), cudaMemcpyDeviceToHost), "download ci");
    cuda_check(cudaMemcpy(A.v.data(), D.v.get(), sizeof(double) * size_t(D.nnz), cudaMemcpyDeviceToHost), "download v");
  }
  return A;
}

// ------------------------------------------------------------------ layouts
namespace {
__global__ void sell_fill_sorted_kernel(int n_slots, const int* rows, const long long* rp, const int* ci, const double* v,
                                        const long long* off, int* cols, double* vals) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= n_slots) return;
  const long long i = rows[q];
  if (i < 0) return;
  const long long base = off[q / kSlice] + (q % kSlice);
  const long long r0 = rp[i], m = rp[i + 1] - r0;
  for (long long k = 0; k < m; ++k) {
    cols[base + k * kSlice] = ci[r0 + k];
    vals[base + k * kSlice] = v[r0 + k];
  }
}
}  // namespace

DSell sell_from(const DCsr& A, cudaStream_t s, bool sorted) {
  DSell D;
  D.n_rows = A.n_rows, D.n_cols = A.n_cols, D.nnz = A.nnz;
  D.n_slices = (A.n_rows + kSlice - 1) / kSlice;
  D.len.alloc(size_t(A.n_rows));
  if (A.n_rows) row_len_kernel<<<grid_for(A.n_rows), kT, 0, s>>>(A.n_rows, A.rp.get(), D.len.get());
  DevBuf<long long> sl(size_t(D.n_slices) + 1);
  D.off.alloc(size_t(D.n_slices) + 1);
  if (sorted && A.n_rows > kSlice) {
    // rows by (window, length descending), then slices of 32: almost no padding per slice
    const int n = A.n_rows;
    DevBuf<int> order{size_t(n)};
    {
      DevBuf<unsigned long long> kin{size_t(n)}, kout{size_t(n)};
      DevBuf<int> vin{size_t(n)};
      bp3_key_kernel<<<grid_for(n), kT, 0, s>>>(n, D.len.get(), kin.get(), vin.get());
      size_t tb = 0;
      cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), vin.get(), order.get(), n, 0, 64, s),
                 "sell sort size");
      DevBuf<unsigned char> tmp(tb);
      cuda_check(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin.get(), kout.get(), vin.get(), order.get(), n, 0, 64, s),
                 "sell sort");
      cuda_check(cudaStreamSynchronize(s), "sell sort");
    }
    D.rows.alloc(size_t(D.n_slices) * kSlice);
    bp3_slots_kernel<<<grid_for(D.n_slices + 1), kT, 0, s>>>(n, D.n_slices, order.get(), D.len.get(), D.rows.get(), sl.get());
    D.slots = exclusive_scan(sl.get(), D.off.get(), D.n_slices, s);
    D.cols.alloc(size_t(D.slots));
    D.vals.alloc(size_t(D.slots));
    if (D.slots) {
      cuda_check(cudaMemsetAsync(D.cols.get(), 0, D.cols.bytes(), s), "memset");
      cuda_check(cudaMemsetAsync(D.vals.get(), 0, D.vals.bytes(), s), "memset");
      sell_fill_sorted_kernel<<<grid_for((long long)D.n_slices * kSlice), kT, 0, s>>>(
          D.n_slices * kSlice, D.rows.get(), A.rp.get(), A.ci.get(), A.v.get(), D.off.get(), D.cols.get(), D.vals.get());
    }
    cuda_check(cudaStreamSynchronize(s), "sell_from");
    return D;
  }
  slice_slots_kernel<<<grid_for(D.n_slices + 1), kT, 0, s>>>(A.n_rows, D.n_slices, D.len.get(), sl.get());
  D.slots = exclusive_scan(sl.get(), D.off.get(), D.n_slices, s);
  D.cols.alloc(size_t(D.slots));
  D.vals.alloc(size_t(D.slots));
  if (D.slots) {
    cuda_check(cudaMemsetAsync(D.cols.get(), 0, D.cols.bytes(), s), "memset");
    cuda_check(cudaMemsetAsync(D.vals.get(), 0, D.vals.bytes(), s), "memset");
    sell_fill_kernel<<<grid_for(A.n_rows), kT, 0, s>>>(A.n_rows, A.rp.get(), A.ci.get(), A.v.get(), D.off.get(),
                                                       D.cols.get(), D.vals.get());
  }
  cuda_check(cudaStreamSynchronize(s), "sell_from");
  return D;
}

namespace {
__global__ void srt_key_kernel(int n, const int* len, unsigned long long* key, int* val) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = ((unsigned long long)(i / kSrtWindow) << 32) | (unsigned)(0x7fffffff - len[i]);
  val[i] = int(i);
}
// slot -> row in sorted order (-1 past the end), and the values of each slice of 8 rows: 256 per round
// of 32 entries of its longest row
__global__ void srt_slots_kernel(int n, int ns, const int* sorted, const int* len, int* row, long long* out) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s > ns) return;
  if (s == ns) {
    out[s] = 0;
    return;
  }
  int mx = 0;
  for (int r = 0; r < kSrtRows; ++r) {
    const long long q = s * kSrtRows + r;
    const int i = q < n ? sorted[q] : -1;
    row[q] = i;
    if (i >= 0) mx = max(mx, len[i]);
  }
  out[s] = (long long)((mx + 31) / 32) * 32 * kSrtRows;
}
__global__ void srt_fill_kernel(int n_slots, const int* row, const long long* rp, const double* v, const long long* off,
                                double* vals) {
  const long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (slot >= n_slots) return;
  const long long r = row[slot];
  if (r < 0) return;
  const int rl = int(slot % kSrtRows);
  const long long base = off[slot / kSrtRows], r0 = rp[r], m = rp[r + 1] - r0;
  for (long long k = 0; k < m; ++k) {
    const long long t = k / 32, q = (k % 32) / 8, u = k % 8;
    vals[base + ((8 * t + u) * kSrtRows + rl) * 4 + q] = v[r0 + k];
  }
}
}  // namespace

DSrt srt_from(const DCsr& A, cudaStream_t s) {
  DSrt D;
  const int n = A.n_rows;
  D.n_rows = n, D.nnz = A.nnz;
  if (n == 0) return D;
  const int ns = (n + kSrtRows - 1) / kSrtRows;
  D.len.alloc(size_t(n));
  row_len_kernel<<<grid_for(n), kT, 0, s>>>(n, A.rp.get(), D.len.get());
  // rows by (window, length descending): a stable sort, so a run of equal-pattern rows stays together
  DevBuf<int> sorted{size_t(n)};
  {
    DevBuf<unsigned long long> kin{size_t(n)}, kout{size_t(n)};
    DevBuf<int> vin{size_t(n)};
    srt_key_kernel<<<grid_for(n), kT, 0, s>>>(n, D.len.get(), kin.get(), vin.get());
    size_t tb = 0;
    cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), vin.get(), sorted.get(), n, 0, 64, s),
               "srt sort size");
    DevBuf<unsigned char> tmp(tb);
    cuda_check(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin.get(), kout.get(), vin.get(), sorted.get(), n, 0, 64, s),
               "srt sort");
    cuda_check(cudaStreamSynchronize(s), "srt sort");
  }
  DevBuf<long long> sl(size_t(ns) + 1);
  D.off.alloc(size_t(ns) + 1);
  D.row.alloc(size_t(ns) * kSrtRows);
  srt_slots_kernel<<<grid_for(ns + 1), kT, 0, s>>>(n, ns, sorted.get(), D.len.get(), D.row.get(), sl.get());
  D.slots = exclusive_scan(sl.get(), D.off.get(), ns, s);
  D.vals.alloc(size_t(D.slots));
  cuda_check(cudaMemsetAsync(D.vals.get(), 0, D.vals.bytes(), s), "memset");
  srt_fill_kernel<<<grid_for((long long)ns * kSrtRows), kT, 0, s>>>(ns * kSrtRows, D.row.get(), A.rp.get(), A.v.get(),
                                                                  D.off.get(), D.vals.get());
  // the columns: shared lists where A has them (share_columns), else its own CSR lists
  D.cp.alloc(size_t(n) + 1);
  if (A.cp.size()) {
    D.nci = A.nci;
    cuda_check(cudaMemcpyAsync(D.cp.get(), A.cp.get(), D.cp.bytes(), cudaMemcpyDeviceToDevice, s), "srt cp");
  } else {
    D.nci = A.nnz;
    cuda_check(cudaMemcpyAsync(D.cp.get(), A.rp.get(), D.cp.bytes(), cudaMemcpyDeviceToDevice, s), "srt cp");
  }
  D.ci.alloc(size_t(D.nci));
  cuda_check(cudaMemcpyAsync(D.ci.get(), A.ci.get(), D.ci.bytes(), cudaMemcpyDeviceToDevice, s), "srt ci");
  cuda_check(cudaStreamSynchronize(s), "srt_from");
  return D;
}

namespace {
__global__ void subset_len_kernel(int m, const int* rows, const long long* rp, long long* cnt) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t > m) return;
  cnt[t] = t < m ? rp[rows[t] + 1] - rp[rows[t]] : 0;
}
// a warp per subset row: values from rp, columns from the row's list (cp with shared lists, else rp)
__global__ void subset_gather_kernel(int m, const int* rows, const long long* rp, const long long* cp, const int* ci,
                                     const double* v, const long long* off, int* oci, double* ov) {
  const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= m) return;
  const long long r = rows[t], r0 = rp[r], len = rp[r + 1] - r0, c0 = cp ? cp[r] : r0, o = off[t];
  for (long long k = lane; k < len; k += 32) oci[o + k] = ci[c0 + k], ov[o + k] = v[r0 + k];
}
}  // namespace

DSrt srt_subset_from(const DCsr& A, const std::vector<int>& rows, cudaStream_t s) {
  const int m = int(rows.size());
  DCsr S;  // the subset as a CSR of its own (plain columns), then the usual builders
  S.n_rows = m, S.n_cols = A.n_cols;
  DevBuf<int> drows;
  drows.upload(rows);
  DevBuf<long long> cnt(size_t(m) + 1);
  S.rp.alloc(size_t(m) + 1);
  subset_len_kernel<<<grid_for(m + 1), kT, 0, s>>>(m, drows.get(), A.rp.get(), cnt.get());
  S.nnz = exclusive_scan(cnt.get(), S.rp.get(), m, s);
  S.ci.alloc(size_t(S.nnz)), S.v.alloc(size_t(S.nnz));
  if (m)
    subset_gather_kernel<<<grid_for((long long)m * 32), kT, 0, s>>>(m, drows.get(), A.rp.get(),
                                                                   A.cp.size() ? A.cp.get() : nullptr, A.ci.get(),
                                                                   A.v.get(), S.rp.get(), S.ci.get(), S.v.get());
  cuda_check(cudaStreamSynchronize(s), "srt subset gather");
  share_columns(S, s);
  DSrt D = srt_from(S, s);
  D.out_row = std::move(drows);
  return D;
}

DBp3 bp3_from(const DCsr& A, cudaStream_t s) {
  DBp3 D;
  if (A.n_rows % 3 != 0 || A.n_rows == 0) return D;
  const int nn = A.n_rows / 3;
  DevBuf<int> ok(1);
  const int one = 1;
  cuda_check(cudaMemcpyAsync(ok.get(), &one, sizeof(int), cudaMemcpyHostToDevice, s), "flag");
  bp3_check_kernel<<<grid_for(nn), kT, 0, s>>>(nn, A.rp.get(), A.ci.get(), ok.get());
  int same = 0;
  cuda_check(cudaMemcpyAsync(&same, ok.get(), sizeof(int), cudaMemcpyDeviceToHost, s), "flag");
  cuda_check(cudaStreamSynchronize(s), "bp3 check");
  if (!same) return D;
  D.n_nodes = nn, D.nnz = A.nnz;
  const int ns = (nn + kSlice - 1) / kSlice;
  D.len.alloc(size_t(nn));
  bp3_len_kernel<<<grid_for(nn), kT, 0, s>>>(nn, A.rp.get(), D.len.get());
  // nodes by (window, length descending): stable radix sort of 64-bit keys
  DevBuf<int> sorted{size_t(nn)};
  {
    DevBuf<unsigned long long> kin{size_t(nn)}, kout{size_t(nn)};
    DevBuf<int> vin{size_t(nn)};
    bp3_key_kernel<<<grid_for(nn), kT, 0, s>>>(nn, D.len.get(), kin.get(), vin.get());
    size_t tb = 0;
    cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), vin.get(), sorted.get(), nn, 0, 64, s),
               "bp3 sort size");
    DevBuf<unsigned char> tmp(tb);
    cuda_check(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin.get(), kout.get(), vin.get(), sorted.get(), nn, 0, 64, s),
               "bp3 sort");
    cuda_check(cudaStreamSynchronize(s), "bp3 sort");
  }
  DevBuf<long long> sl(size_t(ns) + 1);
  D.off.alloc(size_t(ns) + 1);
  D.node.alloc(size_t(ns) * kSlice);
  bp3_slots_kernel<<<grid_for(ns + 1), kT, 0, s>>>(nn, ns, sorted.get(), D.len.get(), D.node.get(), sl.get());
  D.slots = exclusive_scan(sl.get(), D.off.get(), ns, s);
  D.cols.alloc(size_t(D.slots));
  D.vals.alloc(3 * size_t(D.slots));
  if (D.slots) {
    cuda_check(cudaMemsetAsync(D.cols.get(), 0, D.cols.bytes(), s), "memset");
    cuda_check(cudaMemsetAsync(D.vals.get(), 0, D.vals.bytes(), s), "memset");
    bp3_fill_kernel<<<grid_for((long long)ns * kSlice), kT, 0, s>>>(ns * kSlice, D.node.get(), A.rp.get(), A.ci.get(),
                                                                  A.v.get(), D.off.get(), D.cols.get(), D.vals.get());
  }
  cuda_check(cudaStreamSynchronize(s), "bp3_from");
  return D;
}

DBsr3 bsr3_from(const DCsr& A, const std::vector<int>* brows, cudaStream_t s) {
  if (A.n_rows != A.n_cols || A.n_rows % 3 != 0) throw std::invalid_argument("make_bsr3: needs a square matrix with n % 3 == 0");
  DBsr3 D;
  const int nb = brows ? int(brows->size()) : A.n_rows / 3;
  D.n_brows = nb;
  D.n_slices = (nb + kSlice - 1) / kSlice;
  if (brows) D.brow_map.upload(*brows);
  const int* bm = brows ? D.brow_map.get() : nullptr;
  D.len.alloc(size_t(nb));
  if (nb)
    bsr3_rows_kernel<false><<<grid_for(nb), kT, 0, s>>>(nb, bm, A.rp.get(), A.ci.get(), A.v.get(), D.len.get(), nullptr,
                                                        nullptr, nullptr);
  DevBuf<long long> sl(size_t(D.n_slices) + 1);
  D.off.alloc(size_t(D.n_slices) + 1);
  slice_slots_kernel<<<grid_for(D.n_slices + 1), kT, 0, s>>>(nb, D.n_slices, D.len.get(), sl.get());
  D.slots = exclusive_scan(sl.get(), D.off.get(), D.n_slices, s);
  {  // number of blocks (the ledger's byte count)
    std::vector<int> len(static_cast<size_t>(nb));
    if (nb) cuda_check(cudaMemcpy(len.data(), D.len.get(), sizeof(int) * size_t(nb), cudaMemcpyDeviceToHost), "len");
    D.nblocks = std::accumulate(len.begin(), len.end(), int64_t(0));
  }
  D.bcols.alloc(size_t(D.slots));
  D.vals.alloc(size_t(D.slots) * 9);
  if (D.slots) {
    cuda_check(cudaMemsetAsync(D.bcols.get(), 0, D.bcols.bytes(), s), "memset");
    cuda_check(cudaMemsetAsync(D.vals.get(), 0, D.vals.bytes(), s), "memset");
    bsr3_rows_kernel<true><<<grid_for(nb), kT, 0, s>>>(nb, bm, A.rp.get(), A.ci.get(), A.v.get(), D.len.get(),
                                                       D.off.get(), D.bcols.get(), D.vals.get());
  }
  cuda_check(cudaStreamSynchronize(s), "bsr3_from");
  return D;
}

DPipe pipe_from(const DCsr& A, cudaStream_t s) {
  constexpr int kSigma = 4096;  // rows are sorted by length only inside chunks (locality of the gathers)
  DPipe D;
  D.n_rows = A.n_rows, D.nnz = A.nnz;
  D.n_slices = (A.n_rows + kPipeRows - 1) / kPipeRows;
  // the row permutation and the window offsets depend only on the row lengths (host, O(n log))
  std::vector<long long> rp(size_t(A.n_rows) + 1, 0);
  if (A.n_rows)
    cuda_check(cudaMemcpy(rp.data(), A.rp.get(), sizeof(long long) * rp.size(), cudaMemcpyDeviceToHost), "rp");
  auto row_len = [&](int i) { return int(rp[size_t(i) + 1] - rp[i]); };
  std::vector<int> perm(static_cast<size_t>(D.n_slices) * kPipeRows, -1);
  for (int i = 0; i < A.n_rows; ++i) perm[i] = i;
  for (int c0 = 0; c0 < A.n_rows; c0 += kSigma) {
    const int c1 = std::min(A.n_rows, c0 + kSigma);
    std::stable_sort(perm.begin() + c0, perm.begin() + c1, [&](int a, int b) { return row_len(a) > row_len(b); });
  }
  std::vector<int> len(perm.size(), 0);
  std::vector<long long> woff(static_cast<size_t>(D.n_slices) + 1, 0);
  for (int sl = 0; sl < D.n_slices; ++sl) {
    int mx = 0;
    for (int r = 0; r < kPipeRows; ++r) {
      const int i = perm[size_t(sl) * kPipeRows + r];
      len[size_t(sl) * kPipeRows + r] = i >= 0 ? row_len(i) : 0;
      mx = std::max(mx, len[size_t(sl) * kPipeRows + r]);
    }
    woff[sl + 1] = woff[sl] + (mx + kPipeW - 1) / kPipeW;
  }
  constexpr int64_t kWin = int64_t(kPipeRows) * kPipeW;
  D.slots = woff.back() * kWin;
  // persistent CTAs (one per SM) over contiguous slice ranges of equal window count
  int dev = 0, sms = 148;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
  D.n_ctas = std::max(1, std::min(D.n_slices, sms * kPipeCtasPerSm));
  std::vector<int> cs(static_cast<size_t>(D.n_ctas) + 1, D.n_slices);
  cs[0] = 0;
  const long long tot = woff.back();
  for (int b = 1; b < D.n_ctas; ++b) {
    const long long target = (tot * b + D.n_ctas - 1) / D.n_ctas;
    cs[b] = int(std::lower_bound(woff.begin(), woff.end() - 1, target) - woff.begin());
    cs[b] = std::max(cs[b], cs[b - 1]);
  }
  D.cta_slice.upload(cs);
  D.woff.upload(woff);
  D.row.upload(perm);
  D.len.upload(len);
  D.v.alloc(size_t(D.slots));
  D.ci.alloc(size_t(D.slots));
  if (D.slots) {
    cuda_check(cudaMemsetAsync(D.v.get(), 0, D.v.bytes(), s), "memset");
    cuda_check(cudaMemsetAsync(D.ci.get(), 0, D.ci.bytes(), s), "memset");
    pipe_fill_kernel<<<grid_for((long long)D.n_slices * kPipeRows), kT, 0, s>>>(
        D.n_slices, D.row.get(), D.woff.get(), A.rp.get(), A.ci.get(), A.v.get(), D.v.get(), D.ci.get());
  }
  cuda_check(cudaStreamSynchronize(s), "pipe_from");
  return D;
}

DCsr transpose_dev(const DCsr& A, cudaStream_t s) {
  DCsr T;
  T.n_rows = A.n_cols, T.n_cols = A.n_rows, T.nnz = A.nnz;
  DevBuf<unsigned long long> cnt(size_t(A.n_cols) + 1);
  cuda_check(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s), "memset");
  if (A.nnz) col_count_kernel<<<grid_for(A.nnz), kT, 0, s>>>(A.nnz, A.ci.get(), cnt.get());
  T.rp.alloc(size_t(A.n_cols) + 1);
  exclusive_scan(reinterpret_cast<const long long*>(cnt.get()), T.rp.get(), A.n_cols, s);
  T.ci.alloc(size_t(A.nnz));
  T.v.alloc(size_t(A.nnz));
  if (A.nnz) {
    if (A.nnz < (1LL << 31)) transpose_fill<int>(A, T, s);
    else transpose_fill<long long>(A, T, s);
  }
  cuda_check(cudaStreamSynchronize(s), "transpose_dev");
  return T;
}

namespace {
// own[r] = 0 when row r has exactly row r - 1's columns (it will read that row's list), else its
// length; a warp per row.  own[n] = 0 (scan input of n + 1 values).
__global__ void same_cols_kernel(int n, const long long* rp, const int* ci, long long* own) {
  const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r > n) return;
  if (r == n) {
    if (lane == 0) own[r] = 0;
    return;
  }
  const long long b1 = rp[r], len = rp[r + 1] - b1;
  bool same = r > 0 && rp[r] - rp[r - 1] == len;
  if (same) {
    const long long b0 = rp[r - 1];
    for (long long k = lane; same && k < len; k += 32) same = ci[b0 + k] == ci[b1 + k];
  }
  same = __all_sync(0xffffffffu, same);
  if (lane == 0) own[r] = same ? 0 : len;
}
// cp[r] = (lists kept up to and including row r) - len(r): the start of row r's own list, or of the
// list of the first row of its run of equal patterns; rows that own a list copy it there
__global__ void shared_cols_fill_kernel(int n, const long long* rp, const int* ci, const long long* own,
                                        const long long* excl, int* cci, long long* cp) {
  const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const long long b = rp[r], len = rp[r + 1] - b;
  const long long start = excl[r] + own[r] - len;
  if (lane == 0) cp[r] = start;
  if (own[r] != 0)
    for (long long k = lane; k < len; k += 32) cci[start + k] = ci[b + k];
}
}  // namespace

bool share_columns(DCsr& A, cudaStream_t s) {
  if (A.n_rows < 2 || A.nnz == 0 || A.cp.size()) return false;
  const long long n = A.n_rows;
  DevBuf<long long> own(size_t(n) + 1), excl(size_t(n) + 1);
  same_cols_kernel<<<grid_for((n + 1) * 32), kT, 0, s>>>(A.n_rows, A.rp.get(), A.ci.get(), own.get());
  const long long nci = exclusive_scan(own.get(), excl.get(), n, s);
  if (nci > A.nnz - A.nnz / 8) return false;  // under 1/8 of the index bytes saved: keep plain CSR
  DevBuf<int> cci{size_t(nci)};
  A.cp.alloc(size_t(n) + 1);
  shared_cols_fill_kernel<<<grid_for(n * 32), kT, 0, s>>>(A.n_rows, A.rp.get(), A.ci.get(), own.get(), excl.get(),
                                                        cci.get(), A.cp.get());
  cuda_check(cudaMemcpyAsync(A.cp.get() + n, &nci, sizeof(long long), cudaMemcpyHostToDevice, s), "share cp end");
  cuda_check(cudaStreamSynchronize(s), "share_columns");
  A.ci = std::move(cci);
  A.nci = nci;
  return true;
}

bool sell_sorted() {  // FRACPREC_B200_SELL_SORTED=0: plain SELL-32 for the thread-per-row operators
  const char* e = std::getenv("FRACPREC_B200_SELL_SORTED");
  return !(e && std::atoi(e) == 0);
}

DMat mat_from(DCsr&& A, bool few_rows_parallel, bool strided, cudaStream_t s) {
  DMat M;
  if (strided) {  // row_sum = strided32: plain CSR, one warp per row (or window-staged CTAs of R rows)
    M.warp = M.strided = true;
    M.strided_rows = 1;  // one row per CTA: most parallel loads for few-row operators
    M.csr = std::move(A);
    // the warp-row kernel's operators (A_l, R_l of an aggregation hierarchy): the coarse dofs of an
    // aggregate mostly have one column list — a row with exactly its predecessor's columns reads that
    // row's list, so the list is stored (and streamed from HBM) once per run: 12 -> ~8.7 B per entry.
    // FRACPREC_B200_SHARED_COLS=0 keeps plain CSR.
    const char* e = std::getenv("FRACPREC_B200_SHARED_COLS");
    if (M.csr.n_rows >= 2048 && !(e && std::atoi(e) == 0)) share_columns(M.csr, s);
    // enough rows to fill the machine with four lanes per row: the strided32 sums from sorted slices
    // (srt_kernel); the CSR stays for the row-subset launches of the sparse right-hand side.
    // FRACPREC_B200_SRT_MIN_ROWS overrides the threshold (tests force it on small levels; 0 = never).
    long long srt_min = 65536;
    if (const char* q = std::getenv("FRACPREC_B200_SRT_MIN_ROWS")) srt_min = std::atoll(q);
    if (srt_min > 0 && M.csr.n_rows >= srt_min) {
      M.sr = srt_from(M.csr, s);
      M.srt = true;
    }
    return M;
  }
  const double avg = A.n_rows > 0 ? double(A.nnz) / A.n_rows : 0.0;
  // SELL's thread-per-row chains need enough rows to hide latency; below ~64k
  // rows the slice kernel's parallel loads win even for short rows
  M.warp = A.n_rows > 0 && (avg >= 48.0 || (A.n_rows < 65536 && avg >= 8.0) ||
                            (few_rows_parallel && A.n_rows < 2048 && avg >= 2.0));
  if (!M.warp) {
    M.sell = sell_from(A, s, sell_sorted());
    return M;
  }
  M.slice_rows = A.n_rows >= 2048 ? 32 : 8;
  if (M.slice_rows == 32) {
    M.pipe = true;
    M.pm = pipe_from(A, s);
    return M;
  }
  M.csr = std::move(A);
  return M;
}

}  // namespace fpd
