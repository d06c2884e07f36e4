// Device SpGEMM for the preconditioner setup (setup on the
// device): the Galerkin products of amg_setup (D^-1 A P_tent, A P, P^T (A P),
// /root/reference/proj/core/src/amg.cpp:259-268) and the Schur-core products of
// build_tpu / build_tup (precond.cpp:18-36), bit for bit the host's spgemm
// (csrc/host/hcsr.cpp), which restates csr.cpp:139-176:
//   row i of C:  for k in row i of A (ascending), for j in row k of B (ascending):
//                acc[j] = (first touch ? 0.0 : acc[j]) + a_ik * b_kj ; row sorted by j.
// One warp owns a row.  It walks A's entries k in order; for one k the lanes take
// B's row k (all columns distinct), so every output entry receives its products in
// exactly the host's order.  Accumulators live in a per-warp open-addressing hash
// in shared memory; the row is then compacted and sorted by column (bitonic sort in
// shared memory).  Two passes: the symbolic one counts each row's distinct columns
// (the offsets), the numeric one fills values.  A row whose distinct columns exceed
// the hash capacity makes the whole product fall back to the host routine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "../host/hcsr.hpp"
#include "engine.cuh"

namespace fpd {
namespace {

constexpr int kCap = 2048;  // hash slots per warp = max distinct output columns of a row
constexpr int kFill = kCap * 3 / 4;
constexpr int kWarps = 4;   // rows in flight per CTA
constexpr int kThreads = 32 * kWarps;
constexpr size_t kSmem = size_t(kWarps) * kCap * (sizeof(int) + sizeof(double));

struct SpView {
  int n_rows;
  const long long* rp;
  const int* ci;
  const double* v;
};

__device__ __forceinline__ int hslot(int j) { return int((unsigned(j) * 2654435761u) & (kCap - 1)); }

// Find or insert column j; lanes insert distinct keys concurrently.  -1: table full.
__device__ __forceinline__ int hinsert(int* keys, int j, int* count) {
  int s = hslot(j);
  for (int probe = 0; probe < kCap; ++probe) {
    const int prev = atomicCAS(keys + s, -1, j);
    if (prev == -1) {
      atomicAdd(count, 1);
      return s;
    }
    if (prev == j) return s;
    s = (s + 1) & (kCap - 1);
  }
  return -1;
}

// numeric == false: cnt[row] = distinct columns of the row (-1: over kFill, use the host)
// numeric == true : the sorted row at crp[row]
template <bool numeric>
__global__ void __launch_bounds__(kThreads) spgemm_rows(SpView A, SpView B, const double* row_scale, int* cnt,
                                                        const long long* crp, int* cci, double* cv) {
  extern __shared__ unsigned char smem[];
  __shared__ int count[kWarps];
  __shared__ int full[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* keys = reinterpret_cast<int*>(smem) + warp * kCap;
  double* acc = reinterpret_cast<double*>(smem + size_t(kWarps) * kCap * sizeof(int)) + size_t(warp) * kCap;
  for (int row = blockIdx.x * kWarps + warp; row < A.n_rows; row += gridDim.x * kWarps) {
    if (numeric && cnt[row] > kFill) continue;  // a big row (spgemm_big_rows)
    for (int s = lane; s < kCap; s += 32) {
      keys[s] = -1;
      if (numeric) acc[s] = 0.0;  // first accumulation is (0.0 + p), as on the host
    }
    if (lane == 0) count[warp] = 0, full[warp] = 0;
    __syncwarp();
    const double sc = row_scale ? row_scale[row] : 1.0;
    bool overflow = false;
    for (long long ka = A.rp[row]; ka < A.rp[row + 1] && !overflow; ++ka) {
      const int k = A.ci[ka];
      const double av = row_scale ? A.v[ka] * sc : A.v[ka];  // == scale_rows(A, s) entry
      for (long long kb = B.rp[k] + lane; kb < B.rp[k + 1]; kb += 32) {
        const int s = hinsert(keys, B.ci[kb], &count[warp]);
        if (s < 0) {
          full[warp] = 1;
          continue;
        }
        if (numeric) acc[s] = acc[s] + av * B.v[kb];  // one lane per column within a k-step
      }
      __syncwarp();
      overflow = count[warp] > kFill || full[warp];
      __syncwarp();
    }
    if (!numeric) {
      if (lane == 0) cnt[row] = overflow ? -1 : count[warp];
      __syncwarp();
      continue;
    }
    const int n = count[warp];
    // compact the used slots to the front (in slot order; dst <= slot, read-before-write per chunk)
    int base = 0;
    for (int s0 = 0; s0 < kCap; s0 += 32) {
      const int s = s0 + lane;
      const bool has = keys[s] != -1;
      const unsigned mask = __ballot_sync(0xffffffffu, has);
      const int kk = has ? keys[s] : 0;
      const double vv = has ? acc[s] : 0.0;
      __syncwarp();
      if (has) {
        const int dst = base + __popc(mask & ((1u << lane) - 1));
        keys[dst] = kk;
        acc[dst] = vv;
      }
      base += __popc(mask);
      __syncwarp();
    }
    int m = 1;
    while (m < n) m <<= 1;
    for (int s = n + lane; s < m; s += 32) keys[s] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= m; size <<= 1)  // bitonic sort by column (keys distinct)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < m / 2; t += 32) {
          const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const int a = keys[lo], b = keys[hi];
          if ((a > b) == up) {
            keys[lo] = b, keys[hi] = a;
            const double x = acc[lo];
            acc[lo] = acc[hi], acc[hi] = x;
          }
        }
        __syncwarp();
      }
    const long long o = crp[row];
    for (int t = lane; t < n; t += 32) cci[o + t] = keys[t], cv[o + t] = acc[t];
    __syncwarp();
  }
}

// Rows with more distinct columns than a warp's table: one CTA per row, a block-wide table of
// kCapBig slots in shared memory; the k loop stays sequential (a barrier per k) and the threads take
// B's row k (distinct columns), so every entry still receives its products in the host's order.
constexpr int kCapBig = 12288;
constexpr int kFillBig = kCapBig * 3 / 4;
constexpr int kBigThreads = 512;
constexpr size_t kSmemBig = size_t(kCapBig) * (sizeof(int) + sizeof(double));

__device__ __forceinline__ int hslot_big(int j) { return int((unsigned(j) * 2654435761u) % unsigned(kCapBig)); }

__device__ __forceinline__ int hinsert_big(int* keys, int j, int* count) {
  int s = hslot_big(j);
  for (int probe = 0; probe < kCapBig; ++probe) {
    const int prev = atomicCAS(keys + s, -1, j);
    if (prev == -1) {
      atomicAdd(count, 1);
      return s;
    }
    if (prev == j) return s;
    s = s + 1 == kCapBig ? 0 : s + 1;
  }
  return -1;
}

template <bool numeric>
__global__ void __launch_bounds__(kBigThreads) spgemm_big_rows(SpView A, SpView B, const double* row_scale,
                                                              const int* rows, int n_big, int* cnt,
                                                              const long long* crp, int* cci, double* cv) {
  extern __shared__ unsigned char smem[];
  __shared__ int count, full, base;
  int* keys = reinterpret_cast<int*>(smem);
  double* acc = reinterpret_cast<double*>(smem + size_t(kCapBig) * sizeof(int));
  for (int q = blockIdx.x; q < n_big; q += gridDim.x) {
    const int row = rows[q];
    for (int s = threadIdx.x; s < kCapBig; s += blockDim.x) {
      keys[s] = -1;
      if (numeric) acc[s] = 0.0;
    }
    if (threadIdx.x == 0) count = 0, full = 0;
    __syncthreads();
    const double sc = row_scale ? row_scale[row] : 1.0;
    bool overflow = false;
    for (long long ka = A.rp[row]; ka < A.rp[row + 1] && !overflow; ++ka) {
      const int k = A.ci[ka];
      const double av = row_scale ? A.v[ka] * sc : A.v[ka];
      for (long long kb = B.rp[k] + threadIdx.x; kb < B.rp[k + 1]; kb += blockDim.x) {
        const int s = hinsert_big(keys, B.ci[kb], &count);
        if (s < 0) {
          full = 1;
          continue;
        }
        if (numeric) acc[s] = acc[s] + av * B.v[kb];
      }
      __syncthreads();
      overflow = count > kFillBig || full;
      __syncthreads();
    }
    if (!numeric) {
      if (threadIdx.x == 0) cnt[row] = overflow ? -2 : count;
      __syncthreads();
      continue;
    }
    // compact used slots to the front in slot order (block-wide prefix over 512-slot chunks)
    __shared__ int chunk_base;
    if (threadIdx.x == 0) chunk_base = 0;
    __syncthreads();
    const int n = count;
    for (int s0 = 0; s0 < kCapBig; s0 += blockDim.x) {
      const int s = s0 + threadIdx.x;
      const bool has = s < kCapBig && keys[s] != -1;
      const int kk = has ? keys[s] : 0;
      const double vv = has ? acc[s] : 0.0;
      // block-wide exclusive rank of `has`
      __shared__ int warp_tot[kBigThreads / 32];
      const unsigned m = __ballot_sync(0xffffffffu, has);
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      if (lane == 0) warp_tot[w] = __popc(m);
      __syncthreads();
      int before = 0;
      for (int t = 0; t < w; ++t) before += warp_tot[t];
      int tot = 0;
      for (int t = 0; t < int(blockDim.x >> 5); ++t) tot += warp_tot[t];
      const int dst = chunk_base + before + __popc(m & ((1u << lane) - 1));
      __syncthreads();  // every thread has read its slot before any write below
      if (has) keys[dst] = kk, acc[dst] = vv;
      __syncthreads();
      if (threadIdx.x == 0) chunk_base += tot;
      __syncthreads();
    }
    int mm = 1;
    while (mm < n) mm <<= 1;
    for (int s = n + threadIdx.x; s < mm; s += blockDim.x) keys[s] = 0x7fffffff;
    __syncthreads();
    for (int size = 2; size <= mm; size <<= 1)  // bitonic sort by column (keys distinct)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < mm / 2; t += blockDim.x) {
          const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const int a = keys[lo], b = keys[hi];
          if ((a > b) == up) {
            keys[lo] = b, keys[hi] = a;
            const double x = acc[lo];
            acc[lo] = acc[hi], acc[hi] = x;
          }
        }
        __syncthreads();
      }
    const long long o = crp[row];
    for (int t = threadIdx.x; t < n; t += blockDim.x) cci[o + t] = keys[t], cv[o + t] = acc[t];
    __syncthreads();
    (void)base;
  }
}

__global__ void list_big_rows_kernel(int n, const int* cnt, int* rows, int* n_big) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && cnt[i] < 0) rows[atomicAdd(n_big, 1)] = int(i);
}

template <class T>
T* dev_copy(const std::vector<T>& h, std::vector<void*>& owned) {
  T* d = nullptr;
  if (h.empty()) return nullptr;
  cuda_check(cudaMalloc(&d, sizeof(T) * h.size()), "spgemm alloc");
  owned.push_back(d);
  cuda_check(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice), "spgemm upload");
  return d;
}

struct Owned {
  std::vector<void*> p;
  ~Owned() {
    for (void* q : p) cudaFree(q);
  }
};

}  // namespace

// C = diag(row_scale) A B on the device; bitwise fpb::spgemm.  Returns false (C untouched) when a row
// has more distinct columns than the per-warp hash holds.
bool spgemm_device(const fpb::Csr& A, const fpb::Csr& B, std::span<const double> row_scale, fpb::Csr& C) {
  if (A.n_cols != B.n_rows) throw std::invalid_argument("spgemm: dimension mismatch");
  Owned own;
  static bool attr = [] {
    cuda_check(cudaFuncSetAttribute(spgemm_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)),
               "spgemm smem");
    cuda_check(cudaFuncSetAttribute(spgemm_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)),
               "spgemm smem");
    return true;
  }();
  (void)attr;
  const int n = A.n_rows;
  C = fpb::Csr(n, B.n_cols);
  if (n == 0) return true;
  std::vector<long long> arp(A.rp.begin(), A.rp.end()), brp(B.rp.begin(), B.rp.end());
  const SpView dA{n, dev_copy(arp, own.p), dev_copy(A.ci, own.p), dev_copy(A.v, own.p)};
  const SpView dB{B.n_rows, dev_copy(brp, own.p), dev_copy(B.ci, own.p), dev_copy(B.v, own.p)};
  std::vector<double> scale(row_scale.begin(), row_scale.end());
  const double* dscale = row_scale.empty() ? nullptr : dev_copy(scale, own.p);
  int* dcnt = nullptr;
  cuda_check(cudaMalloc(&dcnt, sizeof(int) * size_t(n)), "spgemm alloc");
  own.p.push_back(dcnt);
  int dev = 0, sms = 148;
  cuda_check(cudaGetDevice(&dev), "device");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  const int grid = std::max(1, std::min((n + kWarps - 1) / kWarps, sms * 2));
  spgemm_rows<false><<<grid, kThreads, kSmem>>>(dA, dB, dscale, dcnt, nullptr, nullptr, nullptr);
  cuda_check(cudaGetLastError(), "spgemm symbolic");
  std::vector<int> cnt(static_cast<size_t>(n));
  cuda_check(cudaMemcpy(cnt.data(), dcnt, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost), "spgemm counts");
  for (int i = 0; i < n; ++i) {
    if (cnt[i] < 0) return false;
    C.rp[size_t(i) + 1] = C.rp[i] + cnt[i];
  }
  const int64_t nnz = C.rp[n];
  C.ci.resize(size_t(nnz));
  C.v.resize(size_t(nnz));
  std::vector<long long> crp(C.rp.begin(), C.rp.end());
  long long* dcrp = dev_copy(crp, own.p);
  int* dci = nullptr;
  double* dv = nullptr;
  if (nnz > 0) {
    cuda_check(cudaMalloc(&dci, sizeof(int) * size_t(nnz)), "spgemm alloc");
    own.p.push_back(dci);
    cuda_check(cudaMalloc(&dv, sizeof(double) * size_t(nnz)), "spgemm alloc");
    own.p.push_back(dv);
  }
  spgemm_rows<true><<<grid, kThreads, kSmem>>>(dA, dB, dscale, dcnt, dcrp, dci, dv);
  cuda_check(cudaGetLastError(), "spgemm numeric");
  if (nnz > 0) {
    cuda_check(cudaMemcpy(C.ci.data(), dci, sizeof(int) * size_t(nnz), cudaMemcpyDeviceToHost), "spgemm ci");
    cuda_check(cudaMemcpy(C.v.data(), dv, sizeof(double) * size_t(nnz), cudaMemcpyDeviceToHost), "spgemm v");
  }
  return true;
}

namespace {
__global__ void widen_counts_kernel(int n, const int* cnt, long long* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = cnt[i];
  if (i == n) out[i] = 0;
}
}  // namespace

// The same products with operands and result in HBM (the device setup, dsetup.cu).  A product with
// a row over the hash capacity (none on the BASELINE configs) runs on the host and is uploaded.
DCsr spgemm_dev(const DCsr& A, const DCsr& B, const double* row_scale_dev) {
  if (A.n_cols != B.n_rows) throw std::invalid_argument("spgemm: dimension mismatch");
  static bool attr = [] {
    cuda_check(cudaFuncSetAttribute(spgemm_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)),
               "spgemm smem");
    cuda_check(cudaFuncSetAttribute(spgemm_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)),
               "spgemm smem");
    return true;
  }();
  (void)attr;
  const int n = A.n_rows;
  DCsr C;
  C.n_rows = n, C.n_cols = B.n_cols;
  C.rp.alloc(size_t(n) + 1);
  if (n == 0) {
    C.rp.zero();
    return C;
  }
  const SpView dA{n, A.rp.get(), A.ci.get(), A.v.get()};
  const SpView dB{B.n_rows, B.rp.get(), B.ci.get(), B.v.get()};
  DevBuf<int> cnt(static_cast<size_t>(n));
  int dev = 0, sms = 148;
  cuda_check(cudaGetDevice(&dev), "device");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  const int grid = std::max(1, std::min((n + kWarps - 1) / kWarps, sms * 4));
  spgemm_rows<false><<<grid, kThreads, kSmem>>>(dA, dB, row_scale_dev, cnt.get(), nullptr, nullptr, nullptr);
  cuda_check(cudaGetLastError(), "spgemm symbolic");
  static bool attr_big = [] {
    cuda_check(cudaFuncSetAttribute(spgemm_big_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmemBig)), "spgemm big smem");
    cuda_check(cudaFuncSetAttribute(spgemm_big_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmemBig)), "spgemm big smem");
    return true;
  }();
  (void)attr_big;
  // rows over a warp's table: counted again by one CTA each
  DevBuf<int> big_rows(static_cast<size_t>(n)), n_big_d(1);
  n_big_d.zero();
  list_big_rows_kernel<<<unsigned((n + 255) / 256), 256>>>(n, cnt.get(), big_rows.get(), n_big_d.get());
  int n_big = 0;
  cuda_check(cudaMemcpy(&n_big, n_big_d.get(), sizeof(int), cudaMemcpyDeviceToHost), "big rows");
  const int grid_big = std::max(1, std::min(n_big, sms));
  if (n_big > 0)
    spgemm_big_rows<false><<<grid_big, kBigThreads, kSmemBig>>>(dA, dB, row_scale_dev, big_rows.get(), n_big,
                                                                 cnt.get(), nullptr, nullptr, nullptr);
  int mn = 0;
  {
    DevBuf<int> out(1);
    size_t tb = 0;
    cuda_check(cub::DeviceReduce::Min(nullptr, tb, cnt.get(), out.get(), n), "min size");
    DevBuf<unsigned char> tmp(tb);
    cuda_check(cub::DeviceReduce::Min(tmp.get(), tb, cnt.get(), out.get(), n), "min");
    cuda_check(cudaMemcpy(&mn, out.get(), sizeof(int), cudaMemcpyDeviceToHost), "min");
  }
  if (mn < 0) {  // a row over the block table too: the host routine
    const fpb::Csr hA = download_csr(A), hB = download_csr(B);
    std::vector<double> sc;
    if (row_scale_dev) {
      sc.resize(size_t(n));
      cuda_check(cudaMemcpy(sc.data(), row_scale_dev, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost), "scale");
    }
    return upload_csr(fpb::spgemm(hA, hB, sc));
  }
  DevBuf<long long> wide(size_t(n) + 1);
  widen_counts_kernel<<<unsigned((n + 256) / 256), 256>>>(n, cnt.get(), wide.get());
  size_t tb = 0;
  cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tb, wide.get(), C.rp.get(), n + 1), "scan size");
  {
    DevBuf<unsigned char> tmp(tb);
    cuda_check(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, wide.get(), C.rp.get(), n + 1), "scan");
  }
  long long nnz = 0;
  cuda_check(cudaMemcpy(&nnz, C.rp.get() + n, sizeof(long long), cudaMemcpyDeviceToHost), "nnz");
  C.nnz = nnz;
  C.ci.alloc(size_t(nnz));
  C.v.alloc(size_t(nnz));
  if (nnz > 0) {
    spgemm_rows<true><<<grid, kThreads, kSmem>>>(dA, dB, row_scale_dev, cnt.get(), C.rp.get(), C.ci.get(), C.v.get());
    if (n_big > 0)
      spgemm_big_rows<true><<<grid_big, kBigThreads, kSmemBig>>>(dA, dB, row_scale_dev, big_rows.get(), n_big,
                                                                  cnt.get(), C.rp.get(), C.ci.get(), C.v.get());
  }
  cuda_check(cudaDeviceSynchronize(), "spgemm numeric");
  return C;
}

}  // namespace fpd
