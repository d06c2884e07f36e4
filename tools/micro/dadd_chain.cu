// Latency of a dependent fp64 add chain (the floor of an ordered row sum) and of
// the same chain fed from shared memory, on one warp.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -fmad=false dadd_chain.cu -o dadd_chain
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_reg(int n, double seed, double* out, long long* cyc) {
  double s = 0.0, t = seed;
  long long c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < n; ++k) s = s + t;
  long long c1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

__global__ void chain_smem(int n, double* out, long long* cyc) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 1e-3 * i;
  __syncthreads();
  double s = 0.0;
  long long c0 = clock64();
  for (int k = 0; k < n; k += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = buf[(k + u) & 4095];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = s + t[u];
  }
  long long c1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

// software-pipelined: the next 8 values are loaded while the current 8 are added
__global__ void chain_smem_pipe(int n, double* out, long long* cyc) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 1e-3 * i;
  __syncthreads();
  double s = 0.0, a[8], b[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = buf[u];
  long long c0 = clock64();
  for (int k = 0; k < n; k += 16) {
#pragma unroll
    for (int u = 0; u < 8; ++u) b[u] = buf[(k + 8 + u) & 4095];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = s + a[u];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = buf[(k + 16 + u) & 4095];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = s + b[u];
  }
  long long c1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, sizeof(long long));
  const int n = 1 << 16;
  for (int rep = 0; rep < 2; ++rep) {
    chain_reg<<<1, 32>>>(n, 1e-7, out, cyc);
    cudaDeviceSynchronize();
    printf("register chain: %.2f cycles per dependent DADD\n", double(*cyc) / n);
    chain_smem<<<1, 32>>>(n, out, cyc);
    cudaDeviceSynchronize();
    printf("smem batched-8 chain: %.2f cycles per add\n", double(*cyc) / n);
    chain_smem_pipe<<<1, 32>>>(n, out, cyc);
    cudaDeviceSynchronize();
    printf("smem pipelined chain: %.2f cycles per add\n", double(*cyc) / n);
  }
  return 0;
}
