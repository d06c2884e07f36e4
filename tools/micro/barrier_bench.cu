// Microbenchmark: cost of one grid-wide barrier on B200 (148 CTAs): cooperative_groups
// grid.sync() vs cluster barrier only vs a two-level barrier (cluster barrier + one
// global atomic per cluster + cluster barrier).   nvcc -arch=sm_100a -O3 barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_grid(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) k_cluster(int iters, double* out) {
  cg::cluster_group c = cg::this_cluster();
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; c.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) k_two_level(int iters, unsigned* counter, double* out) {
  cg::cluster_group c = cg::this_cluster();
  const unsigned nclusters = gridDim.x / 8;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    c.sync();
    if (c.block_rank() == 0 && threadIdx.x == 0) {
      const unsigned target = nclusters * (i + 1);
      atomicAdd(counter, 1u);
      for (long long spin = 0; atomicAdd(counter, 0u) < target; ++spin)
        if (spin > (1LL << 24)) { out[1] = -1.0; break; }  // never hang the device
    }
    c.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; unsigned* counter; cudaMalloc(&out, 16); cudaMalloc(&counter, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2000; float ms;
  int grid = sms; void* args[] = {(void*)&iters, (void*)&out};
  cudaLaunchCooperativeKernel((void*)k_grid, grid, 512, args); cudaDeviceSynchronize();
  cudaEventRecord(a); cudaLaunchCooperativeKernel((void*)k_grid, grid, 512, args); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("grid.sync   %d CTAs: %.3f us per barrier (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  int ncl = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(144), cfg.blockDim = dim3(512);
    cudaOccupancyMaxActiveClusters(&ncl, (void*)k_two_level, &cfg);
  }
  const int cgrid = 8 * (ncl < 18 ? ncl : 18);  // only co-resident clusters (the two-level barrier spins)
  printf("co-resident clusters of 8: %d\n", ncl);
  k_cluster<<<cgrid, 512>>>(iters, out); cudaDeviceSynchronize();
  cudaEventRecord(a); k_cluster<<<cgrid, 512>>>(iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("cluster.sync (8) : %.3f us per barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  cudaMemset(counter, 0, 4);
  k_two_level<<<cgrid, 512>>>(iters, counter, out); cudaDeviceSynchronize();
  cudaMemset(counter, 0, 4);
  cudaEventRecord(a); k_two_level<<<cgrid, 512>>>(iters, counter, out); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("two-level (18 clusters x 8): %.3f us per barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
