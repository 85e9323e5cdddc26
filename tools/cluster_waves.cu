// How many 2-CTA clusters of a 1-CTA-per-SM kernel (the pair forward's footprint) run at once
// on this GPU: cudaOccupancyMaxActiveClusters plus an empirical count of clusters that start
// in the first wave.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cw tools/cluster_waves.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) spin2(unsigned long long* t, int* sm) {
  extern __shared__ char s[];
  if (threadIdx.x == 0) {
    t[blockIdx.x] = gtime();
    int id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    sm[blockIdx.x] = id;
    s[0] = 1;
    const unsigned long long t0 = gtime();
    while (gtime() - t0 < 200000) {}
  }
  __syncthreads();
}
__global__ void __launch_bounds__(384, 1) spin1(unsigned long long* t, int* sm) {
  extern __shared__ char s[];
  if (threadIdx.x == 0) {
    t[blockIdx.x] = gtime();
    s[0] = 1;
    const unsigned long long t0 = gtime();
    while (gtime() - t0 < 200000) {}
  }
  __syncthreads();
}
int main() {
  const int smem = 200 * 1024, n = 512;
  cudaFuncSetAttribute(spin2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(spin1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = -1;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)spin2, &cfg);
  printf("cudaOccupancyMaxActiveClusters(2-CTA, 1 CTA/SM) = %d (%s)\n", ncl, cudaGetErrorString(e));
  unsigned long long* t; int* sm;
  cudaMalloc(&t, n * 8); cudaMalloc(&sm, n * 4);
  for (int k = 0; k < 2; ++k) {
    if (k == 0) spin2<<<n, 384, smem>>>(t, sm); else spin1<<<n, 384, smem>>>(t, sm);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(n);
    cudaMemcpy(h.data(), t, n * 8, cudaMemcpyDeviceToHost);
    const unsigned long long m = *std::min_element(h.begin(), h.end());
    int first = 0;
    for (auto x : h) first += (x - m) < 100000;    // started within 100 us of the first
    printf("%s: CTAs started in the first wave: %d of %d\n", k == 0 ? "clusters of 2" : "single CTAs", first, n);
  }
  return 0;
}
