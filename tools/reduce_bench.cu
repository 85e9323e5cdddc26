// Micro-benchmark: throughput of the fp32 reduce-add paths into an L2-resident buffer, as
// used by the backward's dQ drain.  Each CTA (one per SM, or fewer) repeatedly adds a 64 KiB
// smem tile into its own (or a shared) 64 KiB region of a 32 MiB fp32 buffer via
//   mode 0: cp.reduce.async.bulk (1-D bulk, one thread, 2 x 32 KiB per round)
//   mode 1: red.global.add.f32 from registers (all threads, coalesced 128 B per warp)
//   mode 2: red.global.add.v4.f32 from registers
// and reports bytes/clk/SM and total GB/s.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -I../paper_2505_16710_b200/csrc reduce_bench.cu -o reduce_bench
#include <cstdio>

#include "common.cuh"

using namespace seco;

__global__ void __launch_bounds__(512, 1) red_kernel(float* buf, int mode, int rounds, int stride_regions,
                                                     unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  fence_async_smem();
  __syncthreads();
  float* dst = buf + (size_t)(blockIdx.x % stride_regions) * 16384;
  const unsigned long long t0 = clock64();
  if (mode == 0) {
    if (threadIdx.x == 0) {
      for (int r = 0; r < rounds; ++r) {
        bulk_reduce_add_f32(dst, sb, 32768);
        bulk_commit();
        bulk_reduce_add_f32(dst + 8192, sb + 32768, 32768);
        bulk_commit();
        bulk_wait_read<2>();
      }
      bulk_wait0();
    }
  } else if (mode == 1) {
    for (int r = 0; r < rounds; ++r)
      for (int i = threadIdx.x; i < 16384; i += blockDim.x) red_add_f32(dst + i, 1.0f);
  } else {
    for (int r = 0; r < rounds; ++r)
      for (int i = threadIdx.x * 4; i < 16384; i += blockDim.x * 4) red_add_v4_f32(dst + i, 1.f, 1.f, 1.f, 1.f);
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  float* buf;
  unsigned long long* cyc;
  cudaMalloc(&buf, 32u << 20);
  cudaMalloc(&cyc, 148 * 8);
  cudaMemset(buf, 0, 32u << 20);
  cudaFuncSetAttribute(red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int rounds = 200;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int grid : {1, 16, 74, 148}) {
      red_kernel<<<grid, 512, 65536>>>(buf, mode, 4, 512, cyc);
      cudaEventRecord(e0);
      red_kernel<<<grid, 512, 65536>>>(buf, mode, rounds, 512, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[148];
      cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < grid; ++i) avg += h[i];
      avg /= grid;
      const double bytes = 65536.0 * rounds;
      printf("mode %d grid %3d: %6.1f B/clk/SM  total %7.0f GB/s  (%s)\n", mode, grid, bytes / avg,
             bytes * grid / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
