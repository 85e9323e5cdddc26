// Micro-benchmark: softmax-element throughput on one SM for MUFU ex2 vs the FMA-pipe
// polynomial (ex2_emu2) vs mixes.  Per element pair: FFMA2 (x*scale - max), exp2 x2,
// FADD2 (row sum), F2FP pack -- the forward softmax's inner loop without the max pass.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2505_16710_b200/csrc
#include <cstdio>

#include "common.cuh"

using namespace seco;

template <int EMU_OF_16>
__global__ void __launch_bounds__(512, 1) exp_rate(int reps, float* sink, unsigned long long* out) {
  f2_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = f2(-0.01f * i - threadIdx.x * 1e-4f, -0.02f * i);
  f2_t sum = f2(0.f, 0.f);
  uint32_t acc = 0;
  const f2_t sc = f2(0.5f, 0.5f), mx = f2(-1.0f, -1.0f);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const f2_t x = ffma2(v[i], sc, mx);
      f2_t e;
      if ((i % 16) < EMU_OF_16) e = ex2_emu2(x);
      else e = f2(ex2(f2lo(x)), ex2(f2hi(x)));
      sum = fadd2(sum, e);
      acc ^= pack_bf16_f2(e);
      v[i] = e;
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = f2lo(sum) + f2hi(sum);
}

template <int E>
static void run(int threads) {
  const int reps = 400;
  float* s; unsigned long long* d;
  cudaMalloc(&s, 4096); cudaMalloc(&d, 148 * 8);
  exp_rate<E><<<148, threads>>>(reps, s, d);
  exp_rate<E><<<148, threads>>>(reps, s, d);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double elems = (double)reps * 64 * threads;
  printf("emu %2d/16  threads %3d: %6.2f elements/clk/SM  (%s)\n", E, threads, elems / avg,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(s); cudaFree(d);
}

int main() {
  for (int t : {128, 256, 512}) {
    run<0>(t); run<2>(t); run<4>(t); run<6>(t); run<8>(t); run<16>(t);
  }
  return 0;
}
