// Micro-benchmark of tcgen05.mma issue rates on B200 (one CTA per SM, one issuing thread):
// cycles per kind::f16 MMA instruction (K = 16) for SS (A, B in smem) and TS (A in TMEM)
// at M = 128 and several N.  Operands are zero-filled 128B-swizzled tiles; results are not
// checked.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2505_16710_b200/csrc
#include <cstdio>

#include "common.cuh"

using namespace seco;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        if (TS)
          mma_ts(tmem + 256, tmem + kk * 8, make_desc_sw128(sb + 32768 + off, 16, 1024), idesc, kk > 0);
        else
          mma_ss(tmem + 256, make_desc_sw128(sb + off, 16, 1024), make_desc_sw128(sb + 32768 + off, 16, 1024),
                 idesc, kk > 0);
      }
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
static void run(const char* name, int reps) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  mma_rate<N, TS><<<148, 128, 100 * 1024>>>(reps, d);
  mma_rate<N, TS><<<148, 128, 100 * 1024>>>(reps, d);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (reps * 8.0);
  printf("%-18s N=%3d: %7.1f cycles per MMA (ideal %5.1f at 8192 flop/clk/SM)  err=%s\n", name, N, per,
         128.0 * N * 16 * 2 / 8192.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  const int reps = 2000;
  run<64, false>("SS M128", reps);
  run<128, false>("SS M128", reps);
  run<256, false>("SS M128", reps);
  run<64, true>("TS M128", reps);
  run<128, true>("TS M128", reps);
  run<256, true>("TS M128", reps);
  return 0;
}
