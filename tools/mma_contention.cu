// Micro-benchmark: tcgen05.mma (kind::f16, M128, SS N=128 or TS N=128) issue rate on one SM while
// other warps of the CTA generate (mode 1) tcgen05.ld traffic from another TMEM region, (mode 2)
// st.shared traffic, (mode 3) both -- the in-situ conditions of the forward / backward kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2505_16710_b200/csrc
#include <cstdio>

#include "common.cuh"

using namespace seco;

template <bool TS>
__global__ void __launch_bounds__(384, 1) contention(int reps, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); stop = 0; }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0, TS ? 1 : 0);
      const unsigned long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (TS)
            mma_ts(tmem + 256, tmem + kk * 8, make_desc_sw128(sb + 32768 + kk * 2048, 16384, 1024), idesc, kk > 0);
          else
            mma_ss(tmem + 256, make_desc_sw128(sb + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                   make_desc_sw128(sb + 32768 + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024), idesc, kk > 0);
        }
      }
      mma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      out[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (warp >= 4) {
    const int wq = warp % 4;
    const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
    uint32_t acc = 0;
    int it = 0;
    while (!stop) {
      if (mode & 1) {                  // tcgen05.ld of 32 columns in [384, 512)
        uint32_t v[32];
        tmem_ld32(tmem + lane_addr + 384 + 32 * (it & 3), v);
        tmem_wait_ld();
        acc ^= v[lane & 31];
      }
      if (mode & 2) {                  // 4 x 16-B st.shared per thread into [64 KiB, 160 KiB)
        const uint32_t base = sb + 65536 + (uint32_t)((threadIdx.x * 16 + it * 4096) % (96 * 1024 - 64));
#pragma unroll
        for (int q = 0; q < 4; ++q) st_shared_v4(base + q * 16 % 4096, acc, it, q, lane);
      }
      ++it;
    }
    if (acc == 0xdeadbeef) out[1000] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <bool TS>
static void run(const char* name, int mode) {
  unsigned long long* d;
  cudaMalloc(&d, 2048 * sizeof(unsigned long long));
  auto k = contention<TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int reps = 2000;
  k<<<148, 384, 160 * 1024>>>(reps, mode, d);
  k<<<148, 384, 160 * 1024>>>(reps, mode, d);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%s mode %d (%s): %6.1f cycles per MMA  (%s)\n", name, mode,
         mode == 0 ? "alone" : mode == 1 ? "+tcgen05.ld" : mode == 2 ? "+st.shared" : "+both", avg / (reps * 8.0),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int m = 0; m < 4; ++m) run<false>("SS M128N128", m);
  for (int m = 0; m < 4; ++m) run<true>("TS M128N128", m);
  return 0;
}
