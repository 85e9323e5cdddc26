// Micro-benchmark: hand-off latency between warps of one CTA -- the time from a producer's
// arrival (clock64 just before it) to a waiting consumer's wake-up (clock64 just after), for
//   mode 0: consumer lane 0 loops on mbarrier.try_wait (producer: mbarrier.arrive)
//   mode 1: consumer lane 0 loops on mbarrier.test_wait
//   mode 2: named barrier: producer bar.arrive, whole consumer warp bar.sync
// The producer warp waits a random-ish delay before each arrival so the consumer is asleep.
#include <cstdio>

#include "common.cuh"

namespace seco {
SECO_DEV bool mbar_test_wait_(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
}  // namespace seco

using namespace seco;

__global__ void __launch_bounds__(128, 1) wake(int mode, int iters, long long* out) {
  __shared__ uint64_t bar;
  __shared__ long long t_arr[64], t_wake[64];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  __syncthreads();
  for (int i = 0; i < iters; ++i) {
    if (warp == 1) {                                    // producer
      const long long t0 = clock64();
      while (clock64() - t0 < 2000 + (i * 37) % 500) {
      }
      __syncwarp();
      if (mode == 2) {
        if (lane == 0) t_arr[i] = clock64();
        __syncwarp();
        asm volatile("bar.arrive 1, 64;" ::: "memory");
      } else if (lane == 0) {
        t_arr[i] = clock64();
        mbar_arrive(smem_u32(&bar));
      }
    } else if (warp == 0) {                              // consumer
      if (mode == 2) {
        asm volatile("bar.sync 1, 64;" ::: "memory");
        if (lane == 0) t_wake[i] = clock64();
      } else if (lane == 0) {
        if (mode == 0) mbar_wait(smem_u32(&bar), i & 1);
        else while (!mbar_test_wait_(smem_u32(&bar), i & 1)) {}
        t_wake[i] = clock64();
      }
      __syncwarp();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    long long s = 0, mx = 0;
    for (int i = 4; i < iters; ++i) { const long long d = t_wake[i] - t_arr[i]; s += d; mx = d > mx ? d : mx; }
    out[0] = s / (iters - 4);
    out[1] = mx;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int mode = 0; mode < 3; ++mode) {
    wake<<<1, 128>>>(mode, 64, d);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): mean %lld cycles, max %lld  (%s)\n", mode,
           mode == 0 ? "mbarrier try_wait" : mode == 1 ? "mbarrier test_wait spin" : "bar.arrive / bar.sync",
           h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
