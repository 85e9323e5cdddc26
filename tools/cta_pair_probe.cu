// Probe of CTA-pair (cta_group::2) tcgen05 semantics on B200, for the round-2 backward plan
// (DESIGN §12): a cluster of 2 CTAs allocates TMEM with cta_group::2; the leader issues one
// M = 256 (128 A rows per CTA) x N = 128 (64 B rows per CTA, same smem offset in both) x K = 128
// MMA and a multicast commit; then each CTA issues its own cta_group::1 M = 128 x N = 64 MMA into
// other TMEM columns.  Both results are checked exactly against the host (small integer data).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2505_16710_b200/csrc cta_pair_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace seco;

__device__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const float* A, const float* B, float* D2, float* D1, int* flags) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t r = cluster_rank();
  // A: own 128 rows x K=128, two K-major SW128 boxes of [128][128 B] (16 KiB each) at 0, 16 KiB
  // B: own 64 rows (pair N rows [64 r, 64 r + 64)) x K, two boxes of [64][128 B] at 32, 40 KiB
  for (int idx = threadIdx.x; idx < 128 * 128; idx += blockDim.x) {
    const int row = idx / 128, k = idx % 128;
    const uint32_t off = (k / 64) * 16384 + sw128_off(row, (k % 64) / 8) + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = __float2bfloat16(A[((int)r * 128 + row) * 128 + k]);
  }
  for (int idx = threadIdx.x; idx < 64 * 128; idx += blockDim.x) {
    const int row = idx / 128, k = idx % 128;
    const uint32_t off = 32768 + (k / 64) * 8192 + sw128_off(row, (k % 64) / 8) + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = __float2bfloat16(B[((int)r * 64 + row) * 128 + k]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) flags[r] = (int)(sb & 1023);
  if (r == 0 && threadIdx.x == 0) {
    constexpr uint32_t idesc2 = make_idesc_bf16(256, 128, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32, offB = 32768 + (kk / 4) * 8192 + (kk % 4) * 32;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(make_desc_sw128(sb + offA, 16, 1024)), "l"(make_desc_sw128(sb + offB, 16, 1024)), "r"(idesc2),
          "r"(kk > 0 ? 1 : 0)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  // per-CTA cta_group::1 MMA on the pair-allocated TMEM: D1 = A_own (128 x K) B_own^T (64 x K)
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc1 = make_idesc_bf16(128, 64, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32, offB = 32768 + (kk / 4) * 8192 + (kk % 4) * 32;
      mma_ss(tmem + 256, make_desc_sw128(sb + offA, 16, 1024), make_desc_sw128(sb + offB, 16, 1024), idesc1, kk > 0);
    }
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 1);
  tc_fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32, row = 32 * w + lane;
  const uint32_t la = (uint32_t)(32 * w) << 16;
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(tmem + la + 32 * c, v);
    tmem_wait_ld();
    for (int q = 0; q < 32; ++q) D2[((int)r * 128 + row) * 128 + 32 * c + q] = __uint_as_float(v[q]);
  }
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld32(tmem + la + 256 + 32 * c, v);
    tmem_wait_ld();
    for (int q = 0; q < 32; ++q) D1[((int)r * 128 + row) * 64 + 32 * c + q] = __uint_as_float(v[q]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
  std::vector<float> A(2 * 128 * 128), B(128 * 128);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 5 - 2);
  for (auto& x : B) x = (float)(rand() % 5 - 2);
  float *dA, *dB, *dD2, *dD1;
  int* dF;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD2, 2 * 128 * 128 * 4); cudaMalloc(&dD1, 2 * 128 * 64 * 4); cudaMalloc(&dF, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD2, 0xff, 2 * 128 * 128 * 4); cudaMemset(dD1, 0xff, 2 * 128 * 64 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<2, 128, 64 * 1024>>>(dA, dB, dD2, dD1, dF);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> D2(2 * 128 * 128), D1(2 * 128 * 64);
  int F[2];
  cudaMemcpy(D2.data(), dD2, D2.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(D1.data(), dD1, D1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(F, dF, 8, cudaMemcpyDeviceToHost);
  printf("smem misalignment (must be 0): %d %d\n", F[0], F[1]);
  // pair MMA: CTA r rows = A_r rows, N = 128 columns = B rows 0..127 (CTA 0 holds 0-63, CTA 1 64-127)
  int bad2 = 0, bad2_swapped = 0, bad1 = 0;
  for (int r = 0; r < 2; ++r)
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double s = 0, s_sw = 0;
        const int n_sw = (n + 64) % 128;
        for (int k = 0; k < 128; ++k) {
          s += (double)A[(r * 128 + m) * 128 + k] * B[n * 128 + k];
          s_sw += (double)A[(r * 128 + m) * 128 + k] * B[n_sw * 128 + k];
        }
        const float g = D2[(r * 128 + m) * 128 + n];
        bad2 += g != (float)s;
        bad2_swapped += g != (float)s_sw;
      }
  for (int r = 0; r < 2; ++r)
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        double s = 0;
        for (int k = 0; k < 128; ++k) s += (double)A[(r * 128 + m) * 128 + k] * B[(r * 64 + n) * 128 + k];
        bad1 += D1[(r * 128 + m) * 64 + n] != (float)s;
      }
  printf("cta_group::2 M256 N128 K128: %d mismatches (%d if the B halves were swapped) of %d\n", bad2, bad2_swapped,
         2 * 128 * 128);
  printf("cta_group::1 M128 N64 K128 on pair-allocated TMEM: %d mismatches of %d\n", bad1, 2 * 128 * 64);
  return (bad2 == 0 && bad1 == 0) ? 0 : 2;
}
