// Streaming-read microbenchmark (LoRA design question, round 2): per-SM read throughput of
// (a) 1-D bulk copies (cp.async.bulk, TMA engine) of B bytes into a STAGES-deep smem ring and
// (b) 16-B vector loads (ld.global.v4) by W warps, over a 64 MiB buffer, 148 CTAs (one per SM).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* src, size_t per_cta, int bytes, int stages, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[32];
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const int n = (int)(per_cta / bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long acc = 0;
  auto issue = [&](int i) {
    const int s = i % stages;
    const uint32_t bar = smem_u32(&bars[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem + (size_t)s * bytes)),
                 "l"(base + (size_t)i * bytes), "r"(bytes), "r"(bar)
                 : "memory");
  };
  for (int i = 0; i < stages && i < n; ++i) issue(i);
  for (int i = 0; i < n; ++i) {
    const int s = i % stages;
    const uint32_t bar = smem_u32(&bars[s]);
    const uint32_t par = (i / stages) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    acc += smem[(size_t)s * bytes];
    if (i + stages < n) issue(i + stages);
  }
  if (acc == 12345) *sink = acc;
}

__global__ void ldg_kernel(const uint4* src, size_t per_cta, int unroll, unsigned long long* sink) {
  const uint4* base = src + (size_t)blockIdx.x * (per_cta / 16);
  const size_t n = per_cta / 16;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < n; i += (size_t)blockDim.x * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = i + u * blockDim.x < n ? __ldcs(base + i + u * blockDim.x) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 12345) *sink = acc;
}

int main(int argc, char** argv) {
  const size_t total = (argc > 1 ? (size_t)atoll(argv[1]) : 64ull) << 20;
  const int nsm = 148;
  const size_t per_cta = total / nsm / 65536 * 65536;
  uint8_t* buf; unsigned long long* sink;
  cudaMalloc(&buf, total + (1 << 20)); cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, total);
  uint8_t* flush; cudaMalloc(&flush, 256ull << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(flush, r, 256ull << 20);
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < best) best = ms;
    }
    const double bytes = (double)per_cta * nsm;
    printf("%5zu MiB %-34s %8.1f us  %7.0f GB/s  (%5.1f GB/s per SM)  err=%s\n", total >> 20, name, best * 1e3, bytes / best / 1e6,
           bytes / best / 1e6 / nsm, cudaGetErrorString(cudaGetLastError()));
  };
  const bool brief = argc > 2;
  for (int bytes : {1024, 2048, 4096, 8192, 16384, 32768}) {
    if (brief && bytes != 16384) continue;
    for (int stages : {4, 8, 16}) {
      if (brief && stages != 8) continue;
      if ((size_t)bytes * stages > 196 * 1024) continue;
      char nm[64]; snprintf(nm, 64, "bulk %6d B x %2d stages", bytes, stages);
      run(nm, [&] { bulk_kernel<<<nsm, 32, (size_t)bytes * stages>>>(buf, per_cta, bytes, stages, sink); });
    }
  }
  for (int threads : {128, 256, 512, 1024}) {
    if (brief && threads != 1024) continue;
    char nm[64]; snprintf(nm, 64, "ldg.v4 x8 %4d threads", threads);
    run(nm, [&] { ldg_kernel<<<nsm, threads>>>((const uint4*)buf, per_cta, 8, sink); });
  }
  return 0;
}
