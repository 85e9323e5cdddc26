// Device-side helpers for sm_100a: mbarrier, TMA (cp.async.bulk[.tensor]),
// tcgen05 (TMEM alloc / MMA / ld / st / commit) and UMMA descriptors.
// Inline PTX only; no CUTLASS.  Bit layouts of the shared-memory matrix
// descriptor and of the kind::f16 instruction descriptor follow the sm_100
// tcgen05 ISA (descriptor "version 1").
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define SECO_DEV __device__ __forceinline__

// ---------------------------------------------------------------- SECO_CHECK builds
// compute-sanitizer is closed on this pool, so the bounds it would check are
// asserted in-kernel by a separate build (libseco_check.so: -DSECO_CHECK=1, see build.py):
// shared-memory operands and TMA destinations inside the CTA's shared window, tensor-memory
// columns inside the allocation and lanes inside the issuing warp's sub-partition, mbarrier
// alignment, TMA box coordinates inside the tensor, and plain global stores inside their
// buffers (call sites).  A failed check records its id (first failure) and a count in a
// per-translation-unit device word that the host reads through seco_debug_check_word(); the
// kernel carries on, so a failure is reported after the call instead of ending the context.
#ifdef SECO_CHECK
static __device__ unsigned int g_seco_check[2];     // [0] first failing check id, [1] count
#define SECO_CHECK_COND(cond, id)                                   \
  do {                                                              \
    if (!(cond)) {                                                  \
      atomicCAS(&g_seco_check[0], 0u, (unsigned)(id));              \
      atomicAdd(&g_seco_check[1], 1u);                              \
    }                                                               \
  } while (0)
// host: read and clear this translation unit's check word ((count << 32) | first id)
static inline unsigned long long seco_check_read_clear() {
  unsigned int w[2] = {0u, 0u}, z[2] = {0u, 0u};
  cudaMemcpyFromSymbol(w, g_seco_check, sizeof(w));
  cudaMemcpyToSymbol(g_seco_check, z, sizeof(z));
  return ((unsigned long long)w[1] << 32) | w[0];
}
#else
#define SECO_CHECK_COND(cond, id) \
  do {                            \
  } while (0)
static inline unsigned long long seco_check_read_clear() { return 0ull; }
#endif
// check ids: 1xx smem, 2xx tmem, 3xx mbarrier, 4xx TMA coordinates, 5xx global stores

namespace seco {

#ifdef SECO_CHECK
// end of this CTA's shared window: the dynamic block follows any static shared data, so its
// base (every extern __shared__ array aliases it) plus %dynamic_smem_size is the window's end
__device__ __forceinline__ uint32_t smem_window_end() {
  extern __shared__ __align__(16) uint8_t seco_check_dyn_smem[];
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  return static_cast<uint32_t>(__cvta_generic_to_shared(seco_check_dyn_smem)) + dyn;
}
#define SECO_CHECK_SMEM(addr, bytes, id) \
  SECO_CHECK_COND((uint64_t)(addr) + (uint64_t)(bytes) <= (uint64_t)::seco::smem_window_end(), id)
// TMEM address: lane in bits 31:16, column in 15:0; allocations here are at most 512 columns
// and a warp's tcgen05.ld / st reach only the 32 lanes of its sub-partition (warp id % 4)
#define SECO_CHECK_TMEM_COLS(taddr, ncols, id) SECO_CHECK_COND(((taddr) & 0xFFFFu) + (ncols) <= 512u, id)
#define SECO_CHECK_TMEM_WARP(taddr, id) \
  SECO_CHECK_COND(((taddr) >> 16) == 32u * ((threadIdx.x / 32u) % 4u), id)
#else
#define SECO_CHECK_SMEM(addr, bytes, id) SECO_CHECK_COND(true, id)
#define SECO_CHECK_TMEM_COLS(taddr, ncols, id) SECO_CHECK_COND(true, id)
#define SECO_CHECK_TMEM_WARP(taddr, id) SECO_CHECK_COND(true, id)
#endif

SECO_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
SECO_DEV void mbar_init(uint32_t bar, uint32_t count) {
  SECO_CHECK_COND((bar & 7u) == 0u, 301);
  SECO_CHECK_SMEM(bar, 8, 302);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
SECO_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
SECO_DEV void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
SECO_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  SECO_CHECK_SMEM(bar, 8, 303);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
#ifndef SECO_WAIT_HINT
#define SECO_WAIT_HINT 0
#endif
SECO_DEV bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
#if SECO_WAIT_HINT
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
#else
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
#endif
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "n"(0x989680)
      : "memory");
  return ok != 0;
}
SECO_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---------------------------------------------------------------- TMA / bulk copies
SECO_DEV void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 3-D maps have a {64, rows, 1} box of bf16 (rows = 128: 16 KiB; the pair forward's K halves use
// 64-row boxes) with the 128-B swizzle (1024-B aligned)
SECO_DEV void tma_load_3d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2,
                          uint32_t box_bytes = 16384) {
  SECO_CHECK_SMEM(dst, box_bytes, 101);
  SECO_CHECK_COND((dst & 1023u) == 0u, 102);
  SECO_CHECK_COND(c0 >= 0 && c1 >= 0 && c2 >= 0 && (c0 & 63) == 0, 401);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// ---------------------------------------------------------------- CTA pairs (cluster of 2)
// The pair forward (fwd_sm100.cu) issues tcgen05.mma.cta_group::2 from the leader
// (rank 0) on both CTAs' operands and TMEM; TMA loads of either CTA complete on the leader's
// barriers; the leader's commits arrive on both CTAs' barriers (multicast).
SECO_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared::cta offset in CTA `rank` of the cluster
SECO_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
SECO_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
SECO_DEV void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
SECO_DEV void mbar_expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cluster),
               "r"(bytes)
               : "memory");
}
// Cheap cross-CTA hand-off of shared-memory data (round 2): `.release.cluster` on an arrive and
// `.acquire.cluster` on a wait compile to MEMBAR.ALL.GPU (+ ERRBAR, CGAERRBAR) and CCTL.IVALL --
// ~1000 cycles per arrive while global traffic is in flight (tools/trace_lora.py).  When the data
// handed over lives in shared memory only, a fence restricted to shared memory (MEMBAR.ALL.CTA)
// before relaxed arrives, and a shared::cluster acquire fence after a relaxed wait, suffice.
SECO_DEV void fence_release_smem_cluster() {
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
}
SECO_DEV void fence_acquire_smem_cluster() {
  asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}
SECO_DEV void mbar_arrive_remote_relaxed(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// remote arrive with the default semantics (release at CTA scope: no memory fence in SASS), for
// hand-offs ordered by other means (tcgen05 fences for TMEM, as CUTLASS's cluster pipelines do)
SECO_DEV void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
SECO_DEV bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
SECO_DEV void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
// TMA load into this CTA's smem whose completion is counted on a barrier of either CTA of the pair
SECO_DEV void tma_load_3d_pair(uint32_t dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1, int c2,
                               uint32_t box_bytes) {
  SECO_CHECK_SMEM(dst, box_bytes, 108);
  SECO_CHECK_COND((dst & 1023u) == 0u, 109);
  SECO_CHECK_COND(c0 >= 0 && c1 >= 0 && c2 >= 0 && (c0 & 63) == 0, 402);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes.cta_group::2"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

SECO_DEV void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  SECO_CHECK_SMEM(dst, bytes, 103);
  SECO_CHECK_COND((dst & 15u) == 0u && (bytes & 15u) == 0u, 104);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operands)
SECO_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------- tcgen05
template <int NCOLS>
SECO_DEV void tmem_alloc(uint32_t dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
SECO_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}
template <int NCOLS>
SECO_DEV void tmem_alloc_pair(uint32_t dst_smem) {  // whole warp, in both CTAs of the pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int NCOLS>
SECO_DEV void tmem_dealloc_pair(uint32_t taddr) {  // whole warp, in both CTAs of the pair
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
// true in exactly one (the same) lane of a converged warp
SECO_DEV bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
SECO_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SECO_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem desc] * B[smem desc]^T  (kind::f16, fp32 accumulate)
// descriptor start address (bits 13:0, units of 16 B): an operand tile of up to 32 KiB in the window
#define SECO_CHECK_DESC(desc, id) SECO_CHECK_SMEM(((uint32_t)(desc) & 0x3FFFu) << 4, 16 * 128, id)
SECO_DEV void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  SECO_CHECK_TMEM_COLS(d_tmem, (idesc >> 17 & 0x3Fu) << 3, 201);
  SECO_CHECK_COND((d_tmem >> 16) == 0u, 202);
  SECO_CHECK_DESC(a_desc, 105);
  SECO_CHECK_DESC(b_desc, 106);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]^T  (A in tensor memory: lane = row, 2 bf16 per column)
SECO_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  SECO_CHECK_TMEM_COLS(d_tmem, (idesc >> 17 & 0x3Fu) << 3, 203);
  SECO_CHECK_TMEM_COLS(a_tmem, 8, 204);
  SECO_CHECK_COND((d_tmem >> 16) == 0u && (a_tmem >> 16) == 0u, 205);
  SECO_CHECK_DESC(b_desc, 107);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// pair MMAs (issued by the leader CTA only): M = 256 rows, 128 from each CTA's A operand (smem
// descriptor or TMEM at the same address in both), B's N columns split between the two CTAs'
// smem at the same offset; D lands in each CTA's TMEM (its own 128 rows, all N columns)
SECO_DEV void mma_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  SECO_CHECK_TMEM_COLS(d_tmem, (idesc >> 17 & 0x3Fu) << 3, 206);
  SECO_CHECK_DESC(a_desc, 110);
  SECO_CHECK_DESC(b_desc, 111);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
SECO_DEV void mma_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  SECO_CHECK_TMEM_COLS(d_tmem, (idesc >> 17 & 0x3Fu) << 3, 207);
  SECO_CHECK_TMEM_COLS(a_tmem, 8, 208);
  SECO_CHECK_DESC(b_desc, 112);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// arrive on the barrier at this offset in both CTAs of the pair once the leader's MMAs complete
SECO_DEV void mma_commit_pair(uint32_t bar) {
  SECO_CHECK_SMEM(bar, 8, 305);
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

// arrive (once) on an mbarrier when all previously issued tcgen05.mma of this thread complete
SECO_DEV void mma_commit(uint32_t bar) {
  SECO_CHECK_SMEM(bar, 8, 304);
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

#define SECO_R32(a) \
  "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]), \
  "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), \
  "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), \
  "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define SECO_W32(a) \
  "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), \
  "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]), \
  "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]), \
  "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])

// 32 consecutive fp32 columns of this thread's TMEM lane (warp w reads lanes 32*(w%4)..+31)
SECO_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  SECO_CHECK_TMEM_COLS(taddr, 32u, 210);
  SECO_CHECK_TMEM_WARP(taddr, 211);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
      "[%32];"
      : SECO_R32(r)
      : "r"(taddr));
}
SECO_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  SECO_CHECK_TMEM_COLS(taddr, 32u, 212);
  SECO_CHECK_TMEM_WARP(taddr, 213);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
      "%32};" ::"r"(taddr),
      SECO_W32(r)
      : "memory");
}
SECO_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  SECO_CHECK_TMEM_COLS(taddr, 16u, 214);
  SECO_CHECK_TMEM_WARP(taddr, 215);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
SECO_DEV void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  SECO_CHECK_TMEM_COLS(taddr, 8u, 216);
  SECO_CHECK_TMEM_WARP(taddr, 217);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
SECO_DEV void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  SECO_CHECK_TMEM_COLS(taddr, 8u, 218);
  SECO_CHECK_TMEM_WARP(taddr, 219);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
SECO_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  SECO_CHECK_TMEM_COLS(taddr, 16u, 220);
  SECO_CHECK_TMEM_WARP(taddr, 221);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
SECO_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
SECO_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), version 1.
//   K-major operand: rows of 128 B (64 bf16 of K), 8-row atoms 1024 B apart (SBO);
//                    LBO unused (1).  K step of 16 elements = +32 B on the start address.
//   MN-major operand: 128-B rows are K indices holding 64 MN-contiguous elements;
//                    LBO = byte distance between 64-element MN blocks, SBO = 1024 B
//                    between 8-row K groups.  K step of 16 = +2048 B.
SECO_DEV uint64_t make_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, M x N, operand majors (0 = K, 1 = MN)
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                          // D format f32
         | (1u << 7)                        // A bf16
         | (1u << 10)                       // B bf16
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// 128B-swizzled byte offset of 16-byte chunk `c` (0..7) in row `r` of a [rows][128 B] tile
SECO_DEV uint32_t sw128_off(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }

SECO_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
SECO_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
SECO_DEV void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
SECO_DEV void red_add_v4_f32(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
SECO_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SECO_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
SECO_DEV void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// per-warpgroup register budget (all 4 warps of the warpgroup must execute it)
template <int N>
SECO_DEV void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
SECO_DEV void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
SECO_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// ---------------------------------------------------------------- packed fp32 pairs (FFMA2 / FADD2 / FMUL2)
typedef uint64_t f2_t;
SECO_DEV f2_t f2(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
SECO_DEV f2_t f2u(uint32_t lo, uint32_t hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
SECO_DEV float f2lo(f2_t v) { return __uint_as_float((uint32_t)v); }
SECO_DEV float f2hi(f2_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
SECO_DEV f2_t ffma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
SECO_DEV f2_t fadd2(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
SECO_DEV f2_t fsub2(f2_t a, f2_t b) {
  f2_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
SECO_DEV f2_t fmul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a pair on the FMA pipe (offloads the MUFU unit): Cody-Waite split x = j + f,
// j = rint(x) via the 1.5*2^23 shifter, f in [-0.5, 0.5], 2^f by a degree-3 polynomial at
// Chebyshev nodes (max rel. error 1.0e-4, far below bf16's 3.9e-3), then j added to the
// exponent field.  x is clamped to >= -127 (the result underflows to ~0 there).
SECO_DEV f2_t ex2_emu2(f2_t x) {
  const f2_t xc = f2(fmaxf(f2lo(x), -127.f), fmaxf(f2hi(x), -127.f));
  const f2_t magic = f2(12582912.f, 12582912.f);
  const f2_t y = fadd2(xc, magic);
  const f2_t f = fsub2(xc, fsub2(y, magic));
  f2_t p = ffma2(f2(0.05583828315138817f, 0.05583828315138817f), f, f2(0.2426394820213318f, 0.2426394820213318f));
  p = ffma2(p, f, f2(0.6931367516517639f, 0.6931367516517639f));
  p = ffma2(p, f, f2(0.9999245405197144f, 0.9999245405197144f));
  const uint32_t r0 = (uint32_t)p + ((uint32_t)y << 23);
  const uint32_t r1 = (uint32_t)(p >> 32) + ((uint32_t)(y >> 32) << 23);
  return f2u(r0, r1);
}
// bf16x2 pack of a pair (lo in the low half)
SECO_DEV uint32_t pack_bf16_f2(f2_t v) { return pack_bf16(f2lo(v), f2hi(v)); }

// ---------------------------------------------------------------- TMA reduce-add (smem -> global, fp32)
SECO_DEV void tma_reduce_add_2d(const CUtensorMap* m, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
// 1-D bulk reduce-add (smem -> global, fp32), size multiple of 16 B
SECO_DEV void bulk_reduce_add_f32(float* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}
template <int N>
SECO_DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
SECO_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SECO_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SECO_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// relaxed (L1-bypassing, no cache invalidation) poll; pair with fence_acq_rel_gpu() once the
// awaited value is seen -- an ld.acquire in a spin loop invalidates L1 (CCTL.IVALL) per probe
SECO_DEV int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SECO_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
SECO_DEV void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SECO_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SECO_DEV float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
SECO_DEV float ld_shared_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
SECO_DEV void st_shared_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

}  // namespace seco
