// Chunk-local backward on sm_100a tensor cores (Alg. 1 lines 6-7 P:200-201):
// for chunk j, gradients w.r.t. Q_j and w.r.t. every K/V row of cache slots 0..j,
// the latter accumulated in place into the persistent fp32 checkpoint-gradient
// buffer dkv (the requires_grad leaves of App. C.1).
//
// KV-stationary: one CTA owns a 128-key tile of kv-head g (keys [k0, k0+128) in slot
// k0/c <= j) and loops over query tiles of 64 rows of the G q-heads of group g that
// can see those keys (optionally a contiguous share of them: Q-split).  Per query
// tile (5 tcgen05 MMAs, all M = 128, fp32 accumulators in TMEM):
//   S^T  = K Q^T          [128 keys x 64 q]   SS, both K-major
//   dP^T = V dO^T         [128 x 64]
//   P^T  = exp2(S^T sigma log2e - LSE log2e), dS^T = P^T o (dP^T - D)   (CUDA cores, -> smem bf16)
//   dV  += P^T dO         [128 keys x d]      A K-major (smem), B MN-major
//   dK  += dS^T Q         [128 keys x d]
//   dQ^T = K^T dS^T       [d x 64 q]          A and B MN-major; -> smem -> TMA reduce-add into fp32 dQacc
// Warp roles: w0 TMA producer (K,V once; Q,dO,LSE,D per tile through a ring),
// w1 MMA issuer, w2 TMEM allocator, w4-w11 two compute warpgroups (thread = key row,
// 32 query columns each), w12-w15 dQ drain (thread = head-dim lane).
// MMA issue order per tile i: [S^T, dP^T](i+1) -> dV(i), dK(i) -> dQ^T(i), so the
// elementwise work of tile i+1 overlaps the tensor-core work of tile i.
// TMEM columns: S^T [0,64) dP^T [64,128) dQ^T x2 [128,256) dK [256,384) dV [384,512).
// dK/dV leave TMEM once per CTA, scaled (s*sigma, s), through 128B-swizzled smem staging and
// TMA tensor reduce-add (cp.reduce.async.bulk.tensor ... .add) into dkv (slot j was pre-scaled
// by the relay factor gamma in bwd_prep).  All fp32 reductions run in L2, issued by the TMA
// unit, so no thread issues per-element atomics.
#include "common.cuh"
#include "kernels.h"

namespace seco {

#ifdef SECO_TRACE
unsigned long long* seco_trace_buffer = nullptr;
extern "C" void* seco_debug_trace_ptr() { return seco_trace_buffer; }
#endif

cudaError_t launch_prep_bf16(const ChunkGeom& g, const void* o, const void* d_o, float* D, float* dkv,
                             float* dqacc, const float* lse, float* nlse, float relay, cudaStream_t st);
cudaError_t launch_final_bf16(const ChunkGeom& g, const float* dqacc, void* dq, const float* dkv, void* dk_own,
                              void* dv_own, float dq_scale, cudaStream_t st);

namespace bwd {
constexpr int BKV = 128;  // keys per CTA tile (UMMA M)
constexpr int BQ = 64;    // query rows per iteration (UMMA N of S^T / dP^T / dQ^T)
constexpr int D = 128;    // head dim (this kernel)
constexpr int STAGES = 2;
constexpr int kKVBytes = BKV * D * 2;      // K or V tile: 2 boxes [128][128 B]
constexpr int kQBytes = BQ * D * 2;        // Q or dO tile: 2 boxes [64][128 B]
constexpr int kPBytes = BKV * BQ * 2;      // P^T or dS^T: 1 box [128][128 B]
constexpr int kK = 0;
constexpr int kV = kK + kKVBytes;
constexpr int kQ = kV + kKVBytes;                       // [STAGES] Q tiles
constexpr int kDO = kQ + STAGES * kQBytes;              // [STAGES] dO tiles
constexpr int kP = kDO + STAGES * kQBytes;              // [2] P^T
constexpr int kDS = kP + 2 * kPBytes;                   // [2] dS^T
constexpr int kDQ = kDS + 2 * kPBytes;                  // dQ staging: 4 boxes [64 q][32 fp32] (128B swizzle)
constexpr int kDQBytes = BQ * D * 4;
constexpr int kStats = kDQ + kDQBytes;                  // [STAGES][2][BQ] fp32 (LSE, D)
constexpr int kBar = kStats + STAGES * 2 * BQ * 4;
// bars: kv, q_full[ST], q_empty[ST], s_full, ds_ready, dq_full[2], dq_empty[2], acc_full
constexpr int kNumBars = 1 + 2 * STAGES + 1 + 1 + 2 + 2 + 1;
constexpr int kTmemSlot = kBar + 8 * kNumBars;
constexpr int kBytes = kTmemSlot + 16;
constexpr int kAlloc = kBytes + 1024;
constexpr int kThreads = 512;
constexpr int TM_S = 0, TM_DP = 64, TM_DQ = 128, TM_DK = 256, TM_DV = 384;

struct Args {
  int c, j, G, hkv, S;
  int nsplit;
  float scale_log2;   // sigma * log2 e
  float dk_scale;     // s * sigma
  float dv_scale;     // s
  const float* nlse;  // [hq][c]  -LSE * log2(e)   (from bwd_prep)
  const float* Dv;    // [hq][c]  rowsum(dO o O)  (from bwd_prep)
  unsigned long long* trace;  // SECO_TRACE builds only: [kTraceCtas][kTraceSlots][kTraceIters] clock64 stamps
};
constexpr int kTraceCtas = 4, kTraceSlots = 10, kTraceIters = 128;
}  // namespace bwd

__global__ void __launch_bounds__(bwd::kThreads, 1)
    seco_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv,
                          const bwd::Args a) {
  using namespace bwd;
  constexpr int BOX_KV = 128 * 128;  // [128 rows][128 B]
  constexpr int BOX_Q = 64 * 128;    // [64 rows][128 B]
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t sK = sb + kK, sV = sb + kV, sQ = sb + kQ, sDO = sb + kDO, sP = sb + kP, sDS = sb + kDS;
  const uint32_t sDQ = sb + kDQ;
  const uint32_t sStats = sb + kStats;
  const uint32_t b0 = sb + kBar;
  const uint32_t bar_kv = b0;
  auto bar_q_full = [&](int s) { return b0 + 8u * (1 + s); };
  auto bar_q_empty = [&](int s) { return b0 + 8u * (1 + STAGES + s); };
  const uint32_t bar_s_full = b0 + 8u * (1 + 2 * STAGES);
  const uint32_t bar_ds_ready = b0 + 8u * (2 + 2 * STAGES);
  auto bar_dq_full = [&](int q) { return b0 + 8u * (3 + 2 * STAGES + q); };
  auto bar_dq_empty = [&](int q) { return b0 + 8u * (5 + 2 * STAGES + q); };
  const uint32_t bar_acc = b0 + 8u * (7 + 2 * STAGES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kTmemSlot);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#ifdef SECO_TRACE
#define TRACE(slot, i)                                                                                      \
  do {                                                                                                      \
    if (a.trace && blockIdx.x < kTraceCtas && (i) < kTraceIters)                                            \
      a.trace[((size_t)blockIdx.x * kTraceSlots + (slot)) * kTraceIters + (i)] = clock64();                \
  } while (0)
#else
#define TRACE(slot, i) do { } while (0)
#endif
  // block -> (key tile u, split s, kv head g); key tiles in ascending order = longest work first
  const int bid = blockIdx.x;
  const int g = bid % a.hkv;
  const int split = (bid / a.hkv) % a.nsplit;
  const int u = bid / (a.hkv * a.nsplit);
  const int k0 = u * BKV;                                  // first key (absolute position)
  const int nqt = a.c / BQ;
  const int rel = k0 - a.j * a.c;                          // key offset relative to chunk j's first row
  const int qt_min = rel > 0 ? rel / BQ : 0;              // first query tile that sees key k0
  const int n_all = a.G * (nqt - qt_min);
  const int it0 = (int)((int64_t)split * n_all / a.nsplit);
  const int it1 = (int)((int64_t)(split + 1) * n_all / a.nsplit);
  const int n = it1 - it0;
  // iteration i (0-based within this CTA) -> (q-head, query tile): it = it0 + i,
  // head = g*G + it % G, tile = qt_min + it / G; each role walks it incrementally
  struct Walk {
    int hh, qt, G;
    __device__ void next() { if (++hh == G) { hh = 0; ++qt; } }
  };
  const Walk walk0{it0 % a.G, qt_min + it0 / a.G, a.G};

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < STAGES; ++s) { mbar_init(bar_q_full(s), 1); mbar_init(bar_q_empty(s), 1); }
    mbar_init(bar_s_full, 1);
    mbar_init(bar_ds_ready, 256);
    for (int q = 0; q < 2; ++q) { mbar_init(bar_dq_full(q), 1); mbar_init(bar_dq_empty(q), 128); }
    mbar_init(bar_acc, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q); tma_prefetch(&tm_do); tma_prefetch(&tm_k); tma_prefetch(&tm_v);
    tma_prefetch(&tm_dq); tma_prefetch(&tm_dkv);
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (n > 0) {
    if (warp == 0) {
      // -------------------------------------------------------------- TMA producer
      if (lane == 0) {
        mbar_expect_tx(bar_kv, 2 * kKVBytes);
        for (int x = 0; x < D / 64; ++x) {
          tma_load_3d(sK + x * BOX_KV, &tm_k, bar_kv, x * 64, k0, g);
          tma_load_3d(sV + x * BOX_KV, &tm_v, bar_kv, x * 64, k0, g);
        }
        Walk w = walk0;
        for (int i = 0; i < n; ++i, w.next()) {
          const int st = i % STAGES;
          const uint32_t ph = (i / STAGES) & 1;
          const int h = g * a.G + w.hh, qt = w.qt;
          mbar_wait(bar_q_empty(st), ph ^ 1);
          TRACE(0, i);
          mbar_expect_tx(bar_q_full(st), 2 * kQBytes + 2 * BQ * 4);
          for (int x = 0; x < D / 64; ++x) {
            tma_load_3d(sQ + st * kQBytes + x * BOX_Q, &tm_q, bar_q_full(st), x * 64, qt * BQ, h);
            tma_load_3d(sDO + st * kQBytes + x * BOX_Q, &tm_do, bar_q_full(st), x * 64, qt * BQ, h);
          }
          const int64_t ro = (int64_t)h * a.c + qt * BQ;
          bulk_load(sStats + st * 2 * BQ * 4, a.nlse + ro, BQ * 4, bar_q_full(st));
          bulk_load(sStats + st * 2 * BQ * 4 + BQ * 4, a.Dv + ro, BQ * 4, bar_q_full(st));
        }
      }
    } else if (warp == 1) {
      // -------------------------------------------------------------- MMA issuer
      if (lane == 0) {
        constexpr uint32_t idesc_s = make_idesc_bf16(BKV, BQ, 0, 0);
        constexpr uint32_t idesc_kv = make_idesc_bf16(BKV, D, 0, 1);
        constexpr uint32_t idesc_q = make_idesc_bf16(D, BQ, 1, 1);
        auto issue_s_dp = [&](int st) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t okv = (kk / 4) * BOX_KV + (kk % 4) * 32;
            const uint32_t oq = (kk / 4) * BOX_Q + (kk % 4) * 32;
            mma_ss(tmem + TM_S, make_desc_sw128(sK + okv, 16, 1024),
                   make_desc_sw128(sQ + st * kQBytes + oq, 16, 1024), idesc_s, kk > 0);
          }
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t okv = (kk / 4) * BOX_KV + (kk % 4) * 32;
            const uint32_t oq = (kk / 4) * BOX_Q + (kk % 4) * 32;
            mma_ss(tmem + TM_DP, make_desc_sw128(sV + okv, 16, 1024),
                   make_desc_sw128(sDO + st * kQBytes + oq, 16, 1024), idesc_s, kk > 0);
          }
        };
        mbar_wait(bar_kv, 0);
        mbar_wait(bar_q_full(0), 0);
        tc_fence_after();
        issue_s_dp(0);
        mma_commit(bar_s_full);
        for (int i = 0; i < n; ++i) {
          const int st = i % STAGES, pb = i % 2, qb = i % 2;
          mbar_wait(bar_ds_ready, i & 1);
          TRACE(1, i);
          tc_fence_after();
          if (i + 1 < n) {
            const int st1 = (i + 1) % STAGES;
            mbar_wait(bar_q_full(st1), ((i + 1) / STAGES) & 1);
            TRACE(2, i);
            tc_fence_after();
            issue_s_dp(st1);
            mma_commit(bar_s_full);
          }
          // dV += P^T dO ; dK += dS^T Q
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk) {
            mma_ss(tmem + TM_DV, make_desc_sw128(sP + pb * kPBytes + kk * 32, 16, 1024),
                   make_desc_sw128(sDO + st * kQBytes + kk * 2048, BOX_Q, 1024), idesc_kv, (i > 0 || kk > 0));
          }
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk) {
            mma_ss(tmem + TM_DK, make_desc_sw128(sDS + pb * kPBytes + kk * 32, 16, 1024),
                   make_desc_sw128(sQ + st * kQBytes + kk * 2048, BOX_Q, 1024), idesc_kv, (i > 0 || kk > 0));
          }
          mma_commit(bar_q_empty(st));
          // dQ^T = K^T dS^T
          mbar_wait(bar_dq_empty(qb), ((i / 2) & 1) ^ 1);
          TRACE(3, i);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            mma_ss(tmem + TM_DQ + qb * BQ, make_desc_sw128(sK + kk * 2048, BOX_KV, 1024),
                   make_desc_sw128(sDS + pb * kPBytes + kk * 2048, BOX_KV, 1024), idesc_q, kk > 0);
          }
          mma_commit(bar_dq_full(qb));
          TRACE(4, i);
        }
        mma_commit(bar_acc);
      }
    } else if (warp >= 4 && warp < 12) {
      // -------------------------------------------------------------- compute warpgroups
      const int wg = (warp - 4) / 4;            // query columns [32 wg, 32 wg + 32)
      const int wq = warp % 4;
      const int kr = wq * 32 + lane;            // key row within the tile
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      const int key_pos = k0 + kr;
      const float sl2 = a.scale_log2;
      const f2_t sl2x2 = f2(sl2, sl2);
      Walk w = walk0;
      for (int i = 0; i < n; ++i, w.next()) {
        const int st = i % STAGES, pb = i % 2;
        const int qt = w.qt;
        mbar_wait(bar_q_full(st), (i / STAGES) & 1);   // -LSE log2e / D of this tile are in smem
        mbar_wait(bar_s_full, i & 1);
        if (lane == 0 && wq == 0 && wg == 0) TRACE(5, i);
        tc_fence_after();
        uint32_t sv[32], dpv[32];
        tmem_ld32(tmem + lane_addr + TM_S + wg * 32, sv);
        tmem_ld32(tmem + lane_addr + TM_DP + wg * 32, dpv);
        const uint32_t nl_s = sStats + (st * 2 * BQ + wg * 32) * 4;
        const uint32_t d_s = nl_s + BQ * 4;
        const int qpos0 = a.j * a.c + qt * BQ + wg * 32;  // absolute position of column 0
        // causal mask only where this warp's keys can exceed this warpgroup's query positions
        const bool masked = (k0 + wq * 32 + 31) > qpos0;
        tmem_wait_ld();
        uint32_t pp[16], dd[16];
        if (!masked) {
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 L = ld_shared_f4(nl_s + c4 * 16), Dv = ld_shared_f4(d_s + c4 * 16);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int c2 = c4 * 4 + hf * 2;
              const f2_t x = ffma2(f2u(sv[c2], sv[c2 + 1]), sl2x2, hf ? f2(L.z, L.w) : f2(L.x, L.y));
              const f2_t p2 = f2(ex2(f2lo(x)), ex2(f2hi(x)));
              const f2_t ds2 = fmul2(p2, fsub2(f2u(dpv[c2], dpv[c2 + 1]), hf ? f2(Dv.z, Dv.w) : f2(Dv.x, Dv.y)));
              pp[c2 / 2] = pack_bf16_f2(p2);
              dd[c2 / 2] = pack_bf16_f2(ds2);
            }
          }
        } else {
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 L = ld_shared_f4(nl_s + c4 * 16), Dv = ld_shared_f4(d_s + c4 * 16);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int c2 = c4 * 4 + hf * 2;
              const f2_t x = ffma2(f2u(sv[c2], sv[c2 + 1]), sl2x2, hf ? f2(L.z, L.w) : f2(L.x, L.y));
              float p0 = ex2(f2lo(x)), p1 = ex2(f2hi(x));
              if (key_pos > qpos0 + c2) p0 = 0.f;
              if (key_pos > qpos0 + c2 + 1) p1 = 0.f;
              const f2_t p2 = f2(p0, p1);
              const f2_t ds2 = fmul2(p2, fsub2(f2u(dpv[c2], dpv[c2 + 1]), hf ? f2(Dv.z, Dv.w) : f2(Dv.x, Dv.y)));
              pp[c2 / 2] = pack_bf16_f2(p2);
              dd[c2 / 2] = pack_bf16_f2(ds2);
            }
          }
        }
        const uint32_t prow = sP + pb * kPBytes, drow = sDS + pb * kPBytes;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          st_shared_v4(prow + sw128_off(kr, wg * 4 + q), pp[4 * q], pp[4 * q + 1], pp[4 * q + 2], pp[4 * q + 3]);
          st_shared_v4(drow + sw128_off(kr, wg * 4 + q), dd[4 * q], dd[4 * q + 1], dd[4 * q + 2], dd[4 * q + 3]);
        }
        fence_async_smem();
        tc_fence_before();
        if (lane == 0 && wq == 0) TRACE(6 + 3 * wg, i);
        mbar_arrive(bar_ds_ready);
      }
      // final: dK (warpgroup 0) / dV (warpgroup 1): TMEM -> scaled fp32 in smem (128B-swizzled
      // boxes [128 keys][32 fp32]) -> TMA reduce-add into dkv.  The Q/dO ring (dK) and the
      // P/dS buffers (dV) are free once every MMA has completed (bar_acc).
      mbar_wait(bar_acc, 0);
      tc_fence_after();
      const float sc = wg == 0 ? a.dk_scale : a.dv_scale;
      const uint32_t stg = wg == 0 ? sQ : sP;   // 64 KiB each, 1024-B aligned
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_addr + (wg == 0 ? TM_DK : TM_DV) + cc * 32, v);
        tmem_wait_ld();
        const uint32_t box = stg + cc * (BKV * 128);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_shared_v4(box + sw128_off(kr, q), __float_as_uint(sc * __uint_as_float(v[4 * q])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 1])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 2])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 3])));
      }
      fence_async_smem();
      named_bar_sync(2 + wg, 128);
      if (wq == 0 && lane == 0) {
        const int row0 = (wg * a.hkv + g) * a.S + k0;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tma_reduce_add_2d(&tm_dkv, stg + cc * (BKV * 128), cc * 32, row0);
        bulk_commit();
        bulk_wait0();
      }
    } else if (warp >= 12) {
      // -------------------------------------------------------------- dQ drain
      const int wq = warp % 4;
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      const bool leader = (warp == 12 && lane == 0);
      const uint32_t box = sDQ + wq * (BQ * 128);       // this warp's 32 head-dims
      const uint32_t colb = (uint32_t)(lane & 3) * 4;
      Walk w = walk0;
      for (int i = 0; i < n; ++i, w.next()) {
        const int qb = i % 2;
        const int h = g * a.G + w.hh, qt = w.qt;
        mbar_wait(bar_dq_full(qb), (i / 2) & 1);
        if (leader) TRACE(7, i);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32(tmem + lane_addr + TM_DQ + qb * BQ, v0);
        tmem_ld32(tmem + lane_addr + TM_DQ + qb * BQ + 32, v1);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(bar_dq_empty(qb));
        if (leader) bulk_wait_read0();        // previous reduce has finished reading the staging tile
        named_bar_sync(1, 128);
        // element (q row, head-dim dl) -> box wq, row q, 16-B chunk (lane/4) ^ (q%8), word lane%4
#pragma unroll
        for (int q = 0; q < 32; ++q)
          st_shared_f32(box + q * 128 + ((((uint32_t)lane >> 2) ^ (q & 7)) << 4) + colb, __uint_as_float(v0[q]));
#pragma unroll
        for (int q = 0; q < 32; ++q)
          st_shared_f32(box + (32 + q) * 128 + ((((uint32_t)lane >> 2) ^ (q & 7)) << 4) + colb,
                        __uint_as_float(v1[q]));
        fence_async_smem();
        named_bar_sync(1, 128);
        if (leader) {
          const int row0 = h * a.c + qt * BQ;
#pragma unroll
          for (int b = 0; b < D / 32; ++b) tma_reduce_add_2d(&tm_dq, sDQ + b * (BQ * 128), b * 32, row0);
          bulk_commit();
          TRACE(8, i);
        }
      }
      if (leader) bulk_wait0();
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

cudaError_t launch_bwd_sm100(const ChunkGeom& g, const CUtensorMap& tq, const CUtensorMap& tdo,
                             const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tdq,
                             const CUtensorMap& tdkv, const void* o, const void* d_o,
                             const float* lse, float relay, float gscale, float* dkv, void* dq, void* dk_own,
                             void* dv_own, float* ws_dqacc, float* ws_D, cudaStream_t st, int* launches) {
  static_assert(bwd::kAlloc <= 232448, "shared memory budget");
  if (g.d != bwd::D) return cudaErrorInvalidValue;
  cudaError_t e = launch_prep_bf16(g, o, d_o, ws_D, dkv, ws_dqacc, lse, ws_D + (size_t)g.hq * g.c, relay, st);
  if (e != cudaSuccess) return e;
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(seco_bwd_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bwd::kAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  bwd::Args a;
  a.c = g.c; a.j = g.j; a.G = g.hq / g.hkv; a.hkv = g.hkv; a.S = g.c * g.k;
  a.scale_log2 = g.scale * 1.4426950408889634f;
  a.dk_scale = gscale * g.scale;
  a.dv_scale = gscale;
  a.nlse = ws_D + (size_t)g.hq * g.c; a.Dv = ws_D;
  a.trace = nullptr;
#ifdef SECO_TRACE
  {
    static unsigned long long* tbuf = nullptr;
    if (!tbuf) cudaMalloc(&tbuf, sizeof(unsigned long long) * bwd::kTraceCtas * bwd::kTraceSlots * bwd::kTraceIters);
    cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * bwd::kTraceCtas * bwd::kTraceSlots * bwd::kTraceIters, st);
    a.trace = tbuf;
    seco_trace_buffer = tbuf;
  }
#endif
  const int ntiles = (g.j + 1) * g.c / bwd::BKV;
  // Q-split when the chunk offers fewer key tiles than ~2 waves of SMs; each split keeps
  // at least 2*G query tiles (the shortest diagonal tile has 2*G of them).
  int nsplit = (2 * 148 + ntiles * g.hkv - 1) / (ntiles * g.hkv);
  if (nsplit > 2 * a.G) nsplit = 2 * a.G;
  if (nsplit < 1) nsplit = 1;
  a.nsplit = nsplit;
  dim3 grid(ntiles * nsplit * g.hkv);
  seco_bwd_sm100_kernel<<<grid, bwd::kThreads, bwd::kAlloc, st>>>(tq, tdo, tk, tv, tdq, tdkv, a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  e = launch_final_bf16(g, ws_dqacc, dq, dkv, dk_own, dv_own, gscale * g.scale, st);
  *launches = 2 + 1;
  return e;
}

}  // namespace seco
