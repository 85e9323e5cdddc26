// Chunk-local backward on sm_100a tensor cores (Alg. 1 lines 6-7 P:200-201):
// for chunk j, gradients w.r.t. Q_j and w.r.t. every K/V row of cache slots 0..j,
// the latter accumulated in place into the persistent fp32 checkpoint-gradient
// buffer dkv (the requires_grad leaves of App. C.1).
//
// KV-stationary: one CTA owns a 128-key tile of kv-head g (keys [k0, k0+128) in slot
// k0/c <= j) and loops over 128-row query tiles of the G q-heads of group g that can
// see those keys (optionally a contiguous share of them: Q-split).  Per query tile,
// five tcgen05 MMAs, all M = 128, N = 128, fp32 accumulators in TMEM:
//   S^T  = K Q^T     -> R0            SS (K, Q K-major)
//   dP^T = V dO^T    -> R1            SS
//   P^T  = exp2(S^T sigma log2e - LSE log2e), dS^T = P^T o (dP^T - D)
//          (CUDA cores; bf16 P^T over R0, bf16 dS^T over R1, dS^T also to smem)
//   dV  += P^T dO    A = P^T from TMEM (TS), B = dO MN-major
//   dK  += dS^T Q    A = dS^T from TMEM (TS), B = Q MN-major
//   dQ^T = K^T dS^T  -> R0 (after dV has consumed P^T), A and B MN-major in smem;
//          drained to smem (swizzled) and TMA reduce-added into the fp32 dQ accumulator
// TMEM columns: R0 [0,128)  R1 [128,256)  dK [256,384)  dV [384,512).
// MMA issue order per tile i: dV(i) dK(i) dQ^T(i) dP(i+1) [R0 drained] S(i+1).
// Warp roles: w0 TMA producer (K,V once; Q,dO double-buffered, LSE/D with Q), w1 MMA
// issuer, w2 TMEM allocator, w3 lane 0 issues the dQ TMA reduce-adds, w4-w19 four compute
// warpgroups (thread = key row; WG w owns query columns [16w, 16w+16) of each 64-column
// half -- four warps per SM sub-partition hide the MUFU / TMEM latencies; between tiles the
// same warps read dQ^T out of R0 and stage it).
// The dQ staging tile (64 KiB fp32) borrows the current Q and dO buffers, both dead once
// dQ^T(i) has started (dK(i), dV(i) consumed them); their next loads wait for the drain
// (measured: one SM drains reduce-adds at 25.6 B/clk, so the 64 KiB take ~2600 cycles, as
// long as the tile's MMAs), the dO half first since dP^T(i+2) is issued before S^T(i+2).
// dK/dV leave TMEM once per CTA, scaled (s sigma,
// s), through swizzled smem staging and TMA reduce-add into dkv; slot j of dkv was
// pre-scaled by the relay factor gamma in bwd_prep (grad_hook).
// All fp32 reductions are issued by the TMA unit: no per-element atomics.
//
// This header describes v1 (seco_bwd_sm100_kernel, the deterministic-mode kernel).  The default
// kernel is v2 (seco_bwd2_sm100_kernel, further down): same regions and MMAs in the CUTLASS /
// FlashAttention-4 issue order, see its own header and DESIGN §6.2.
//
// mbarrier waits in this translation unit pass a suspend-time hint to try_wait: fewer polling
// wavefronts on the shared-memory pipe, which the backward keeps ~90 % busy (+1.7-3 % per call;
// the forward, compiled separately, measured -0.5 % with it and keeps the plain wait).
#ifndef SECO_BWD_PAIR_DEFAULT
#define SECO_BWD_PAIR_DEFAULT 0
#endif
#ifndef SECO_BWD_MMA_WARP
#define SECO_BWD_MMA_WARP 1
#endif
#ifndef SECO_WAIT_HINT
#define SECO_WAIT_HINT 1
#endif
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace seco {

#ifdef SECO_TRACE
unsigned long long* seco_trace_buffer = nullptr;
extern "C" void* seco_debug_trace_ptr() { return seco_trace_buffer; }
#endif

cudaError_t launch_prep_bf16(const ChunkGeom& g, const void* o, const void* d_o, float* D, float* dkv,
                             float* dqacc, const float* lse, float* nlse, float relay, cudaStream_t st,
                             int* order);
cudaError_t launch_final_bf16(const ChunkGeom& g, const float* dqacc, void* dq, const float* dkv, void* dk_own,
                              void* dv_own, float dq_scale, cudaStream_t st);

namespace bwd {
constexpr int BKV = 128;  // keys per CTA tile (UMMA M)
constexpr int BQ = 128;   // query rows per iteration (UMMA N)
constexpr int D = 128;    // head dim (this kernel)
constexpr int kTile = 128 * 128 * 2;            // bf16 [128][128] tile = 2 boxes [128 rows][128 B]
constexpr int kBox = 128 * 128;                 // one [128 rows][128 B] box
constexpr int kK = 0;
constexpr int kV = kK + kTile;
constexpr int kQD = kV + kTile;                 // stage s: Q tile at kQD + 2s*kTile, dO tile right after it
constexpr int kDS = kQD + 4 * kTile;            // dS^T [128 keys][128 q] bf16 (2 boxes by q half)
constexpr int kStats = kDS + kTile;             // [2][2][BQ] fp32 (-LSE log2e, D)
constexpr int kBar = kStats + 2 * 2 * BQ * 4;
// bars: kv, q_full[2], q_empty[2], do_full[2], do_empty[2], s_full, ds_half[0], dq_full, dq_empty,
//       stg_half[0], acc_full, drain_done, ds_half[1], stg_half[1]
constexpr int kNumBars = 1 + 8 + 9;
constexpr int kTmemSlot = kBar + 8 * kNumBars;
constexpr int kBytes = kTmemSlot + 16;
constexpr int kThreads = 640;   // 4 role warps + 4 compute warpgroups
constexpr int kWG = 4;          // compute warpgroups; WG w owns query columns {16w + 64hf}
// dQ drain: one thread issues TMA bulk reduce-adds.  (Tried: warps 2-3 moving the tile with
// ld.shared + red.global.add.v4 to keep the TMA unit free for loads -- 10-15 % slower, the
// reds clog the MIO queue that the mbarrier traffic of every role also uses.)

constexpr int R0 = 0, R1 = 128, TM_DK = 256, TM_DV = 384;

struct Args {
  int c, j, G, hkv, S;
  int cp;             // rows per head of nlse / Dv / dqacc: c rounded up to BQ (ragged last tile)
  // work list (launch_bwd_sm100 / choose_schedule): blocks [0, n0) take whole units, the next
  // n1 units are split into f1 query-range pieces each, the remaining units into f2 pieces.
  // Unit U = (key tile U / hkv, kv head U % hkv); ascending key tiles = descending work.
  int n0, n1, f1, f2;
  float scale_log2;   // sigma * log2 e
  float dk_scale;     // s * sigma
  float dv_scale;     // s
  const float* nlse;  // [hq][cp]  -LSE * log2(e)   (from bwd_prep; -inf on padded rows)
  const float* Dv;    // [hq][cp]  rowsum(dO o O)  (from bwd_prep; 0 on padded rows)
  float* dqacc;       // [hq][cp][D] fp32 dQ accumulator (zeroed by bwd_prep)
  int* dq_order;      // deterministic mode: [hq][ceil(c/BQ)] count of key tiles that have added their
                      // dQ share of query tile (h, qt) (zeroed by bwd_prep); null otherwise
  int* ticket;        // deterministic mode: work-unit ticket counter (zeroed by bwd_prep); null otherwise
  int* err;           // set to 1 if the dynamic smem window is not 1024-B aligned
  unsigned long long* trace;  // SECO_TRACE builds only: [kTraceCtas][kTraceSlots][kTraceIters] clock64
};
#ifdef SECO_TRACE
constexpr int kTraceCtas = 4, kTraceSlots = 20, kTraceIters = 128;
#endif
}  // namespace bwd

__global__ void __launch_bounds__(bwd::kThreads, 1)
    seco_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv,
                          const bwd::Args a) {
  using namespace bwd;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  if (sb & 1023) {   // the 128B-swizzle atoms need 1024-B alignment; never observed, checked anyway
    if (threadIdx.x == 0 && a.err) atomicExch(a.err, 1);
    return;
  }
  const uint32_t sK = sb + kK, sV = sb + kV, sDS = sb + kDS;
  // stage st: [Q tile][dO tile] contiguous (64 KiB) -- also the dQ staging [128 q][128 d] fp32
  auto qbuf = [&](int st) { return sb + kQD + (uint32_t)st * 2 * kTile; };
  auto dobuf = [&](int st) { return sb + kQD + (uint32_t)st * 2 * kTile + kTile; };
  const uint32_t sStats = sb + kStats;
  const uint32_t b0 = sb + kBar;
  const uint32_t bar_kv = b0;
  auto bar_q_full = [&](int s) { return b0 + 8u * (1 + s); };
  auto bar_q_empty = [&](int s) { return b0 + 8u * (3 + s); };
  auto bar_do_full = [&](int s) { return b0 + 8u * (5 + s); };
  auto bar_do_empty = [&](int s) { return b0 + 8u * (7 + s); };
  const uint32_t bar_s_full = b0 + 8u * 9;
  // ds_half(h): P^T / dS^T of query half h (columns [64h, 64h+64)) are in TMEM and smem
  auto bar_ds_half = [&](int h) { return b0 + 8u * (h == 0 ? 10 : 16); };
  const uint32_t bar_dq_full = b0 + 8u * 11;
  const uint32_t bar_dq_empty = b0 + 8u * 12;
  // stg_half(h): dQ^T rows [64h, 64h+64) staged (the 4 warps of compute warpgroup h)
  auto bar_stg_half = [&](int h) { return b0 + 8u * (h == 0 ? 13 : 17); };
  const uint32_t bar_acc = b0 + 8u * 14;
  const uint32_t bar_drain_done = b0 + 8u * 15;
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
  // block -> (unit U, piece of f); units in ascending key-tile order = longest work first,
  // the split (shorter) pieces at the end of the list fill the last wave.  Deterministic mode
  // takes its work item from a ticket drawn when the CTA starts: a unit's dQ adds wait only for
  // lower units, which were claimed by CTAs already running, so progress does not depend on
  // the order in which the hardware dispatches blocks.
  int bid = blockIdx.x;
  if (a.ticket) {    // broadcast through the dynamic window (static smem would not fit beside it)
    volatile int* s_ticket = reinterpret_cast<volatile int*>(smem + kTmemSlot + 8);
    if (threadIdx.x == 0) *s_ticket = atomicAdd(a.ticket, 1);
    __syncthreads();
    bid = *s_ticket;
  }
  int U, piece, f;
  if (bid < a.n0) {
    U = bid; piece = 0; f = 1;
  } else if (bid < a.n0 + a.n1 * a.f1) {
    const int r = bid - a.n0;
    U = a.n0 + r / a.f1; piece = r % a.f1; f = a.f1;
  } else {
    const int r = bid - a.n0 - a.n1 * a.f1;
    U = a.n0 + a.n1 + r / a.f2; piece = r % a.f2; f = a.f2;
  }
  const int g = U % a.hkv;
  const int u = U / a.hkv;
  const int k0 = u * BKV;                                  // first key (absolute position)
  const int nqt = (a.c + BQ - 1) / BQ;
  const int rel = k0 - a.j * a.c;                          // key offset relative to chunk j's first row
  const int qt_min = rel > 0 ? rel / BQ : 0;               // first query tile that sees key k0
  const int n_all = a.G * (nqt - qt_min);
  const int it0 = (int)((int64_t)piece * n_all / f);
  const int it1 = (int)((int64_t)(piece + 1) * n_all / f);
  const int n = it1 - it0;
  // iteration i -> (q-head g*G + hh, query tile qt); each role walks it incrementally
  struct Walk {
    int hh, qt, G;
    __device__ void next() { if (++hh == G) { hh = 0; ++qt; } }
  };
  const Walk walk0{it0 % a.G, qt_min + it0 / a.G, a.G};

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_q_full(s), 1);
      mbar_init(bar_q_empty(s), 2);     // dK has consumed Q, and the dQ drain has read it
      mbar_init(bar_do_full(s), 1);
      mbar_init(bar_do_empty(s), 2);    // dV has consumed dO, and the dQ drain has read it
    }
    mbar_init(bar_s_full, 1);
    mbar_init(bar_ds_half(0), 4 * kWG);  // one elected lane per compute warp
    mbar_init(bar_ds_half(1), 4 * kWG);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 4 * kWG);   // one elected lane per compute warp (they read R0 out)
    mbar_init(bar_stg_half(0), 2 * 4);  // the 8 warps staging dQ rows [64h, 64h + 64)
    mbar_init(bar_stg_half(1), 2 * 4);
    mbar_init(bar_acc, 1);
    mbar_init(bar_drain_done, 1);
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
        mbar_expect_tx(bar_kv, 2 * kTile);
        SECO_CHECK_COND(k0 < (a.j + 1) * a.c && g < a.hkv, 410);   // key tile inside slots 0..j
        for (int x = 0; x < D / 64; ++x) {
          tma_load_3d(sK + x * kBox, &tm_k, bar_kv, x * 64, k0, g);
          tma_load_3d(sV + x * kBox, &tm_v, bar_kv, x * 64, k0, g);
        }
        Walk w = walk0;
        for (int i = 0; i < n; ++i, w.next()) {
          const int st = i & 1;
          const uint32_t ph = (i >> 1) & 1;
          const int h = g * a.G + w.hh, qt = w.qt;
          SECO_CHECK_COND(qt * BQ < a.c && w.hh < a.G, 411);       // query tile inside chunk j
          // dO first: dP^T(i) is issued before S^T(i), and its buffer frees earlier (dV(i-2))
          mbar_wait(bar_do_empty(st), ph ^ 1);
          mbar_expect_tx(bar_do_full(st), kTile);
          for (int x = 0; x < D / 64; ++x)
            tma_load_3d(dobuf(st) + x * kBox, &tm_do, bar_do_full(st), x * 64, qt * BQ, h);
          TRACE(19, i);
          mbar_wait(bar_q_empty(st), ph ^ 1);
          mbar_expect_tx(bar_q_full(st), kTile + 2 * BQ * 4);
          for (int x = 0; x < D / 64; ++x)
            tma_load_3d(qbuf(st) + x * kBox, &tm_q, bar_q_full(st), x * 64, qt * BQ, h);
          const int64_t ro = (int64_t)h * a.cp + qt * BQ;
          bulk_load(sStats + st * 2 * BQ * 4, a.nlse + ro, BQ * 4, bar_q_full(st));
          bulk_load(sStats + st * 2 * BQ * 4 + BQ * 4, a.Dv + ro, BQ * 4, bar_q_full(st));
          TRACE(0, i);
        }
      }
    } else if (warp == 1) {
      // -------------------------------------------------------------- MMA issuer
#if SECO_BWD_MMA_WARP
      const bool issuer = elect_one_sync();               // converged warp, one elected lane issues
      {
#else
      const bool issuer = true;
      if (lane == 0) {
#endif
        constexpr uint32_t idesc_s = make_idesc_bf16(BKV, BQ, 0, 0);    // S^T, dP^T
        constexpr uint32_t idesc_kv = make_idesc_bf16(BKV, D, 0, 1);    // dV, dK: A TMEM (K-major), B MN-major
        constexpr uint32_t idesc_q = make_idesc_bf16(D, BQ, 1, 1);      // dQ^T: A, B MN-major
        auto issue_sdp = [&](uint32_t a_base, uint32_t b_base, uint32_t d_col) {
          const uint64_t da = make_desc_sw128(a_base, 16, 1024), db = make_desc_sw128(b_base, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk / 4) * kBox + (kk % 4) * 32) >> 4;
            if (issuer) mma_ss(tmem + d_col, da + off, db + off, idesc_s, kk > 0);
          }
        };
        // A operand (P^T or dS^T, bf16 in TMEM): query k-step kk (queries 16kk..16kk+15) lives
        // packed in columns base + 16kk .. +7 (over the S^T / dP^T columns of those queries, which
        // their compute warp has already read); query half hf = k-steps 4hf .. 4hf+3
        auto issue_kv = [&](uint32_t a_col, uint32_t b_base, uint32_t d_col, int hf, bool acc) {
          const uint64_t db = make_desc_sw128(b_base, kBox, 1024);
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = 4 * hf + k4;
            if (issuer)
              mma_ts(tmem + d_col, tmem + a_col + 16 * kk, db + (uint32_t)(kk * 2048 >> 4), idesc_kv,
                     (acc || kk > 0) ? 1u : 0u);
          }
        };
        auto commit = [&](uint32_t bar) { if (issuer) mma_commit(bar); };
        const uint64_t dk_mn = make_desc_sw128(sK, kBox, 1024), dds_mn = make_desc_sw128(sDS, kBox, 1024);
        mbar_wait(bar_kv, 0);
        mbar_wait(bar_do_full(0), 0);
        mbar_wait(bar_q_full(0), 0);
        tc_fence_after();
        issue_sdp(sV, dobuf(0), R1);
        issue_sdp(sK, qbuf(0), R0);
        commit(bar_s_full);
        for (int i = 0; i < n; ++i) {
          const int st = i & 1;
          // dV += P^T dO ; dK += dS^T Q, query half 0 while the compute warps finish half 1
          mbar_wait(bar_ds_half(0), i & 1);
          TRACE(1, i);
          tc_fence_after();
          issue_kv(R0, dobuf(st), TM_DV, 0, i > 0);
          issue_kv(R1, qbuf(st), TM_DK, 0, i > 0);
          mbar_wait(bar_ds_half(1), i & 1);
          TRACE(16, i);
          tc_fence_after();
          issue_kv(R0, dobuf(st), TM_DV, 1, true);
          commit(bar_do_empty(st));
          issue_kv(R1, qbuf(st), TM_DK, 1, true);
          commit(bar_q_empty(st));
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)             // dQ^T = K^T dS^T -> R0
            if (issuer)
              mma_ss(tmem + R0, dk_mn + (uint32_t)(kk * 2048 >> 4), dds_mn + (uint32_t)(kk * 2048 >> 4), idesc_q,
                     kk > 0);
          commit(bar_dq_full);
          TRACE(2, i);
          if (i + 1 < n) {
            const int st1 = (i + 1) & 1;
            const uint32_t ph1 = ((i + 1) >> 1) & 1;
            mbar_wait(bar_do_full(st1), ph1);
            tc_fence_after();
            issue_sdp(sV, dobuf(st1), R1);                  // dP^T(i+1) -> R1 (dS^T(i) consumed by dK(i))
            TRACE(17, i);
            mbar_wait(bar_dq_empty, i & 1);                 // R0 drained
            TRACE(3, i);
            mbar_wait(bar_q_full(st1), ph1);
            tc_fence_after();
            issue_sdp(sK, qbuf(st1), R0);                   // S^T(i+1) -> R0
            commit(bar_s_full);
            TRACE(4, i);
          }
        }
        commit(bar_acc);
      }
    } else if (warp >= 4) {
      // -------------------------------------------------------------- compute warpgroups
      const int wg = (warp - 4) / 4;            // query columns [16 wg, +16) of each half
      const int wq = warp % 4;
      const int kr = wq * 32 + lane;            // key row within the tile
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      const int key_pos = k0 + kr;
      const f2_t sl2x2 = f2(a.scale_log2, a.scale_log2);
      Walk w = walk0;
      for (int i = 0; i < n; ++i, w.next()) {
        const int st = i & 1;
        mbar_wait(bar_q_full(st), (i >> 1) & 1);  // -LSE log2e / D of this tile are in smem
        mbar_wait(bar_s_full, i & 1);
        if (lane == 0 && wq == 0 && wg == 0) TRACE(5, i);
        tc_fence_after();
        const int qbase = a.j * a.c + w.qt * BQ;   // absolute position of query column 0
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int c = 64 * hf + 16 * wg;        // this warp's 16 query columns of half hf
          uint32_t sv[16], dpv[16];
          tmem_ld16(tmem + lane_addr + R0 + c, sv);
          tmem_ld16(tmem + lane_addr + R1 + c, dpv);
          const uint32_t nl_s = sStats + (st * 2 * BQ + c) * 4;
          const uint32_t d_s = nl_s + BQ * 4;
          const int qpos0 = qbase + c;
          const bool masked = (k0 + wq * 32 + 31) > qpos0;
          tmem_wait_ld();
          if (lane == 0 && wq == 0 && wg == 0) TRACE(10 + 2 * hf, i);
          uint32_t pp[8], dd[8];
          if (!masked) {
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const float4 L = ld_shared_f4(nl_s + c4 * 16), Dv = ld_shared_f4(d_s + c4 * 16);
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const int c2 = c4 * 4 + h2 * 2;
                const f2_t x = ffma2(f2u(sv[c2], sv[c2 + 1]), sl2x2, h2 ? f2(L.z, L.w) : f2(L.x, L.y));
                const f2_t p2 = f2(ex2(f2lo(x)), ex2(f2hi(x)));
                const f2_t ds2 = fmul2(p2, fsub2(f2u(dpv[c2], dpv[c2 + 1]), h2 ? f2(Dv.z, Dv.w) : f2(Dv.x, Dv.y)));
                pp[c2 / 2] = pack_bf16_f2(p2);
                dd[c2 / 2] = pack_bf16_f2(ds2);
              }
            }
          } else {
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const float4 L = ld_shared_f4(nl_s + c4 * 16), Dv = ld_shared_f4(d_s + c4 * 16);
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const int c2 = c4 * 4 + h2 * 2;
                const f2_t x = ffma2(f2u(sv[c2], sv[c2 + 1]), sl2x2, h2 ? f2(L.z, L.w) : f2(L.x, L.y));
                float p0 = ex2(f2lo(x)), p1 = ex2(f2hi(x));
                if (key_pos > qpos0 + c2) p0 = 0.f;
                if (key_pos > qpos0 + c2 + 1) p1 = 0.f;
                const f2_t p2 = f2(p0, p1);
                const f2_t ds2 = fmul2(p2, fsub2(f2u(dpv[c2], dpv[c2 + 1]), h2 ? f2(Dv.z, Dv.w) : f2(Dv.x, Dv.y)));
                pp[c2 / 2] = pack_bf16_f2(p2);
                dd[c2 / 2] = pack_bf16_f2(ds2);
              }
            }
          }
          if (lane == 0 && wq == 0 && wg == 0) TRACE(11 + 2 * hf, i);
          // P^T, dS^T (bf16 pairs) over this warp's own S^T / dP^T columns just read: [c, c + 8)
          tmem_st8(tmem + lane_addr + R0 + c, pp);
          tmem_st8(tmem + lane_addr + R1 + c, dd);
          // dS^T to smem for dQ^T: box hf (query half), row kr, 16-B chunks 2 wg, 2 wg + 1
          const uint32_t drow = sDS + hf * kBox;
          st_shared_v4(drow + sw128_off(kr, 2 * wg), dd[0], dd[1], dd[2], dd[3]);
          st_shared_v4(drow + sw128_off(kr, 2 * wg + 1), dd[4], dd[5], dd[6], dd[7]);
          tmem_wait_st();
          fence_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0 && wq == 0 && wg == 0 && hf == 1) TRACE(6, i);
          if (lane == 0) mbar_arrive(bar_ds_half(hf));
        }
        // dQ^T(i) read-out (the compute warps are idle until S^T(i+1) lands): lane = head dim
        // d = 32 wq + lane, this warpgroup's 32 query columns [32 wg, +32) -> registers -> R0
        // released -> row-major [128 q][128 d] fp32 staging over the Q(i) and dO(i) buffers
        // (contiguous; rows 0-63 in Q's, 64-127 in dO's), both dead once dQ^T(i) completed.
        mbar_wait(bar_dq_full, i & 1);
        if (lane == 0 && wq == 0 && wg == 0) TRACE(14, i);
        tc_fence_after();
        uint32_t qa[32];
        tmem_ld32(tmem + lane_addr + R0 + 32 * wg, qa);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_dq_empty);
        if (lane == 0 && wq == 0 && wg == 0) TRACE(15, i);
        // 32 lanes store 128 contiguous bytes of one row (conflict-free)
        const uint32_t rowb = qbuf(st) + (uint32_t)(32 * wg) * 512 + (uint32_t)(32 * wq + lane) * 4;
#pragma unroll
        for (int q = 0; q < 32; ++q) st_shared_f32(rowb + q * 512, __uint_as_float(qa[q]));
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_stg_half(wg >> 1));
      }
      // final: dK (warpgroups 0, 1) / dV (warpgroups 2, 3), two 32-column chunks each: TMEM ->
      // scaled fp32 in smem (128B-swizzled boxes [128 keys][32 fp32]) -> TMA reduce-add into
      // dkv.  dK stages in the Q buffers, dV in the dO buffers: free once every MMA has
      // completed and the drain is done.
      mbar_wait(bar_acc, 0);
      mbar_wait(bar_drain_done, 0);
      tc_fence_after();
      const int mat = wg >> 1;                  // 0 = dK, 1 = dV
      const float sc = mat == 0 ? a.dk_scale : a.dv_scale;
      auto stg_box = [&](int cc) { return (mat == 0 ? qbuf(cc >> 1) : dobuf(cc >> 1)) + (uint32_t)(cc & 1) * kBox; };
#pragma unroll 1
      for (int c2 = 0; c2 < 2; ++c2) {
        const int cc = 2 * (wg & 1) + c2;
        uint32_t v[32];
        tmem_ld32(tmem + lane_addr + (mat == 0 ? TM_DK : TM_DV) + cc * 32, v);
        tmem_wait_ld();
        const uint32_t box = stg_box(cc);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_shared_v4(box + sw128_off(kr, q), __float_as_uint(sc * __uint_as_float(v[4 * q])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 1])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 2])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 3])));
      }
      fence_async_smem();
      named_bar_sync(2 + mat, 256);
      if ((wg & 1) == 0 && wq == 0 && lane == 0) {
        const int row0 = (mat * a.hkv + g) * a.S + k0;
        SECO_CHECK_COND(k0 < (a.j + 1) * a.c && row0 < 2 * a.hkv * a.S, 510);   // dKV rows
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tma_reduce_add_2d(&tm_dkv, stg_box(cc), cc * 32, row0);
        bulk_commit();
        bulk_wait0();
      }
    } else if (warp == 3) {
      // -------------------------------------------------------------- dQ reduce
      // once the compute warps have staged dQ^T(i) (Q(i) and dO(i) buffers), one thread
      // issues the TMA reduce-add into dQacc rows [h c + 128 qt, +128) and, when the TMA
      // has read the staging, releases both buffers to the producer.
      if (lane == 0) {
        Walk w = walk0;
        for (int i = 0; i < n; ++i, w.next()) {
          const int st = i & 1;
          const int h = g * a.G + w.hh, qt = w.qt;
          float* dst = a.dqacc + ((int64_t)h * a.cp + qt * BQ) * D;  // 128 contiguous dQacc rows
          // rows 64-127 (in dO(i)'s buffer) first: dP(i+2) needs that buffer before S(i+2) needs Q's
          // (the TMA unit serves requests in order and loads queue behind these; issuing the
          // tile in 4-16 KiB pieces with <= 2 in flight measured 2-20 % slower)
          int* ctr = a.dq_order ? a.dq_order + (int64_t)h * nqt + qt : nullptr;
          mbar_wait(bar_stg_half(1), i & 1);
          TRACE(7, i);
          if (ctr) {
            // deterministic mode: the key tiles seeing query tile qt are 0 .. j c / BKV + qt;
            // add after tiles 0 .. u-1 have (fixed fp32 summation order).  Both staging
            // phases are consumed before the (possibly long) wait, so the compute warps can
            // never run a full phase ahead of this thread on the stg barriers.
            mbar_wait(bar_stg_half(0), i & 1);
            while (ld_relaxed_gpu(ctr) != u) {
            }
            fence_acq_rel_gpu();
            fence_proxy_async_global();      // ... before this thread's TMA reduce-adds
          }
          SECO_CHECK_COND(dst >= a.dqacc && dst + 128 * D <= a.dqacc + (int64_t)a.G * a.hkv * a.cp * D, 511);
          bulk_reduce_add_f32(dst + 64 * D, dobuf(st), kTile);
          bulk_commit();
          if (!ctr) mbar_wait(bar_stg_half(0), i & 1);
          bulk_reduce_add_f32(dst, qbuf(st), kTile);
          bulk_commit();
          bulk_wait_read<1>();
          TRACE(18, i);
          mbar_arrive(bar_do_empty(st));
          bulk_wait_read<0>();
          TRACE(8, i);
          mbar_arrive(bar_q_empty(st));
          if (ctr) {
            bulk_wait0();                    // the reduce-adds have been performed in L2
            fence_proxy_async_global();
            st_release_gpu(ctr, u + 1);
          }
        }
        bulk_wait0();
        mbar_arrive(bar_drain_done);
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================================ backward v2
// Same work decomposition, TMEM regions and MMAs as seco_bwd_sm100_kernel, with the issue order
// of the CUTLASS / FlashAttention-4 Blackwell backward: per query tile i the MMA warp issues
//   S^T(i+1) -> R0,  dK(i) += dS^T(i) Q(i),  dQ^T(i) -> R1,  dP^T(i+1) -> R1,  dV(i+1) += P^T(i+1) dO(i+1)
// so the exponentials of tile i+1 (P^T, phase A) run while dK(i) / dQ^T(i) execute, and only
// dQ^T drain -> dP^T(i+1) -> dS^T(i+1) (phase B) -> dK(i+1) -> dQ^T(i+1) stays serial.  dQ^T
// lives in R1 (the dP^T region: dP^T(i) is dead once dS^T(i) is formed) and is drained by a
// dedicated warpgroup into a two-slot 16 KiB staging ring (32 query rows x 128 d fp32 each),
// from which one thread issues 1-D bulk reduce-adds; dO is single-buffered to make room.
// Warps: w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w3 dQ reduce issuer, w4-w7 dQ^T
// drain (lane = d), w8-w15 two compute warpgroups (thread = key row, WG c owns query columns
// [64c, 64c+64)).  Non-deterministic mode only (the deterministic mode keeps the v1 kernel).
namespace bwd2 {
constexpr int BKV = 128, BQ = 128, D = 128;
constexpr int kTile = 128 * 128 * 2;           // bf16 [128][128]
constexpr int kBox = 128 * 128;                // one [128 rows][128 B] box
constexpr int kK = 0;
constexpr int kV = kK + kTile;
constexpr int kQ = kV + kTile;                 // two stages
constexpr int kDO = kQ + 2 * kTile;            // one stage
constexpr int kSTG = kDO + kTile;              // dQ staging: 2 slots x 16 KiB (contiguous after dO)
constexpr int kSlot = 32 * D * 4;
constexpr int kDS = kSTG + 2 * kSlot;          // dS^T [128 keys][128 q] bf16 (2 boxes by q half)
constexpr int kStats = kDS + kTile;            // [2 stages][2][BQ] fp32 (-LSE log2e, D)
constexpr int kBar = kStats + 2 * 2 * BQ * 4;
constexpr int kNumBars = 20;
constexpr int kTmemSlot = kBar + 8 * kNumBars;
constexpr int kBytes = kTmemSlot + 16;
constexpr int kThreads = 512;
constexpr int R0 = 0, R1 = 128, TM_DK = 256, TM_DV = 384;
}  // namespace bwd2

__global__ void __launch_bounds__(bwd2::kThreads, 1)
    seco_bwd2_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                           const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                           const __grid_constant__ CUtensorMap tm_dkv, const bwd::Args a) {
  using namespace bwd2;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  if (sb & 1023) {
    if (threadIdx.x == 0 && a.err) atomicExch(a.err, 1);
    return;
  }
  const uint32_t sK = sb + kK, sV = sb + kV, sDO = sb + kDO, sDS = sb + kDS, sSTG = sb + kSTG;
  auto qbuf = [&](int st) { return sb + kQ + (uint32_t)st * kTile; };
  const uint32_t sStats = sb + kStats;
  const uint32_t b0 = sb + kBar;
  const uint32_t bar_kv = b0;
  auto bar_q_full = [&](int s) { return b0 + 8u * (1 + s); };
  auto bar_q_empty = [&](int s) { return b0 + 8u * (3 + s); };
  const uint32_t bar_do_full = b0 + 8u * 5, bar_do_empty = b0 + 8u * 6;
  const uint32_t bar_s_full = b0 + 8u * 7, bar_p_ready = b0 + 8u * 8;
  const uint32_t bar_dp_full = b0 + 8u * 9, bar_ds_ready = b0 + 8u * 10;
  const uint32_t bar_dq_full = b0 + 8u * 11, bar_dq_empty = b0 + 8u * 12;
  auto bar_stg_full = [&](int s) { return b0 + 8u * (13 + s); };
  auto bar_stg_free = [&](int s) { return b0 + 8u * (15 + s); };
  const uint32_t bar_acc = b0 + 8u * 17, bar_drain_done = b0 + 8u * 18;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kTmemSlot);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#ifdef SECO_TRACE
#define V2TRACE(slot, i)                                                                                   \
  do {                                                                                                     \
    if (a.trace && blockIdx.x < bwd::kTraceCtas && (i) < bwd::kTraceIters)                                \
      a.trace[((size_t)blockIdx.x * bwd::kTraceSlots + (slot)) * bwd::kTraceIters + (i)] = clock64();     \
  } while (0)
#else
#define V2TRACE(slot, i) do { } while (0)
#endif

  // work decode: identical to seco_bwd_sm100_kernel (balanced list of units / query-range pieces)
  const int bid = blockIdx.x;
  int U, piece, f;
  if (bid < a.n0) {
    U = bid; piece = 0; f = 1;
  } else if (bid < a.n0 + a.n1 * a.f1) {
    const int r = bid - a.n0;
    U = a.n0 + r / a.f1; piece = r % a.f1; f = a.f1;
  } else {
    const int r = bid - a.n0 - a.n1 * a.f1;
    U = a.n0 + a.n1 + r / a.f2; piece = r % a.f2; f = a.f2;
  }
  const int g = U % a.hkv;
  const int u = U / a.hkv;
  const int k0 = u * BKV;
  const int nqt = (a.c + BQ - 1) / BQ;
  const int rel = k0 - a.j * a.c;
  const int qt_min = rel > 0 ? rel / BQ : 0;
  const int n_all = a.G * (nqt - qt_min);
  const int it0 = (int)((int64_t)piece * n_all / f);
  const int it1 = (int)((int64_t)(piece + 1) * n_all / f);
  const int n = it1 - it0;
  struct Walk {
    int hh, qt, G;
    __device__ void next() { if (++hh == G) { hh = 0; ++qt; } }
  };
  const Walk walk0{it0 % a.G, qt_min + it0 / a.G, a.G};

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_q_full(s), 1);
      mbar_init(bar_q_empty(s), 1);
      mbar_init(bar_stg_full(s), 4);    // the 4 drain warps
      mbar_init(bar_stg_free(s), 1);
    }
    mbar_init(bar_do_full, 1);
    mbar_init(bar_do_empty, 1);
    mbar_init(bar_s_full, 1);
    mbar_init(bar_p_ready, 8);          // the 8 compute warps
    mbar_init(bar_dp_full, 1);
    mbar_init(bar_ds_ready, 8);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 4);         // the 4 drain warps
    mbar_init(bar_acc, 1);
    mbar_init(bar_drain_done, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q); tma_prefetch(&tm_do); tma_prefetch(&tm_k); tma_prefetch(&tm_v);
    tma_prefetch(&tm_dkv);
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
        mbar_expect_tx(bar_kv, 2 * kTile);
        SECO_CHECK_COND(k0 < (a.j + 1) * a.c && g < a.hkv, 410);   // key tile inside slots 0..j
        for (int x = 0; x < D / 64; ++x) {
          tma_load_3d(sK + x * kBox, &tm_k, bar_kv, x * 64, k0, g);
          tma_load_3d(sV + x * kBox, &tm_v, bar_kv, x * 64, k0, g);
        }
        Walk w = walk0;
        for (int i = 0; i < n; ++i, w.next()) {
          const int st = i & 1;
          const uint32_t ph = (i >> 1) & 1;
          const int h = g * a.G + w.hh, qt = w.qt;
          SECO_CHECK_COND(qt * BQ < a.c && w.hh < a.G, 412);       // query tile inside chunk j
          mbar_wait(bar_q_empty(st), ph ^ 1);
          mbar_expect_tx(bar_q_full(st), kTile + 2 * BQ * 4);
          for (int x = 0; x < D / 64; ++x)
            tma_load_3d(qbuf(st) + x * kBox, &tm_q, bar_q_full(st), x * 64, qt * BQ, h);
          const int64_t ro = (int64_t)h * a.cp + qt * BQ;
          bulk_load(sStats + st * 2 * BQ * 4, a.nlse + ro, BQ * 4, bar_q_full(st));
          bulk_load(sStats + st * 2 * BQ * 4 + BQ * 4, a.Dv + ro, BQ * 4, bar_q_full(st));
          V2TRACE(0, i);
          mbar_wait(bar_do_empty, (i & 1) ^ 1);
          mbar_expect_tx(bar_do_full, kTile);
          for (int x = 0; x < D / 64; ++x)
            tma_load_3d(sDO + x * kBox, &tm_do, bar_do_full, x * 64, qt * BQ, h);
          V2TRACE(1, i);
        }
      }
    } else if (warp == 1) {
      // -------------------------------------------------------------- MMA issuer
#if SECO_BWD_MMA_WARP
      // converged warp: every lane waits, one elected lane issues (operands stay warp-uniform)
      const bool issuer = elect_one_sync();
      {
#else
      const bool issuer = true;
      if (lane == 0) {
#endif
        constexpr uint32_t idesc_s = make_idesc_bf16(BKV, BQ, 0, 0);
        constexpr uint32_t idesc_kv = make_idesc_bf16(BKV, D, 0, 1);
        constexpr uint32_t idesc_q = make_idesc_bf16(D, BQ, 1, 1);
        // descriptors per tile base; a k-step adds its byte offset / 16 to the start-address field
        auto issue_sdp = [&](uint32_t a_base, uint32_t b_base, uint32_t d_col) {
          const uint64_t da = make_desc_sw128(a_base, 16, 1024), db = make_desc_sw128(b_base, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk / 4) * kBox + (kk % 4) * 32) >> 4;
            if (issuer) mma_ss(tmem + d_col, da + off, db + off, idesc_s, kk > 0);
          }
        };
        // A = P^T / dS^T packed in TMEM (query k-step kk at columns base + 16 kk .. +7)
        auto issue_kv = [&](uint32_t a_col, uint32_t b_base, uint32_t d_col, bool acc) {
          const uint64_t db = make_desc_sw128(b_base, kBox, 1024);
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)
            if (issuer)
              mma_ts(tmem + d_col, tmem + a_col + 16 * kk, db + (uint32_t)(kk * 2048 >> 4), idesc_kv,
                     (acc || kk > 0) ? 1u : 0u);
        };
        auto commit = [&](uint32_t bar) { if (issuer) mma_commit(bar); };
        const uint64_t dk_mn = make_desc_sw128(sK, kBox, 1024), dds_mn = make_desc_sw128(sDS, kBox, 1024);
        const uint64_t dds_k = make_desc_sw128(sDS, 16, 1024);
        mbar_wait(bar_kv, 0);
        mbar_wait(bar_q_full(0), 0);
        tc_fence_after();
        issue_sdp(sK, qbuf(0), R0);                       // S^T(0)
        commit(bar_s_full);
        mbar_wait(bar_do_full, 0);
        tc_fence_after();
        issue_sdp(sV, sDO, R1);                           // dP^T(0)
        commit(bar_dp_full);
        mbar_wait(bar_p_ready, 0);
        tc_fence_after();
        issue_kv(R0, sDO, TM_DV, false);                  // dV = P^T(0) dO(0)
        commit(bar_do_empty);
        for (int i = 0; i < n; ++i) {
          const int st = i & 1;
          const bool more = i + 1 < n;
          if (more) {                                     // S^T(i+1) -> R0 (P^T(i) consumed by dV(i))
            mbar_wait(bar_q_full(st ^ 1), ((i + 1) >> 1) & 1);
            tc_fence_after();
            issue_sdp(sK, qbuf(st ^ 1), R0);
            commit(bar_s_full);
            V2TRACE(2, i);
          }
          mbar_wait(bar_ds_ready, i & 1);
          V2TRACE(3, i);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)           // dQ^T(i) = K^T dS^T(i) -> R1 (first: it
            if (issuer)                                   // heads the serial chain)
              mma_ss(tmem + R1, dk_mn + (uint32_t)(kk * 2048 >> 4), dds_mn + (uint32_t)(kk * 2048 >> 4), idesc_q,
                     kk > 0);
          commit(bar_dq_full);
          V2TRACE(4, i);
          const uint64_t dq_mn = make_desc_sw128(qbuf(st), kBox, 1024);
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)            // dK(i) += dS^T(i) Q(i), A = dS^T from smem
            if (issuer)
              mma_ss(tmem + TM_DK, dds_k + (uint32_t)(((kk / 4) * kBox + (kk % 4) * 32) >> 4),
                     dq_mn + (uint32_t)(kk * 2048 >> 4), idesc_kv, (i > 0 || kk > 0) ? 1u : 0u);
          commit(bar_q_empty(st));
          if (more) {
            mbar_wait(bar_dq_empty, i & 1);               // dQ^T(i) drained from R1
            V2TRACE(5, i);
            mbar_wait(bar_do_full, (i + 1) & 1);
            V2TRACE(6, i);
            tc_fence_after();
            issue_sdp(sV, sDO, R1);                       // dP^T(i+1)
            commit(bar_dp_full);
            mbar_wait(bar_p_ready, (i + 1) & 1);
            V2TRACE(7, i);
            tc_fence_after();
            issue_kv(R0, sDO, TM_DV, true);               // dV += P^T(i+1) dO(i+1)
            commit(bar_do_empty);
          }
        }
        commit(bar_acc);
      }
    } else if (warp == 3) {
      // -------------------------------------------------------------- dQ reduce issuer
      if (lane == 0) {
        Walk w = walk0;
        int m = 0;                                        // staged chunk sequence number
        for (int i = 0; i < n; ++i, w.next()) {
          const int h = g * a.G + w.hh, qt = w.qt;
          float* dst = a.dqacc + ((int64_t)h * a.cp + qt * BQ) * D;
          for (int c = 0; c < 4; ++c, ++m) {
            const int s = c & 1;
            mbar_wait(bar_stg_full(s), (m >> 1) & 1);
            SECO_CHECK_COND(dst >= a.dqacc && dst + 32 * (c + 1) * D <= a.dqacc + (int64_t)a.G * a.hkv * a.cp * D, 512);
            bulk_reduce_add_f32(dst + 32 * c * D, sSTG + s * kSlot, kSlot);
            bulk_commit();
            if (c == 0) V2TRACE(16, i);
            if (c == 3) V2TRACE(17, i);
            if (m > 0) {
              bulk_wait_read<1>();                        // the previous chunk's slot was read
              mbar_arrive(bar_stg_free(s ^ 1));
            }
          }
        }
        bulk_wait_read<0>();
        mbar_arrive(bar_stg_free((m - 1) & 1));
        bulk_wait0();
        mbar_arrive(bar_drain_done);
      }
    } else if (warp >= 4 && warp < 8) {
      // -------------------------------------------------------------- dQ^T drain (lane = d)
      const int wq = warp % 4;
      const int dr = wq * 32 + lane;
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      int m = 0;
      auto stage = [&](const uint32_t (&v)[32], int s) {
        mbar_wait(bar_stg_free(s), ((m >> 1) & 1) ^ 1);
        const uint32_t base = sSTG + s * kSlot + dr * 4;
#pragma unroll
        for (int q = 0; q < 32; ++q) st_shared_f32(base + q * (D * 4), __uint_as_float(v[q]));
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_stg_full(s));
        ++m;
      };
      for (int i = 0; i < n; ++i) {
        mbar_wait(bar_dq_full, i & 1);
        if (lane == 0 && wq == 0) V2TRACE(13, i);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32(tmem + lane_addr + R1, v0);
        tmem_wait_ld();
        stage(v0, 0);
        tmem_ld32(tmem + lane_addr + R1 + 32, v1);
        tmem_wait_ld();
        stage(v1, 1);
        tmem_ld32(tmem + lane_addr + R1 + 64, v0);
        tmem_ld32(tmem + lane_addr + R1 + 96, v1);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_dq_empty);        // R1 free for dP^T(i+1)
        if (lane == 0 && wq == 0) V2TRACE(14, i);
        stage(v0, 0);
        stage(v1, 1);
        if (lane == 0 && wq == 0) V2TRACE(15, i);
      }
    } else if (warp >= 8) {
      // -------------------------------------------------------------- compute warpgroups
      const int cw = (warp - 8) / 4;                      // query columns [64 cw, 64 cw + 64)
      const int wq = warp % 4;
      const int kr = wq * 32 + lane;                      // key row within the tile
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      const int key_pos = k0 + kr;
      const f2_t sl2x2 = f2(a.scale_log2, a.scale_log2);
      Walk w = walk0;
      for (int i = 0; i < n; ++i, w.next()) {
        const int st = i & 1;
        const int qbase = a.j * a.c + w.qt * BQ;
        uint32_t pk[32];                                  // P^T of this thread's 64 queries, bf16 pairs
        // ---- phase A: P^T = exp2(S^T sigma log2e - LSE log2e) -> bf16 over R0
        mbar_wait(bar_q_full(st), (i >> 1) & 1);
        mbar_wait(bar_s_full, i & 1);
        if (lane == 0 && wq == 0 && cw == 0) V2TRACE(8, i);
        tc_fence_after();
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int c = 64 * cw + 32 * sub;
          uint32_t sv[32];
          float p[32];
          tmem_ld32(tmem + lane_addr + R0 + c, sv);
          tmem_wait_ld();
          const uint32_t nl_s = sStats + (st * 2 * BQ + c) * 4;
          const int qpos0 = qbase + c;
          const bool masked = (k0 + wq * 32 + 31) > qpos0;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 L = ld_shared_f4(nl_s + c4 * 16);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int c2 = c4 * 4 + h2 * 2;
              const f2_t x = ffma2(f2u(sv[c2], sv[c2 + 1]), sl2x2, h2 ? f2(L.z, L.w) : f2(L.x, L.y));
              float p0 = ex2(f2lo(x)), p1 = ex2(f2hi(x));
              if (masked) {
                if (key_pos > qpos0 + c2) p0 = 0.f;
                if (key_pos > qpos0 + c2 + 1) p1 = 0.f;
              }
              p[c2] = p0;
              p[c2 + 1] = p1;
            }
          }
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {               // query k-steps c/16 + k2 -> columns 16 kk .. +7
            uint32_t pp[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              pp[q] = pack_bf16(p[16 * k2 + 2 * q], p[16 * k2 + 2 * q + 1]);
              pk[16 * sub + 8 * k2 + q] = pp[q];
            }
            tmem_st8(tmem + lane_addr + R0 + c + 16 * k2, pp);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p_ready);
        if (lane == 0 && wq == 0 && cw == 0) V2TRACE(9, i);
        // ---- phase B: dS^T = P^T o (dP^T - D) (P^T as rounded for the dV MMA) -> bf16 to smem,
        // the A operand of dK and the B operand of dQ^T
        mbar_wait(bar_dp_full, i & 1);
        if (lane == 0 && wq == 0 && cw == 0) V2TRACE(10, i);
        tc_fence_after();
        uint32_t dpv[64];
        tmem_ld32(tmem + lane_addr + R1 + 64 * cw, *reinterpret_cast<uint32_t(*)[32]>(dpv));
        tmem_ld32(tmem + lane_addr + R1 + 64 * cw + 32, *reinterpret_cast<uint32_t(*)[32]>(dpv + 32));
        tmem_wait_ld();
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int c = 64 * cw + 32 * sub;
          const uint32_t d_s = sStats + (st * 2 * BQ + BQ + c) * 4;
          uint32_t dd[16];
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 Dv = ld_shared_f4(d_s + c4 * 16);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int c2 = c4 * 4 + h2 * 2;
              const uint32_t pw = pk[16 * sub + c2 / 2];
              const f2_t p2 = f2(__uint_as_float(pw << 16), __uint_as_float(pw & 0xffff0000u));
              const f2_t ds2 = fmul2(p2, fsub2(f2u(dpv[32 * sub + c2], dpv[32 * sub + c2 + 1]),
                                               h2 ? f2(Dv.z, Dv.w) : f2(Dv.x, Dv.y)));
              dd[c2 / 2] = pack_bf16_f2(ds2);
            }
          }
          // dS^T to smem: box c / 64 (query half), row kr, 16-B chunks (c % 64) / 8 .. +3
          const uint32_t drow = sDS + (c / 64) * kBox;
          const int ch = (c % 64) / 8;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(drow + sw128_off(kr, ch + q), dd[4 * q], dd[4 * q + 1], dd[4 * q + 2], dd[4 * q + 3]);
        }
        tmem_wait_st();
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_ds_ready);
        if (lane == 0 && wq == 0) V2TRACE(cw == 0 ? 11 : 12, i);
      }
      // ---- epilogue: WG 0 -> dK, WG 1 -> dV: TMEM -> scaled fp32 swizzled boxes -> TMA reduce-add
      mbar_wait(bar_acc, 0);
      mbar_wait(bar_drain_done, 0);
      tc_fence_after();
      const int mat = cw;
      const float sc = mat == 0 ? a.dk_scale : a.dv_scale;
      auto stg_box = [&](int cc) { return (mat == 0 ? sb + kQ : sDO) + (uint32_t)cc * kBox; };
#pragma unroll 1
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_addr + (mat == 0 ? TM_DK : TM_DV) + cc * 32, v);
        tmem_wait_ld();
        const uint32_t box = stg_box(cc);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_shared_v4(box + sw128_off(kr, q), __float_as_uint(sc * __uint_as_float(v[4 * q])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 1])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 2])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 3])));
      }
      fence_async_smem();
      named_bar_sync(2 + mat, 128);
      if (wq == 0 && lane == 0) {
        const int row0 = (mat * a.hkv + g) * a.S + k0;
        SECO_CHECK_COND(k0 < (a.j + 1) * a.c && row0 < 2 * a.hkv * a.S, 510);   // dKV rows
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tma_reduce_add_2d(&tm_dkv, stg_box(cc), cc * 32, row0);
        bulk_commit();
        bulk_wait0();
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================================ backward v3 (CTA pairs)
// seco_bwd3_sm100_kernel: the v2 algorithm (same MMAs, issue order, TMEM regions, drain and compute
// warps) on clusters of 2 CTAs = two adjacent key tiles (2u, 2u + 1) of one kv head that walk the
// same query tiles.  Four of the five MMAs per block run as tcgen05.mma.cta_group::2 with M = 256
// (each CTA's 128 keys), issued by the leader:
//   S^T  = K Q^T    B = Q^T: each CTA holds its 64 query rows of Q(i) (Qr)
//   dP^T = V dO^T   B = dO^T: its 64 query rows of dO(i) (dOr)
//   dV  += P^T dO   B = dO: its 64 d columns of dO(i), every query row (dOc)
//   dK  += dS^T Q   B = Q: its 64 d columns of Q(i) (Qc)
// so each SM reads half of every B operand from shared memory; dQ^T = K^T dS^T contracts over the
// keys and stays per CTA (cta_group::1, issued by each CTA's own MMA warp).  Hand-offs to the
// leader's MMA warp (both CTAs' P^T ready, dS^T ready, dQ^T drained) are remote mbarrier arrives
// with CTA-scope semantics (TMEM / smem data ordered by the tcgen05 fences and the proxy fence);
// the leader's commits reach both CTAs by multicast.  DESIGN §6.2.
namespace bwd3 {
constexpr int BKV = 128, BQ = 128, D = 128;
constexpr int kTile = 128 * 128 * 2;           // bf16 [128][128]
constexpr int kBox = 128 * 128;                // one [128 rows][128 B] box
constexpr int kHalf = 64 * 128;                // one [64 rows][128 B] box
constexpr int kK = 0;
constexpr int kV = kK + kTile;
constexpr int kQ = kV + kTile;                 // two stages of {Qr: 2 x [64][64], Qc: [128][64]}
constexpr int kQStage = 2 * kHalf + kBox;      // 32 KiB
constexpr int kDO = kQ + 2 * kQStage;          // one stage of {dOr, dOc}
constexpr int kSTG = kDO + kQStage;            // dQ staging: 2 slots x 16 KiB
constexpr int kSlot = 32 * D * 4;
constexpr int kDS = kSTG + 2 * kSlot;          // dS^T [128 keys][128 q] bf16 (2 boxes by q half)
constexpr int kStats = kDS + kTile;            // [2 stages][2][BQ] fp32 (-LSE log2e, D)
constexpr int kBar = kStats + 2 * 2 * BQ * 4;
constexpr int kNumBars = 24;
constexpr int kTmemSlot = kBar + 8 * kNumBars;
constexpr int kBytes = kTmemSlot + 16;
constexpr int kThreads = 512;
constexpr int R0 = 0, R1 = 128, TM_DK = 256, TM_DV = 384;
}  // namespace bwd3

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(bwd3::kThreads, 1)
    seco_bwd3_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                           const __grid_constant__ CUtensorMap tm_q64, const __grid_constant__ CUtensorMap tm_do64,
                           const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                           const __grid_constant__ CUtensorMap tm_dkv, const bwd::Args a) {
  using namespace bwd3;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  const uint32_t sK = sb + kK, sV = sb + kV, sDO = sb + kDO, sDS = sb + kDS, sSTG = sb + kSTG;
  auto qbuf = [&](int st) { return sb + kQ + (uint32_t)st * kQStage; };   // Qr at +0, Qc at +2 kHalf
  const uint32_t sStats = sb + kStats;
  const uint32_t b0 = sb + kBar;
  const uint32_t bar_kv = b0;
  auto bar_q_full = [&](int s) { return b0 + 8u * (1 + s); };      // leader: both CTAs' Q halves
  auto bar_q_empty = [&](int s) { return b0 + 8u * (3 + s); };     // local, multicast release
  const uint32_t bar_do_full = b0 + 8u * 5, bar_do_empty = b0 + 8u * 6;
  const uint32_t bar_s_full = b0 + 8u * 7;                          // local, multicast commit
  const uint32_t bar_p_ready = b0 + 8u * 8;                         // leader: 16 compute warps
  const uint32_t bar_dp_full = b0 + 8u * 9;                         // local, multicast commit
  const uint32_t bar_ds_ready = b0 + 8u * 10;                       // local: own dQ^T
  const uint32_t bar_dq_full = b0 + 8u * 11;                        // local: own dQ^T done
  const uint32_t bar_dq_empty = b0 + 8u * 12;                       // leader: 8 drain warps
  auto bar_stg_full = [&](int s) { return b0 + 8u * (13 + s); };
  auto bar_stg_free = [&](int s) { return b0 + 8u * (15 + s); };
  const uint32_t bar_acc = b0 + 8u * 17, bar_drain_done = b0 + 8u * 18;
  const uint32_t bar_ds_pair = b0 + 8u * 19;                        // leader: 16 compute warps
  auto bar_st_full = [&](int s) { return b0 + 8u * (20 + s); };    // local: this CTA's stats
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kTmemSlot);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = (int)cluster_ctarank();
  const bool leader = rank == 0;
  constexpr uint16_t kPair = 3;

  // work decode over pair units (clusters = blockIdx / 2); the pair walks its first tile's queries
  const int bid = (int)blockIdx.x >> 1;
  int U, piece, f;
  if (bid < a.n0) {
    U = bid; piece = 0; f = 1;
  } else if (bid < a.n0 + a.n1 * a.f1) {
    const int r = bid - a.n0;
    U = a.n0 + r / a.f1; piece = r % a.f1; f = a.f1;
  } else {
    const int r = bid - a.n0 - a.n1 * a.f1;
    U = a.n0 + a.n1 + r / a.f2; piece = r % a.f2; f = a.f2;
  }
  const int g = U % a.hkv;
  const int u = 2 * (U / a.hkv) + rank;
  const int k0 = u * BKV;
  const int nqt = (a.c + BQ - 1) / BQ;
  const int rel = 2 * (U / a.hkv) * BKV - a.j * a.c;
  const int qt_min = rel > 0 ? rel / BQ : 0;
  const int n_all = a.G * (nqt - qt_min);
  const int it0 = (int)((int64_t)piece * n_all / f);
  const int it1 = (int)((int64_t)(piece + 1) * n_all / f);
  const int n = it1 - it0;
  struct Walk {
    int hh, qt, G;
    __device__ void next() { if (++hh == G) { hh = 0; ++qt; } }
  };
  const Walk walk0{it0 % a.G, qt_min + it0 / a.G, a.G};

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_q_full(s), 1);
      mbar_init(bar_q_empty(s), 1);
      mbar_init(bar_stg_full(s), 4);    // the 4 drain warps
      mbar_init(bar_stg_free(s), 1);
      mbar_init(bar_st_full(s), 1);
    }
    mbar_init(bar_do_full, 1);
    mbar_init(bar_do_empty, 1);
    mbar_init(bar_s_full, 1);
    mbar_init(bar_p_ready, 16);         // 8 compute warps x 2 CTAs (leader's copy)
    mbar_init(bar_dp_full, 1);
    mbar_init(bar_ds_ready, 8);         // this CTA's 8 compute warps
    mbar_init(bar_ds_pair, 16);
    mbar_init(bar_dq_full, 1);
    mbar_init(bar_dq_empty, 8);         // 4 drain warps x 2 CTAs (leader's copy)
    mbar_init(bar_acc, 1);
    mbar_init(bar_drain_done, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q); tma_prefetch(&tm_do); tma_prefetch(&tm_q64); tma_prefetch(&tm_do64);
    tma_prefetch(&tm_k); tma_prefetch(&tm_v); tma_prefetch(&tm_dkv);
  }
  if (warp == 2) tmem_alloc_pair<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  cluster_sync();                      // both CTAs' barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (n > 0) {
    if (warp == 0) {
      // -------------------------------------------------------------- TMA producer (both CTAs)
      if (lane == 0) {
        mbar_expect_tx(bar_kv, 2 * kTile);
        SECO_CHECK_COND(k0 < (a.j + 1) * a.c && g < a.hkv, 413);
        for (int x = 0; x < D / 64; ++x) {
          tma_load_3d(sK + x * kBox, &tm_k, bar_kv, x * 64, k0, g);
          tma_load_3d(sV + x * kBox, &tm_v, bar_kv, x * 64, k0, g);
        }
        Walk w = walk0;
        for (int i = 0; i < n; ++i, w.next()) {
          const int st = i & 1;
          const uint32_t ph = (i >> 1) & 1;
          const int h = g * a.G + w.hh, qt = w.qt;
          SECO_CHECK_COND(qt * BQ < a.c && w.hh < a.G, 414);
          mbar_wait(bar_q_empty(st), ph ^ 1);
          if (leader) mbar_expect_tx(bar_q_full(st), 2 * kQStage);
          const uint32_t bq = mapa_shared(bar_q_full(st), 0);
          for (int x = 0; x < D / 64; ++x)      // Qr: this CTA's 64 query rows, all d
            tma_load_3d_pair(qbuf(st) + x * kHalf, &tm_q64, bq, x * 64, qt * BQ + 64 * rank, h, kHalf);
          tma_load_3d_pair(qbuf(st) + 2 * kHalf, &tm_q, bq, 64 * rank, qt * BQ, h, kBox);   // Qc
          const int64_t ro = (int64_t)h * a.cp + qt * BQ;
          mbar_expect_tx(bar_st_full(st), 2 * BQ * 4);
          bulk_load(sStats + st * 2 * BQ * 4, a.nlse + ro, BQ * 4, bar_st_full(st));
          bulk_load(sStats + st * 2 * BQ * 4 + BQ * 4, a.Dv + ro, BQ * 4, bar_st_full(st));
          mbar_wait(bar_do_empty, (i & 1) ^ 1);
          if (leader) mbar_expect_tx(bar_do_full, 2 * kQStage);
          const uint32_t bdo = mapa_shared(bar_do_full, 0);
          for (int x = 0; x < D / 64; ++x)
            tma_load_3d_pair(sDO + x * kHalf, &tm_do64, bdo, x * 64, qt * BQ + 64 * rank, h, kHalf);
          tma_load_3d_pair(sDO + 2 * kHalf, &tm_do, bdo, 64 * rank, qt * BQ, h, kBox);
        }
        // the leader's last multicast releases have landed in this CTA before the pair may exit
        for (int i = n; i < n + 2; ++i) mbar_wait(bar_q_empty(i & 1), ((i >> 1) & 1) ^ 1);
        mbar_wait(bar_do_empty, (n & 1) ^ 1);
      }
    } else if (warp == 1) {
      // -------------------------------------------------------------- MMA issuer
      // converged warp, one elected lane issues.  Leader: the pair's S^T, dP^T, dV, dK (M = 256)
      // and its own dQ^T; follower: its own dQ^T only.
      const bool issuer = elect_one_sync();
      constexpr uint32_t idesc_s = make_idesc_bf16(2 * BKV, BQ, 0, 0);
      constexpr uint32_t idesc_kv = make_idesc_bf16(2 * BKV, D, 0, 1);
      constexpr uint32_t idesc_q = make_idesc_bf16(D, BQ, 1, 1);
      const uint64_t dk_mn = make_desc_sw128(sK, kBox, 1024), dds_mn = make_desc_sw128(sDS, kBox, 1024);
      auto issue_dq = [&]() {                          // dQ^T = K^T dS^T -> R1 (this CTA)
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          if (issuer)
            mma_ss(tmem + R1, dk_mn + (uint32_t)(kk * 2048 >> 4), dds_mn + (uint32_t)(kk * 2048 >> 4), idesc_q,
                   kk > 0);
        if (issuer) mma_commit(bar_dq_full);
      };
      if (!leader) {
        for (int i = 0; i < n; ++i) {
          mbar_wait(bar_ds_ready, i & 1);
          tc_fence_after();
          issue_dq();
        }
      } else {
        // A = K / V (this CTA's 128 keys, K-major boxes of 128 rows); B = the 64-row halves
        auto issue_sdp = [&](uint32_t a_base, uint32_t b_base, uint32_t d_col) {
          const uint64_t da = make_desc_sw128(a_base, 16, 1024), db = make_desc_sw128(b_base, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            if (issuer)
              mma_ss_pair(tmem + d_col, da + (uint32_t)(((kk / 4) * kBox + (kk % 4) * 32) >> 4),
                          db + (uint32_t)(((kk / 4) * kHalf + (kk % 4) * 32) >> 4), idesc_s, kk > 0);
        };
        // A = P^T (TMEM, packed bf16); B = the d-column half (one [128 q][64 d] box, MN-major)
        auto issue_kv = [&](uint32_t a_col, uint32_t b_base, uint32_t d_col, bool acc) {
          const uint64_t db = make_desc_sw128(b_base, kBox, 1024);
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)
            if (issuer)
              mma_ts_pair(tmem + d_col, tmem + a_col + 16 * kk, db + (uint32_t)(kk * 2048 >> 4), idesc_kv,
                          (acc || kk > 0) ? 1u : 0u);
        };
        auto commit2 = [&](uint32_t bar) { if (issuer) mma_commit_pair(bar); };
        const uint64_t dds_k = make_desc_sw128(sDS, 16, 1024);
        mbar_wait(bar_kv, 0);
        mbar_wait(bar_q_full(0), 0);
        tc_fence_after();
        issue_sdp(sK, qbuf(0), R0);                       // S^T(0)
        commit2(bar_s_full);
        mbar_wait(bar_do_full, 0);
        tc_fence_after();
        issue_sdp(sV, sDO, R1);                           // dP^T(0)
        commit2(bar_dp_full);
        mbar_wait(bar_p_ready, 0);
        tc_fence_after();
        issue_kv(R0, sDO + 2 * kHalf, TM_DV, false);      // dV = P^T(0) dO(0)
        commit2(bar_do_empty);
        for (int i = 0; i < n; ++i) {
          const int st = i & 1;
          const bool more = i + 1 < n;
          if (more) {                                     // S^T(i+1) -> R0 (P^T(i) consumed by dV(i))
            mbar_wait(bar_q_full(st ^ 1), ((i + 1) >> 1) & 1);
            tc_fence_after();
            issue_sdp(sK, qbuf(st ^ 1), R0);
            commit2(bar_s_full);
          }
          mbar_wait(bar_ds_ready, i & 1);                 // own dS^T(i): own dQ^T first (heads the chain)
          tc_fence_after();
          issue_dq();
          mbar_wait(bar_ds_pair, i & 1);                  // both CTAs' dS^T(i)
          tc_fence_after();
          const uint64_t dq_mn = make_desc_sw128(qbuf(st) + 2 * kHalf, kBox, 1024);
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)            // dK(i) += dS^T(i) Q(i) (pair)
            if (issuer)
              mma_ss_pair(tmem + TM_DK, dds_k + (uint32_t)(((kk / 4) * kBox + (kk % 4) * 32) >> 4),
                          dq_mn + (uint32_t)(kk * 2048 >> 4), idesc_kv, (i > 0 || kk > 0) ? 1u : 0u);
          commit2(bar_q_empty(st));
          if (more) {
            mbar_wait(bar_dq_empty, i & 1);               // both CTAs' dQ^T(i) drained from R1
            mbar_wait(bar_do_full, (i + 1) & 1);
            tc_fence_after();
            issue_sdp(sV, sDO, R1);                       // dP^T(i+1)
            commit2(bar_dp_full);
            mbar_wait(bar_p_ready, (i + 1) & 1);
            tc_fence_after();
            issue_kv(R0, sDO + 2 * kHalf, TM_DV, true);   // dV += P^T(i+1) dO(i+1)
            commit2(bar_do_empty);
          }
        }
        commit2(bar_acc);
      }
    } else if (warp == 3) {
      // -------------------------------------------------------------- dQ reduce issuer
      if (lane == 0) {
        Walk w = walk0;
        int m = 0;
        for (int i = 0; i < n; ++i, w.next()) {
          const int h = g * a.G + w.hh, qt = w.qt;
          float* dst = a.dqacc + ((int64_t)h * a.cp + qt * BQ) * D;
          for (int c = 0; c < 4; ++c, ++m) {
            const int s = c & 1;
            mbar_wait(bar_stg_full(s), (m >> 1) & 1);
            SECO_CHECK_COND(dst >= a.dqacc && dst + 32 * (c + 1) * D <= a.dqacc + (int64_t)a.G * a.hkv * a.cp * D, 513);
            bulk_reduce_add_f32(dst + 32 * c * D, sSTG + s * kSlot, kSlot);
            bulk_commit();
            if (m > 0) {
              bulk_wait_read<1>();
              mbar_arrive(bar_stg_free(s ^ 1));
            }
          }
        }
        bulk_wait_read<0>();
        mbar_arrive(bar_stg_free((m - 1) & 1));
        bulk_wait0();
        mbar_arrive(bar_drain_done);
      }
    } else if (warp >= 4 && warp < 8) {
      // -------------------------------------------------------------- dQ^T drain (lane = d)
      const int wq = warp % 4;
      const int dr = wq * 32 + lane;
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      const uint32_t dq_empty_l = mapa_shared(bar_dq_empty, 0);
      int m = 0;
      auto stage = [&](const uint32_t (&v)[32], int s) {
        mbar_wait(bar_stg_free(s), ((m >> 1) & 1) ^ 1);
        const uint32_t base = sSTG + s * kSlot + dr * 4;
#pragma unroll
        for (int q = 0; q < 32; ++q) st_shared_f32(base + q * (D * 4), __uint_as_float(v[q]));
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_stg_full(s));
        ++m;
      };
      for (int i = 0; i < n; ++i) {
        mbar_wait(bar_dq_full, i & 1);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32(tmem + lane_addr + R1, v0);
        tmem_wait_ld();
        stage(v0, 0);
        tmem_ld32(tmem + lane_addr + R1 + 32, v1);
        tmem_wait_ld();
        stage(v1, 1);
        tmem_ld32(tmem + lane_addr + R1 + 64, v0);
        tmem_ld32(tmem + lane_addr + R1 + 96, v1);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(dq_empty_l);   // R1 free for the pair's dP^T(i+1)
        stage(v0, 0);
        stage(v1, 1);
      }
    } else if (warp >= 8) {
      // -------------------------------------------------------------- compute warpgroups (as v2)
      const int cw = (warp - 8) / 4;
      const int wq = warp % 4;
      const int kr = wq * 32 + lane;
      const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
      const int key_pos = k0 + kr;
      const f2_t sl2x2 = f2(a.scale_log2, a.scale_log2);
      const uint32_t p_ready_l = mapa_shared(bar_p_ready, 0), ds_pair_l = mapa_shared(bar_ds_pair, 0);
      Walk w = walk0;
      for (int i = 0; i < n; ++i, w.next()) {
        const int st = i & 1;
        const int qbase = a.j * a.c + w.qt * BQ;
        uint32_t pk[32];
        // ---- phase A: P^T = exp2(S^T sigma log2e - LSE log2e) -> bf16 over R0
        mbar_wait(bar_st_full(st), (i >> 1) & 1);
        mbar_wait(bar_s_full, i & 1);
        tc_fence_after();
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int c = 64 * cw + 32 * sub;
          uint32_t sv[32];
          float p[32];
          tmem_ld32(tmem + lane_addr + R0 + c, sv);
          tmem_wait_ld();
          const uint32_t nl_s = sStats + (st * 2 * BQ + c) * 4;
          const int qpos0 = qbase + c;
          const bool masked = (k0 + wq * 32 + 31) > qpos0;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 L = ld_shared_f4(nl_s + c4 * 16);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int c2 = c4 * 4 + h2 * 2;
              const f2_t x = ffma2(f2u(sv[c2], sv[c2 + 1]), sl2x2, h2 ? f2(L.z, L.w) : f2(L.x, L.y));
              float p0 = ex2(f2lo(x)), p1 = ex2(f2hi(x));
              if (masked) {
                if (key_pos > qpos0 + c2) p0 = 0.f;
                if (key_pos > qpos0 + c2 + 1) p1 = 0.f;
              }
              p[c2] = p0;
              p[c2 + 1] = p1;
            }
          }
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {
            uint32_t pp[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              pp[q] = pack_bf16(p[16 * k2 + 2 * q], p[16 * k2 + 2 * q + 1]);
              pk[16 * sub + 8 * k2 + q] = pp[q];
            }
            tmem_st8(tmem + lane_addr + R0 + c + 16 * k2, pp);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(p_ready_l);
        // ---- phase B: dS^T = P^T o (dP^T - D) -> bf16 to smem
        mbar_wait(bar_dp_full, i & 1);
        tc_fence_after();
        uint32_t dpv[64];
        tmem_ld32(tmem + lane_addr + R1 + 64 * cw, *reinterpret_cast<uint32_t(*)[32]>(dpv));
        tmem_ld32(tmem + lane_addr + R1 + 64 * cw + 32, *reinterpret_cast<uint32_t(*)[32]>(dpv + 32));
        tmem_wait_ld();
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int c = 64 * cw + 32 * sub;
          const uint32_t d_s = sStats + (st * 2 * BQ + BQ + c) * 4;
          uint32_t dd[16];
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 Dv = ld_shared_f4(d_s + c4 * 16);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int c2 = c4 * 4 + h2 * 2;
              const uint32_t pw = pk[16 * sub + c2 / 2];
              const f2_t p2 = f2(__uint_as_float(pw << 16), __uint_as_float(pw & 0xffff0000u));
              const f2_t ds2 = fmul2(p2, fsub2(f2u(dpv[32 * sub + c2], dpv[32 * sub + c2 + 1]),
                                               h2 ? f2(Dv.z, Dv.w) : f2(Dv.x, Dv.y)));
              dd[c2 / 2] = pack_bf16_f2(ds2);
            }
          }
          const uint32_t drow = sDS + (c / 64) * kBox;
          const int ch = (c % 64) / 8;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(drow + sw128_off(kr, ch + q), dd[4 * q], dd[4 * q + 1], dd[4 * q + 2], dd[4 * q + 3]);
        }
        tmem_wait_st();
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(bar_ds_ready);
          mbar_arrive_remote(ds_pair_l);
        }
      }
      // ---- epilogue: WG 0 -> dK, WG 1 -> dV (this CTA's keys)
      mbar_wait(bar_acc, 0);
      mbar_wait(bar_drain_done, 0);
      tc_fence_after();
      const int mat = cw;
      const float sc = mat == 0 ? a.dk_scale : a.dv_scale;
      auto stg_box = [&](int cc) { return (mat == 0 ? sb + kQ : sDO) + (uint32_t)cc * kBox; };
#pragma unroll 1
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_addr + (mat == 0 ? TM_DK : TM_DV) + cc * 32, v);
        tmem_wait_ld();
        const uint32_t box = stg_box(cc);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_shared_v4(box + sw128_off(kr, q), __float_as_uint(sc * __uint_as_float(v[4 * q])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 1])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 2])),
                       __float_as_uint(sc * __uint_as_float(v[4 * q + 3])));
      }
      fence_async_smem();
      named_bar_sync(2 + mat, 128);
      if (wq == 0 && lane == 0) {
        const int row0 = (mat * a.hkv + g) * a.S + k0;
        SECO_CHECK_COND(k0 < (a.j + 1) * a.c && row0 < 2 * a.hkv * a.S, 514);
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tma_reduce_add_2d(&tm_dkv, stg_box(cc), cc * 32, row0);
        bulk_commit();
        bulk_wait0();
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();                      // neither CTA leaves while the pair still uses its smem / TMEM
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
}

namespace {
// ---- work list for one backward call (host side) ------------------------------------------
// Units (key tile u of kv-head g) cost G * (query tiles that see the tile) 128x128 blocks: the
// cache-slot tiles all G c / 128, the diagonal slot's tiles G c / 128 ... G.  One CTA runs per
// SM and the hardware hands blocks out in index order, so the call's time is that of list
// scheduling the work list on the SMs.  Whole units first (longest first), then the last units
// split into f1, then f2 query-range pieces (each piece reduce-adds its own dK/dV share), so the
// last wave is made of short pieces.  (n0, n1, f1, f2) minimise the simulated makespan with a
// per-piece overhead of kItemOverhead blocks (prologue, K/V load, dK/dV epilogue);
// deterministic mode keeps whole units (one owner per dK/dV tile).
struct Schedule { int n0, n1, f1, f2, grid; };

float item_overhead() {
  static const float o = [] {
    const char* e = std::getenv("SECO_BWD_ITEM_OVERHEAD");   // tuning experiments only
    return e ? (float)std::atof(e) : 3.0f;
  }();
  return o;
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
                                                cudaSuccess || n <= 0)
    return 148;
  return n;
}

// makespan of list-scheduling `pieces` (in order) onto P machines whose busy-until times are `t0`
float list_makespan(std::vector<float> t, const std::vector<float>& pieces) {
  std::make_heap(t.begin(), t.end(), std::greater<float>());
  for (float p : pieces) {
    std::pop_heap(t.begin(), t.end(), std::greater<float>());
    t.back() += p;
    std::push_heap(t.begin(), t.end(), std::greater<float>());
  }
  return *std::max_element(t.begin(), t.end());
}

// pair = true: units are pairs of adjacent key tiles run by a cluster of 2 CTAs (P / 2 machines),
// costed by the query walk of their first tile
Schedule compute_schedule(int c, int j, int hkv, int G, int P, bool pair = false) {
  const int nqt = (c + bwd::BQ - 1) / bwd::BQ, ntiles = ((j + 1) * c + bwd::BKV - 1) / bwd::BKV / (pair ? 2 : 1),
            N = ntiles * hkv;
  if (pair) P /= 2;
  const float o = item_overhead();
  auto unit_blocks = [&](int U) {
    const int rel = (U / hkv) * bwd::BKV * (pair ? 2 : 1) - j * c;
    return G * (nqt - (rel > 0 ? rel / bwd::BQ : 0));
  };
  auto add_pieces = [&](std::vector<float>& out, int U, int f) {
    const int nb = unit_blocks(U);
    for (int p = 0; p < f; ++p) {
      const int b = (int)((int64_t)(p + 1) * nb / f - (int64_t)p * nb / f);
      out.push_back(b > 0 ? b + o : 0.25f * o);
    }
  };
  Schedule best{N, 0, 1, 1, N};
  float best_t;
  {
    std::vector<float> all;
    for (int U = 0; U < N; ++U) add_pieces(all, U, 1);
    best_t = list_makespan(std::vector<float>(P, 0.f), all);
  }
  // split candidates: the last n12 units (all of them if the call has <= 2 waves of units,
  // then in steps of 8); the
  // busy-until state after the whole-unit prefix is extended incrementally as n12 shrinks
  const int kStep = 8;
  const int max12 = std::min(N, 2 * P);
  static const int kF[][2] = {{2, 2}, {4, 4}, {8, 8}, {2, 4}, {2, 8}, {4, 8}};
  std::vector<float> t(P, 0.f), head, tail;
  auto push_all = [&](const std::vector<float>& pcs) {
    for (float p : pcs) {
      std::pop_heap(t.begin(), t.end(), std::greater<float>());
      t.back() += p;
      std::push_heap(t.begin(), t.end(), std::greater<float>());
    }
  };
  std::make_heap(t.begin(), t.end(), std::greater<float>());
  for (int U = 0; U < N - max12; ++U) add_pieces(head, U, 1);
  push_all(head);
  for (int n12 = max12; n12 >= 1; n12 -= kStep) {
    const int n0 = N - n12;
    if (n12 < max12) {
      head.clear();
      for (int U = n0 - kStep; U < n0; ++U) add_pieces(head, U, 1);
      push_all(head);
    }
    for (const auto& ff : kF) {
      for (int n2 = 0; n2 <= n12; n2 += 2 * kStep) {
        if (ff[0] == ff[1] && n2 > 0) break;   // one split factor: n2 is immaterial
        tail.clear();
        for (int U = n0; U < n0 + n12 - n2; ++U) add_pieces(tail, U, ff[0]);
        for (int U = n0 + n12 - n2; U < N; ++U) add_pieces(tail, U, ff[1]);
        const float m = list_makespan(t, tail);
        if (m < best_t * 0.999f) {
          best_t = m;
          best = Schedule{n0, n12 - n2, ff[0], ff[1], n0 + (n12 - n2) * ff[0] + n2 * ff[1]};
        }
      }
    }
  }
  return best;
}

Schedule choose_schedule(int c, int j, int hkv, int G, int P, bool pair = false) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int>, Schedule> cache;
  const auto key = std::make_tuple(c, j, hkv, G, P, (int)pair);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const Schedule s = compute_schedule(c, j, hkv, G, P, pair);
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, s);
  return s;
}
}  // namespace

extern "C" int32_t seco_debug_bwd_schedule(int32_t c, int32_t j, int32_t hkv, int32_t G, int32_t P, int32_t* out4) {
  const Schedule s = choose_schedule(c, j, hkv, G, P);
  out4[0] = s.n0; out4[1] = s.n1; out4[2] = s.f1; out4[3] = s.f2;
  return s.grid;
}

cudaError_t launch_bwd_sm100(const ChunkGeom& g, const CUtensorMap& tq, const CUtensorMap& tdo,
                             const CUtensorMap& tq64, const CUtensorMap& tdo64,
                             const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tdq,
                             const CUtensorMap& tdkv, const void* o, const void* d_o,
                             const float* lse, float relay, float gscale, float* dkv, void* dq, void* dk_own,
                             void* dv_own, float* ws_dqacc, float* ws_D, cudaStream_t st, int* launches) {
  static_assert(bwd::kBytes <= 232448 && bwd2::kBytes <= 232448 && bwd3::kBytes <= 232448, "shared memory budget");
  // d = 64 runs on zero-padded 128-column tiles (TMA out-of-bounds fill on load; the dK/dV
  // reduce-add boxes past column 64 are dropped by the same bounds check; dQacc rows are 128)
  if (g.d > bwd::D || g.d % 32 || g.cp % bwd::BQ) return cudaErrorInvalidValue;
  int* order = g.det ? reinterpret_cast<int*>(ws_D + 2 * (size_t)g.hq * g.cp) : nullptr;
  cudaError_t e = launch_prep_bf16(g, o, d_o, ws_D, dkv, ws_dqacc, lse, ws_D + (size_t)g.hq * g.cp, relay, st, order);
  if (e != cudaSuccess) return e;
  static std::atomic<unsigned long long> attr_done{0}, attr_done2{0};
  static const bool v2 = [] {
    const char* e2 = std::getenv("SECO_BWD_V2");   // A/B switch: SECO_BWD_V2=0 selects the v1 kernel
    return e2 == nullptr || e2[0] != '0';
  }();
  const bool use_v2 = v2 && !g.det;
  if ((e = use_v2 ? ensure_smem_attr(seco_bwd2_sm100_kernel, bwd2::kBytes, attr_done2)
                  : ensure_smem_attr(seco_bwd_sm100_kernel, bwd::kBytes, attr_done)) != cudaSuccess)
    return e;
  bwd::Args a;
  a.c = g.c; a.j = g.j; a.G = g.hq / g.hkv; a.hkv = g.hkv; a.S = g.c * g.k; a.cp = g.cp;
  a.scale_log2 = g.scale * 1.4426950408889634f;
  a.dk_scale = gscale * g.scale;
  a.dv_scale = gscale;
  a.nlse = ws_D + (size_t)g.hq * g.cp; a.Dv = ws_D; a.dqacc = ws_dqacc; a.dq_order = order;
  a.ticket = order ? order + (size_t)g.hq * ((g.c + bwd::BQ - 1) / bwd::BQ) : nullptr;   // zeroed with the counters
  a.err = nullptr;
  a.trace = nullptr;
#ifdef SECO_TRACE
  {
    static unsigned long long* tbuf = nullptr;
    const size_t nb = sizeof(unsigned long long) * bwd::kTraceCtas * bwd::kTraceSlots * bwd::kTraceIters;
    if (!tbuf) cudaMalloc(&tbuf, nb);
    cudaMemsetAsync(tbuf, 0, nb, st);
    a.trace = tbuf;
    seco_trace_buffer = tbuf;
  }
#endif
  const int ntiles = ((g.j + 1) * g.c + bwd::BKV - 1) / bwd::BKV;
  // CTA pairs (v3, cta_group::2 MMAs over two adjacent key tiles) need an even number of key tiles
  const bool pair = use_v2 && ntiles % 2 == 0 && bwd_uses_pair(g);
  static std::atomic<unsigned long long> attr_done3{0};
  if (pair && (e = ensure_smem_attr(seco_bwd3_sm100_kernel, bwd3::kBytes, attr_done3)) != cudaSuccess) return e;
  const Schedule sc = g.det ? Schedule{ntiles * g.hkv, 0, 1, 1, ntiles * g.hkv}   // one owner per dK/dV tile
                           : choose_schedule(g.c, g.j, g.hkv, a.G, num_sms(), pair);
  a.n0 = sc.n0; a.n1 = sc.n1; a.f1 = sc.f1; a.f2 = sc.f2;
  dim3 grid(sc.grid * (pair ? 2 : 1));
  if (pair)
    seco_bwd3_sm100_kernel<<<grid, bwd3::kThreads, bwd3::kBytes, st>>>(tq, tdo, tq64, tdo64, tk, tv, tdkv, a);
  else if (use_v2)
    seco_bwd2_sm100_kernel<<<grid, bwd2::kThreads, bwd2::kBytes, st>>>(tq, tdo, tk, tv, tdkv, a);
  else
    seco_bwd_sm100_kernel<<<grid, bwd::kThreads, bwd::kBytes, st>>>(tq, tdo, tk, tv, tdq, tdkv, a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  e = launch_final_bf16(g, ws_dqacc, dq, dkv, dk_own, dv_own, gscale * g.scale, st);
  *launches = 2 + 1;
  return e;
}

bool bwd_uses_pair(const ChunkGeom& g) {
  // SECO_BWD_PAIR=1 selects the CTA-pair backward (v3), =0 the single-CTA v2 (A/B switch)
  static const int mode = [] {
    const char* e = std::getenv("SECO_BWD_PAIR");
    return e == nullptr ? -1 : (e[0] == '0' ? 0 : 1);
  }();
  const bool on = mode >= 0 ? mode == 1 : SECO_BWD_PAIR_DEFAULT != 0;
  return on && !g.det && g.d <= 128 && g.d % 32 == 0 && g.c % 128 == 0;   // whole query tiles only
}

unsigned long long check_word_bwd() { return seco_check_read_clear(); }

}  // namespace seco
