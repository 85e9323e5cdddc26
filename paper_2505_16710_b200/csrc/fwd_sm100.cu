// Chunk forward on sm_100a tensor cores: O_j, LSE_j of chunk j against KV-cache
// slots 0..j (Eq. 1; Alg. 1 lines 2 and 5), bf16 in, fp32
// accumulate, online softmax.
//
// One CTA = one 128-row query tile of chunk j for NH q-heads of the same kv-head
// group (GQA: the NH tiles share every K/V tile loaded into shared memory).
// Warp roles (warp-uniform dispatch):
//   warp 0        TMA producer: Q tiles once, then K_t, V_t through a STAGES-deep ring
//   warp 1        MMA issuer (converged warp, one elected lane issues): S_b = Q_b K_t^T (SS) and
//                 O_b += P_b V_t (TS: P_b
//                 is read straight from tensor memory)
//   warp 2        TMEM allocator
//   warps 4..     one 128-thread softmax warpgroup per q-head tile b (thread = query row):
//                 tcgen05.ld S_b, online softmax in the log2 domain, P_b (bf16) written back
//                 over S_b's first 64 TMEM columns with tcgen05.st, lazy O rescale in TMEM,
//                 epilogue O/l -> global, LSE.  A fixed share of the exponentials runs as a
//                 polynomial on the FMA pipe (ex2_emu2) to relieve the MUFU unit.
// MMA issue order ping-pongs the NH tiles: PV_0(t), S_0(t+1), PV_1(t), S_1(t+1), ...
// so the softmax of one tile overlaps tensor-core work of the other.  S_b(t+1) may
// overwrite P_b(t) because tcgen05.mma from one thread executes in issue order.
// TMEM: S_b / P_b at columns [128b, 128b+128), O_b at [128 NH + D b, ... + D).
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

#ifndef SECO_FWD_PAIR_STAGES
#define SECO_FWD_PAIR_STAGES 8   // K / V half-tile ring slots of the pair kernel (16 KiB each)
#endif

namespace seco {

#ifdef SECO_TRACE
unsigned long long* seco_fwd_trace_buffer = nullptr;
extern "C" void* seco_debug_fwd_trace_ptr() { return seco_fwd_trace_buffer; }
#endif

namespace fwd {
constexpr int BM = 128;  // query rows per tile (= UMMA M)
constexpr int BN = 128;  // keys per K/V tile (= UMMA N of S, K of PV)
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only when the max grows by > 2^8
#ifndef SECO_FWD_EMU
#define SECO_FWD_EMU 2
#endif
constexpr int kEmuPairs = SECO_FWD_EMU;     // of every 8 exponential pairs, this many use ex2_emu2
#ifndef SECO_FWD_EMU2
#define SECO_FWD_EMU2 0
#endif
constexpr int kEmuPairs2 = SECO_FWD_EMU2;   // the same for the part released second (MUFU only)
#ifndef SECO_FWD_PDL
#define SECO_FWD_PDL 1
#endif
constexpr int kSMs = 148;                  // B200
#ifndef SECO_FWD_SPLIT
#define SECO_FWD_SPLIT 3
#endif
#ifndef SECO_FWD_NAMED_P
#define SECO_FWD_NAMED_P 1
#endif
#ifndef SECO_FWD_MMA_WARP
#define SECO_FWD_MMA_WARP 1
#endif
#ifndef SECO_FWD_MAXCH
#define SECO_FWD_MAXCH 4
#endif
#ifndef SECO_FWD_PROD_SLEEP
#define SECO_FWD_PROD_SLEEP 200
#endif
#ifndef SECO_FWD_LSUM_AFTER
#define SECO_FWD_LSUM_AFTER 1
#endif
// P is released to the MMA warp in two parts: 32-key chunks [0, kSplit) and [kSplit, 4)
constexpr int kSplit = SECO_FWD_SPLIT;

template <int NH, int D, int STAGES>
struct Layout {
  static constexpr int kTileBytes = BM * D * 2;       // Q tile, K tile, V tile (bf16)
  static constexpr int kQ = 0;
  static constexpr int kKV = kQ + NH * kTileBytes;
  static constexpr int kBar = kKV + STAGES * kTileBytes;
  // barriers: q[NH], kv_full[STAGES], kv_empty[STAGES], s_full[NH], p_half[NH][2], o_full[NH]
  static constexpr int kNumBars = NH + 2 * STAGES + 4 * NH;
  static constexpr int kTmemSlot = kBar + 8 * kNumBars;
  static constexpr int kBytes = kTmemSlot + 16;
  static constexpr int kAlloc = kBytes + 1024;  // slack for 1024-B alignment
  static constexpr int kTmemCols = (NH * (BN + D) <= 256) ? 256 : 512;
  static constexpr int kThreads = 128 + 128 * NH;
};

struct Args {
  int c, j, hq, G, nqt, nhp;  // chunk size, chunk index, q heads, group size, q tiles, head packs
  int cp;                     // rows per head of the split-KV partials: c rounded up to 128
  int nsplit;                 // split-KV factor of the units past n_full (1: no split)
  int n_full;                 // work items [0, n_full) are whole units (final O / LSE written
                              // directly); the rest are nsplit key-range pieces per unit
  int n_units;                // work units (query tile x head pack, or x head quad for pairs)
  int merge;                  // 1: the split units' last pieces merge in-kernel (DP + split
                              // tail); 0: the combine kernel merges (sub-wave split)
  int d_out;                  // head dim of the O buffer (64: the D = 128 tile is zero-padded)
  int wait_prev;              // PDL launch without SECO_FLAG_PREV_INDEPENDENT: wait for the
                              // predecessor grid before the first global access
  float scale_log2;           // sigma * log2(e)
  int64_t qh, qr;             // o strides (elements)
  float* part_o;              // nsplit > 1: [nsplit][hq][c][D] fp32 normalised partial O
  float* part_lse;            // nsplit > 1: [nsplit][hq][c] partial LSE (natural log)
  int* cnt;                   // nsplit > 1: pieces done per split CTA-unit (zeroed before launch)
  unsigned long long* trace;  // SECO_TRACE builds only: [kTraceCtas][kTraceSlots][kTraceIters]
};
#ifdef SECO_TRACE
constexpr int kTraceCtas = 2, kTraceSlots = 24, kTraceIters = 256;
#endif

// weak global loads that skip L1: data other CTAs of this grid wrote (after the acquire fence).
// __ldcg compiles to a strong (LDG.STRONG.GPU) load, which ptxas does not batch.
__device__ __forceinline__ float4 ld_na_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_na_f32(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ctaid_x() {   // a fresh read (volatile: not CSE'd with earlier ones)
  uint32_t x;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(x));
  return x;
}

// work item w -> (unit, key-range piece, pieces of that unit): [0, n_full) whole units, then
// the pieces of the remaining units, piece-major (every unit's first key range, then every
// unit's second, ...) so the CTAs running at the same time stream the same K/V tiles
// through L2, as the whole units of a wave do
struct Work {
  int unit, split, ns;
};
__device__ __forceinline__ Work decode_work(int w, const Args& a) {
  if (w < a.n_full) return Work{w, 0, 1};
  const int r = w - a.n_full, rem = a.n_units - a.n_full;
  return Work{a.n_full + r % rem, r / rem, a.nsplit};
}

// Split-KV merge (§8 a9), in two steps.  piece_done: every softmax thread (NH warpgroups) of a
// piece calls it after storing its normalised partial rows (O_s, LSE_s); the piece that
// completes its CTA-unit last (counter ci) sets the flag.  Release: every thread fences its own
// stores before the barrier that precedes the counter increment; acquire: the last piece's
// counting thread fences after observing the count, and every merging thread fences again.
template <int NH>
__device__ __forceinline__ void piece_done(const Args& a, int ci, int ns, volatile int* s_flag) {
  constexpr uint32_t kBarMerge = 7;
  __threadfence();
  named_bar_sync(kBarMerge, 128 * NH);
  if (threadIdx.x % (128 * NH) == 0) {
    const bool last = atomicAdd(a.cnt + ci, 1) == ns - 1;
    if (last) __threadfence();
    *s_flag = last ? 1 : 0;
  }
}
// merge_rows: after the CTA's final barrier, the last piece merges rows of heads h_first ..
// h_first + NH - 1, query rows row0 .. row0 + 127:
//   O = sum_s e^{LSE_s - LSE} O_s,  LSE = log sum_s e^{LSE_s},
// reading all parts back in part order, so the result does not depend on which piece came
// last (the stage-2 rebuild reproduces stage 1 bit for bit).  The parts, written by other SMs
// (possibly on the other die), come in by bulk copies into the now idle shared memory (sbuf,
// >= 2 x 66 KiB + 16 B): 32-row chunks of every part's O rows and LSE, double-buffered; then
// one warp per row, each lane 4 of the 128 columns.  (Register-staged loads of the same data
// took ~15 us per merging CTA: too few bytes in flight to cover the cross-die latency.)
template <int NH>
__device__ __forceinline__ void merge_rows(const Args& a, int ns, int h_first, int row0, uint32_t sbuf,
                                           __nv_bfloat16* __restrict__ o, float* __restrict__ lse) {
  constexpr int kRows = 32, kChunks = NH * 128 / kRows;
  constexpr uint32_t kPartO = kRows * 128 * 4;               // one part's O rows of a chunk (16 KiB)
  constexpr uint32_t kBuf = 4 * kPartO + 4 * kRows * 4;       // <= 4 parts' O rows + LSE
  const uint32_t bar = sbuf + 2 * kBuf;
  const int64_t plane = (int64_t)a.hq * a.cp;              // parts: [ns][hq][cp] rows
  auto first_row = [&](int ch) { return (int64_t)(h_first + ch * kRows / 128) * a.cp + row0 + ch * kRows % 128; };
  auto issue = [&](int ch) {                                  // one thread
    const int64_t w0 = first_row(ch);
    const uint32_t b = bar + 8 * (ch & 1), dst = sbuf + (ch & 1) * kBuf;
    mbar_expect_tx(b, ns * (kPartO + kRows * 4));
    for (int p = 0; p < ns; ++p) {
      bulk_load(dst + p * kPartO, a.part_o + (p * plane + w0) * 128, kPartO, b);
      bulk_load(dst + 4 * kPartO + p * kRows * 4, a.part_lse + p * plane + w0, kRows * 4, b);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    fence_barrier_init();
    __threadfence();                                          // acquire, as the counting thread did
    fence_proxy_async_global();                               // other SMs' generic stores -> bulk reads
    issue(0);
    if (kChunks > 1) issue(1);
  }
  __syncthreads();
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32, nw = blockDim.x / 32;
#pragma unroll 1
  for (int ch = 0; ch < kChunks; ++ch) {
    mbar_wait(bar + 8 * (ch & 1), (ch >> 1) & 1);
    const uint32_t src = sbuf + (ch & 1) * kBuf;
    const int64_t w0 = first_row(ch);
#pragma unroll 1
    for (int k = wid; k < kRows; k += nw) {
      float lp[4], mx = -INFINITY, den = 0.f;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        lp[p] = p < ns ? ld_shared_f32(src + 4 * kPartO + (p * kRows + k) * 4) : -INFINITY;
        mx = fmaxf(mx, lp[p]);
      }
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (p >= ns) break;
        const float wk = __expf(lp[p] - mx);
        den += wk;
        const float4 v = ld_shared_f4(src + p * kPartO + k * 512 + 16 * lane);
        acc.x += wk * v.x; acc.y += wk * v.y; acc.z += wk * v.z; acc.w += wk * v.w;
      }
      const float inv = 1.f / den;
      const int64_t w = w0 + k;                               // = h * cp + row (a chunk stays in one head)
      const int64_t h = w / a.cp, row = w % a.cp;
      if (row >= a.c) continue;                               // padded rows of a ragged last tile
      if (4 * lane < a.d_out)
        *reinterpret_cast<uint2*>(o + h * a.qh + row * a.qr + 4 * lane) =
            make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
      if (lane == 0) lse[h * a.c + row] = mx + __logf(den);
    }
    __syncthreads();                                          // buffer ch & 1 consumed
    if (threadIdx.x == 0 && ch + 2 < kChunks) issue(ch + 2);
  }
}
}  // namespace fwd

template <int NH, int D, int STAGES>
__global__ void __launch_bounds__(fwd::Layout<NH, D, STAGES>::kThreads, 1)
    seco_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ o,
                          float* __restrict__ lse, const fwd::Args a) {
  using L = fwd::Layout<NH, D, STAGES>;
  constexpr int HALVES = D / 64;       // 64-element (128 B) swizzle boxes per row
  constexpr int BOX = 128 * 128;       // bytes of one [128 rows][128 B] box
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase + L::kQ, sKV = sbase + L::kKV;
  const uint32_t bar0 = sbase + L::kBar;
  auto bar_q = [&](int b) { return bar0 + 8u * b; };
  auto bar_kv_full = [&](int s) { return bar0 + 8u * (NH + s); };
  auto bar_kv_empty = [&](int s) { return bar0 + 8u * (NH + STAGES + s); };
  auto bar_s_full = [&](int b) { return bar0 + 8u * (NH + 2 * STAGES + b); };
  // p_half(b, 0/1): P_b for keys [0, 32 kSplit) / [32 kSplit, 128) is in TMEM (one arrival per
  // softmax warp)
  auto bar_p_half = [&](int b, int hf) { return bar0 + 8u * (2 * NH + 2 * STAGES + 2 * b + hf); };
  auto bar_o_full = [&](int b) { return bar0 + 8u * (4 * NH + 2 * STAGES + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#ifdef SECO_TRACE
#define FTRACE(slot, i)                                                                                      \
  do {                                                                                                       \
    if (a.trace && blockIdx.x < fwd::kTraceCtas && (i) < fwd::kTraceIters)                                   \
      a.trace[((size_t)blockIdx.x * fwd::kTraceSlots + (slot)) * fwd::kTraceIters + (i)] = clock64();       \
  } while (0)
#else
#define FTRACE(slot, i) do { } while (0)
#endif
  // heavier query tiles first (longest-processing-time order): whole units, then the pieces of
  // the split ones (split-KV part innermost)
  const fwd::Work wk = fwd::decode_work((int)blockIdx.x, a);
  const int unit = wk.unit, split = wk.split, ns = wk.ns;
  const int qt = a.nqt - 1 - unit / a.nhp;
  const int hp = unit % a.nhp;
  const int h0 = hp * NH, g = h0 / a.G;
  const int q0 = a.j * a.c + qt * fwd::BM;  // absolute position of the tile's first row
  const int nvalid = min(fwd::BM, a.c - qt * fwd::BM);   // rows inside the chunk (ragged last tile)
  const int T = (q0 + nvalid - 1) / fwd::BN + 1;         // K/V tiles 0..T-1 (the last one or two
                                                         // straddle the causal diagonal)
  const int t0 = T * split / ns;            // this CTA's K/V tiles: [t0, t0 + nT)
  const int nT = T * (split + 1) / ns - t0;

  if (threadIdx.x == 0) {
    *reinterpret_cast<volatile int*>(smem + L::kTmemSlot + 8) = 0;   // split-KV: "this piece merges"
    for (int b = 0; b < NH; ++b) mbar_init(bar_q(b), 1);
    for (int s = 0; s < STAGES; ++s) { mbar_init(bar_kv_full(s), 1); mbar_init(bar_kv_empty(s), 1); }
    for (int b = 0; b < NH; ++b) {
      mbar_init(bar_s_full(b), 1);
      mbar_init(bar_p_half(b, 0), 4);
      mbar_init(bar_p_half(b, 1), 4);
      mbar_init(bar_o_full(b), 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tm_q); tma_prefetch(&tm_k); tma_prefetch(&tm_v); }
#if SECO_FWD_PDL
  // Programmatic dependent launch: the next kernel in the stream may start on SMs this grid
  // leaves idle (its last, partial wave).  A following forward launched with
  // SECO_FLAG_PREV_INDEPENDENT (the next chunk's forward in stage 1) fills this tail; any
  // other follower either waits (griddepcontrol.wait) or is a plain launch, which starts
  // only after this grid completed.  A forward that must wait for its own predecessor
  // triggers only after that wait (below), so a flagged follower -- which trusts this grid,
  // not the one before it -- never starts while that earlier kernel may still be writing.
  if (!a.wait_prev) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  if (warp == 2) tmem_alloc<L::kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#if SECO_FWD_PDL
  // Without the caller's SECO_FLAG_PREV_INDEPENDENT promise the predecessor may still be
  // writing Q / K / V (or reading O / LSE): only the prologue above overlaps it.
  if (a.wait_prev) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
#endif

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      SECO_CHECK_COND(qt * fwd::BM < a.c && h0 + NH <= a.hq, 420);                // query tile inside chunk j
      SECO_CHECK_COND(t0 >= 0 && (t0 + nT - 1) * fwd::BN < (a.j + 1) * a.c, 421); // key tiles inside slots 0..j
      for (int b = 0; b < NH; ++b) {
        mbar_expect_tx(bar_q(b), L::kTileBytes);
        for (int x = 0; x < HALVES; ++x)
          tma_load_3d(sQ + b * L::kTileBytes + x * BOX, &tm_q, bar_q(b), x * 64, qt * fwd::BM, h0 + b);
      }
      int slot = 0;
      uint32_t phase = 0;
      for (int t = t0; t < t0 + nT; ++t) {
        for (int w = 0; w < 2; ++w) {  // K_t then V_t
#if SECO_FWD_PROD_SLEEP
          // the ring runs STAGES / 2 tiles ahead: back off instead of spinning on the issue
          // slots this warp's SM sub-partition shares with two softmax warps
          while (!mbar_try_wait(bar_kv_empty(slot), phase ^ 1)) __nanosleep(SECO_FWD_PROD_SLEEP);
#else
          mbar_wait(bar_kv_empty(slot), phase ^ 1);
#endif
          mbar_expect_tx(bar_kv_full(slot), L::kTileBytes);
          const CUtensorMap* m = w == 0 ? &tm_k : &tm_v;
          for (int x = 0; x < HALVES; ++x)
            tma_load_3d(sKV + slot * L::kTileBytes + x * BOX, m, bar_kv_full(slot), x * 64, t * fwd::BN, g);
          FTRACE(16 + w, t - t0);
          if (++slot == STAGES) { slot = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
#if SECO_FWD_MMA_WARP
    // converged warp: every lane waits, one elected lane issues (operands stay warp-uniform)
    const bool issuer = elect_one_sync();
    {
#else
    const bool issuer = true;
    if (lane == 0) {
#endif
      constexpr uint32_t idesc_s = make_idesc_bf16(fwd::BM, fwd::BN, 0, 0);  // Q K-major, K K-major
      constexpr uint32_t idesc_pv = make_idesc_bf16(fwd::BM, D, 0, 1);       // P (TMEM) K-major, V MN-major
      // descriptors: one per tile base; a k-step adds its byte offset / 16 to the 14-bit start
      // address field (shared-memory offsets stay below 256 KiB, so the field never carries)
      auto issue_s = [&](int b, int slot) {
        const uint64_t dq = make_desc_sw128(sQ + b * L::kTileBytes, 16, 1024);
        const uint64_t dk = make_desc_sw128(sKV + slot * L::kTileBytes, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk / 4) * BOX + (kk % 4) * 32) >> 4;
          if (issuer) mma_ss(tmem + b * fwd::BN, dq + off, dk + off, idesc_s, kk > 0);
        }
      };
      auto issue_pv_half = [&](int b, int slot, int hf, bool acc) {   // part hf: k16 steps [k0, k1)
        const uint64_t dv = make_desc_sw128(sKV + slot * L::kTileBytes, BOX, 1024);
        const int k0 = hf ? 2 * fwd::kSplit : 0, k1 = hf ? fwd::BN / 16 : 2 * fwd::kSplit;
#pragma unroll
        for (int kk = k0; kk < k1; ++kk)
          if (issuer)
            mma_ts(tmem + NH * fwd::BN + b * D, tmem + b * fwd::BN + kk * 8, dv + (uint32_t)(kk * 2048 >> 4), idesc_pv,
                   (acc || kk > 0) ? 1u : 0u);
      };
      auto commit = [&](uint32_t bar) { if (issuer) mma_commit(bar); };
      for (int b = 0; b < NH; ++b) mbar_wait(bar_q(b), 0);
      int slot = 0;
      uint32_t phase = 0;
      // prologue: S_b(0)
      mbar_wait(bar_kv_full(slot), phase);
      tc_fence_after();
      for (int b = 0; b < NH; ++b) { issue_s(b, slot); commit(bar_s_full(b)); }
      commit(bar_kv_empty(slot));
      if (++slot == STAGES) { slot = 0; phase ^= 1; }
      for (int t = 0; t < nT; ++t) {   // t counts this CTA's tiles
        const int vslot = slot;
        mbar_wait(bar_kv_full(vslot), phase);
        FTRACE(10, t);
        if (++slot == STAGES) { slot = 0; phase ^= 1; }
        const int kslot = slot;
        const bool more = t + 1 < nT;
        for (int b = 0; b < NH; ++b) {
          if (b == 0) FTRACE(18, t);
#if SECO_FWD_NAMED_P
          named_bar_sync(1 + 2 * b, 128 + 32);
#else
          mbar_wait(bar_p_half(b, 0), t & 1);
#endif
          FTRACE(0 + b, t);
          tc_fence_after();
          issue_pv_half(b, vslot, 0, t > 0);
#if SECO_FWD_NAMED_P
          named_bar_sync(2 + 2 * b, 128 + 32);
#else
          mbar_wait(bar_p_half(b, 1), t & 1);
#endif
          FTRACE(11 + 3 * b, t);
          tc_fence_after();
          issue_pv_half(b, vslot, 1, true);
          commit(bar_o_full(b));
          if (more) {
            if (b == 0) { mbar_wait(bar_kv_full(kslot), phase); tc_fence_after(); }
            issue_s(b, kslot);
            commit(bar_s_full(b));
            FTRACE(2 + b, t);
          }
        }
        commit(bar_kv_empty(vslot));
        if (more) {
          commit(bar_kv_empty(kslot));
          if (++slot == STAGES) { slot = 0; phase ^= 1; }
        }
        FTRACE(15, t);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax warpgroups
    const int b = (warp - 4) / 4;
    const int wq = warp % 4;                 // TMEM lane quarter this warp may access
    const int r = wq * 32 + lane;            // row within the tile
    const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
    const uint32_t tS = tmem + lane_addr + b * fwd::BN;
    const uint32_t tO = tmem + lane_addr + NH * fwd::BN + b * D;
    const float sl2 = a.scale_log2;
    const f2_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    for (int t = 0; t < nT; ++t) {   // t counts this CTA's tiles; global tile index t0 + t
      mbar_wait(bar_s_full(b), t & 1);
      if (lane == 0 && wq == 0) FTRACE(4 + b, t);
      tc_fence_after();
      const int kb = (t0 + t) * fwd::BN - q0;  // the tile's first key relative to the query tile's first row
      const bool diag = kb + fwd::BN - 1 > 0;  // keys beyond row 0: the causal mask applies
      // the whole 128-column row of S_b in registers (4 loads, one wait)
      uint32_t v[fwd::BN];
#pragma unroll
      for (int cc = 0; cc < fwd::BN / 32; ++cc) tmem_ld32(tS + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(v + cc * 32));
      tmem_wait_ld();
      if (diag) {
#pragma unroll
        for (int i = 0; i < fwd::BN; ++i)
          if (i + kb > r) v[i] = __float_as_uint(-INFINITY);
      }
#if SECO_FWD_MAXCH == 4
      // four independent FMNMX3 chains: half the dependent-latency depth of two
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int i = 0; i < fwd::BN; i += 8) {
        mx0 = fmax3(mx0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        mx1 = fmax3(mx1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        mx2 = fmax3(mx2, __uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
        mx3 = fmax3(mx3, __uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
      }
      mx0 = fmax3(mx0, mx1, fmaxf(mx2, mx3));
#else
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int i = 0; i < fwd::BN; i += 4) {
        mx0 = fmax3(mx0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        mx1 = fmax3(mx1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
      }
      mx0 = fmaxf(mx0, mx1);
#endif
      if (lane == 0 && wq == 0) FTRACE(6 + b, t);
      const float m_new = fmaxf(m, mx0 * sl2);
      const bool need = m_new > m + fwd::kRescaleThreshold;
      const float m_use = need ? m_new : m;
      const float alpha = need ? ex2(m - m_new) : 1.f;
      l *= alpha;
      // lazy O rescale: only when some row's max grew by > 2^8, and before PV_b(t) accumulates.
      // PV_b(t-1) is complete here (S_b(t), issued after it, has completed).
      if (t > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int cc = 0; cc < D / 8; ++cc) {   // 8 columns at a time: S_b's row is live in registers
          uint32_t ov[8];
          tmem_ld8(tO + cc * 8, ov);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st8(tO + cc * 8, ov);
        }
      }
      m = m_use;
      // P = exp2(S sigma log2e - m) -> bf16 -> TMEM columns [16cc, 16cc+16) of S_b's block, in two
      // parts (keys [0, 96) and [96, 128) by default), each released to the MMA warp as soon as it is stored, so
      // PV on the first half overlaps the exponentials of the second.  Masked entries hold -inf
      // and give exactly 0 through MUFU.
      const f2_t negm = f2(-m_use, -m_use);
      f2_t lsum0 = f2(0.f, 0.f), lsum1 = f2(0.f, 0.f);
      auto exp_half = [&](int hf, auto emu_pairs) {   // part hf: 32-key chunks [c0, c1)
        constexpr int EMU = decltype(emu_pairs)::value;
        const int c0 = hf ? fwd::kSplit : 0, c1 = hf ? fwd::BN / 32 : fwd::kSplit;
#pragma unroll
        for (int cc = c0; cc < c1; ++cc) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const f2_t x = ffma2(f2u(v[cc * 32 + i], v[cc * 32 + i + 1]), sl2x2, negm);
            // EMU of the 16 pairs, evenly spread, run on the FMA pipe (ex2_emu2)
            // EMU of every 8 pairs, evenly spread, run on the FMA pipe (ex2_emu2); the MUFU unit
            // then has slack beside the tensor pipe (2 of 8 measured best)
            const int p8 = (i / 2) % 8;
            const bool emu = (p8 * EMU) / 8 != ((p8 + 1) * EMU) / 8;
            const f2_t p2 = emu ? ex2_emu2(x) : f2(ex2(f2lo(x)), ex2(f2hi(x)));
#if SECO_FWD_LSUM_AFTER
            v[cc * 32 + i] = (uint32_t)p2; v[cc * 32 + i + 1] = (uint32_t)(p2 >> 32);   // row sum after release
#else
            if ((i / 2) & 1) lsum1 = fadd2(lsum1, p2); else lsum0 = fadd2(lsum0, p2);
#endif
            pk[i / 2] = pack_bf16_f2(p2);
          }
          tmem_st16(tS + cc * 16, pk);
        }
        tmem_wait_st();
        tc_fence_before();
#if SECO_FWD_NAMED_P
        named_bar_arrive(1 + 2 * b + hf, 128 + 32);   // the warpgroup's 128 threads + the MMA warp
#else
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p_half(b, hf));
#endif
        if (hf == 0 && lane == 0 && wq == 0) FTRACE(12 + b, t);
      };
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        if (diag) exp_half(hf, std::integral_constant<int, 0>{});
        else if (hf == 0) exp_half(hf, std::integral_constant<int, fwd::kEmuPairs>{});
        else exp_half(hf, std::integral_constant<int, fwd::kEmuPairs2>{});
      }
      if (lane == 0 && wq == 0) FTRACE(8 + b, t);
#if SECO_FWD_LSUM_AFTER
#pragma unroll
      for (int i = 0; i < fwd::BN; i += 4) {
        lsum0 = fadd2(lsum0, f2u(v[i], v[i + 1]));
        lsum1 = fadd2(lsum1, f2u(v[i + 2], v[i + 3]));
      }
#endif
      const f2_t lsum = fadd2(lsum0, lsum1);
      l += f2lo(lsum) + f2hi(lsum);
    }
    mbar_wait(bar_o_full(b), (nT - 1) & 1);
    tc_fence_after();
    // epilogue: O = acc / l, LSE = (m + log2 l) ln 2 -- bf16 O directly, or (split-KV) the
    // normalised fp32 partial for the in-kernel merge.  Indices re-derived from the block index:
    // keeps them out of the registers of the softmax loop (168-register cap)
    const fwd::Work we = fwd::decode_work((int)fwd::ctaid_x(), a);
    const int hf = (we.unit % a.nhp) * NH, row0 = (a.nqt - 1 - we.unit / a.nhp) * fwd::BM;
    const int h = hf + b, row = row0 + r;
    const float inv_l = 1.f / l;
    const float lse_v = (m + __log2f(l)) * 0.69314718055994531f;
    if (we.ns == 1) {
      __nv_bfloat16* orow = o + (int64_t)h * a.qh + (int64_t)row * a.qr;
      const bool in_chunk = row < a.c;       // rows of a ragged last tile past the chunk: not stored
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        if (cc * 32 >= a.d_out) break;       // warp-uniform
        uint32_t v[32];
        tmem_ld32(tO + cc * 32, v);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(v[8 * q + 0]) * inv_l, __uint_as_float(v[8 * q + 1]) * inv_l);
          w.y = pack_bf16(__uint_as_float(v[8 * q + 2]) * inv_l, __uint_as_float(v[8 * q + 3]) * inv_l);
          w.z = pack_bf16(__uint_as_float(v[8 * q + 4]) * inv_l, __uint_as_float(v[8 * q + 5]) * inv_l);
          w.w = pack_bf16(__uint_as_float(v[8 * q + 6]) * inv_l, __uint_as_float(v[8 * q + 7]) * inv_l);
          if (in_chunk) dst[q] = w;
        }
      }
      SECO_CHECK_COND(h < a.hq, 520);
      if (in_chunk) lse[(int64_t)h * a.c + row] = lse_v;
    } else {
      const int64_t prow = ((int64_t)we.split * a.hq + h) * a.cp + row;
      SECO_CHECK_COND(prow < (int64_t)a.nsplit * a.hq * a.cp, 521);
      float4* dst = reinterpret_cast<float4*>(a.part_o + prow * D);
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(tO + cc * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          dst[cc * 8 + q] = make_float4(__uint_as_float(v[4 * q]) * inv_l, __uint_as_float(v[4 * q + 1]) * inv_l,
                                        __uint_as_float(v[4 * q + 2]) * inv_l, __uint_as_float(v[4 * q + 3]) * inv_l);
      }
      a.part_lse[prow] = lse_v;
      if (a.merge)
        fwd::piece_done<NH>(a, we.unit - a.n_full, we.ns, reinterpret_cast<volatile int*>(smem + L::kTmemSlot + 8));
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<L::kTmemCols>(tmem);
  if (*reinterpret_cast<volatile int*>(smem + L::kTmemSlot + 8)) {   // the last piece of a split unit
    const fwd::Work we = fwd::decode_work((int)fwd::ctaid_x(), a);
    fwd::merge_rows<NH>(a, we.ns, (we.unit % a.nhp) * NH, (a.nqt - 1 - we.unit / a.nhp) * fwd::BM, sbase, o,
                        lse);
  }
#if SECO_FWD_PDL
  // do not complete before the kernel this one may have overlapped: keeps "this grid is done"
  // implying "everything before it in the stream is done" for the plain launches that follow
  if (threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// ============================================================================ CTA-pair forward
// seco_fwd2_sm100_kernel: the same algorithm as seco_fwd_sm100_kernel (NH = 2 heads per CTA,
// single-pass online softmax, P in TMEM, lazy rescale, ping-pong MMA order), issued as
// tcgen05.mma.cta_group::2 on a cluster of 2 CTAs.  The pair covers one 128-row query tile of
// the 4 q-heads of one kv-head group (CTA r: heads 4 quad + 2 r, +1), so both CTAs see the same
// K/V tiles and the same causal mask.  Per K/V tile each CTA loads only half of K (keys
// [64 r, 64 r + 64), all d: the N half of S's B operand) and half of V (all keys, d columns
// [64 r, 64 r + 64): the N half of PV's B operand), and each M = 256 MMA reads only that half
// from each CTA's shared memory: per CTA and K/V tile 2 x 48 KiB of S operands + 2 x 16 KiB of
// PV operands + 32 KiB of TMA writes, against 2 x 64 + 2 x 32 + 64 KiB unpaired -- the
// unpaired kernel's shared-memory port was ~98 % busy.
// Roles: the leader's warp 1 issues every MMA of the pair; the producers of both CTAs load into
// their own smem and complete on the leader's q / kv_full barriers (TMA .cta_group::2); the
// leader's commits arrive on both CTAs' s_full / o_full / kv_empty (multicast); both CTAs'
// softmax warps arrive on the leader's p_half barriers (8 arrivals: 4 warps x 2 CTAs).
namespace fwd2 {
constexpr int NH = 2, D = 128, BM = 128, BN = 128;
constexpr int kQBytes = BM * D * 2;                  // one head's Q tile (32 KiB)
constexpr int kStage = 64 * D * 2;                   // a K half or a V half (16 KiB)
template <int STAGES>
struct Layout {
  static constexpr int kQ = 0;
  static constexpr int kKV = kQ + NH * kQBytes;
  static constexpr int kBar = kKV + STAGES * kStage;
  // barriers: q[NH], kv_full[STAGES], kv_empty[STAGES], s_full[NH], p_half[NH][2], o_full[NH]
  static constexpr int kNumBars = NH + 2 * STAGES + 4 * NH;
  static constexpr int kTmemSlot = kBar + 8 * kNumBars;
  static constexpr int kBytes = kTmemSlot + 16;
  static constexpr int kAlloc = kBytes + 1024;
  static constexpr int kThreads = 128 + 128 * NH;
};
}  // namespace fwd2

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(fwd2::Layout<STAGES>::kThreads, 1)
    seco_fwd2_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ o,
                           float* __restrict__ lse, const fwd::Args a) {
  using namespace fwd2;
  using L = Layout<STAGES>;
  constexpr int BOX = 128 * 128;                     // one [128 rows][128 B] box (Q)
  constexpr int HBOX = 64 * 128;                     // one [64 rows][128 B] box (K half)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase + L::kQ, sKV = sbase + L::kKV;
  const uint32_t bar0 = sbase + L::kBar;
  auto bar_q = [&](int b) { return bar0 + 8u * b; };
  auto bar_kv_full = [&](int s) { return bar0 + 8u * (NH + s); };
  auto bar_kv_empty = [&](int s) { return bar0 + 8u * (NH + STAGES + s); };
  auto bar_s_full = [&](int b) { return bar0 + 8u * (NH + 2 * STAGES + b); };
  auto bar_p_half = [&](int b, int hf) { return bar0 + 8u * (2 * NH + 2 * STAGES + 2 * b + hf); };
  auto bar_o_full = [&](int b) { return bar0 + 8u * (4 * NH + 2 * STAGES + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // heavier query tiles first, whole units before pieces (split-KV part innermost); the pair
  // shares (query tile, head quad)
  const fwd::Work wk = fwd::decode_work((int)blockIdx.x / 2, a);
  const int unit = wk.unit, split = wk.split, ns = wk.ns;
  const int nquad = a.hq / 4;
  const int qt = a.nqt - 1 - unit / nquad;
  const int quad = unit % nquad;
  const int h0 = quad * 4 + 2 * (int)rank, g = (quad * 4) / a.G;
  const int q0 = a.j * a.c + qt * BM;
  const int nvalid = min(BM, a.c - qt * BM);         // rows inside the chunk (ragged last tile)
  const int T = (q0 + nvalid - 1) / BN + 1;
  const int t0 = T * split / ns;
  const int nT = T * (split + 1) / ns - t0;

  if (threadIdx.x == 0) {
    *reinterpret_cast<volatile int*>(smem + L::kTmemSlot + 8) = 0;   // split-KV: "this piece merges"
    for (int b = 0; b < NH; ++b) mbar_init(bar_q(b), 1);
    for (int s = 0; s < STAGES; ++s) { mbar_init(bar_kv_full(s), 1); mbar_init(bar_kv_empty(s), 1); }
    for (int b = 0; b < NH; ++b) {
      mbar_init(bar_s_full(b), 1);
      mbar_init(bar_p_half(b, 0), 8);                // 4 softmax warps of each CTA (leader's copy)
      mbar_init(bar_p_half(b, 1), 8);
      mbar_init(bar_o_full(b), 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tm_q); tma_prefetch(&tm_k); tma_prefetch(&tm_v); }
#if SECO_FWD_PDL
  if (!a.wait_prev) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  if (warp == 2) tmem_alloc_pair<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  cluster_sync();                                    // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#if SECO_FWD_PDL
  if (a.wait_prev) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
#endif

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      SECO_CHECK_COND(qt * BM < a.c && h0 + NH <= a.hq, 422);
      SECO_CHECK_COND(t0 >= 0 && (t0 + nT - 1) * BN < (a.j + 1) * a.c, 423);
      for (int b = 0; b < NH; ++b) {
        if (leader) mbar_expect_tx(bar_q(b), 2 * kQBytes);     // both CTAs' Q_b
        const uint32_t bq = mapa_shared(bar_q(b), 0);
        for (int x = 0; x < 2; ++x)
          tma_load_3d_pair(sQ + b * kQBytes + x * BOX, &tm_q, bq, x * 64, qt * BM, h0 + b, BOX);
      }
      int slot = 0;
      uint32_t phase = 0;
      for (int t = t0; t < t0 + nT; ++t) {
        for (int w = 0; w < 2; ++w) {  // K_t half then V_t half
#if SECO_FWD_PROD_SLEEP
          while (!mbar_try_wait(bar_kv_empty(slot), phase ^ 1)) __nanosleep(SECO_FWD_PROD_SLEEP);
#else
          mbar_wait(bar_kv_empty(slot), phase ^ 1);
#endif
          if (leader) mbar_expect_tx(bar_kv_full(slot), 2 * kStage);
          const uint32_t bf = mapa_shared(bar_kv_full(slot), 0);
          const uint32_t dst = sKV + slot * kStage;
          if (w == 0) {   // keys [64 r, 64 r + 64) of tile t, d in two 64-column boxes
            for (int x = 0; x < 2; ++x)
              tma_load_3d_pair(dst + x * HBOX, &tm_k, bf, x * 64, t * BN + 64 * (int)rank, g, HBOX);
          } else {        // every key of tile t, d columns [64 r, 64 r + 64)
            tma_load_3d_pair(dst, &tm_v, bf, 64 * (int)rank, t * BN, g, BOX);
          }
          if (++slot == STAGES) { slot = 0; phase ^= 1; }
        }
      }
      // teardown: every slot's last release (a multicast commit from the leader) has landed in this
      // CTA's barriers before the pair may exit
      for (int s2 = 0; s2 < STAGES; ++s2) {
        mbar_wait(bar_kv_empty(slot), phase ^ 1);
        if (++slot == STAGES) { slot = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    // converged warp, one elected lane issues (operands in uniform registers); the waits use
    // CTA-scope acquire like CUTLASS's cluster pipelines: the data handed over lives in TMEM or
    // arrives by TMA, both ordered by the tcgen05 fences and the mbarrier transaction counts
    const bool issuer = elect_one_sync();
    if (leader) {
      constexpr uint32_t idesc_s = make_idesc_bf16(2 * BM, BN, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t idesc_pv = make_idesc_bf16(2 * BM, D, 0, 1);   // P (TMEM), V MN-major
      auto issue_s = [&](int b, int slot) {
        const uint64_t dq = make_desc_sw128(sQ + b * kQBytes, 16, 1024);
        const uint64_t dk = make_desc_sw128(sKV + slot * kStage, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          if (issuer)
            mma_ss_pair(tmem + b * BN, dq + (uint32_t)(((kk / 4) * BOX + (kk % 4) * 32) >> 4),
                        dk + (uint32_t)(((kk / 4) * HBOX + (kk % 4) * 32) >> 4), idesc_s, kk > 0);
      };
      auto issue_pv_part = [&](int b, int slot, int hf, bool acc) {   // part hf: k16 steps [k0, k1)
        const uint64_t dv = make_desc_sw128(sKV + slot * kStage, BOX, 1024);
        const int k0 = hf ? 2 * fwd::kSplit : 0, k1 = hf ? BN / 16 : 2 * fwd::kSplit;
#pragma unroll
        for (int kk = k0; kk < k1; ++kk)
          if (issuer)
            mma_ts_pair(tmem + NH * BN + b * D, tmem + b * BN + kk * 8, dv + (uint32_t)(kk * 2048 >> 4), idesc_pv,
                        (acc || kk > 0) ? 1u : 0u);
      };
      auto commit = [&](uint32_t bar) { if (issuer) mma_commit_pair(bar); };
      for (int b = 0; b < NH; ++b) mbar_wait(bar_q(b), 0);
      int slot = 0;
      uint32_t phase = 0;
      mbar_wait(bar_kv_full(slot), phase);
      tc_fence_after();
      for (int b = 0; b < NH; ++b) { issue_s(b, slot); commit(bar_s_full(b)); }
      commit(bar_kv_empty(slot));
      if (++slot == STAGES) { slot = 0; phase ^= 1; }
      for (int t = 0; t < nT; ++t) {
        const int vslot = slot;
        mbar_wait(bar_kv_full(vslot), phase);
        if (++slot == STAGES) { slot = 0; phase ^= 1; }
        const int kslot = slot;
        const bool more = t + 1 < nT;
        for (int b = 0; b < NH; ++b) {
          mbar_wait(bar_p_half(b, 0), t & 1);
          tc_fence_after();
          issue_pv_part(b, vslot, 0, t > 0);
          mbar_wait(bar_p_half(b, 1), t & 1);
          tc_fence_after();
          issue_pv_part(b, vslot, 1, true);
          commit(bar_o_full(b));
          if (more) {
            if (b == 0) { mbar_wait(bar_kv_full(kslot), phase); tc_fence_after(); }
            issue_s(b, kslot);
            commit(bar_s_full(b));
          }
        }
        commit(bar_kv_empty(vslot));
        if (more) {
          commit(bar_kv_empty(kslot));
          if (++slot == STAGES) { slot = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax warpgroups (both CTAs)
    const int b = (warp - 4) / 4;
    const int wq = warp % 4;
    const int r = wq * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
    const uint32_t tS = tmem + lane_addr + b * BN;
    const uint32_t tO = tmem + lane_addr + NH * BN + b * D;
    const float sl2 = a.scale_log2;
    const f2_t sl2x2 = f2(sl2, sl2);
    float m = -INFINITY, l = 0.f;
    for (int t = 0; t < nT; ++t) {
      mbar_wait(bar_s_full(b), t & 1);
      tc_fence_after();
      const int kb = (t0 + t) * BN - q0;     // the tile's first key relative to the query tile's first row
      const bool diag = kb + BN - 1 > 0;
      uint32_t v[BN];
#pragma unroll
      for (int cc = 0; cc < BN / 32; ++cc) tmem_ld32(tS + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(v + cc * 32));
      tmem_wait_ld();
      if (diag) {
#pragma unroll
        for (int i = 0; i < BN; ++i)
          if (i + kb > r) v[i] = __float_as_uint(-INFINITY);
      }
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int i = 0; i < BN; i += 8) {
        mx0 = fmax3(mx0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        mx1 = fmax3(mx1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        mx2 = fmax3(mx2, __uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
        mx3 = fmax3(mx3, __uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
      }
      const float m_new = fmaxf(m, fmax3(mx0, mx1, fmaxf(mx2, mx3)) * sl2);
      const bool need = m_new > m + fwd::kRescaleThreshold;
      const float m_use = need ? m_new : m;
      const float alpha = need ? ex2(m - m_new) : 1.f;
      l *= alpha;
      // PV_b(t-1) is complete: S_b(t), issued after it by the same (leader) thread, has completed
      if (t > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int cc = 0; cc < D / 8; ++cc) {
          uint32_t ov[8];
          tmem_ld8(tO + cc * 8, ov);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st8(tO + cc * 8, ov);
        }
      }
      m = m_use;
      const f2_t negm = f2(-m_use, -m_use);
      f2_t lsum0 = f2(0.f, 0.f), lsum1 = f2(0.f, 0.f);
      // as in seco_fwd_sm100_kernel: P released in two parts (32-key chunks [0, kSplit), then the
      // rest) to the leader's MMA warp, 2 of 8 exponential pairs of the first part on the FMA
      // pipe (not on the diagonal tile), the row sum after the releases
      auto exp_part = [&](int hf, auto emu_pairs) {
        constexpr int EMU = decltype(emu_pairs)::value;
        const int c0 = hf ? fwd::kSplit : 0, c1 = hf ? BN / 32 : fwd::kSplit;
#pragma unroll
        for (int cc = c0; cc < c1; ++cc) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const f2_t x = ffma2(f2u(v[cc * 32 + i], v[cc * 32 + i + 1]), sl2x2, negm);
            const int p8 = (i / 2) % 8;
            const bool emu = (p8 * EMU) / 8 != ((p8 + 1) * EMU) / 8;
            const f2_t p2 = emu ? ex2_emu2(x) : f2(ex2(f2lo(x)), ex2(f2hi(x)));
            v[cc * 32 + i] = (uint32_t)p2;
            v[cc * 32 + i + 1] = (uint32_t)(p2 >> 32);
            pk[i / 2] = pack_bf16_f2(p2);
          }
          tmem_st16(tS + cc * 16, pk);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(mapa_shared(bar_p_half(b, hf), 0));
      };
      if (diag) {
        exp_part(0, std::integral_constant<int, 0>{});
        exp_part(1, std::integral_constant<int, 0>{});
      } else {
        exp_part(0, std::integral_constant<int, fwd::kEmuPairs>{});
        exp_part(1, std::integral_constant<int, fwd::kEmuPairs2>{});
      }
#pragma unroll
      for (int i = 0; i < BN; i += 4) {
        lsum0 = fadd2(lsum0, f2u(v[i], v[i + 1]));
        lsum1 = fadd2(lsum1, f2u(v[i + 2], v[i + 3]));
      }
      const f2_t lsum = fadd2(lsum0, lsum1);
      l += f2lo(lsum) + f2hi(lsum);
    }
    mbar_wait(bar_o_full(b), (nT - 1) & 1);
    tc_fence_after();
    // epilogue indices re-derived from the block index: keeps them out of the registers of the
    // softmax loop (this kernel sits at its 168-register cap)
    const fwd::Work we = fwd::decode_work((int)fwd::ctaid_x() / 2, a);
    const int row = (a.nqt - 1 - we.unit / (a.hq / 4)) * BM + r;
    const int h = (we.unit % (a.hq / 4)) * 4 + 2 * (int)cluster_ctarank() + b;
    const float inv_l = 1.f / l;
    const float lse_v = (m + __log2f(l)) * 0.69314718055994531f;
    if (we.ns == 1) {
      __nv_bfloat16* orow = o + (int64_t)h * a.qh + (int64_t)row * a.qr;
      const bool in_chunk = row < a.c;       // rows of a ragged last tile past the chunk: not stored
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        if (cc * 32 >= a.d_out) break;
        uint32_t v[32];
        tmem_ld32(tO + cc * 32, v);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(v[8 * q + 0]) * inv_l, __uint_as_float(v[8 * q + 1]) * inv_l);
          w.y = pack_bf16(__uint_as_float(v[8 * q + 2]) * inv_l, __uint_as_float(v[8 * q + 3]) * inv_l);
          w.z = pack_bf16(__uint_as_float(v[8 * q + 4]) * inv_l, __uint_as_float(v[8 * q + 5]) * inv_l);
          w.w = pack_bf16(__uint_as_float(v[8 * q + 6]) * inv_l, __uint_as_float(v[8 * q + 7]) * inv_l);
          if (in_chunk) dst[q] = w;
        }
      }
      SECO_CHECK_COND(h < a.hq, 522);
      if (in_chunk) lse[(int64_t)h * a.c + row] = lse_v;
    } else {
      const int64_t prow = ((int64_t)we.split * a.hq + h) * a.cp + row;
      SECO_CHECK_COND(prow < (int64_t)a.nsplit * a.hq * a.cp, 523);
      float4* dst = reinterpret_cast<float4*>(a.part_o + prow * D);
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(tO + cc * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          dst[cc * 8 + q] = make_float4(__uint_as_float(v[4 * q]) * inv_l, __uint_as_float(v[4 * q + 1]) * inv_l,
                                        __uint_as_float(v[4 * q + 2]) * inv_l, __uint_as_float(v[4 * q + 3]) * inv_l);
      }
      a.part_lse[prow] = lse_v;
      if (a.merge)
        fwd::piece_done<NH>(a, 2 * (we.unit - a.n_full) + (int)cluster_ctarank(), we.ns,
                            reinterpret_cast<volatile int*>(smem + L::kTmemSlot + 8));
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();                                    // neither CTA leaves while the pair still uses its smem / TMEM
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
  if (*reinterpret_cast<volatile int*>(smem + L::kTmemSlot + 8)) {   // the last piece of a split CTA-unit
    const fwd::Work we = fwd::decode_work((int)fwd::ctaid_x() / 2, a);
    fwd::merge_rows<NH>(a, we.ns, (we.unit % (a.hq / 4)) * 4 + 2 * (int)cluster_ctarank(),
                        (a.nqt - 1 - we.unit / (a.hq / 4)) * BM, sbase, o, lse);
  }
#if SECO_FWD_PDL
  if (threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

namespace fwd {
// float offset of the split-KV piece counters in the workspace: after the partial O
// [sp][hq][cp][128] and partial LSE [sp][hq][cp]
inline size_t split_counter_offset(const ChunkGeom& g, int sp) { return (size_t)sp * g.hq * g.cp * (128 + 1); }

// Split-KV plan of one forward call (§8 row a9).  A sub-wave grid (fewer units than work slots:
// head-sharded ranks, short chunks) cuts every unit into nsplit key ranges and merges the parts
// with the combine kernel.  A multi-wave grid runs DP + split tail: the first n_full units (as
// many whole waves as the grid fills) run whole, the remaining ones are cut into nsplit key
// ranges whose pieces fill the last waves, and the piece that finishes a unit last merges its
// parts in-kernel (there the merges overlap other pieces' work; in a sub-wave grid every merge
// would sit on the critical path, where the combine kernel spreads it over all SMs).  Cost in
// K/V-tile times per work slot (an SM, or a cluster for the pair kernel): kOver tiles of
// prologue / epilogue per CTA; the combine ~0.15 of a unit; kMerge per round of pieces for the
// partial rows and the in-kernel merge (measured).  SECO_FWD_NSPLIT=s forces s;
// SECO_FWD_SLOTS=n pretends n SMs (tests reach the DP + tail form on small shapes).
struct SplitPlan {
  int units, n_full, nsplit, merge;
  int items() const { return n_full + (units - n_full) * nsplit; }
};
inline SplitPlan split_plan(const ChunkGeom& g, int units, bool pair, bool have_ws, size_t ws_floats,
                            int sms = 0) {
  constexpr double kOver = 8.0, kMerge = 7.0;
  static const int forced = [] {
    const char* e = std::getenv("SECO_FWD_NSPLIT");
    return e == nullptr ? 0 : std::atoi(e);
  }();
  static const int slots_env = [] {
    const char* e = std::getenv("SECO_FWD_SLOTS");
    return e == nullptr ? 0 : std::atoi(e);
  }();
  const int sm_slots = sms > 0 ? sms : slots_env > 0 ? slots_env : kSMs;
  const int slots = pair ? (sm_slots + 1) / 2 : sm_slots;
  const int t_min = g.j * g.c / BN + 1;                // K/V tiles of the lightest unit
  const int waves_full = units / slots;
  const int n_full = waves_full * slots, rem = units - n_full;
  int best = 1;
  double best_cost = (double)((units + slots - 1) / slots) * (t_min + kOver);
  for (int sp = 2; sp <= 4 && rem > 0; ++sp) {
    if (t_min < 8 * sp || g.j == 0 || !have_ws || split_counter_offset(g, sp) + (size_t)2 * units > ws_floats) break;
    const int rounds = (rem * sp + slots - 1) / slots;
    const double cost = waves_full * (t_min + kOver) + rounds * ((double)t_min / sp + kOver) +
                        (waves_full == 0 ? 0.15 * t_min : kMerge * rounds);
    if (forced ? sp == forced : cost < best_cost) { best_cost = cost; best = sp; }
  }
  if (forced == 1) best = 1;
  return SplitPlan{units, best > 1 ? n_full : units, best, best > 1 && n_full > 0 ? 1 : 0};
}
}  // namespace fwd

cudaError_t launch_fwd_combine(const ChunkGeom& g, int nsplit, const float* part_o, const float* part_lse, void* o,
                               float* lse, cudaStream_t st);

template <int NH, int D, int STAGES, bool PAIR>
static cudaError_t launch_fwd_impl(const ChunkGeom& g, const CUtensorMap& tq, const CUtensorMap& tk,
                                   const CUtensorMap& tv, void* o, float* lse, float* ws, size_t ws_floats,
                                   cudaStream_t st, int* launches) {
  using L = typename std::conditional<PAIR, fwd2::Layout<STAGES>, fwd::Layout<NH, D, STAGES>>::type;
  static_assert(L::kAlloc <= 232448, "shared memory budget");
  static_assert(!PAIR || (NH == 2 && D == 128), "the pair kernel is NH = 2, D = 128");
  auto kern = [] {
    if constexpr (PAIR) return seco_fwd2_sm100_kernel<STAGES>;
    else return seco_fwd_sm100_kernel<NH, D, STAGES>;
  }();
  static std::atomic<unsigned long long> attr_done{0};
  {
    cudaError_t e = ensure_smem_attr(kern, L::kAlloc, attr_done);
    if (e != cudaSuccess) return e;
  }
  fwd::Args a;
  a.c = g.c; a.j = g.j; a.hq = g.hq; a.G = g.hq / g.hkv;
  a.nqt = (g.c + fwd::BM - 1) / fwd::BM; a.nhp = g.hq / NH; a.cp = g.cp;
  a.scale_log2 = g.scale * 1.4426950408889634f;
  a.qh = g.qh; a.qr = g.qr; a.d_out = g.d;
  a.wait_prev = g.prev_indep ? 0 : 1;
  const fwd::SplitPlan pl = fwd::split_plan(g, a.nqt * a.nhp / (PAIR ? 2 : 1), PAIR, ws != nullptr, ws_floats);
  const int units = pl.units, best = pl.nsplit;
  a.nsplit = best;
  a.n_full = pl.n_full;
  a.n_units = units;
  a.merge = pl.merge;
  auto cnt_off = [&](int sp) { return fwd::split_counter_offset(g, sp); };
  a.part_o = ws;
  a.part_lse = ws ? ws + (size_t)best * g.hq * g.cp * D : nullptr;
  a.cnt = ws ? reinterpret_cast<int*>(ws + cnt_off(best)) : nullptr;
  a.trace = nullptr;
#ifdef SECO_TRACE
  {
    static unsigned long long* tbuf = nullptr;
    const size_t n = (size_t)fwd::kTraceCtas * fwd::kTraceSlots * fwd::kTraceIters;
    if (!tbuf) cudaMalloc(&tbuf, sizeof(unsigned long long) * n);
    cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * n, st);
    a.trace = tbuf;
    seco_fwd_trace_buffer = tbuf;
  }
#endif
  const int items = a.n_full + (units - a.n_full) * a.nsplit;
  dim3 grid(items * (PAIR ? 2 : 1));
  cudaError_t e;
  if (a.merge) {   // one counter per split CTA-unit (pairs: per CTA of the pair)
    e = cudaMemsetAsync(a.cnt, 0, sizeof(int) * 2 * (size_t)units, st);
    if (e != cudaSuccess) return e;
  }
  if (SECO_FWD_PDL && a.nsplit == 1) {
    // the split path writes fp32 partials into the workspace, which a preceding backward's
    // final kernel may still be reading: only the unsplit forward may overlap its predecessor
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(L::kThreads);
    cfg.dynamicSmemBytes = L::kAlloc;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, reinterpret_cast<__nv_bfloat16*>(o), lse, a);
    if (e != cudaSuccess) return e;
  } else {
    kern<<<grid, L::kThreads, L::kAlloc, st>>>(tq, tk, tv, reinterpret_cast<__nv_bfloat16*>(o), lse, a);
  }
  e = cudaGetLastError();
  *launches = 1;
  if (e == cudaSuccess && a.nsplit > 1 && !a.merge) {
    e = launch_fwd_combine(g, a.nsplit, a.part_o, a.part_lse, o, lse, st);
    *launches = 2;
  }
  return e;
}

bool fwd_uses_pair(const ChunkGeom& g) {
  // CTA pairs halve each SM's shared-memory operand and TMA traffic; per call they run level
  // with the unpaired kernel and, at the lower power, +0.4 % on the power-capped cfg3 step, but
  // their 4-head work units are coarser: with fewer unsplit units than SMs (head-sharded ranks,
  // short chunks) they lose ~1 %.  SECO_FWD_PAIR=0 / 1 forces the choice (A/B).
  static const int mode = [] {
    const char* e = std::getenv("SECO_FWD_PAIR");
    return e == nullptr ? -1 : (e[0] == '0' ? 0 : 1);
  }();
  const bool shape_ok = g.d <= 128 && g.d % 32 == 0 && (g.hq / g.hkv) % 4 == 0;
  if (mode >= 0) return mode == 1 && shape_ok;
  return shape_ok && (g.c + fwd::BM - 1) / fwd::BM * (g.hq / 2) >= fwd::kSMs;
}

int32_t fwd_debug_plan(const ChunkGeom& g, size_t ws_floats, int sms, int32_t* out5) {
  const bool pair = fwd_uses_pair(g);
  const int NH = pair || (g.hq / g.hkv) % 2 == 0 ? 2 : 1;
  const int nqt = (g.c + fwd::BM - 1) / fwd::BM;
  const fwd::SplitPlan pl = fwd::split_plan(g, nqt * (g.hq / NH) / (pair ? 2 : 1), pair, true, ws_floats, sms);
  out5[0] = pair ? 1 : 0; out5[1] = pl.units; out5[2] = pl.n_full; out5[3] = pl.nsplit; out5[4] = pl.merge;
  return pl.items() * (pair ? 2 : 1);
}

cudaError_t launch_fwd_sm100(const ChunkGeom& g, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, void* o, float* lse, float* ws, size_t ws_floats,
                             cudaStream_t st, int* launches) {
  const int G = g.hq / g.hkv;
  // d = 32, 64, 96 run the D = 128 kernel on zero-padded tiles: the tensor maps describe
  // d-column rows, so the TMA fills the columns past d with zeros (they add 0 to every dot
  // product, and the epilogues store only the first d columns)
  if (g.d <= 128 && g.d % 32 == 0) {
    // groups of 4 q-heads per kv head (LLaMA): CTA pairs over the 4 heads of a group, K / V
    // halves per CTA (tk must then have 64-row boxes: seco_api.cpp asks fwd_uses_pair)
    if (fwd_uses_pair(g))
      return launch_fwd_impl<2, 128, SECO_FWD_PAIR_STAGES, true>(g, tq, tk, tv, o, lse, ws, ws_floats, st, launches);
    if (G % 2 == 0) return launch_fwd_impl<2, 128, 5, false>(g, tq, tk, tv, o, lse, ws, ws_floats, st, launches);
    return launch_fwd_impl<1, 128, 6, false>(g, tq, tk, tv, o, lse, ws, ws_floats, st, launches);
  }
  return cudaErrorInvalidValue;
}

unsigned long long check_word_fwd() { return seco_check_read_clear(); }

}  // namespace seco
