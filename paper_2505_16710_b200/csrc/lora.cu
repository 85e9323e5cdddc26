// LoRA gradient accumulation for one adapted projection and one chunk (LoRA
// on q, k, v, o of every layer).  For Y = X W + (X A) B and the output cotangent dY:
//   u   = dY B^T   [rows][R]      -> u_out (fp32; the caller forms dX = dY W^T + u A^T)
//   t   = X A      [rows][R]      (workspace)
//   dA += X^T u    [n_in][R]      fp32 accumulator
//   dB += t^T dY   [R][n_out]     fp32 accumulator
// Rank-R skinny contractions: HBM-bound on X and dY (R = 8 gives 8 FLOP per loaded element),
// so CUDA cores with coalesced loads, not tensor cores.  Three kernels, all deterministic:
//   rows   (twice: t from X, u from dY) a block reduces 8 rows against A / B (L1-resident),
//          16-B vector loads
//   cols   a thread owns four columns of X / dY over a contiguous share of the rows (u / t
//          of those rows staged in smem); per-split partial sums of dA / dB to the workspace
//   reduce partials added in split order into dA / dB
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace seco {

namespace lora {

SECO_DEV float to_f(float v) { return v; }
SECO_DEV float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

// R contiguous elements (a row of A) as floats, with the widest aligned vector loads
template <typename T, int R>
SECO_DEV void load_row(const T* p, float (&out)[R]) {
  constexpr int BYTES = R * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
    constexpr int NV = BYTES / 16, PER = 16 / sizeof(T);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      T tmp[PER];
      *reinterpret_cast<uint4*>(tmp) = __ldg(reinterpret_cast<const uint4*>(p) + v);
#pragma unroll
      for (int e = 0; e < PER; ++e) out[v * PER + e] = to_f(tmp[e]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < R; ++k) out[k] = to_f(p[k]);
  }
}

SECO_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
}  // namespace lora

// Z[row][k] = sum_i M[row][i] P(i, k) for a [rows][n] matrix M (row stride ldm): P(i, k) =
// A[i][k] (t = X A) or B[k][i] (u = dY B^T).  A block of 4 warps takes RW = 4 rows; its 128
// lanes stride over 16-B vectors of those rows, each vector's P values coming from L1 (A and
// B are at most a few hundred KiB), RW x R FMAs per loaded element of P; lane and warp
// partial sums are reduced through shuffles and smem.
template <typename T, int R>
__global__ void __launch_bounds__(128) lora_rows_kernel(const T* __restrict__ m, int64_t ldm,
                                                        const T* __restrict__ P, bool p_is_b, int rows, int n,
                                                        float* __restrict__ z) {
  constexpr int VEC = 16 / sizeof(T);           // elements per 16-B vector
  constexpr int RW = 4;                         // rows per block (register budget: RW x R accumulators)
  constexpr int NT = 128, NW = NT / 32;         // threads / warps per block
  __shared__ float red[NW][RW][R];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r0 = blockIdx.x * RW;
  float acc[RW][R];
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int k = 0; k < R; ++k) acc[q][k] = 0.f;
  for (int i0 = threadIdx.x * VEC; i0 < n; i0 += NT * VEC) {
    T xv[RW][VEC];
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      if (r0 + q < rows)
        *reinterpret_cast<uint4*>(xv[q]) = *reinterpret_cast<const uint4*>(m + (int64_t)(r0 + q) * ldm + i0);
      else
        *reinterpret_cast<uint4*>(xv[q]) = make_uint4(0, 0, 0, 0);
    }
    if (!p_is_b) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        float pv[R];
        lora::load_row<T, R>(P + (int64_t)(i0 + e) * R, pv);
#pragma unroll
        for (int q = 0; q < RW; ++q) {
          const float xq = lora::to_f(xv[q][e]);
#pragma unroll
          for (int k = 0; k < R; ++k) acc[q][k] = fmaf(xq, pv[k], acc[q][k]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        T bv[VEC];
        *reinterpret_cast<uint4*>(bv) = *reinterpret_cast<const uint4*>(P + (int64_t)k * n + i0);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const float b = lora::to_f(bv[e]);
#pragma unroll
          for (int q = 0; q < RW; ++q) acc[q][k] = fmaf(lora::to_f(xv[q][e]), b, acc[q][k]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const float v = lora::warp_sum(acc[q][k]);
      if (lane == 0) red[warp][q][k] = v;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < RW * R; e += blockDim.x) {
    const int q = e / R, k = e - q * R;
    if (r0 + q >= rows) continue;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) v += red[w][q][k];
    z[(int64_t)(r0 + q) * R + k] = v;
  }
}

// part[s][col][k]: columns [0, n_in) of X against u (-> dA), then [n_in, n_in + n_out) of dY
// against t (-> dB^T), over rows [s * rows / S, (s + 1) * rows / S).  A thread owns CPT = 4
// adjacent columns (one 8- or 16-B load per row, coalesced across the block, rows unrolled
// by 4 for loads in flight); the split's rows of u and t are staged in smem (broadcasts).
template <typename T, int R>
__global__ void __launch_bounds__(256) lora_cols_kernel(const T* __restrict__ x, int64_t ldx,
                                                        const T* __restrict__ dy, int64_t ldy,
                                                        const float* __restrict__ t, const float* __restrict__ u,
                                                        int rows, int n_in, int n_out, int nsplit,
                                                        float* __restrict__ part) {
  constexpr int CPT = 4;
  using V = typename std::conditional<sizeof(T) == 2, uint2, uint4>::type;   // CPT elements
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int s = blockIdx.y;
  const int r0 = (int)((int64_t)s * rows / nsplit), r1 = (int)((int64_t)(s + 1) * rows / nsplit);
  float* su = reinterpret_cast<float*>(smem_raw);          // [rows of the split][R] of u, then of t
  float* st = su + (r1 - r0) * R;
  for (int e = threadIdx.x; e < (r1 - r0) * R; e += blockDim.x) {
    su[e] = u[(int64_t)r0 * R + e];
    st[e] = t[(int64_t)r0 * R + e];
  }
  __syncthreads();
  const int ncol = n_in + n_out;
  const int col = (blockIdx.x * 256 + threadIdx.x) * CPT;  // this thread's CPT columns
  if (col >= ncol) return;
  const bool isA = col < n_in;                             // n_in % CPT == 0: no straddling
  const float* sw = isA ? su : st;
  const T* src = isA ? x + col : dy + (col - n_in);
  const int64_t ld_src = isA ? ldx : ldy;
  float acc[CPT][R];
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int k = 0; k < R; ++k) acc[c][k] = 0.f;
  int row = r0;
  for (; row + 4 <= r1; row += 4) {
    T v[4][CPT];
#pragma unroll
    for (int q = 0; q < 4; ++q) *reinterpret_cast<V*>(v[q]) = *reinterpret_cast<const V*>(src + (int64_t)(row + q) * ld_src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float* wr = sw + (row + q - r0) * R;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const float wk = wr[k];
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[c][k] = fmaf(lora::to_f(v[q][c]), wk, acc[c][k]);
      }
    }
  }
  for (; row < r1; ++row) {
    T v[CPT];
    *reinterpret_cast<V*>(v) = *reinterpret_cast<const V*>(src + (int64_t)row * ld_src);
    const float* wr = sw + (row - r0) * R;
#pragma unroll
    for (int k = 0; k < R; ++k)
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[c][k] = fmaf(lora::to_f(v[c]), wr[k], acc[c][k]);
  }
  float* out = part + ((int64_t)s * ncol + col) * R;
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int k = 0; k < R; ++k) out[c * R + k] = acc[c][k];
}

// dA[i][k] += sum_s part[s][i][k];  dB[k][j] += sum_s part[s][n_in + j][k]
template <int R>
__global__ void __launch_bounds__(256) lora_reduce_kernel(const float* __restrict__ part, int n_in, int n_out,
                                                          int nsplit, float* __restrict__ dA, float* __restrict__ dB) {
  const int ncol = n_in + n_out;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ncol * R; e += gridDim.x * blockDim.x) {
    const int col = e / R, k = e - col * R;
    float acc = 0.f;
    for (int s = 0; s < nsplit; ++s) acc += part[((int64_t)s * ncol + col) * R + k];
    if (col < n_in) dA[(int64_t)col * R + k] += acc;
    else dB[(int64_t)k * n_out + (col - n_in)] += acc;
  }
}

constexpr size_t kColsSmem = 96 * 1024;   // smem cap of lora_cols_kernel (u, t rows of a split)

int lora_splits(const LoraGeom& g) {
  const int col_blocks = (g.n_in + g.n_out + 1023) / 1024;
  int s = (2 * 148 + col_blocks - 1) / col_blocks;
  s = s < 1 ? 1 : s;
  const int max_s = g.rows / 64 > 0 ? g.rows / 64 : 1;   // at least ~64 rows per split
  s = s > max_s ? max_s : s;
  // the column pass stages u and t of a split's rows in smem: keep that under kColsSmem
  while ((size_t)2 * ((g.rows + s - 1) / s + 1) * g.rank * 4 > kColsSmem) ++s;
  return s;
}

size_t lora_tc_ws_floats(const LoraGeom& g);

size_t lora_ws_floats(const LoraGeom& g) {
  const size_t simt = (size_t)g.rows * g.rank + (size_t)lora_splits(g) * (g.n_in + g.n_out) * g.rank;
  const size_t tc = lora_tc_ws_floats(g);
  return simt > tc ? simt : tc;
}

template <typename T, int R>
static cudaError_t launch_lora_impl(const LoraGeom& g, const void* x, const void* dy, const void* a, const void* b,
                                    float* da, float* db, float* u, float* ws, cudaStream_t st) {
  const T* X = static_cast<const T*>(x);
  const T* dY = static_cast<const T*>(dy);
  float* t = ws;
  float* part = ws + (size_t)g.rows * R;
  cudaError_t e;
  const int blocks = (g.rows + 3) / 4;
  lora_rows_kernel<T, R><<<blocks, 128, 0, st>>>(X, g.ldx, static_cast<const T*>(a), false, g.rows, g.n_in, t);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  lora_rows_kernel<T, R><<<blocks, 128, 0, st>>>(dY, g.ldy, static_cast<const T*>(b), true, g.rows, g.n_out, u);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int nsplit = lora_splits(g);
  const int max_rows = (g.rows + nsplit - 1) / nsplit + 1;
  auto cols_k = lora_cols_kernel<T, R>;
  static std::atomic<unsigned long long> attr_done{0};
  if ((e = ensure_smem_attr(cols_k, (int)kColsSmem, attr_done)) != cudaSuccess) return e;
  dim3 grid((g.n_in + g.n_out + 1023) / 1024, nsplit);
  cols_k<<<grid, 256, (size_t)2 * max_rows * R * 4, st>>>(X, g.ldx, dY, g.ldy, t, u, g.rows, g.n_in, g.n_out, nsplit,
                                                      part);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int rb = ((g.n_in + g.n_out) * R + 255) / 256;
  lora_reduce_kernel<R><<<rb < 296 ? rb : 296, 256, 0, st>>>(part, g.n_in, g.n_out, nsplit, da, db);
  return cudaGetLastError();
}

// ============================================================================ bf16 tensor-core path
// Used when the inputs are bf16 and n_in, n_out are multiples of 256 (every LLaMA projection).
// The contractions are rank-R skinny GEMMs whose operands are read once from HBM; at R = 8 they
// are 16 FLOP per loaded element per pass, which the CUDA cores (FFMA, fp32 inputs converted
// from bf16) cannot sustain at HBM rate, so both passes issue warp-level mma.sync.m16n8k16
// (bf16 in, fp32 accumulate; N = 8 = R matches the instruction, while a tcgen05 MMA would need
// N >= 16 and a TMEM round trip for a 16 x 8 result).  Two kernels, each a cluster of 8 CTAs
// whose partial sums are reduced in a fixed order through distributed shared memory, so the
// result is deterministic and no partial ever reaches global memory:
//   tu  : grid (8 column chunks, 64-row blocks, {X.A -> t, dY.B^T -> u}).  A warp owns 4 m16
//         tiles (64 rows) and k32 steps of its CTA's column chunk; X / dY fragments come from
//         16-B global loads with the k index permuted inside each 32-column step (thread q owns
//         physical columns 8q..8q+7; mma 0 takes 8q..8q+3, mma 1 8q+4..8q+7, logical k pairs
//         (2q, 2q+1) / (2q+8, 2q+9) mapped to consecutive physical pairs), and the same
//         permutation selects the B fragments (staged in smem in mma order: A columns packed in k
//         pairs, B rows as loaded).  The 8 chunk partials are summed through DSMEM; the result is
//         written as fp32 (u_out) and as bf16 hi + lo mma B fragments (x = hi + lo to 2^-16).
//   grad: grid (8 row splits, 256-column groups of [X | dY]).  dA = X^T u, dB = t^T dY with the
//         columns of X / dY as M (a thread's 16-B row vectors of 4 rows are re-paired into
//         k = row fragments with PRMT) and rows as K; hi and lo fragments give two MMAs.  The 8
//         row-split partials are summed through DSMEM and added into dA / dB.
// Both kernels read X and dY once each (the second kernel mostly from L2).
namespace lora_tc {
constexpr int kCluster = 8;
constexpr int kThreads = 128;          // 4 warps per CTA
constexpr int kRowsTU = 64;            // rows per tu CTA (4 m16 tiles per warp)
constexpr int kColsG = 256;            // columns per grad CTA (64 per warp, 4 m16 tiles)

SECO_DEV void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 16-B read-only load, zero when !ok.  asm volatile keeps the loads of a batch in program order
// ahead of the (also volatile) MMAs that consume them: the compiler would otherwise sink each
// load next to its first use and leave only a few of them in flight
SECO_DEV uint4 ldg16(const __nv_bfloat16* p, bool ok) {
  uint4 v;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "r"((int)ok));
  return v;
}
// bf16 hi / lo split of two fp32 values (lower k in the low half): x ~= hi + lo
SECO_DEV void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
  const __nv_bfloat16 l0 = __float2bfloat16_rn(x0 - __bfloat162float(h0));
  const __nv_bfloat16 l1 = __float2bfloat16_rn(x1 - __bfloat162float(h1));
  hi = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
  lo = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
}

struct Args {
  const __nv_bfloat16 *x, *dy, *a, *b;
  int64_t ldx, ldy;
  int rows, n_in, n_out;
  int nsteps;               // ceil(rows / 16)
  float *da, *db, *u;       // accumulators, u_out
  uint4* frag;              // [2 (0: t, 1: u)][nsteps][NT][32] hi/lo B fragments
};

// ---------------------------------------------------------------- shared-memory staging
// cp.async (16 B, L2 -> smem, zero-filled when !ok): each warp copies whole row segments, so
// every load instruction reads contiguous 512 B of a row (HBM-friendly), and a CTA has its
// whole tile in flight at once without spending registers on it
SECO_DEV void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
SECO_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SECO_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
SECO_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SECO_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// ---------------------------------------------------------------- pass 1: t = X A, u = dY B^T
// CTA (chunk c of the cluster, 64-row block, tensor): the [64 rows][n / 8 columns] tile goes to
// smem in one burst of cp.async (rows padded by 16 B: conflict-free ldmatrix); warp w then owns
// rows [16 w, 16 w + 16) and walks the chunk in k16 steps (ldmatrix A fragment, B fragments of
// the A / B slice staged in mma order).  The 8 chunk partials of a row block are summed in
// rank order through DSMEM.
template <int R>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads)
    lora_tu_kernel(const Args p) {
  constexpr int NT = (R + 7) / 8, RP = 8 * NT;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int tau = blockIdx.z;                       // 0: X A -> t, 1: dY B^T -> u
  const int n = tau ? p.n_out : p.n_in;
  const int chunk = n / kCluster;                   // columns of this CTA (multiple of 32)
  const int col_c = (int)cluster.block_rank() * chunk;
  const int row0 = blockIdx.y * kRowsTU;
  const __nv_bfloat16* M = tau ? p.dy : p.x;
  const int64_t ld = tau ? p.ldy : p.ldx;
  const int rstride = chunk * 2 + 16;               // bytes per staged row
  const int nk16 = chunk / 16;
  // smem: X / dY tile [64][chunk] | B fragments [k16 step][NT][lane] (uint2) | CTA partial [64][RP]
  //       | one 16-row step [16][RP] | raw A / B slice of the chunk
  uint8_t* sx = smem_raw;
  uint2* sfrag = reinterpret_cast<uint2*>(smem_raw + kRowsTU * rstride);
  float* part = reinterpret_cast<float*>(sfrag + nk16 * NT * 32);
  float* stepv = part + kRowsTU * RP;
  __nv_bfloat16* sraw = reinterpret_cast<__nv_bfloat16*>(stepv + 16 * RP);   // raw A / B slice
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, q = lane % 4;
  // group 0: the chunk's slice of A ([chunk][R], contiguous) or B ([R][chunk] rows of n_out)
  if constexpr (R % 8 == 0) {
    const uint32_t sr = smem_u32(sraw);
    if (tau == 0) {
      for (int e = threadIdx.x; e < chunk * R / 8; e += kThreads)
        cp_async16(sr + e * 16, p.a + (int64_t)col_c * R + e * 8, true);
    } else {
      const int vpr = chunk / 8;
      for (int e = threadIdx.x; e < R * vpr; e += kThreads) {
        const int k = e / vpr, v = e % vpr;
        cp_async16(sr + (k * chunk + v * 8) * 2, p.b + (int64_t)k * p.n_out + col_c + v * 8, true);
      }
    }
  } else {
    for (int e = threadIdx.x; e < chunk * R; e += kThreads)
      sraw[e] = tau == 0 ? p.a[(int64_t)col_c * R + e] : p.b[(int64_t)(e / chunk) * p.n_out + col_c + e % chunk];
  }
  cp_async_commit();
  // group 1: the [64 rows][chunk] X / dY tile, whole row segments per warp instruction
  {
    const uint32_t sxa = smem_u32(sx);
    const int vpr = chunk / 8;                      // 16-B vectors per row
    for (int e = threadIdx.x; e < kRowsTU * vpr; e += kThreads) {
      const int r = e / vpr, v = e % vpr;
      const bool ok = row0 + r < p.rows;
      cp_async16(sxa + r * rstride + v * 16, M + (int64_t)(ok ? row0 + r : 0) * ld + col_c + v * 8, ok);
    }
    cp_async_commit();
  }
  cp_async_wait<1>();                               // the slice has landed; the tile streams on
  __syncthreads();
  // B fragments in mma order, standard k order: lane (g, q) of step s needs k = 16 s + {2q, 2q+1}
  // (b0) and {2q+8, 2q+9} (b1) at n = 8 nt + g
  for (int e = threadIdx.x; e < nk16 * NT * 32; e += kThreads) {
    const int ln = e % 32, nt = (e / 32) % NT, s = e / (32 * NT);
    const int nn = 8 * nt + ln / 4, k0 = 16 * s + 2 * (ln % 4);
    uint2 f = make_uint2(0u, 0u);
    if (nn < R) {
      if (tau == 0) {   // A slice [chunk][R]
        f.x = (uint32_t)__bfloat16_as_ushort(sraw[k0 * R + nn]) |
              ((uint32_t)__bfloat16_as_ushort(sraw[(k0 + 1) * R + nn]) << 16);
        f.y = (uint32_t)__bfloat16_as_ushort(sraw[(k0 + 8) * R + nn]) |
              ((uint32_t)__bfloat16_as_ushort(sraw[(k0 + 9) * R + nn]) << 16);
      } else {          // B slice [R][chunk]
        f.x = *reinterpret_cast<const uint32_t*>(sraw + nn * chunk + k0);
        f.y = *reinterpret_cast<const uint32_t*>(sraw + nn * chunk + k0 + 8);
      }
    }
    sfrag[e] = f;
  }
  cp_async_wait<0>();
  __syncthreads();
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
  // ldmatrix row address of this lane: rows 16 w + (lane % 16), k offset 8 (lane / 16)
  const uint32_t arow = smem_u32(sx) + (16 * warp + lane % 16) * rstride + (lane / 16) * 16;
#pragma unroll 4
  for (int s = 0; s < nk16; ++s) {
    uint32_t a0, a1, a2, a3;
    ldsm_x4(arow + s * 32, a0, a1, a2, a3);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint2 f = sfrag[(s * NT + nt) * 32 + lane];
      mma16816(acc[nt], a0, a1, a2, a3, f.x, f.y);
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float* w0 = part + (16 * warp + g) * RP + 8 * nt + 2 * q;
    w0[0] = acc[nt][0]; w0[1] = acc[nt][1];
    w0[8 * RP] = acc[nt][2]; w0[8 * RP + 1] = acc[nt][3];
  }
  cluster.sync();                                   // every chunk's partial is visible
  const int rank = (int)cluster.block_rank();
  if (rank < kRowsTU / 16) {                        // ranks 0..3: one 16-row step each
    const int step = blockIdx.y * (kRowsTU / 16) + rank;
    for (int e = threadIdx.x; e < 16 * RP; e += kThreads) {
      float v = 0.f;
#pragma unroll
      for (int c = 0; c < kCluster; ++c) v += cluster.map_shared_rank(part, c)[16 * rank * RP + e];
      stepv[e] = v;
      const int r = 16 * step + e / RP, k = e % RP;
      if (tau == 1 && k < R && r < p.rows) p.u[(int64_t)r * R + k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 32 && step < p.nsteps) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int k = 8 * nt + g;
        uint4 f;
        split2(stepv[(2 * q) * RP + k], stepv[(2 * q + 1) * RP + k], f.x, f.z);
        split2(stepv[(2 * q + 8) * RP + k], stepv[(2 * q + 9) * RP + k], f.y, f.w);
        p.frag[(((int64_t)tau * p.nsteps + step) * NT + nt) * 32 + lane] = f;   // {hi0, hi1, lo0, lo1}
      }
    }
  }
  cluster.sync();                                   // keep smem alive until every rank has read it
}

// ---------------------------------------------------------------- pass 2: dA += X^T u, dB += t^T dY
// CTA (row split r of the cluster, 256-column group of [X | dY]): 64-row slabs of the group go
// to smem through a 3-deep cp.async ring; warp w owns columns [64 w, 64 w + 64) (4 m16 tiles:
// columns are M, rows are K) and takes its A fragments with ldmatrix.trans; the B fragments are
// pass 1's hi / lo fragments of u (for X) or t (for dY).  The 8 row-split partials are summed in
// rank order through DSMEM and added into dA / dB.
template <int R>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads)
    lora_grad_kernel(const Args p) {
  constexpr int NT = (R + 7) / 8, RP = 8 * NT;
  constexpr int SLAB = 64, NSTAGE = 3;
  constexpr int RS = kColsG * 2 + 16;               // bytes per staged row
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float* part = reinterpret_cast<float*>(smem_raw);                    // [256 columns][RP]
  uint8_t* ring = smem_raw + kColsG * RP * 4;                          // [NSTAGE][SLAB][RS]
  // the slab's hi / lo B fragments ride in the same ring stage: [NSTAGE][SLAB / 16][NT][32] uint4
  uint8_t* fring = ring + NSTAGE * SLAB * RS;
  const int rank = (int)cluster.block_rank();
  const int gcol = blockIdx.y * kColsG;             // global column of [X | dY]
  const bool isA = gcol < p.n_in;
  const __nv_bfloat16* M = isA ? p.x : p.dy;
  const int64_t ld = isA ? p.ldx : p.ldy;
  const int col0 = isA ? gcol : gcol - p.n_in;
  const uint4* frag = p.frag + (int64_t)(isA ? 1 : 0) * p.nsteps * NT * 32;   // X^T u, t^T dY
  const int s0 = rank * p.nsteps / kCluster, s1 = (rank + 1) * p.nsteps / kCluster;
  const int r_begin = 16 * s0, r_end = 16 * s1;     // this split's rows (padded to 16)
  const int nslab = (r_end - r_begin + SLAB - 1) / SLAB;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, q = lane % 4;
  const uint32_t ring_a = smem_u32(ring);
  auto load_slab = [&](int sl) {
    const uint32_t base = ring_a + (sl % NSTAGE) * SLAB * RS;
    for (int e = threadIdx.x; e < SLAB * (kColsG / 8); e += kThreads) {
      const int r = e / (kColsG / 8), v = e % (kColsG / 8);
      const int row = r_begin + sl * SLAB + r;
      const bool ok = row < r_end && row < p.rows;
      cp_async16(base + r * RS + v * 16, M + (int64_t)(ok ? row : 0) * ld + col0 + v * 8, ok);
    }
    const uint32_t fb = smem_u32(fring) + (sl % NSTAGE) * (SLAB / 16) * NT * 32 * 16;
    const int sfirst = (r_begin + sl * SLAB) / 16;
    for (int e = threadIdx.x; e < (SLAB / 16) * NT * 32; e += kThreads) {
      const int st = sfirst + e / (NT * 32);
      cp_async16(fb + e * 16, frag + (int64_t)(st < s1 ? st : s0) * NT * 32 + e % (NT * 32), st < s1);
    }
    cp_async_commit();
  };
  float acc[4][NT][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][nt][e] = 0.f;
  for (int sl = 0; sl < NSTAGE - 1; ++sl) {
    if (sl < nslab) load_slab(sl); else cp_async_commit();
  }
  // ldmatrix.trans: matrix i = lane / 8 covers stored rows (K) 8 (i / 2) .. +7 of the k16 step at
  // stored columns (M) 16 j + 8 (i % 2); lane supplies row lane % 8 of it
  const int li = lane / 8, lr = lane % 8;
  const uint32_t lane_off = (uint32_t)((8 * (li / 2) + lr) * RS + (64 * warp + 8 * (li % 2)) * 2);
  for (int sl = 0; sl < nslab; ++sl) {
    if (sl + NSTAGE - 1 < nslab) load_slab(sl + NSTAGE - 1); else cp_async_commit();
    cp_async_wait<NSTAGE - 1>();
    __syncthreads();
    const uint32_t base = ring_a + (sl % NSTAGE) * SLAB * RS + lane_off;
#pragma unroll
    for (int kk = 0; kk < SLAB / 16; ++kk) {
      const int s = (r_begin + sl * SLAB) / 16 + kk;   // global 16-row step
      if (s >= s1) break;
      uint4 f[NT];
      const uint4* sf = reinterpret_cast<const uint4*>(fring) + ((sl % NSTAGE) * (SLAB / 16) + kk) * NT * 32;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) f[nt] = sf[nt * 32 + lane];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(base + kk * 16 * RS + j * 32, a0, a1, a2, a3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mma16816(acc[j][nt], a0, a1, a2, a3, f[nt].x, f[nt].y);   // hi
          mma16816(acc[j][nt], a0, a1, a2, a3, f[nt].z, f[nt].w);   // lo
        }
      }
    }
    __syncthreads();                                // the slab's stage may be refilled next
  }
  cp_async_wait<0>();
  // CTA partial [256 columns][RP]: tile j of warp w covers columns 64 w + 16 j + {g, g + 8}
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float* d0 = part + (64 * warp + 16 * j + g) * RP + 8 * nt + 2 * q;
      d0[0] = acc[j][nt][0]; d0[1] = acc[j][nt][1];
      d0[8 * RP] = acc[j][nt][2]; d0[8 * RP + 1] = acc[j][nt][3];
    }
  cluster.sync();
  // rank r adds columns [32 r, 32 r + 32) of the 8 row-split partials, in rank order
  for (int e = threadIdx.x; e < 32 * R; e += kThreads) {
    const int cl = 32 * rank + e / R, k = e % R;
    float v = 0.f;
#pragma unroll
    for (int c = 0; c < kCluster; ++c) v += cluster.map_shared_rank(part, c)[cl * RP + k];
    if (isA) p.da[(int64_t)(col0 + cl) * R + k] += v;
    else p.db[(int64_t)k * p.n_out + col0 + cl] += v;
  }
  cluster.sync();
}

template <int R>
size_t tu_smem(int n_in, int n_out) {
  constexpr int NT = (R + 7) / 8, RP = 8 * NT;
  const int chunk = (n_in > n_out ? n_in : n_out) / kCluster;
  return (size_t)kRowsTU * (chunk * 2 + 16) + (size_t)(chunk / 16) * NT * 32 * 8 + (size_t)(kRowsTU + 16) * RP * 4 +
         (size_t)chunk * R * 2;
}
template <int R>
constexpr size_t grad_smem() {
  return (size_t)kColsG * 8 * ((R + 7) / 8) * 4 + (size_t)3 * 64 * (kColsG * 2 + 16) +
         (size_t)3 * 4 * ((R + 7) / 8) * 32 * 16;
}
}  // namespace lora_tc

// ============================================================================ fused persistent path
// lora_fused_kernel: one launch that reads X and dY exactly once (round 2).  A
// cluster of CS CTAs splits the columns: CTA r of a cluster owns columns [r n_in / CS, ...) of X
// and [r n_out / CS, ...) of dY, so the A / B slices it contracts against stay in registers for
// the whole launch and its share of dA / dB accumulates in registers too.  Clusters are
// persistent (as many as are co-resident) and walk contiguous ranges of 16-row blocks.  Per block:
//   1. a producer warp streams the CTA's 16 X rows and 16 dY rows (one row per lane, 1-D bulk
//      copies) into a STAGES-deep ring, completing on an mbarrier;
//   2. the NW compute warps form the CTA's partial t = X A and u = dY B^T over its columns
//      (mma.sync m16n8k16, ldmatrix from the ring), sum them across warps, and push the CTA
//      partial into slot [rank] of every peer's receive buffer with st.async (remote shared-
//      memory stores that complete_tx on the peer's mbarrier: no cross-CTA round trip);
//   3. once the CS partials have landed, every lane sums the values its mma fragments need in
//      rank order (so every CTA sees bit-identical t, u; rank 0 writes u_out), splits them into
//      bf16 hi + lo (x = hi + lo to 2^-16) and adds X^T u and dY^T t for its columns -- from the
//      same ring stage, so nothing is read twice -- into its register accumulators.
// The receive buffers alternate between blocks; a peer can refill one only after it received
// this CTA's partial of the next block, which this CTA sends after it finished reading it.
// At the end each CTA writes its dA / dB share to the workspace ([cluster][n_in + n_out][R]),
// publishes a per-launch epoch flag, and -- once the CTAs of its rank in every cluster have
// published -- adds the ncl cluster partials of its share of the rank's columns in cluster order
// into dA / dB: deterministic, no atomics, one launch.
// R <= 8: clusters of 4 with 16 compute warps (1024 columns of X and dY per CTA); R = 16 (twice
// the registers per fragment): clusters of 8 with 8 compute warps.
namespace lora_fz {
constexpr int kRB = 16;                      // rows per block (one m16 tile)
constexpr int KW = 4;                        // k16 steps (pass 1) / m16 tiles (pass 2) per warp
constexpr int kMaxN = 4096;                  // n_in, n_out bound of the fused path
constexpr int kMaxClusters = 40;             // workspace bound (148 SMs: at most 37 clusters of 4)

template <int R> struct Cfg {
  static constexpr int CS = R > 8 ? 8 : 4;                  // CTAs per cluster
  static constexpr int NW = R > 8 ? 8 : 16;                 // compute warps
  static constexpr int kThreads = 32 * (NW + 1);            // + one producer warp
  static constexpr int STAGES = R > 8 ? 4 : 3;
  static constexpr int NT = (R + 7) / 8, RP = 8 * NT;
  static constexpr int NE = 2 * kRB * RP;                   // t and u of one block
  static_assert(kMaxN / CS == 16 * NW * KW, "columns per CTA = k16 steps of the warps");
};

struct Args {
  const __nv_bfloat16 *x, *dy, *a, *b;
  int64_t ldx, ldy;
  int rows, n_in, n_out, nblk, ncl;
  float* u;                                  // u_out [rows][R]
  float* part;                               // deterministic: [ncl][n_in R | R n_out] cluster partials
  float *da, *db;                            // accumulators
  int deterministic;
};

#ifdef SECO_LORA_TRACE
// experiment build only (SECO_DEFINES=-DSECO_LORA_TRACE=1): clock64 per phase and block of CTA 0
constexpr int kTrBlocks = 32, kTrPts = 12;
__device__ unsigned long long g_lora_trace[kTrBlocks * kTrPts];
#define LTRACE(pt, i)                                                                        \
  do {                                                                                       \
    if (blockIdx.x == 0 && (i) < kTrBlocks) g_lora_trace[(i) * kTrPts + (pt)] = clock64();   \
  } while (0)
#else
#define LTRACE(pt, i) do { } while (0)
#endif

// remote shared-memory store of 16 B whose bytes complete_tx on the destination CTA's mbarrier
SECO_DEV void st_async_v4(uint32_t dst_cluster, float4 v, uint32_t bar_cluster) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(dst_cluster), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar_cluster)
               : "memory");
}

template <int R>
inline size_t smem_bytes(int n_in, int n_out) {
  using C = Cfg<R>;
  const size_t stage = (size_t)kRB * ((n_in / C::CS) * 2 + 16 + (n_out / C::CS) * 2 + 16);
  return C::STAGES * stage + (size_t)(C::NW + 2 * C::CS + 1) * C::NE * 4 + (2 * C::STAGES + 2) * 8;
}

template <int R>
__global__ void __launch_bounds__(Cfg<R>::kThreads, 1) lora_fused_kernel(const Args p) {
  using lora_tc::ldsm_x4;
  using lora_tc::ldsm_x4_t;
  using lora_tc::mma16816;
  using lora_tc::split2;
  using C = Cfg<R>;
  constexpr int CS = C::CS, NW = C::NW, STAGES = C::STAGES, NT = C::NT, RP = C::RP, NE = C::NE;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, q = lane % 4;
  const int rank = (int)cluster_ctarank();
  const int cl = (int)blockIdx.x / CS;
  const int cx = p.n_in / CS, cy = p.n_out / CS;             // columns of this CTA
  const int colx = rank * cx, coly = rank * cy;
  const int rsx = cx * 2 + 16, rsy = cy * 2 + 16;            // staged row bytes (+16: ldmatrix banks)
  const int stage_bytes = kRB * (rsx + rsy);
  const uint32_t ring = smem_u32(smem);
  float* wpart = reinterpret_cast<float*>(smem + STAGES * stage_bytes);    // [NW][NE]
  float* recv = wpart + NW * NE;                                            // [2][CS][NE]
  float* tu = recv + 2 * CS * NE;                                           // [t | u][n][row]
  const uint32_t bar0 = smem_u32(tu + NE);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto rfull = [&](int b) { return bar0 + 8u * (2 * STAGES + b); };
  const int b0 = cl * p.nblk / p.ncl, nb = (cl + 1) * p.nblk / p.ncl - b0;

  if (threadIdx.x == 0) LTRACE(10, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), NW); }
    mbar_init(rfull(0), 1);
    mbar_init(rfull(1), 1);
    fence_barrier_init();
  }
  cluster_sync();                            // every peer's barriers exist before the first remote store

  if (warp == NW) {
    // ------------------------------------------------------------ producer: one row per lane
    const int r = lane % kRB;
    const bool isy = lane >= kRB;
    const int bytes = isy ? cy * 2 : cx * 2;
    for (int i = 0; i < nb; ++i) {
      const int s = i % STAGES;
      const int row0 = (b0 + i) * kRB;
      const int nvalid = min(kRB, p.rows - row0);
      if (lane == 0) mbar_wait(empty(s), ((i / STAGES) & 1) ^ 1);
      __syncwarp();
      const uint32_t dst = ring + s * stage_bytes + (isy ? kRB * rsx + r * rsy : r * rsx);
      if (r >= nvalid) {                     // ragged tail: zero rows
        for (int o = 0; o < bytes; o += 16) st_shared_v4(dst + o, 0u, 0u, 0u, 0u);
        fence_async_smem();
      }
      __syncwarp();
      if (lane == 0) mbar_expect_tx(full(s), (uint32_t)nvalid * (cx + cy) * 2);
      __syncwarp();
      if (lane == 0) LTRACE(7, i);
      if (r < nvalid) {
        const __nv_bfloat16* src = isy ? p.dy + (int64_t)(row0 + r) * p.ldy + coly
                                       : p.x + (int64_t)(row0 + r) * p.ldx + colx;
        bulk_load(dst, src, (uint32_t)bytes, full(s));
      }
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int tid = threadIdx.x;
    const int nkx = cx / 16, nky = cy / 16;  // k16 steps of pass 1 = m16 tiles of pass 2
    // pass-1 B fragments (lane (g, q): k = 16 ks + {2q, 2q+1} / {2q+8, 2q+9}, n = 8 nt + g):
    // A [n_in][R] for t = X A, B^T for u = dY B^T; columns n >= R stay zero
    uint32_t fa[KW][NT][2], fb[KW][NT][2];
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
      const int ks = warp + NW * kk;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int n = 8 * nt + g;
        fa[kk][nt][0] = fa[kk][nt][1] = fb[kk][nt][0] = fb[kk][nt][1] = 0u;
        if (n < R && ks < nkx) {
          const __nv_bfloat16* ap = p.a + (int64_t)(colx + 16 * ks + 2 * q) * R + n;
          fa[kk][nt][0] = (uint32_t)__bfloat16_as_ushort(ap[0]) | ((uint32_t)__bfloat16_as_ushort(ap[R]) << 16);
          fa[kk][nt][1] = (uint32_t)__bfloat16_as_ushort(ap[8 * R]) | ((uint32_t)__bfloat16_as_ushort(ap[9 * R]) << 16);
        }
        if (n < R && ks < nky) {
          const __nv_bfloat16* bp = p.b + (int64_t)n * p.n_out + coly + 16 * ks + 2 * q;
          fb[kk][nt][0] = *reinterpret_cast<const uint32_t*>(bp);
          fb[kk][nt][1] = *reinterpret_cast<const uint32_t*>(bp + 8);
        }
      }
    }
    float accA[KW][NT][4], accB[KW][NT][4];
#pragma unroll
    for (int kk = 0; kk < KW; ++kk)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) accA[kk][nt][e] = accB[kk][nt][e] = 0.f;
    if (tid == 0) LTRACE(10, 1);
    const int li = lane / 8, lr = lane % 8;
    const uint32_t offx = (uint32_t)((lane % 16) * rsx + (lane / 16) * 16);    // ldmatrix (rows = M)
    const uint32_t offy = (uint32_t)((lane % 16) * rsy + (lane / 16) * 16);
    const uint32_t toffx = (uint32_t)((8 * (li / 2) + lr) * rsx + 8 * (li % 2) * 2);   // .trans (rows = K)
    const uint32_t toffy = (uint32_t)((8 * (li / 2) + lr) * rsy + 8 * (li % 2) * 2);
    const uint32_t recv_a = smem_u32(recv);
    for (int i = 0; i < nb; ++i) {
      const int s = i % STAGES, pb = i & 1;
      const int row0 = (b0 + i) * kRB;
      const uint32_t xs = ring + s * stage_bytes, ys = xs + kRB * rsx;
      if (tid == 0) mbar_expect_tx(rfull(pb), (uint32_t)(CS * NE * 4));   // this block's CS partials
      mbar_wait(full(s), (i / STAGES) & 1);
      if (tid == 0) LTRACE(0, i);
      // pass 1: this warp's share of the CTA partial of t and u
      float ct[NT][4], cu[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) ct[nt][e] = cu[nt][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KW; ++kk) {
        const int ks = warp + NW * kk;
        uint32_t a0, a1, a2, a3;
        if (ks < nkx) {
          ldsm_x4(xs + offx + ks * 32, a0, a1, a2, a3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma16816(ct[nt], a0, a1, a2, a3, fa[kk][nt][0], fa[kk][nt][1]);
        }
        if (ks < nky) {
          ldsm_x4(ys + offy + ks * 32, a0, a1, a2, a3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma16816(cu[nt], a0, a1, a2, a3, fb[kk][nt][0], fb[kk][nt][1]);
        }
      }
      if (tid == 0) LTRACE(1, i);
      float* wp = wpart + warp * NE;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c0 = 8 * nt + 2 * q;
        *reinterpret_cast<float2*>(wp + g * RP + c0) = make_float2(ct[nt][0], ct[nt][1]);
        *reinterpret_cast<float2*>(wp + (g + 8) * RP + c0) = make_float2(ct[nt][2], ct[nt][3]);
        *reinterpret_cast<float2*>(wp + kRB * RP + g * RP + c0) = make_float2(cu[nt][0], cu[nt][1]);
        *reinterpret_cast<float2*>(wp + kRB * RP + (g + 8) * RP + c0) = make_float2(cu[nt][2], cu[nt][3]);
      }
      named_bar_sync(1, 32 * NW);
      if (tid == 0) LTRACE(2, i);
      // CTA partial (warps summed in order), 4 values per thread, pushed to slot [rank] of
      // every peer's receive buffer (this CTA's own included)
      static_assert(NE / 4 <= 32 * NW, "one float4 of the CTA partial per thread");
      if (tid < NE / 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const float4 x = reinterpret_cast<const float4*>(wpart + w * NE)[tid];
          v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
        }
        const uint32_t dst = recv_a + (uint32_t)((pb * CS + rank) * NE + 4 * tid) * 4u;
#pragma unroll
        for (int c = 0; c < CS; ++c) st_async_v4(mapa_shared(dst, (uint32_t)c), v, mapa_shared(rfull(pb), (uint32_t)c));
      }
      if (tid == 0) LTRACE(3, i);
      // acquire at cluster scope: the peers' stores (and, through them, their reads of the
      // buffer this block's stores may reuse two blocks later) are ordered before what follows
      mbar_wait_cluster(rfull(pb), (i >> 1) & 1);
      if (tid == 0) LTRACE(4, i);
      // t, u of the block: the CS partials summed in rank order, once per value (every CTA of the
      // cluster forms bit-identical sums); stored n-major so a lane's fragment rows are adjacent
      for (int e = tid; e < NE; e += 32 * NW) {
        const float* rb = recv + pb * CS * NE;
        float v = 0.f;
#pragma unroll
        for (int c = 0; c < CS; ++c) v += rb[c * NE + e];
        const int isu = e / (kRB * RP), row = (e / RP) % kRB, n = e % RP;
        tu[isu * kRB * RP + n * kRB + row] = v;
        if (isu && rank == 0 && n < R && row0 + row < p.rows) p.u[(int64_t)(row0 + row) * R + n] = v;
      }
      named_bar_sync(1, 32 * NW);
      // pass 2 B fragments: u (for X^T u) and t (for dY^T t); k = row, n = rank; hi + lo
      uint32_t fu[NT][4], ft[NT][4];   // {hi0, hi1, lo0, lo1}
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int n = 8 * nt + g;
        const float2 t01 = *reinterpret_cast<const float2*>(tu + n * kRB + 2 * q);
        const float2 t89 = *reinterpret_cast<const float2*>(tu + n * kRB + 2 * q + 8);
        const float2 u01 = *reinterpret_cast<const float2*>(tu + kRB * RP + n * kRB + 2 * q);
        const float2 u89 = *reinterpret_cast<const float2*>(tu + kRB * RP + n * kRB + 2 * q + 8);
        split2(u01.x, u01.y, fu[nt][0], fu[nt][2]);
        split2(u89.x, u89.y, fu[nt][1], fu[nt][3]);
        split2(t01.x, t01.y, ft[nt][0], ft[nt][2]);
        split2(t89.x, t89.y, ft[nt][1], ft[nt][3]);
      }
      if (tid == 0) LTRACE(5, i);
#pragma unroll
      for (int kk = 0; kk < KW; ++kk) {
        const int mt = warp + NW * kk;
        uint32_t a0, a1, a2, a3;
        if (mt < nkx) {
          ldsm_x4_t(xs + toffx + mt * 32, a0, a1, a2, a3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma16816(accA[kk][nt], a0, a1, a2, a3, fu[nt][0], fu[nt][1]);
            mma16816(accA[kk][nt], a0, a1, a2, a3, fu[nt][2], fu[nt][3]);
          }
        }
        if (mt < nky) {
          ldsm_x4_t(ys + toffy + mt * 32, a0, a1, a2, a3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma16816(accB[kk][nt], a0, a1, a2, a3, ft[nt][0], ft[nt][1]);
            mma16816(accB[kk][nt], a0, a1, a2, a3, ft[nt][2], ft[nt][3]);
          }
        }
      }
      __syncwarp();
      if (tid == 0) LTRACE(6, i);
      if (lane == 0) mbar_arrive(empty(s));
    }
    if (tid == 0) LTRACE(11, 0);
    // this cluster's share of dA (columns of X, [col][R] as in dA) and dB (columns of dY,
    // [R][col] as in dB), staged in the (now idle) ring and moved with 1-D bulk copies: 1 + R
    // contiguous runs.  Default: TMA reduce-add straight into dA / dB (cluster order unfixed,
    // like the attention backward's dQ / dKV deposits).  Deterministic: the runs go to the
    // workspace and lora_fused_reduce_kernel adds the clusters in order.
    named_bar_sync(1, 32 * NW);                               // every warp is done with the ring
    float* stg = reinterpret_cast<float*>(smem);              // [cx][R] | [R][cy]
    float* stgy = stg + cx * R;
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
      const int mt = warp + NW * kk;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = 8 * nt + 2 * q + e;
            if (k >= R) continue;
            if (mt < nkx) stg[(16 * mt + g + 8 * h) * R + k] = accA[kk][nt][2 * h + e];
            if (mt < nky) stgy[k * cy + 16 * mt + g + 8 * h] = accB[kk][nt][2 * h + e];
          }
    }
    fence_async_smem();                                       // generic smem writes -> bulk copies
    named_bar_sync(1, 32 * NW);
    if (tid == 0) {
      float* oa = p.deterministic ? p.part + (int64_t)cl * (p.n_in + p.n_out) * R : p.da;
      float* ob = p.deterministic ? oa + (int64_t)p.n_in * R : p.db;
      if (p.deterministic) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(oa + (int64_t)colx * R), "r"(smem_u32(stg)), "r"(cx * R * 4) : "memory");
        for (int k = 0; k < R; ++k)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(ob + (int64_t)k * p.n_out + coly), "r"(smem_u32(stgy + k * cy)), "r"(cy * 4) : "memory");
      } else {
        bulk_reduce_add_f32(oa + (int64_t)colx * R, smem_u32(stg), cx * R * 4);
        for (int k = 0; k < R; ++k) bulk_reduce_add_f32(ob + (int64_t)k * p.n_out + coly, smem_u32(stgy + k * cy), cy * 4);
      }
      bulk_commit();
      bulk_wait0();
      LTRACE(11, 1);
    }
  }
  cluster_sync();                            // no CTA leaves while a peer may still store into it
}

// Deterministic mode: dA / dB (as one flat [n_in R | R n_out] array) += the ncl cluster partials
// in a fixed association -- thread row cr takes clusters cr, cr + 8, ... in order, then the 8 row
// sums in row order.  Launched with programmatic stream serialization behind the fused kernel.
__global__ void __launch_bounds__(256) lora_fused_reduce_kernel(const float* __restrict__ part, int n_a, int n_b,
                                                                int ncl, float* __restrict__ dA, float* __restrict__ dB) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the fused kernel's partials are complete
  constexpr int G = 32, CR = 8, MAXC = (kMaxClusters + CR - 1) / CR;
  __shared__ float4 red[CR][G];
  const int n = n_a + n_b;                             // floats; n_a, n_b multiples of 4
  const int gi = threadIdx.x % G, cr = threadIdx.x / G;
  const int e = (blockIdx.x * G + gi) * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e < n) {
    float4 v[MAXC];
#pragma unroll
    for (int m = 0; m < MAXC; ++m)
      if (cr + CR * m < ncl) v[m] = *reinterpret_cast<const float4*>(part + (int64_t)(cr + CR * m) * n + e);
#pragma unroll
    for (int m = 0; m < MAXC; ++m)
      if (cr + CR * m < ncl) { acc.x += v[m].x; acc.y += v[m].y; acc.z += v[m].z; acc.w += v[m].w; }
  }
  red[cr][gi] = acc;
  __syncthreads();
  if (cr == 0 && e < n) {
#pragma unroll
    for (int r = 1; r < CR; ++r) {
      const float4 x = red[r][gi];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    float4* d = e < n_a ? reinterpret_cast<float4*>(dA + e) : reinterpret_cast<float4*>(dB + (e - n_a));
    float4 o = *d;
    o.x += acc.x; o.y += acc.y; o.z += acc.z; o.w += acc.w;
    *d = o;
  }
}
}  // namespace lora_fz

#ifdef SECO_LORA_TRACE
extern "C" int seco_debug_lora_trace(unsigned long long* host, int n) {
  const int m = n < lora_fz::kTrBlocks * lora_fz::kTrPts ? n : lora_fz::kTrBlocks * lora_fz::kTrPts;
  return (int)cudaMemcpyFromSymbol(host, lora_fz::g_lora_trace, m * sizeof(unsigned long long));
}
#endif

bool lora_fused_ok(const LoraGeom& g) {
  static const bool enabled = [] {
    const char* e = std::getenv("SECO_LORA_FUSED");  // A/B switch: SECO_LORA_FUSED=0 selects the 2-pass kernels
    return e == nullptr || e[0] != '0';
  }();
  const int cs = g.rank > 8 ? 8 : 4;
  return enabled && g.n_in % (16 * cs) == 0 && g.n_out % (16 * cs) == 0 && g.n_in <= lora_fz::kMaxN &&
         g.n_out <= lora_fz::kMaxN && g.ldx % 8 == 0 && g.ldy % 8 == 0 &&
         (g.rank == 1 || g.rank == 2 || g.rank == 4 || g.rank == 8 || g.rank == 16);
}

size_t lora_fused_ws_floats(const LoraGeom& g) {   // deterministic mode's cluster partials
  return (size_t)lora_fz::kMaxClusters * (g.n_in + g.n_out) * g.rank;
}

template <int R>
static cudaError_t launch_lora_fused(const LoraGeom& g, const void* x, const void* dy, const void* a, const void* b,
                                     float* da, float* db, float* u, float* ws, cudaStream_t st) {
  using namespace lora_fz;
  using C = Cfg<R>;
  const int max_smem = (int)smem_bytes<R>(kMaxN, kMaxN);
  static std::atomic<unsigned long long> attr_done{0};
  cudaError_t e = ensure_smem_attr(lora_fused_kernel<R>, max_smem, attr_done);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute cattr[1];
  cattr[0].id = cudaLaunchAttributeClusterDimension;
  cattr[0].val.clusterDim.x = C::CS; cattr[0].val.clusterDim.y = 1; cattr[0].val.clusterDim.z = 1;
  // persistent clusters: as many as are co-resident (queried once per device at the largest
  // shared-memory footprint, so a smaller shape never exceeds it)
  static std::atomic<int> max_cl[64];
  int dev = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  int ncl = max_cl[dev & 63].load(std::memory_order_relaxed);
  if (ncl == 0) {
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3(C::CS * kMaxClusters); qc.blockDim = dim3(C::kThreads); qc.dynamicSmemBytes = max_smem;
    qc.attrs = cattr; qc.numAttrs = 1;
    if ((e = cudaOccupancyMaxActiveClusters(&ncl, lora_fused_kernel<R>, &qc)) != cudaSuccess) return e;
    ncl = ncl < 1 ? 1 : (ncl > kMaxClusters ? kMaxClusters : ncl);
    max_cl[dev & 63].store(ncl, std::memory_order_relaxed);
    if (std::getenv("SECO_LORA_DEBUG")) fprintf(stderr, "lora_fused: %d co-resident clusters of %d\n", ncl, C::CS);
  }
  Args p;
  p.x = static_cast<const __nv_bfloat16*>(x); p.dy = static_cast<const __nv_bfloat16*>(dy);
  p.a = static_cast<const __nv_bfloat16*>(a); p.b = static_cast<const __nv_bfloat16*>(b);
  p.ldx = g.ldx; p.ldy = g.ldy; p.rows = g.rows; p.n_in = g.n_in; p.n_out = g.n_out;
  p.nblk = (g.rows + kRB - 1) / kRB;
  p.ncl = ncl < p.nblk ? ncl : p.nblk;
  p.u = u; p.part = ws; p.da = da; p.db = db; p.deterministic = g.deterministic;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C::CS * p.ncl); cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = smem_bytes<R>(g.n_in, g.n_out); cfg.stream = st;
  cfg.attrs = cattr; cfg.numAttrs = 1;
  if ((e = cudaLaunchKernelEx(&cfg, lora_fused_kernel<R>, p)) != cudaSuccess || !g.deterministic) return e;
  // deterministic: cluster partials -> dA, dB in cluster order (its launch overlaps the tail)
  cudaLaunchAttribute rattr[1];
  rattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  rattr[0].val.programmaticStreamSerializationAllowed = 1;
  const int n = (g.n_in + g.n_out) * R;
  cudaLaunchConfig_t rc = {};
  rc.gridDim = dim3((n / 4 + 31) / 32); rc.blockDim = dim3(256); rc.stream = st; rc.attrs = rattr; rc.numAttrs = 1;
  return cudaLaunchKernelEx(&rc, lora_fused_reduce_kernel, (const float*)ws, g.n_in * R, g.n_out * R, p.ncl, da, db);
}

bool lora_tc_ok(const LoraGeom& g) {
  static const bool enabled = [] {
    const char* e = std::getenv("SECO_LORA_TC");     // A/B switch: SECO_LORA_TC=0 selects the CUDA-core kernels
    return e == nullptr || e[0] != '0';
  }();
  return enabled && g.n_in % 256 == 0 && g.n_out % 256 == 0 && g.ldx % 8 == 0 && g.ldy % 8 == 0 &&
         (g.rank == 1 || g.rank == 2 || g.rank == 4 || g.rank == 8 || g.rank == 16) &&
         lora_tc::tu_smem<16>(g.n_in, g.n_out) <= 200 * 1024;
}

size_t lora_tc_ws_floats(const LoraGeom& g) {
  const int nt = g.rank > 8 ? 2 : 1;
  const size_t tc = (size_t)2 * ((g.rows + 15) / 16) * nt * 32 * 4;
  const size_t fz = lora_fused_ws_floats(g);
  return tc > fz ? tc : fz;
}

template <int R>
static cudaError_t launch_lora_tc(const LoraGeom& g, const void* x, const void* dy, const void* a, const void* b,
                                  float* da, float* db, float* u, float* ws, cudaStream_t st) {
  lora_tc::Args p;
  p.x = static_cast<const __nv_bfloat16*>(x); p.dy = static_cast<const __nv_bfloat16*>(dy);
  p.a = static_cast<const __nv_bfloat16*>(a); p.b = static_cast<const __nv_bfloat16*>(b);
  p.ldx = g.ldx; p.ldy = g.ldy; p.rows = g.rows; p.n_in = g.n_in; p.n_out = g.n_out;
  p.nsteps = (g.rows + 15) / 16;
  p.da = da; p.db = db; p.u = u;
  p.frag = reinterpret_cast<uint4*>(ws);
  const size_t smem = lora_tc::tu_smem<R>(g.n_in, g.n_out);
  static std::atomic<unsigned long long> attr_done{0};
  cudaError_t e = ensure_smem_attr(lora_tc::lora_tu_kernel<R>, 200 * 1024, attr_done);
  if (e != cudaSuccess) return e;
  dim3 g1(lora_tc::kCluster, (g.rows + lora_tc::kRowsTU - 1) / lora_tc::kRowsTU, 2);
  lora_tc::lora_tu_kernel<R><<<g1, lora_tc::kThreads, smem, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  static std::atomic<unsigned long long> attr_done2{0};
  if ((e = ensure_smem_attr(lora_tc::lora_grad_kernel<R>, (int)lora_tc::grad_smem<R>(), attr_done2)) != cudaSuccess)
    return e;
  dim3 g2(lora_tc::kCluster, (g.n_in + g.n_out) / lora_tc::kColsG);
  lora_tc::lora_grad_kernel<R><<<g2, lora_tc::kThreads, lora_tc::grad_smem<R>(), st>>>(p);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_lora_t(const LoraGeom& g, const void* x, const void* dy, const void* a, const void* b,
                                 float* da, float* db, float* u, float* ws, cudaStream_t st) {
  switch (g.rank) {
    case 1: return launch_lora_impl<T, 1>(g, x, dy, a, b, da, db, u, ws, st);
    case 2: return launch_lora_impl<T, 2>(g, x, dy, a, b, da, db, u, ws, st);
    case 4: return launch_lora_impl<T, 4>(g, x, dy, a, b, da, db, u, ws, st);
    case 8: return launch_lora_impl<T, 8>(g, x, dy, a, b, da, db, u, ws, st);
    case 16: return launch_lora_impl<T, 16>(g, x, dy, a, b, da, db, u, ws, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_lora_grad(const LoraGeom& g, bool bf16, const void* x, const void* dy, const void* a,
                             const void* b, float* da, float* db, float* u, float* ws, cudaStream_t st,
                             int* launches) {
  if (bf16 && lora_fused_ok(g)) {
    *launches = g.deterministic ? 2 : 1;
    switch (g.rank) {
      case 1: return launch_lora_fused<1>(g, x, dy, a, b, da, db, u, ws, st);
      case 2: return launch_lora_fused<2>(g, x, dy, a, b, da, db, u, ws, st);
      case 4: return launch_lora_fused<4>(g, x, dy, a, b, da, db, u, ws, st);
      case 8: return launch_lora_fused<8>(g, x, dy, a, b, da, db, u, ws, st);
      default: return launch_lora_fused<16>(g, x, dy, a, b, da, db, u, ws, st);
    }
  }
  if (bf16 && lora_tc_ok(g)) {
    *launches = 2;
    switch (g.rank) {
      case 1: return launch_lora_tc<1>(g, x, dy, a, b, da, db, u, ws, st);
      case 2: return launch_lora_tc<2>(g, x, dy, a, b, da, db, u, ws, st);
      case 4: return launch_lora_tc<4>(g, x, dy, a, b, da, db, u, ws, st);
      case 8: return launch_lora_tc<8>(g, x, dy, a, b, da, db, u, ws, st);
      default: return launch_lora_tc<16>(g, x, dy, a, b, da, db, u, ws, st);
    }
  }
  *launches = 4;
  return bf16 ? launch_lora_t<__nv_bfloat16>(g, x, dy, a, b, da, db, u, ws, st)
              : launch_lora_t<float>(g, x, dy, a, b, da, db, u, ws, st);
}

unsigned long long check_word_lora() { return seco_check_read_clear(); }

}  // namespace seco
