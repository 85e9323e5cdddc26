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

int lora_splits(const LoraGeom& g) {
  const int col_blocks = (g.n_in + g.n_out + 1023) / 1024;
  int s = (2 * 148 + col_blocks - 1) / col_blocks;
  s = s < 1 ? 1 : s;
  const int max_s = g.rows / 64 > 0 ? g.rows / 64 : 1;   // at least ~64 rows per split
  return s > max_s ? max_s : s;
}

size_t lora_ws_floats(const LoraGeom& g) {
  return (size_t)g.rows * g.rank + (size_t)lora_splits(g) * (g.n_in + g.n_out) * g.rank;
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
  e = cudaFuncSetAttribute(cols_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * max_rows * R * 4);
  if (e != cudaSuccess) return e;
  dim3 grid((g.n_in + g.n_out + 1023) / 1024, nsplit);
  cols_k<<<grid, 256, (size_t)2 * max_rows * R * 4, st>>>(X, g.ldx, dY, g.ldy, t, u, g.rows, g.n_in, g.n_out, nsplit,
                                                      part);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int rb = ((g.n_in + g.n_out) * R + 255) / 256;
  lora_reduce_kernel<R><<<rb < 296 ? rb : 296, 256, 0, st>>>(part, g.n_in, g.n_out, nsplit, da, db);
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
  *launches = 4;
  return bf16 ? launch_lora_t<__nv_bfloat16>(g, x, dy, a, b, da, db, u, ws, st)
              : launch_lora_t<float>(g, x, dy, a, b, da, db, u, ws, st);
}

}  // namespace seco
