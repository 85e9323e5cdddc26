// LoRA gradient accumulation for one adapted projection and one chunk (LoRA
// on q, k, v, o of every layer).  For Y = X W + (X A) B and the output cotangent dY:
//   u   = dY B^T   [rows][R]      -> u_out (fp32; the caller forms dX = dY W^T + u A^T)
//   t   = X A      [rows][R]      (workspace)
//   dA += X^T u    [n_in][R]      fp32 accumulator
//   dB += t^T dY   [R][n_out]     fp32 accumulator
// Rank-R skinny contractions: HBM-bound on X and dY (R = 8 gives 8 FLOP per loaded element),
// so CUDA cores with coalesced loads, not tensor cores.  Three kernels, all deterministic:
//   rows   one warp per row: t, u as warp-reduced dot products (A and B, a few hundred KiB at
//          most, stay in L1 / L2)
//   cols   one thread per column of X / dY over a contiguous share of the rows; per-split
//          partial sums of dA / dB to the workspace
//   reduce partials added in split order into dA / dB
#include "common.cuh"
#include "kernels.h"

namespace seco {

namespace lora {
constexpr int kRowsPerBlock = 8;     // warps per block in the row pass (one row each, strided)
constexpr int kColThreads = 256;

template <typename T> SECO_DEV float ld(const T* p);
template <> SECO_DEV float ld<float>(const float* p) { return __ldg(p); }
template <> SECO_DEV float ld<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

SECO_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
}  // namespace lora

// t[row][k] = sum_i X[row][i] A[i][k];  u[row][k] = sum_j dY[row][j] B[k][j]
template <typename T, int R>
__global__ void __launch_bounds__(256) lora_rows_kernel(const T* __restrict__ x, int64_t ldx, const T* __restrict__ dy,
                                                        int64_t ldy, const T* __restrict__ A, const T* __restrict__ B,
                                                        int rows, int n_in, int n_out, float* __restrict__ t,
                                                        float* __restrict__ u) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int row = blockIdx.x * lora::kRowsPerBlock + warp; row < rows; row += gridDim.x * lora::kRowsPerBlock) {
    float at[R], au[R];
#pragma unroll
    for (int k = 0; k < R; ++k) at[k] = au[k] = 0.f;
    const T* xr = x + (int64_t)row * ldx;
    for (int i = lane; i < n_in; i += 32) {
      const float xv = lora::ld(xr + i);
#pragma unroll
      for (int k = 0; k < R; ++k) at[k] = fmaf(xv, lora::ld(A + (int64_t)i * R + k), at[k]);
    }
    const T* gr = dy + (int64_t)row * ldy;
    for (int j = lane; j < n_out; j += 32) {
      const float gv = lora::ld(gr + j);
#pragma unroll
      for (int k = 0; k < R; ++k) au[k] = fmaf(gv, lora::ld(B + (int64_t)k * n_out + j), au[k]);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const float st = lora::warp_sum(at[k]), su = lora::warp_sum(au[k]);
      if (lane == 0) { t[(int64_t)row * R + k] = st; u[(int64_t)row * R + k] = su; }
    }
  }
}

// part[s][col][k]: columns [0, n_in) of X against u (-> dA), then [n_in, n_in + n_out) of dY
// against t (-> dB^T), each over rows [s * rows / S, (s + 1) * rows / S)
template <typename T, int R>
__global__ void __launch_bounds__(lora::kColThreads) lora_cols_kernel(const T* __restrict__ x, int64_t ldx,
                                                                      const T* __restrict__ dy, int64_t ldy,
                                                                      const float* __restrict__ t,
                                                                      const float* __restrict__ u, int rows, int n_in,
                                                                      int n_out, int nsplit, float* __restrict__ part) {
  const int col = blockIdx.x * lora::kColThreads + threadIdx.x;
  const int s = blockIdx.y;
  const int r0 = (int)((int64_t)s * rows / nsplit), r1 = (int)((int64_t)(s + 1) * rows / nsplit);
  const int ncol = n_in + n_out;
  if (col >= ncol) return;
  const bool isA = col < n_in;
  const T* src = isA ? x + col : dy + (col - n_in);
  const int64_t ld_src = isA ? ldx : ldy;
  const float* w = isA ? u : t;
  float acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.f;
  for (int row = r0; row < r1; ++row) {
    const float v = lora::ld(src + (int64_t)row * ld_src);
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = fmaf(v, __ldg(w + (int64_t)row * R + k), acc[k]);
  }
  float* out = part + ((int64_t)s * ncol + col) * R;
#pragma unroll
  for (int k = 0; k < R; ++k) out[k] = acc[k];
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
  const int col_blocks = (g.n_in + g.n_out + lora::kColThreads - 1) / lora::kColThreads;
  int s = (2 * 148 + col_blocks - 1) / col_blocks;
  s = s < 1 ? 1 : s;
  const int max_s = g.rows / 32 > 0 ? g.rows / 32 : 1;   // at least ~32 rows per split
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
  int blocks = (g.rows + lora::kRowsPerBlock - 1) / lora::kRowsPerBlock;
  if (blocks > 148) blocks = 148;
  lora_rows_kernel<T, R><<<blocks, 32 * lora::kRowsPerBlock, 0, st>>>(X, g.ldx, dY, g.ldy, static_cast<const T*>(a),
                                                         static_cast<const T*>(b), g.rows, g.n_in, g.n_out, t, u);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int nsplit = lora_splits(g);
  dim3 grid((g.n_in + g.n_out + lora::kColThreads - 1) / lora::kColThreads, nsplit);
  lora_cols_kernel<T, R><<<grid, lora::kColThreads, 0, st>>>(X, g.ldx, dY, g.ldy, t, u, g.rows, g.n_in, g.n_out,
                                                             nsplit, part);
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
  *launches = 3;
  return bf16 ? launch_lora_t<__nv_bfloat16>(g, x, dy, a, b, da, db, u, ws, st)
              : launch_lora_t<float>(g, x, dy, a, b, da, db, u, ws, st);
}

}  // namespace seco
