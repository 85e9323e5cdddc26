// Memory-bound helper kernels of the chunk backward, shared by the bf16 and the
// fp32-debug paths, and the fp32 SIMT "debug" forward/backward kernels.
//
//   bwd_prep   : D_j = rowsum(dO_j o O_j)  [hq][c] fp32;
//                relay: dkv[:, :, slot j] *= gamma  (Alg. 2 line 6 P:334; grad_hook P:551 --
//                the relayed checkpoint gradient is pre-scaled so that the own-slot
//                deposits of the main kernel complete "grad + base * scaler");
//                zero the fp32 dQ accumulator.
//   bwd_final  : dQ_j = T(s * sigma * dQacc) and dk_own/dv_own = T(dkv[:, :, slot j]).
//   fwd_fp32 / bwd_fp32_dq / bwd_fp32_dkv : plain FFMA reference kernels for the
//                SECO_FP32_DEBUG dtype (any d <= 256, any chunk size).
#include "common.cuh"
#include "kernels.h"

// Grid sizes of the memory-bound helpers for large chunk calls (>= kBigRows query rows; smaller
// calls keep 296 blocks, which measured faster on the 8-rank per-rank shape): multiples of the
// 148 SMs, measured at cfg3 with tools/launch_gaps.py: prep 17.2 -> 14.0 us,
// final 13.4 -> 10.7 us against 296 blocks and 4 rows in flight
#ifndef SECO_FINAL_U
#define SECO_FINAL_U 8          // bwd_final, d = 128: rows in flight per thread
#endif
#ifndef SECO_FINAL_BLOCKS
#define SECO_FINAL_BLOCKS 592   // bwd_final dQ blocks (4 per SM)
#endif
#ifndef SECO_PREP_BLOCKS
#define SECO_PREP_BLOCKS 888    // bwd_prep blocks per task (D rows; dQacc zeroing), 6 per SM
#endif
constexpr int kBigRows = 32768;  // hq * c

namespace seco {

template <typename T> SECO_DEV float ldf(const T* p);
template <> SECO_DEV float ldf<float>(const float* p) { return *p; }
template <> SECO_DEV float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T> SECO_DEV void stf(T* p, float v);
template <> SECO_DEV void stf<float>(float* p, float v) { *p = v; }
template <> SECO_DEV void stf<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

SECO_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct PrepArgs {
  int hq, hkv, c, d, j, S;
  int cp;          // rows per head of D / nlse / dQacc (c, or c rounded up to 128 on the bf16 path)
  int64_t qh, qr;
  float relay;
  int nD, nR, nZ;  // block counts of the three tasks
  int ldq;         // dQacc row stride (floats)
  int* order;      // deterministic mode: dQ order counters [hq][c/128] to zero (else null)
  int n_order;
  int vec;         // Task A on 16-B vectors (bf16, d in {64, 128}; nD is then a grid-stride count)
};

// Task A (blocks [0,nD)): one warp per (h, row): D = sum_x dO*O (and -LSE log2 e for the
// tensor-core kernel, which evaluates P = exp2(S sigma log2 e - LSE log2 e) with one FFMA).
// Task B (blocks [nD,nD+nR)): scale slot j of dkv (both dK and dV) by relay.
// Task C (rest): zero dQacc [hq][c][d].
template <typename T>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const T* __restrict__ o, const T* __restrict__ d_o,
                                                       float* __restrict__ D, float* __restrict__ dkv,
                                                       float* __restrict__ dqacc, const float* __restrict__ lse,
                                                       float* __restrict__ nlse, PrepArgs a) {
  const int bid = blockIdx.x;
  if (bid < a.nD && a.vec) {
    // bf16 rows of d in {64, 128} (16-B aligned, checked by the ABI): d/8 lanes per row, one
    // 16-B load of O and of dO per lane, 4 row groups of a warp in flight per step (grid-stride)
    const int lpr = a.d / 8, rpw = 32 / lpr;
    const int lane = threadIdx.x % 32, sub = lane / lpr, x = (lane % lpr) * 8;
    const int nrows = a.hq * a.c;
    const int gw = bid * 8 + threadIdx.x / 32, nw = a.nD * 8;
    constexpr int B = 4;
    for (int w0 = gw * rpw * B; w0 < nrows; w0 += nw * rpw * B) {
      uint4 ov[B], dv[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int w = w0 + u * rpw + sub;
        if (w < nrows) {
          const int h = w / a.c, r = w % a.c;
          ov[u] = *reinterpret_cast<const uint4*>(o + (int64_t)h * a.qh + (int64_t)r * a.qr + x);
          dv[u] = *reinterpret_cast<const uint4*>(d_o + (int64_t)h * a.qh + (int64_t)r * a.qr + x);
        } else {
          ov[u] = dv[u] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const uint32_t* op = &ov[u].x;
        const uint32_t* dp = &dv[u].x;
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc += __uint_as_float(op[e] << 16) * __uint_as_float(dp[e] << 16) +
                 __uint_as_float(op[e] & 0xffff0000u) * __uint_as_float(dp[e] & 0xffff0000u);
        for (int off = lpr / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        const int w = w0 + u * rpw + sub;
        if (lane % lpr == 0 && w < nrows) {
          const int h = w / a.c, r = w % a.c;
          D[(int64_t)h * a.cp + r] = acc;
          if (nlse) nlse[(int64_t)h * a.cp + r] = -1.4426950408889634f * lse[w];
        }
      }
    }
  } else if (bid < a.nD) {
    const int w = bid * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (w >= a.hq * a.c) return;
    const int h = w / a.c, r = w % a.c;
    const T* orow = o + (int64_t)h * a.qh + (int64_t)r * a.qr;
    const T* drow = d_o + (int64_t)h * a.qh + (int64_t)r * a.qr;
    float acc = 0.f;
    for (int x = lane; x < a.d; x += 32) acc += ldf(orow + x) * ldf(drow + x);
    acc = warp_sum(acc);
    if (lane == 0) {
      D[(int64_t)h * a.cp + r] = acc;
      if (nlse) nlse[(int64_t)h * a.cp + r] = -1.4426950408889634f * lse[(int64_t)h * a.c + r];
    }
  } else if (bid < a.nD + a.nR) {
    if (a.relay == 1.f) return;
    const int64_t per = (int64_t)a.c * a.d;                 // one slot of one head
    const int64_t total = 2 * (int64_t)a.hkv * per / 4;     // float4 units
    const int64_t stride = (int64_t)a.nR * blockDim.x;
    constexpr int U = 4;                                    // float4s in flight per thread
    for (int64_t i0 = (int64_t)(bid - a.nD) * blockDim.x + threadIdx.x; i0 < total; i0 += U * stride) {
      float4* p[U];
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride, e = (i < total ? i : 0) * 4;
        const int64_t th = e / per, off = e % per;            // th = tensor*hkv + g
        p[u] = reinterpret_cast<float4*>(dkv + th * (int64_t)a.S * a.d + (int64_t)a.j * per + off);
        if (i < total) v[u] = *p[u];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u * stride >= total) break;
        v[u].x *= a.relay; v[u].y *= a.relay; v[u].z *= a.relay; v[u].w *= a.relay;
        *p[u] = v[u];
      }
    }
  } else {
    if (bid == a.nD + a.nR) {
      if (a.order)
        for (int i = threadIdx.x; i < a.n_order; i += blockDim.x) a.order[i] = 0;
      // padded rows of a ragged last query tile: P = exp2(S sigma log2 e - inf) = 0, dS = 0
      const int pad = a.cp - a.c;
      for (int i = threadIdx.x; i < a.hq * pad; i += blockDim.x) {
        const int64_t w = (int64_t)(i / pad) * a.cp + a.c + i % pad;
        D[w] = 0.f;
        if (nlse) nlse[w] = -INFINITY;
      }
    }
    if (dqacc == nullptr) return;
    const int64_t total = (int64_t)a.hq * a.cp * a.ldq / 4;
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = (int64_t)(bid - a.nD - a.nR) * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)a.nZ * blockDim.x)
      reinterpret_cast<float4*>(dqacc)[i] = z;
  }
}

struct FinalArgs {
  int hq, hkv, c, d, j, S;
  int cp;          // rows per head of dQacc
  int ldq;         // dQacc row stride (floats)
  int64_t qh, qr;
  float dq_scale;  // s * sigma
  int nQ, nO;
};

// Task A (blocks [0,nQ)): dq = T(dq_scale * dqacc) (skipped when dqacc == null).
// Task B: dk_own / dv_own = T(dkv slot j).  Both move 4 consecutive elements per thread
// step (d % 4 == 0 is required by the ABI), so index arithmetic is paid once per 4.
template <typename T> struct Vec4;
template <> struct Vec4<float> {
  static SECO_DEV void store(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
};
template <> struct Vec4<__nv_bfloat16> {
  static SECO_DEV void store(__nv_bfloat16* p, float4 v) {
    uint2 w;
    w.x = pack_bf16(v.x, v.y);
    w.y = pack_bf16(v.z, v.w);
    *reinterpret_cast<uint2*>(p) = w;
  }
};

template <typename T>
__global__ void __launch_bounds__(256) bwd_final_kernel(const float* __restrict__ dqacc, T* __restrict__ dq,
                                                        const float* __restrict__ dkv, T* __restrict__ dk_own,
                                                        T* __restrict__ dv_own, FinalArgs a) {
  const int bid = blockIdx.x;
  const int dv4 = a.d / 4, ld4 = a.ldq / 4;
  const int lane = threadIdx.x % 32;
  if (bid < a.nQ) {
    if (dqacc == nullptr) return;
    if (dv4 == 32) {
      // d = 128: one float4 per (row, lane); a thread keeps U rows' loads in flight before its
      // stores (32-bit index math: row = idx >> 5)
      const int rows = a.hq * a.c, total = rows * 32, stride = a.nQ * (int)blockDim.x;
      constexpr int U = SECO_FINAL_U;
      for (int base = bid * (int)blockDim.x + (int)threadIdx.x; base < total; base += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * stride;
          if (idx < total) {
            const int row = idx >> 5, h = row / a.c, r = row - h * a.c;
            v[u] = reinterpret_cast<const float4*>(dqacc)[((int64_t)h * a.cp + r) * ld4 + (idx & 31)];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * stride;
          if (idx >= total) break;
          const int row = idx >> 5, h = row / a.c, r = row - h * a.c;
          float4 w = v[u];
          w.x *= a.dq_scale; w.y *= a.dq_scale; w.z *= a.dq_scale; w.w *= a.dq_scale;
          Vec4<T>::store(dq + (int64_t)h * a.qh + (int64_t)r * a.qr + 4 * (idx & 31), w);
        }
      }
      return;
    }
    // one warp per row (h, r) in a grid-stride loop, 4 rows in flight; lanes stride the row's
    // float4s (no 64-bit index divisions in the loop)
    const int rows = a.hq * a.c;
    const int gw = bid * 8 + threadIdx.x / 32, nw = a.nQ * 8;
    constexpr int B = 4;
    for (int row0 = gw * B; row0 < rows; row0 += nw * B) {
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int row = row0 + u;
        if (row >= rows) break;
        const int h = row / a.c, r = row - h * a.c;
        const float4* src = reinterpret_cast<const float4*>(dqacc) + ((int64_t)h * a.cp + r) * ld4;
        T* dst = dq + (int64_t)h * a.qh + (int64_t)r * a.qr;
        for (int x4 = lane; x4 < dv4; x4 += 32) {
          float4 v = src[x4];
          v.x *= a.dq_scale; v.y *= a.dq_scale; v.z *= a.dq_scale; v.w *= a.dq_scale;
          Vec4<T>::store(dst + 4 * x4, v);
        }
      }
    }
  } else {
    if (dk_own == nullptr && dv_own == nullptr) return;
    if (dv4 == 32 && dk_own != nullptr && dv_own != nullptr) {
      // d = 128, both copies: flat float4 index over (tensor x kv head, row, lane), 4 in flight
      const int rows = 2 * a.hkv * a.c, total = rows * 32, stride = a.nO * (int)blockDim.x;
      constexpr int U = 4;
      for (int base = (bid - a.nQ) * (int)blockDim.x + (int)threadIdx.x; base < total; base += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * stride;
          if (idx < total) {
            const int row = idx >> 5, th = row / a.c, r = row - th * a.c;
            v[u] = reinterpret_cast<const float4*>(dkv + (int64_t)th * a.S * a.d + ((int64_t)a.j * a.c + r) * a.d)[idx & 31];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * stride;
          if (idx >= total) break;
          const int row = idx >> 5, th = row / a.c, r = row - th * a.c;
          T* own = th < a.hkv ? dk_own : dv_own;
          Vec4<T>::store(own + ((int64_t)(th % a.hkv) * a.c + r) * a.d + 4 * (idx & 31), v[u]);
        }
      }
      return;
    }
    // rows of slot j: (tensor, kv head, row) -> own copy [hkv][c][d]
    const int rows = 2 * a.hkv * a.c;
    const int gw = (bid - a.nQ) * 8 + threadIdx.x / 32, nw = a.nO * 8;
    for (int row = gw; row < rows; row += nw) {
      const int th = row / a.c, r = row - th * a.c;            // th = tensor * hkv + g
      T* own = th < a.hkv ? dk_own : dv_own;
      if (own == nullptr) continue;
      const float4* src = reinterpret_cast<const float4*>(dkv + (int64_t)th * a.S * a.d + ((int64_t)a.j * a.c + r) * a.d);
      T* dst = own + ((int64_t)(th % a.hkv) * a.c + r) * a.d;
      for (int x4 = lane; x4 < dv4; x4 += 32) Vec4<T>::store(dst + 4 * x4, src[x4]);
    }
  }
}

template <typename T>
static cudaError_t launch_prep(const ChunkGeom& g, const T* o, const T* d_o, float* D, float* dkv, float* dqacc,
                               const float* lse, float* nlse, float relay, cudaStream_t st, int* order = nullptr) {
  PrepArgs a;
  a.hq = g.hq; a.hkv = g.hkv; a.c = g.c; a.d = g.d; a.j = g.j; a.S = g.c * g.k;
  a.cp = g.cp > 0 ? g.cp : g.c;
  a.qh = g.qh; a.qr = g.qr; a.relay = relay;
  a.vec = (sizeof(T) == 2 && (g.d == 64 || g.d == 128)) ? 1 : 0;
  const int blocks = g.hq * g.c >= kBigRows ? SECO_PREP_BLOCKS : 296;
  a.nD = a.vec ? blocks : (g.hq * g.c + 7) / 8;
  a.nR = relay == 1.f ? 0 : 296;
  a.nZ = dqacc ? blocks : 0;
  a.order = order;
  a.ldq = g.ldq ? g.ldq : g.d;
  a.n_order = g.hq * ((g.c + 127) / 128) + 1;   // order counters + the deterministic-mode work ticket
  bwd_prep_kernel<T><<<a.nD + a.nR + a.nZ, 256, 0, st>>>(o, d_o, D, dkv, dqacc, lse, nlse, a);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_final(const ChunkGeom& g, const float* dqacc, T* dq, const float* dkv, T* dk_own,
                                T* dv_own, float dq_scale, cudaStream_t st) {
  FinalArgs a;
  a.hq = g.hq; a.hkv = g.hkv; a.c = g.c; a.d = g.d; a.j = g.j; a.S = g.c * g.k;
  a.qh = g.qh; a.qr = g.qr; a.dq_scale = dq_scale; a.ldq = g.ldq ? g.ldq : g.d;
  a.cp = g.cp > 0 ? g.cp : g.c;
  a.nQ = dqacc ? (g.hq * g.c >= kBigRows ? SECO_FINAL_BLOCKS : 296) : 0;
  a.nO = (dk_own || dv_own) ? 148 : 0;
  if (a.nQ + a.nO == 0) return cudaSuccess;
  bwd_final_kernel<T><<<a.nQ + a.nO, 256, 0, st>>>(dqacc, dq, dkv, dk_own, dv_own, a);
  return cudaGetLastError();
}

// bf16 path helpers, used by launch_bwd_sm100
cudaError_t launch_prep_bf16(const ChunkGeom& g, const void* o, const void* d_o, float* D, float* dkv,
                             float* dqacc, const float* lse, float* nlse, float relay, cudaStream_t st,
                             int* order) {
  return launch_prep<__nv_bfloat16>(g, reinterpret_cast<const __nv_bfloat16*>(o),
                                    reinterpret_cast<const __nv_bfloat16*>(d_o), D, dkv, dqacc, lse, nlse, relay,
                                    st, order);
}
cudaError_t launch_final_bf16(const ChunkGeom& g, const float* dqacc, void* dq, const float* dkv, void* dk_own,
                              void* dv_own, float dq_scale, cudaStream_t st) {
  return launch_final<__nv_bfloat16>(g, dqacc, reinterpret_cast<__nv_bfloat16*>(dq), dkv,
                                     reinterpret_cast<__nv_bfloat16*>(dk_own),
                                     reinterpret_cast<__nv_bfloat16*>(dv_own), dq_scale, st);
}

// ===================================================================== SECO_CHECK self-test
// One failing check (id 999) so a test can see that a check build reports failures.
__global__ void check_selftest_kernel(int v) { SECO_CHECK_COND(v == 0, 999); }
cudaError_t launch_check_selftest(cudaStream_t st) {
  check_selftest_kernel<<<1, 1, 0, st>>>(1);
  return cudaGetLastError();
}

// ===================================================================== SpaCO skipped chunk
// Alg. 2 line 5 ("for i in I") never visits a chunk outside the sample: its dQ, own
// dK / dV are zero and the deposits later chunks made into its checkpoint slot are dropped
// (reading Z11).  Blocks [0, nQ): dq rows (strided, element type T) = 0; the rest: dkv slot j
// (both tensors, every kv head, fp32) = 0 and the optional own copies = 0.  16-B stores
// (d % 4 == 0 on every path, so a dkv slot and a dense own copy are 16-B aligned whenever
// their base pointers are -- checked by the ABI).
struct SkipArgs {
  int hq, hkv, c, d, j, S;
  int64_t qh, qr;
  int nQ, nK;
  int vec;   // 1: dq rows and strides are 16-B aligned (always on the bf16 path) -> 16-B stores
};
template <typename T>
__global__ void __launch_bounds__(256) chunk_skip_kernel(float* __restrict__ dkv, T* __restrict__ dq,
                                                         T* __restrict__ dk_own, T* __restrict__ dv_own,
                                                         SkipArgs a) {
  const int bid = blockIdx.x;
  const int dv4 = a.d / 4;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (bid < a.nQ) {
    // one warp per row (h, r), grid-stride; 16-B stores when the rows allow, else 4 elements
    constexpr int E = 16 / sizeof(T);          // elements per 16-B store
    const int per = a.vec ? E : 4;
    const int lane = threadIdx.x % 32;
    const int rows = a.hq * a.c;
    for (int row = bid * 8 + threadIdx.x / 32; row < rows; row += a.nQ * 8) {
      const int h = row / a.c, r = row - h * a.c;
      T* base = dq + (int64_t)h * a.qh + (int64_t)r * a.qr;
      for (int x = lane * per; x < a.d; x += 32 * per) {
        T* dst = base + x;
        if (a.vec) {
          *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
        } else {                                // element stores: fp32 dq strides need no 16-B alignment
#pragma unroll
          for (int e = 0; e < 4; ++e) stf(dst + e, 0.f);
        }
      }
    }
  } else {
    const int64_t per4 = (int64_t)a.c * dv4;
    const int64_t total = 2 * (int64_t)a.hkv * per4;
    for (int64_t i = (int64_t)(bid - a.nQ) * blockDim.x + threadIdx.x; i < total; i += (int64_t)a.nK * blockDim.x) {
      const int64_t th = i / per4, off4 = i - th * per4;
      reinterpret_cast<float4*>(dkv + th * (int64_t)a.S * a.d + (int64_t)a.j * a.c * a.d)[off4] = z;
      T* own = th < a.hkv ? dk_own : dv_own;
      if (own) Vec4<T>::store(own + (th % a.hkv) * per4 * 4 + off4 * 4, z);
    }
  }
}

cudaError_t launch_chunk_skip(const ChunkGeom& g, bool bf16, float* dkv, void* dq, void* dk_own, void* dv_own,
                              cudaStream_t st) {
  SkipArgs a;
  a.hq = g.hq; a.hkv = g.hkv; a.c = g.c; a.d = g.d; a.j = g.j; a.S = g.c * g.k;
  a.qh = g.qh; a.qr = g.qr;
  a.nQ = 296;
  a.nK = 296;
  const size_t el = bf16 ? 2 : 4;
  a.vec = (reinterpret_cast<uintptr_t>(dq) % 16 == 0 && (g.qh * el) % 16 == 0 && (g.qr * el) % 16 == 0 &&
           (g.d * el) % 16 == 0) ? 1 : 0;
  if (bf16)
    chunk_skip_kernel<__nv_bfloat16><<<a.nQ + a.nK, 256, 0, st>>>(
        dkv, reinterpret_cast<__nv_bfloat16*>(dq), reinterpret_cast<__nv_bfloat16*>(dk_own),
        reinterpret_cast<__nv_bfloat16*>(dv_own), a);
  else
    chunk_skip_kernel<float><<<a.nQ + a.nK, 256, 0, st>>>(dkv, reinterpret_cast<float*>(dq),
                                                          reinterpret_cast<float*>(dk_own),
                                                          reinterpret_cast<float*>(dv_own), a);
  return cudaGetLastError();
}

// ===================================================================== split-KV combine (§8 a9)
// O = sum_s exp(LSE_s - LSE) O_s,  LSE = log sum_s exp(LSE_s)   (exact merge of softmax partials
// over disjoint key ranges).  One warp per (head, row); each lane owns 4 of the d = 128 columns.
struct CombArgs {
  int hq, c, cp, nsplit, d;   // cp: rows per head of the partials (c rounded up to 128)
  int64_t qh, qr;
};
__global__ void __launch_bounds__(256) fwd_combine_kernel(const float* __restrict__ part_o,
                                                          const float* __restrict__ part_lse,
                                                          __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                                                          CombArgs a) {
  const int w = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (w >= a.hq * a.c) return;
  const int h = w / a.c, r = w % a.c;
  const int64_t plane = (int64_t)a.hq * a.cp, pw = (int64_t)h * a.cp + r;   // partial row
  // every part's LSE and O slice requested before any is used (nsplit <= 4)
  float lp[4];
  float4 v[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    lp[s] = s < a.nsplit ? part_lse[s * plane + pw] : -INFINITY;
    v[s] = s < a.nsplit ? reinterpret_cast<const float4*>(part_o + (s * plane + pw) * 128)[lane]
                        : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float mx = -INFINITY;
#pragma unroll
  for (int s = 0; s < 4; ++s) mx = fmaxf(mx, lp[s]);
  float den = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s >= a.nsplit) break;
    const float wt = __expf(lp[s] - mx);
    den += wt;
    acc.x += wt * v[s].x; acc.y += wt * v[s].y; acc.z += wt * v[s].z; acc.w += wt * v[s].w;
  }
  const float inv = 1.f / den;
  if (4 * lane >= a.d) { if (lane == 0) lse[w] = mx + __logf(den); return; }
  uint2 pk;
  pk.x = pack_bf16(acc.x * inv, acc.y * inv);
  pk.y = pack_bf16(acc.z * inv, acc.w * inv);
  *reinterpret_cast<uint2*>(o + (int64_t)h * a.qh + (int64_t)r * a.qr + 4 * lane) = pk;
  if (lane == 0) lse[w] = mx + __logf(den);
}

cudaError_t launch_fwd_combine(const ChunkGeom& g, int nsplit, const float* part_o, const float* part_lse, void* o,
                               float* lse, cudaStream_t st) {
  CombArgs a;
  a.hq = g.hq; a.c = g.c; a.cp = g.cp; a.nsplit = nsplit; a.qh = g.qh; a.qr = g.qr; a.d = g.d;
  fwd_combine_kernel<<<(g.hq * g.c + 7) / 8, 256, 0, st>>>(part_o, part_lse, reinterpret_cast<__nv_bfloat16*>(o),
                                                            lse, a);
  return cudaGetLastError();
}

// ===================================================================== fp32 debug path
struct DbgArgs {
  int hq, hkv, G, c, d, j;
  float scale;
  int64_t qh, qr, kh, kr;
};

// one warp per query row; online softmax over the visible keys (FFMA, expf/logf)
template <int DPL>
__global__ void __launch_bounds__(256) fwd_fp32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                       const float* __restrict__ v, float* __restrict__ o,
                                                       float* __restrict__ lse, DbgArgs a) {
  const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32, h = blockIdx.y;
  if (r >= a.c) return;
  const int g = h / a.G, pos = a.j * a.c + r;
  const float* qrow = q + (int64_t)h * a.qh + (int64_t)r * a.qr;
  float qv[DPL], acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int x = lane + 32 * i;
    qv[i] = x < a.d ? qrow[x] : 0.f;
    acc[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int key = 0; key <= pos; ++key) {
    const float* krow = k + (int64_t)g * a.kh + (int64_t)key * a.kr;
    const float* vrow = v + (int64_t)g * a.kh + (int64_t)key * a.kr;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int x = lane + 32 * i;
      if (x < a.d) s += qv[i] * krow[x];
    }
    s = warp_sum(s) * a.scale;
    const float m_new = fmaxf(m, s);
    const float alpha = expf(m - m_new), p = expf(s - m_new);
    l = l * alpha + p;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int x = lane + 32 * i;
      acc[i] = acc[i] * alpha + (x < a.d ? p * vrow[x] : 0.f);
    }
    m = m_new;
  }
  float* orow = o + (int64_t)h * a.qh + (int64_t)r * a.qr;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int x = lane + 32 * i;
    if (x < a.d) orow[x] = acc[i] / l;
  }
  if (lane == 0) lse[(int64_t)h * a.c + r] = m + logf(l);
}

// dQ: one warp per query row
template <int DPL>
__global__ void __launch_bounds__(256) bwd_fp32_dq_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                          const float* __restrict__ v, const float* __restrict__ d_o,
                                                          const float* __restrict__ lse, const float* __restrict__ D,
                                                          float* __restrict__ dq, float gscale, DbgArgs a) {
  const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32, h = blockIdx.y;
  if (r >= a.c) return;
  const int g = h / a.G, pos = a.j * a.c + r;
  const float* qrow = q + (int64_t)h * a.qh + (int64_t)r * a.qr;
  const float* drow = d_o + (int64_t)h * a.qh + (int64_t)r * a.qr;
  float qv[DPL], dv[DPL], acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int x = lane + 32 * i;
    qv[i] = x < a.d ? qrow[x] : 0.f;
    dv[i] = x < a.d ? drow[x] : 0.f;
    acc[i] = 0.f;
  }
  const float L = lse[(int64_t)h * a.c + r], Dr = D[(int64_t)h * a.c + r];
  for (int key = 0; key <= pos; ++key) {
    const float* krow = k + (int64_t)g * a.kh + (int64_t)key * a.kr;
    const float* vrow = v + (int64_t)g * a.kh + (int64_t)key * a.kr;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int x = lane + 32 * i;
      if (x < a.d) { s += qv[i] * krow[x]; dp += dv[i] * vrow[x]; }
    }
    s = warp_sum(s) * a.scale;
    dp = warp_sum(dp);
    const float p = expf(s - L), ds = p * (dp - Dr);
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int x = lane + 32 * i;
      if (x < a.d) acc[i] += ds * krow[x];
    }
  }
  float* out = dq + (int64_t)h * a.qh + (int64_t)r * a.qr;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int x = lane + 32 * i;
    if (x < a.d) out[x] = gscale * a.scale * acc[i];
  }
}

// dK/dV: one warp per key (kv-head g, key position in [0, (j+1)c)); loops over the
// G q-heads of the group and the chunk's rows that see the key; adds the key's
// contribution into dkv (slot j was pre-scaled by the relay factor in bwd_prep).
template <int DPL>
__global__ void __launch_bounds__(256) bwd_fp32_dkv_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                           const float* __restrict__ v, const float* __restrict__ d_o,
                                                           const float* __restrict__ lse, const float* __restrict__ D,
                                                           float* __restrict__ dkv, float gscale, int S, DbgArgs a) {
  const int key = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32, g = blockIdx.y;
  const int end = (a.j + 1) * a.c;
  if (key >= end) return;
  const float* krow = k + (int64_t)g * a.kh + (int64_t)key * a.kr;
  const float* vrow = v + (int64_t)g * a.kh + (int64_t)key * a.kr;
  float kv[DPL], vv[DPL], dk[DPL], dvv[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int x = lane + 32 * i;
    kv[i] = x < a.d ? krow[x] : 0.f;
    vv[i] = x < a.d ? vrow[x] : 0.f;
    dk[i] = 0.f;
    dvv[i] = 0.f;
  }
  const int r0 = key > a.j * a.c ? key - a.j * a.c : 0;  // first row of the chunk that sees `key`
  for (int hh = 0; hh < a.G; ++hh) {
    const int h = g * a.G + hh;
    for (int r = r0; r < a.c; ++r) {
      const float* qrow = q + (int64_t)h * a.qh + (int64_t)r * a.qr;
      const float* drow = d_o + (int64_t)h * a.qh + (int64_t)r * a.qr;
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        const int x = lane + 32 * i;
        if (x < a.d) { s += kv[i] * qrow[x]; dp += vv[i] * drow[x]; }
      }
      s = warp_sum(s) * a.scale;
      dp = warp_sum(dp);
      const float p = expf(s - lse[(int64_t)h * a.c + r]);
      const float ds = p * (dp - D[(int64_t)h * a.c + r]);
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        const int x = lane + 32 * i;
        if (x < a.d) { dk[i] += ds * qrow[x]; dvv[i] += p * drow[x]; }
      }
    }
  }
  float* pk = dkv + ((int64_t)g * S + key) * a.d;
  float* pv = dkv + ((int64_t)(a.hkv + g) * S + key) * a.d;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int x = lane + 32 * i;
    if (x < a.d) {
      pk[x] += gscale * a.scale * dk[i];
      pv[x] += gscale * dvv[i];
    }
  }
}

static DbgArgs dbg_args(const ChunkGeom& g) {
  DbgArgs a;
  a.hq = g.hq; a.hkv = g.hkv; a.G = g.hq / g.hkv; a.c = g.c; a.d = g.d; a.j = g.j;
  a.scale = g.scale; a.qh = g.qh; a.qr = g.qr; a.kh = g.kh; a.kr = g.kr;
  return a;
}


cudaError_t launch_fwd_fp32(const ChunkGeom& g, const float* q, const float* k, const float* v, float* o,
                            float* lse, cudaStream_t st) {
  DbgArgs a = dbg_args(g);
  dim3 grid((g.c + 7) / 8, g.hq);
  if (g.d <= 32) fwd_fp32_kernel<1><<<grid, 256, 0, st>>>(q, k, v, o, lse, a);
  else if (g.d <= 64) fwd_fp32_kernel<2><<<grid, 256, 0, st>>>(q, k, v, o, lse, a);
  else if (g.d <= 128) fwd_fp32_kernel<4><<<grid, 256, 0, st>>>(q, k, v, o, lse, a);
  else fwd_fp32_kernel<8><<<grid, 256, 0, st>>>(q, k, v, o, lse, a);
  return cudaGetLastError();
}

cudaError_t launch_bwd_fp32(const ChunkGeom& g, const float* q, const float* k, const float* v, const float* o,
                            const float* d_o, const float* lse, float relay, float gscale, float* dkv, float* dq,
                            float* dk_own, float* dv_own, float* ws_D, cudaStream_t st, int* launches) {
  cudaError_t e = launch_prep<float>(g, o, d_o, ws_D, dkv, nullptr, lse, nullptr, relay, st);
  if (e != cudaSuccess) return e;
  DbgArgs a = dbg_args(g);
  dim3 gq((g.c + 7) / 8, g.hq);
  if (g.d <= 32) bwd_fp32_dq_kernel<1><<<gq, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dq, gscale, a);
  else if (g.d <= 64) bwd_fp32_dq_kernel<2><<<gq, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dq, gscale, a);
  else if (g.d <= 128) bwd_fp32_dq_kernel<4><<<gq, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dq, gscale, a);
  else bwd_fp32_dq_kernel<8><<<gq, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dq, gscale, a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int S = g.c * g.k;
  dim3 gk(((g.j + 1) * g.c + 7) / 8, g.hkv);
  if (g.d <= 32) bwd_fp32_dkv_kernel<1><<<gk, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dkv, gscale, S, a);
  else if (g.d <= 64) bwd_fp32_dkv_kernel<2><<<gk, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dkv, gscale, S, a);
  else if (g.d <= 128) bwd_fp32_dkv_kernel<4><<<gk, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dkv, gscale, S, a);
  else bwd_fp32_dkv_kernel<8><<<gk, 256, 0, st>>>(q, k, v, d_o, lse, ws_D, dkv, gscale, S, a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  e = launch_final<float>(g, nullptr, dq, dkv, dk_own, dv_own, 1.f, st);
  *launches = 3 + ((dk_own || dv_own) ? 1 : 0);
  return e;
}

unsigned long long check_word_aux() { return seco_check_read_clear(); }

}  // namespace seco
