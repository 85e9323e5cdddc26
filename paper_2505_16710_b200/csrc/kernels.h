// Internal launcher interface between the C-ABI host layer (seco_api.cpp) and the
// CUDA kernels.  Not part of the public ABI.
#pragma once
#include <atomic>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace seco {

struct ChunkGeom {
  int hq, hkv, d, c, k, j;   // heads, head dim, chunk size, #chunks, chunk index
  float scale;               // softmax scale sigma
  int64_t qh, qr;            // q/o/do/dq strides (elements)
  int64_t kh, kr;            // k/v cache strides (elements)
  bool det = false;          // SECO_FLAG_DETERMINISTIC: ordered dQ reduction, no Q-split
  int ldq = 0;               // row stride (floats) of the dQ accumulator: 128 on the bf16 path
                             // (d = 64 runs zero-padded to 128), d on the fp32 path
  int cp = 0;                // rows per head of the per-chunk workspace arrays (dQacc, D, -LSE
                             // log2 e, split-KV partials): c rounded up to the 128-row tile on
                             // the bf16 path (a ragged last query tile stays inside its head's
                             // rows), c on the fp32 path
  bool prev_indep = false;   // SECO_FLAG_PREV_INDEPENDENT: the forward may load before its
                             // predecessor kernel completes (programmatic dependent launch)
};

// ---- SECO_CHECK builds (common.cuh): per-translation-unit check words, read and cleared ----
unsigned long long check_word_fwd();
unsigned long long check_word_bwd();
unsigned long long check_word_aux();
unsigned long long check_word_lora();
cudaError_t launch_check_selftest(cudaStream_t st);

// ---- SpaCO non-sampled chunk (reading Z11): dq = 0, dkv slot j = 0, own copies = 0 ---
cudaError_t launch_chunk_skip(const ChunkGeom& g, bool bf16, float* dkv, void* dq, void* dk_own, void* dv_own,
                              cudaStream_t st);

// ---- fp32 debug path (SIMT FFMA, any d <= 256, any c) -------------------------------
cudaError_t launch_fwd_fp32(const ChunkGeom& g, const float* q, const float* k, const float* v, float* o,
                            float* lse, cudaStream_t st);
cudaError_t launch_bwd_fp32(const ChunkGeom& g, const float* q, const float* k, const float* v,
                            const float* o, const float* d_o, const float* lse, float relay, float gscale,
                            float* dkv, float* dq, float* dk_own, float* dv_own, float* ws_D,
                            cudaStream_t st, int* launches);

// ---- bf16 tensor-core path (tcgen05 / TMEM / TMA) -----------------------------------
// the forward runs as CTA pairs (tk must then be encoded with 64-row boxes, see seco_api.cpp)
bool fwd_uses_pair(const ChunkGeom& g);
cudaError_t launch_fwd_sm100(const ChunkGeom& g, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, void* o, float* lse, float* ws, size_t ws_floats,
                             cudaStream_t st, int* launches);
bool bwd_uses_pair(const ChunkGeom& g);   // CTA-pair backward (v3) selected
cudaError_t launch_bwd_sm100(const ChunkGeom& g, const CUtensorMap& tq, const CUtensorMap& tdo,
                             const CUtensorMap& tq64, const CUtensorMap& tdo64,
                             const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tdq,
                             const CUtensorMap& tdkv, const void* o, const void* d_o,
                             const float* lse, float relay, float gscale, float* dkv, void* dq,
                             void* dk_own, void* dv_own, float* ws_dqacc, float* ws_D, cudaStream_t st,
                             int* launches);

// the forward's work plan for a call (seco_debug_fwd_schedule): out5 = {pair kernel, units,
// whole units n_full, pieces per split unit, in-kernel merge}; returns the grid size in CTAs
int32_t fwd_debug_plan(const ChunkGeom& g, size_t ws_floats, int sms, int32_t* out5);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device), thread-safe:
// `done` holds one bit per device ordinal (the attribute is per device).
template <typename Kernel>
inline cudaError_t ensure_smem_attr(Kernel kern, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// ---- LoRA gradient accumulation (lora.cu) ------------------------------------------------
struct LoraGeom {
  int rows, n_in, n_out, rank;
  int64_t ldx, ldy;
  int deterministic;
};
size_t lora_ws_floats(const LoraGeom& g);
cudaError_t launch_lora_grad(const LoraGeom& g, bool bf16, const void* x, const void* dy, const void* a,
                             const void* b, float* da, float* db, float* u, float* ws, cudaStream_t st,
                             int* launches);

}  // namespace seco
