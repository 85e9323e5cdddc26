// C-ABI host layer of libseco.so (see include/seco.h for the contract).
// Validates arguments, encodes TMA tensor maps, picks the kernel variant and
// enqueues it on the caller's stream.  Also the host SpaCO sampler.
#include "seco.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "kernels.h"

namespace {

thread_local char g_err[512] = "";
thread_local int32_t g_launches = 0;

seco_status fail(seco_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
seco_status fail(seco_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

seco_status cuda_fail(cudaError_t e, const char* where) {
  return fail(SECO_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// ---- cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
  static std::once_flag once;
  static EncodeFn fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// ---- tensor-map cache (seco.h "Host-side state").  Encoding is pure host arithmetic on
// (pointer, sizes, strides, box); a map holds no data, so a cached entry stays exact for any
// buffer that later occupies the same address with the same geometry.  Bounded: cleared when
// it reaches kMapCacheMax entries.
struct MapKey {
  uintptr_t ptr;
  int64_t a, b, c, d, e, f, g;   // kind-specific geometry
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && a == o.a && b == o.b && c == o.c && d == o.d && e == o.e && f == o.f && g == o.g;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ k.ptr;
    for (int64_t v : {k.a, k.b, k.c, k.d, k.e, k.f, k.g}) h = (h ^ (uint64_t)v) * 0x100000001B3ull + (h >> 29);
    return (size_t)h;
  }
};
constexpr size_t kMapCacheMax = 4096;
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash>& map_cache() {
  static auto* m = new std::unordered_map<MapKey, CUtensorMap, MapKeyHash>();
  return *m;
}
template <typename Encode>
bool cached_map(CUtensorMap* m, const MapKey& key, Encode&& encode) {
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = map_cache().find(key);
    if (it != map_cache().end()) { *m = it->second; return true; }
  }
  if (!encode(m)) return false;
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (map_cache().size() >= kMapCacheMax) map_cache().clear();
  map_cache().emplace(key, *m);
  return true;
}

// 3-D bf16 tensor map over [heads][rows][d], box {64, box_rows, 1}, 128-B swizzle
bool encode_3d(CUtensorMap* m, const void* ptr, int d, int rows, int heads, int64_t row_stride,
               int64_t head_stride, int box_rows) {
  const MapKey key{reinterpret_cast<uintptr_t>(ptr), 3, d, rows, heads, row_stride, head_stride, box_rows};
  return cached_map(m, key, [&](CUtensorMap* out) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)rows, (cuuint64_t)heads};
    cuuint64_t strides[2] = {(cuuint64_t)row_stride * 2, (cuuint64_t)head_stride * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  });
}

// 2-D fp32 tensor map over a dense [rows][cols] matrix, box {32, box_rows}, 128-B swizzle
// (the TMA reduce-add targets: dQ accumulator and dKV).  Boxes of 32 columns; a box past
// `cols` is skipped by the TMA's bounds check, which is how a zero-padded d = 64 tile
// reduces into a d = 64 buffer.
bool encode_f32_rows(CUtensorMap* m, const void* ptr, int64_t rows, int box_rows, int cols = 128) {
  const MapKey key{reinterpret_cast<uintptr_t>(ptr), 2, rows, box_rows, cols, 0, 0, 0};
  return cached_map(m, key, [&](CUtensorMap* out) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  });
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Rows of d elements, `rows` per head, `heads` heads never share an element when either
// heads are outermost ([h][r][d]: rs >= d, hs >= rows*rs) or rows are outermost with the
// heads interleaved inside a row ([r][h][d], e.g. a QKV projection output: hs >= d,
// rs >= heads*hs).
bool disjoint(int64_t d, int64_t rows, int64_t heads, int64_t rs, int64_t hs) {
  if (rs >= d && hs >= rows * rs) return true;
  return hs >= d && rs >= heads * hs;
}

seco_status check_shape(const seco_shape* s, int32_t j) {
  if (!s) return fail(SECO_ERR_ARG, "shape is NULL");
  if (s->hq <= 0 || s->hkv <= 0 || s->d <= 0 || s->chunk <= 0 || s->num_chunks <= 0)
    return fail(SECO_ERR_ARG, "non-positive size (hq=%d hkv=%d d=%d c=%d k=%d)", s->hq, s->hkv, s->d, s->chunk,
                s->num_chunks);
  if (s->hq % s->hkv) return fail(SECO_ERR_ARG, "hq %% hkv != 0 (hq=%d hkv=%d)", s->hq, s->hkv);
  if (j < 0 || j >= s->num_chunks) return fail(SECO_ERR_ARG, "chunk index j=%d out of [0,%d)", j, s->num_chunks);
  if (!disjoint(s->d, s->chunk, s->hq, s->q_row_stride, s->q_head_stride) ||
      !disjoint(s->d, (int64_t)s->chunk * s->num_chunks, s->hkv, s->kv_row_stride, s->kv_head_stride))
    return fail(SECO_ERR_ARG, "strides overlap rows/heads (need head-major or row-major-interleaved rows)");
  if (s->dtype == SECO_BF16) {
    if (s->d > 128 || s->d % 32)
      return fail(SECO_ERR_UNSUPPORTED, "bf16 path implements d in {32, 64, 96, 128} (got %d)", s->d);
    if ((s->q_row_stride * 2) % 16 || (s->q_head_stride * 2) % 16 || (s->kv_row_stride * 2) % 16 ||
        (s->kv_head_stride * 2) % 16)
      return fail(SECO_ERR_ARG, "bf16 strides must be multiples of 16 bytes");
  } else if (s->dtype == SECO_FP32_DEBUG) {
    if (s->d > 256 || s->d % 4) return fail(SECO_ERR_UNSUPPORTED, "fp32 debug path needs d <= 256, d %% 4 == 0");
  } else {
    return fail(SECO_ERR_ARG, "unknown dtype %d", (int)s->dtype);
  }
  if (s->flags & ~(SECO_FLAG_DETERMINISTIC | SECO_FLAG_PREV_INDEPENDENT))
    return fail(SECO_ERR_ARG, "unknown flags 0x%x", (unsigned)s->flags);
  return SECO_OK;
}

// the bf16 kernels work on 128-wide head dims (d = 64 is zero-padded by the TMA's
// out-of-bounds fill), so their fp32 dQ accumulator rows are 128 floats
int dq_ld(const seco_shape* s) { return s->dtype == SECO_BF16 ? 128 : s->d; }
// rows per head of the per-chunk workspace arrays: the bf16 kernels work on 128-row query tiles,
// so a ragged chunk (c % 128 != 0) pads each head's rows to the next tile
int64_t ws_rows(const seco_shape* s) { return s->dtype == SECO_BF16 ? (s->chunk + 127) / 128 * 128 : s->chunk; }

seco::ChunkGeom geom(const seco_shape* s, int32_t j) {
  seco::ChunkGeom g;
  g.hq = s->hq; g.hkv = s->hkv; g.d = s->d; g.c = s->chunk; g.k = s->num_chunks; g.j = j;
  g.scale = s->softmax_scale > 0.f ? s->softmax_scale : 1.0f / std::sqrt((float)s->d);
  g.qh = s->q_head_stride; g.qr = s->q_row_stride; g.kh = s->kv_head_stride; g.kr = s->kv_row_stride;
  g.det = (s->flags & SECO_FLAG_DETERMINISTIC) != 0;
  g.prev_indep = (s->flags & SECO_FLAG_PREV_INDEPENDENT) != 0;
  g.ldq = dq_ld(s);
  g.cp = (int)ws_rows(s);
  return g;
}

size_t ws_floats(const seco_shape* s) {
  // (cp = ws_rows: c, or on the bf16 path c rounded up to the 128-row tile)
  // backward: dQ accumulator [hq][cp][d] + D [hq][cp] + (-LSE log2 e) [hq][cp]
  //           + (deterministic mode) dQ order counters [hq][ceil(c/128)] int32 + a work ticket
  // forward (split-KV, up to 4 parts): partial O [4][hq][cp][d] + partial LSE [4][hq][cp]
  //           + piece counters, two per 128-row query tile and head
  const size_t cp = (size_t)ws_rows(s);
  const size_t bwd = (size_t)s->hq * cp * dq_ld(s) + 2 * (size_t)s->hq * cp +
                     (size_t)s->hq * ((s->chunk + 127) / 128) + 1;
  const size_t fwd = 4 * (size_t)s->hq * cp * (dq_ld(s) + 1) + 2 * (size_t)s->hq * ((s->chunk + 127) / 128);
  return bwd > fwd ? bwd : fwd;
}

// ---- splitmix64 (Steele, Lea & Flood 2014), state = seed
struct SplitMix64 {
  uint64_t x;
  uint64_t next() {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};
inline uint64_t mulhi64(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }

}  // namespace

extern "C" {

const char* seco_status_string(seco_status s) {
  switch (s) {
    case SECO_OK: return "SECO_OK";
    case SECO_ERR_ARG: return "SECO_ERR_ARG";
    case SECO_ERR_UNSUPPORTED: return "SECO_ERR_UNSUPPORTED";
    case SECO_ERR_CUDA: return "SECO_ERR_CUDA";
  }
  return "SECO_UNKNOWN_STATUS";
}

const char* seco_last_error(void) { return g_err; }
int32_t seco_last_launch_count(void) { return g_launches; }

size_t seco_workspace_size(const seco_shape* s) {
  if (!s || s->hq <= 0 || s->chunk <= 0 || s->d <= 0) return 0;
  return (ws_floats(s) * 4 + 255) & ~(size_t)255;
}

seco_status seco_chunk_forward(const seco_shape* s, int32_t j, const void* q, const void* k, const void* v, void* o,
                               float* lse, void* ws, size_t ws_bytes, seco_stream_t stream) {
  g_launches = 0;
  seco_status st = check_shape(s, j);
  if (st != SECO_OK) return st;
  if (!q || !k || !v || !o || !lse) return fail(SECO_ERR_ARG, "NULL tensor pointer");
  const seco::ChunkGeom g = geom(s, j);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (s->dtype == SECO_FP32_DEBUG) {
    e = seco::launch_fwd_fp32(g, (const float*)q, (const float*)k, (const float*)v, (float*)o, lse, cs);
    if (e != cudaSuccess) return cuda_fail(e, "fwd_fp32");
    g_launches = 1;
    return SECO_OK;
  }
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(SECO_ERR_ARG, "bf16 tensors must be 16-byte aligned");
  const int S_used = (j + 1) * s->chunk;
  CUtensorMap tq, tk, tv;
  if (!encode_3d(&tq, q, s->d, s->chunk, s->hq, s->q_row_stride, s->q_head_stride, 128) ||
      !encode_3d(&tk, k, s->d, S_used, s->hkv, s->kv_row_stride, s->kv_head_stride,
                 seco::fwd_uses_pair(g) ? 64 : 128) ||   // CTA pairs load K in 64-key halves
      !encode_3d(&tv, v, s->d, S_used, s->hkv, s->kv_row_stride, s->kv_head_stride, 128))
    return fail(SECO_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (ws && !aligned16(ws)) return fail(SECO_ERR_ARG, "ws must be 16-byte aligned");
  int launches = 0;
  e = seco::launch_fwd_sm100(g, tq, tk, tv, o, lse, reinterpret_cast<float*>(ws), ws ? ws_bytes / 4 : 0, cs,
                             &launches);
  if (e != cudaSuccess) return cuda_fail(e, "fwd_sm100");
  g_launches = launches;
  return SECO_OK;
}

seco_status seco_chunk_backward(const seco_shape* s, int32_t j, const void* q, const void* k, const void* v,
                                const void* o, const void* d_o, const float* lse, float relay_scale,
                                float grad_scale, float* dkv, void* dq, void* dk_own, void* dv_own, void* ws,
                                size_t ws_bytes, seco_stream_t stream) {
  g_launches = 0;
  seco_status st = check_shape(s, j);
  if (st != SECO_OK) return st;
  if (!q || !k || !v || !o || !d_o || !lse || !dkv || !dq) return fail(SECO_ERR_ARG, "NULL tensor pointer");
  if (!ws || ws_bytes < seco_workspace_size(s)) return fail(SECO_ERR_ARG, "workspace too small");
  if (!aligned16(dkv) || !aligned16(ws)) return fail(SECO_ERR_ARG, "dkv / ws must be 16-byte aligned");
  if (!std::isfinite(relay_scale) || !std::isfinite(grad_scale)) return fail(SECO_ERR_ARG, "non-finite scale");
  const seco::ChunkGeom g = geom(s, j);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  float* wsf = reinterpret_cast<float*>(ws);
  float* ws_dqacc = wsf;
  float* ws_D = wsf + (size_t)s->hq * ws_rows(s) * dq_ld(s);
  int launches = 0;
  cudaError_t e;
  if (s->dtype == SECO_FP32_DEBUG) {
    e = seco::launch_bwd_fp32(g, (const float*)q, (const float*)k, (const float*)v, (const float*)o,
                              (const float*)d_o, lse, relay_scale, grad_scale, dkv, (float*)dq, (float*)dk_own,
                              (float*)dv_own, ws_D, cs, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "bwd_fp32");
    g_launches = launches;
    return SECO_OK;
  }
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(d_o) || !aligned16(dq))
    return fail(SECO_ERR_ARG, "bf16 tensors must be 16-byte aligned");
  const int S_used = (j + 1) * s->chunk;
  CUtensorMap tq, tdo, tq64, tdo64, tk, tv, tdq, tdkv;
  const int64_t S = (int64_t)s->chunk * s->num_chunks;
  // 64-row boxes of Q / dO: the CTA-pair backward loads each CTA's query half (seco::bwd_uses_pair)
  const bool bpair = seco::bwd_uses_pair(g);
  if (!encode_3d(&tq, q, s->d, s->chunk, s->hq, s->q_row_stride, s->q_head_stride, 128) ||
      !encode_3d(&tdo, d_o, s->d, s->chunk, s->hq, s->q_row_stride, s->q_head_stride, 128) ||
      (bpair && !encode_3d(&tq64, q, s->d, s->chunk, s->hq, s->q_row_stride, s->q_head_stride, 64)) ||
      (bpair && !encode_3d(&tdo64, d_o, s->d, s->chunk, s->hq, s->q_row_stride, s->q_head_stride, 64)) ||
      !encode_3d(&tk, k, s->d, S_used, s->hkv, s->kv_row_stride, s->kv_head_stride, 128) ||
      !encode_3d(&tv, v, s->d, S_used, s->hkv, s->kv_row_stride, s->kv_head_stride, 128) ||
      !encode_f32_rows(&tdq, ws_dqacc, (int64_t)s->hq * ws_rows(s), 128) ||
      !encode_f32_rows(&tdkv, dkv, 2 * (int64_t)s->hkv * S, 128, s->d))
    return fail(SECO_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (!bpair) { tq64 = tq; tdo64 = tdo; }
  e = seco::launch_bwd_sm100(g, tq, tdo, tq64, tdo64, tk, tv, tdq, tdkv, o, d_o, lse, relay_scale, grad_scale, dkv, dq, dk_own, dv_own,
                             ws_dqacc, ws_D, cs, &launches);
  if (e != cudaSuccess) return cuda_fail(e, "bwd_sm100");
  g_launches = launches;
  return SECO_OK;
}

int32_t seco_debug_fwd_schedule(const seco_shape* s, int32_t j, int32_t num_sms, int32_t* out5) {
  if (check_shape(s, j) != SECO_OK || s->dtype != SECO_BF16 || !out5) return -1;
  return seco::fwd_debug_plan(geom(s, j), ws_floats(s), num_sms, out5);
}

seco_status spaco_chunk_skip(const seco_shape* s, int32_t j, float* dkv, void* dq, void* dk_own, void* dv_own,
                             seco_stream_t stream) {
  g_launches = 0;
  seco_status st = check_shape(s, j);
  if (st != SECO_OK) return st;
  if (!dkv || !dq) return fail(SECO_ERR_ARG, "NULL tensor pointer");
  if (!aligned16(dkv) || (dk_own && !aligned16(dk_own)) || (dv_own && !aligned16(dv_own)))
    return fail(SECO_ERR_ARG, "dkv / dk_own / dv_own must be 16-byte aligned");
  if (s->dtype == SECO_BF16 && !aligned16(dq)) return fail(SECO_ERR_ARG, "bf16 tensors must be 16-byte aligned");
  if (s->d % 4) return fail(SECO_ERR_UNSUPPORTED, "d %% 4 != 0");
  cudaError_t e = seco::launch_chunk_skip(geom(s, j), s->dtype == SECO_BF16, dkv, dq, dk_own, dv_own,
                                          reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "chunk_skip");
  g_launches = 1;
  return SECO_OK;
}

uint64_t seco_debug_check_word(void) {
  const unsigned long long w[4] = {seco::check_word_fwd(), seco::check_word_bwd(), seco::check_word_aux(),
                                   seco::check_word_lora()};
  uint64_t count = 0, first = 0;
  for (unsigned long long x : w) {
    count += x >> 32;
    if (!first) first = x & 0xFFFFFFFFull;
  }
  return (count << 32) | first;
}

int32_t seco_debug_check_enabled(void) {
#ifdef SECO_CHECK
  return 1;
#else
  return 0;
#endif
}

seco_status seco_debug_check_selftest(seco_stream_t stream) {
  cudaError_t e = seco::launch_check_selftest(reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SECO_OK : cuda_fail(e, "check_selftest");
}

static bool lora_geom(const seco_lora_shape* s, seco::LoraGeom* g) {
  if (!s || s->rows <= 0 || s->n_in <= 0 || s->n_out <= 0 || s->rank <= 0) return false;
  g->rows = s->rows; g->n_in = s->n_in; g->n_out = s->n_out; g->rank = s->rank;
  g->ldx = s->ldx; g->ldy = s->ldy;
  g->deterministic = (s->flags & SECO_FLAG_DETERMINISTIC) != 0;
  return true;
}

size_t seco_lora_workspace_size(const seco_lora_shape* s) {
  seco::LoraGeom g;
  if (!lora_geom(s, &g)) return 0;
  return seco::lora_ws_floats(g) * sizeof(float);
}

seco_status seco_lora_grad(const seco_lora_shape* s, const void* x, const void* dy, const void* a, const void* b,
                           float* da, float* db, float* u_out, void* ws, size_t ws_bytes, seco_stream_t stream) {
  g_launches = 0;
  seco::LoraGeom g;
  if (!lora_geom(s, &g)) return fail(SECO_ERR_ARG, "lora: NULL shape or non-positive size");
  if (!x || !dy || !a || !b || !da || !db || !u_out || !ws) return fail(SECO_ERR_ARG, "lora: NULL pointer");
  if (s->ldx < s->n_in || s->ldy < s->n_out) return fail(SECO_ERR_ARG, "lora: row stride shorter than the row");
  if (s->dtype != SECO_BF16 && s->dtype != SECO_FP32_DEBUG) return fail(SECO_ERR_ARG, "lora: unknown dtype");
  if (s->rank != 1 && s->rank != 2 && s->rank != 4 && s->rank != 8 && s->rank != 16)
    return fail(SECO_ERR_UNSUPPORTED, "lora: rank must be 1, 2, 4, 8 or 16 (got %d)", s->rank);
  if (ws_bytes < seco_lora_workspace_size(s)) return fail(SECO_ERR_ARG, "lora: workspace too small");
  const int vec = s->dtype == SECO_BF16 ? 8 : 4;           // 16-B vectors of the row pass
  if (s->n_in % vec || s->n_out % vec || s->ldx % vec || s->ldy % vec)
    return fail(SECO_ERR_ARG, "lora: n_in, n_out and row strides must be multiples of %d elements", vec);
  if (!aligned16(x) || !aligned16(dy)) return fail(SECO_ERR_ARG, "lora: x / dy must be 16-byte aligned");
  if (!aligned16(a) || !aligned16(b)) return fail(SECO_ERR_ARG, "lora: a / b must be 16-byte aligned");
  int launches = 0;
  cudaError_t e = seco::launch_lora_grad(g, s->dtype == SECO_BF16, x, dy, a, b, da, db, u_out,
                                         reinterpret_cast<float*>(ws), reinterpret_cast<cudaStream_t>(stream),
                                         &launches);
  if (e != cudaSuccess) return cuda_fail(e, "lora_grad");
  g_launches = launches;
  return SECO_OK;
}

seco_status spaco_sample_and_scale(int32_t k, int32_t t, uint64_t seed, float cap, spaco_mode mode,
                                   int32_t* idx_out, int32_t* n_out, float* relay_scale_out,
                                   float* seed_scale_out) {
  if (!idx_out || !n_out || !relay_scale_out || !seed_scale_out) return fail(SECO_ERR_ARG, "NULL output");
  if (k < 1 || t < 1 || t > k) return fail(SECO_ERR_ARG, "need 1 <= t <= k (k=%d t=%d)", k, t);
  if (mode == SPACO_HT && t < 2) return fail(SECO_ERR_ARG, "SPACO_HT needs t >= 2");
  if (mode != SPACO_PAPER && mode != SPACO_HT && mode != SPACO_BERNOULLI)
    return fail(SECO_ERR_ARG, "unknown mode %d", (int)mode);
  SplitMix64 rng{seed};
  int32_t n = 0;
  if (mode == SPACO_BERNOULLI) {
    for (int32_t i = 0; i < k; ++i)
      if (mulhi64(rng.next(), (uint64_t)k) < (uint64_t)t) idx_out[n++] = i;
  } else {
    // partial Fisher-Yates over a = [0..k-1] held in idx_out
    for (int32_t i = 0; i < k; ++i) idx_out[i] = i;
    for (int32_t r = 0; r < t; ++r) {
      const int32_t jj = r + (int32_t)mulhi64(rng.next(), (uint64_t)(k - r));
      std::swap(idx_out[r], idx_out[jj]);
    }
    n = t;
  }
  std::sort(idx_out, idx_out + n, [](int32_t a, int32_t b) { return a > b; });
  double gamma, sscale;
  if (mode == SPACO_PAPER) { gamma = (double)k / t; sscale = 1.0; }
  else if (mode == SPACO_HT) { gamma = (double)(k - 1) / (t - 1); sscale = (double)k / t; }
  else { gamma = (double)k / t; sscale = (double)k / t; }
  float g32 = (float)gamma;
  if (cap > 0.f) g32 = std::min(g32, cap);
  *relay_scale_out = g32;
  *seed_scale_out = (float)sscale;
  *n_out = n;
  return SECO_OK;
}

}  // extern "C"
