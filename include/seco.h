/*
 * seco.h -- C ABI of libseco.so: the data-parallel hot path of SeCO / SpaCO
 * (Sequential / Sparse Chunk-wise Optimization, arXiv 2505.16710) for one
 * causal GQA attention layer on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = PAPER.md line n.  The operations follow the paper's
 * problem statement: a sequence of k chunks of size c (Eq. 1);
 * chunk j's forward reads the KV cache of all earlier chunks (Eq. 1, Alg. 1
 * line 2 P:196); the chunk-local backward runs in reverse chunk order and
 * deposits gradients into every preceding checkpoint (Alg. 1
 * lines 4-7 P:199-202); SpaCO samples t of the k chunks and scales the relayed
 * checkpoint gradient by the compensation factor k/t (Alg. 2, capped
 * per P:415).
 *
 * Conventions (readings Z1-Z4 of DESIGN.md §3):
 *   - chunk index j is 0-based; query row r of chunk j is at absolute position
 *     p = j*c + r and sees every key position q <= p (cache slots 0..j-1 fully,
 *     its own slot j causally);
 *   - q-head h reads kv-head g = h / (hq/hkv);
 *   - logits are softmax_scale * <q, k>, softmax_scale <= 0 means 1/sqrt(d);
 *   - LSE is the natural-log log-sum-exp of the scaled logits, float32.
 *
 * Layouts (all row-major, innermost dimension d contiguous, strides in ELEMENTS):
 *   q, o, d_o, dq : [hq][c][d]   element (h, r, x) at h*q_head_stride + r*q_row_stride + x
 *                  (heads outermost, or rows outermost with heads interleaved, i.e.
 *                  the [c][hq][d] output of a projection: q_head_stride = d,
 *                  q_row_stride = hq*d; the same two choices for the KV cache)
 *   k_cache, v_cache : [hkv][S][d], S = c*num_chunks, element (g, q, x) at
 *                  g*kv_head_stride + q*kv_row_stride + x; slot j = rows [j*c, (j+1)*c)
 *   lse           : [hq][c] float32, dense
 *   dkv           : [2][hkv][S][d] float32, dense (index 0 = dK, 1 = dV): the
 *                   persistent checkpoint-gradient buffer m'.grad
 *   dk_own, dv_own: [hkv][c][d], dense, same element type as q
 * Element type: bf16 for SECO_BF16, float32 for SECO_FP32_DEBUG.
 *
 * Ownership: the caller owns every buffer (device memory), including dkv, which
 * the caller zeroes once per training step.  The library never allocates device
 * memory, never synchronises, and enqueues all work on `stream`.  Host-side
 * state: mutex-guarded caches of kernel attributes, backward work lists and TMA
 * tensor maps (keyed by pointer, sizes and strides; a tensor map holds no data, so
 * a cached map of a freed and re-allocated buffer with the same key is still
 * exact).  All functions are reentrant.
 *
 * Errors: return codes only, nothing throws across the ABI.  Arguments are
 * validated on the host before any launch (SECO_ERR_ARG: null pointer, j out of
 * range, hq % hkv != 0, non-positive sizes, misaligned pointer or stride;
 * SECO_ERR_UNSUPPORTED: a shape the bf16 tensor-core path does not implement --
 * it needs d in {32, 64, 96, 128} (d < 128 runs on zero-padded 128-wide tiles)
 * and 16-byte aligned rows; any chunk size c works (a ragged c % 128 != 0 leaves the last
 * query tile of each chunk partial: its rows past the chunk are zero-filled on
 * load, masked out of every softmax and never stored); the fp32 debug
 * path accepts any d <= 256 and any c).  Launch failures return SECO_ERR_CUDA;
 * faults during execution surface at the caller's next synchronisation.
 */
#ifndef SECO_H_
#define SECO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* seco_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum { SECO_OK = 0, SECO_ERR_ARG = 1, SECO_ERR_UNSUPPORTED = 2, SECO_ERR_CUDA = 3 } seco_status;
typedef enum { SECO_BF16 = 0, SECO_FP32_DEBUG = 1 } seco_dtype;
typedef enum { SPACO_PAPER = 0, SPACO_HT = 1, SPACO_BERNOULLI = 2 } spaco_mode;

typedef struct {
  int32_t hq, hkv, d;       /* q heads, kv heads, head dim                        */
  int32_t chunk;            /* c: rows per chunk (the paper's chunk size)         */
  int32_t num_chunks;       /* k: number of chunks, S = c * k                     */
  float softmax_scale;      /* <= 0 -> 1/sqrt(d)                                  */
  seco_dtype dtype;
  int64_t q_head_stride, q_row_stride;   /* for q, o, d_o, dq                     */
  int64_t kv_head_stride, kv_row_stride; /* for k_cache, v_cache                  */
  int32_t flags;            /* SECO_FLAG_* (0 = default)                          */
} seco_shape;

/* flags: SECO_FLAG_DETERMINISTIC makes every call bit-reproducible for identical
 * inputs (the paper attributes its SeCO-vs-baseline mismatch to
 * atomic accumulation).  The backward then adds the per-key-tile dQ
 * partials of each query tile in ascending key-tile order (per-tile counters in
 * the workspace, one owner per dK/dV tile, no Q-split); the forward is
 * deterministic in every mode (one writer per output, fixed-order split-KV
 * combine).  Costs backward throughput: the first wave of CTAs orders itself. */
#define SECO_FLAG_DETERMINISTIC 1

/* flags: SECO_FLAG_PREV_INDEPENDENT is the caller's promise, for seco_chunk_forward,
 * that the kernel enqueued on `stream` immediately before the call writes none of the
 * call's inputs (q, k_cache, v_cache) and reads none of its outputs (o, lse) -- e.g.
 * the previous chunk's forward in stage 1 (Alg. 1 lines 1-3 P:195-197).  The forward
 * may then load its inputs while that kernel's last wave drains (programmatic
 * dependent launch).  Without the flag the forward still overlaps its prologue
 * (barrier init, TMEM allocation) with the predecessor, but waits for the
 * predecessor's completion and memory visibility before its first global load or
 * store.  In both cases the forward completes only after its predecessor did, so
 * work enqueued after it sees normal stream order.  Ignored by the other calls. */
#define SECO_FLAG_PREV_INDEPENDENT 2

/* Bytes of device workspace `ws` the two chunk calls need (dQ accumulator,
 * row statistics).  Same for every j. */
size_t seco_workspace_size(const seco_shape* shape);

/* Chunk forward (Eq. 1; Alg. 1 lines 2 and 5): for the c
 * query rows of chunk j, attend to cache slots 0..j (own slot causally) with
 * an online softmax; write O_j (o) and LSE_j (lse).  Slot j of k_cache/v_cache
 * must already hold chunk j's keys/values.  `ws` is optional: when it is given
 * (ws_bytes >= seco_workspace_size()), long chunks may split each query tile's
 * key range over several CTAs (split-KV) and merge the partial results with the
 * exact LSE-weighted combine -- by a second kernel when the grid is smaller
 * than one wave, in-kernel by the last piece of each query tile otherwise (the
 * call then also enqueues a cudaMemsetAsync of its piece counters in ws); with
 * ws == NULL no split is used.  ws is scratch: its contents on entry do not
 * matter and are clobbered; two calls that share a ws must be stream-ordered.
 * Deterministic for a given (shape, j, ws != NULL): the stage-2 rebuild
 * reproduces stage 1 bit for bit (parts are merged in part order). */
seco_status seco_chunk_forward(const seco_shape* shape, int32_t j,
                               const void* q, const void* k_cache, const void* v_cache,
                               void* o, float* lse,
                               void* ws, size_t ws_bytes, seco_stream_t stream);

/* Chunk-local backward (Alg. 1 lines 6-7 P:200-201; Alg. 2 lines 6-7
 * P:334-335; relay = grad_hook(grad, base, scaler) P:551-552).  Inputs: the
 * chunk's q, o (from seco_chunk_forward), d_o (cotangent of o), lse.  Effects,
 * with s = grad_scale (loss seed scale; 1 for SeCO and Alg. 2 as printed) and
 * gamma = relay_scale (1 for SeCO, the compensation factor for SpaCO):
 *   dq                    = s * dQ_j                          (overwritten)
 *   dkv[:, :, slot i < j] += s * dK^(j->i), s * dV^(j->i)     (deposits into earlier checkpoints)
 *   dkv[:, :, slot j]      = gamma * dkv[:, :, slot j] + s * dK^(j->j)   (relay + own block)
 *   dk_own, dv_own         = dkv[0|1, :, slot j] converted to the element type (skipped if NULL)
 * Preconditions: every later chunk's backward that should deposit into slot j
 * was enqueued earlier on `stream` (descending order, reading Z10).  Summation
 * order of the fp32 deposits is not fixed (atomics; reading Z14). */
seco_status seco_chunk_backward(const seco_shape* shape, int32_t j,
                                const void* q, const void* k_cache, const void* v_cache,
                                const void* o, const void* d_o, const float* lse,
                                float relay_scale, float grad_scale,
                                float* dkv, void* dq, void* dk_own, void* dv_own,
                                void* ws, size_t ws_bytes, seco_stream_t stream);

/* SpaCO, a chunk j that is NOT in the sampled set I (Alg. 2 line 5 "for i in I"
 * skips it; reading Z11): its gradients are zero and its checkpoint gradient is
 * never relayed.  Effects, enqueued on `stream`:
 *   dq                    = 0   ([hq][c][d] chunk view, q strides of `shape`)
 *   dkv[:, :, slot j]     = 0   (the deposits of later chunks into slot j are dropped)
 *   dk_own, dv_own        = 0   (skipped if NULL)
 * Call it at chunk j's place in the descending stage-2 walk, i.e. after every
 * sampled chunk > j has run its backward (those are the only depositors into slot
 * j).  After a SpaCO step dkv then holds exactly the per-chunk own gradients.
 * Errors: as seco_chunk_backward (SECO_ERR_ARG for a NULL dq / dkv, bad shape, j out
 * of range, misaligned pointer). */
seco_status spaco_chunk_skip(const seco_shape* shape, int32_t j, float* dkv, void* dq, void* dk_own,
                             void* dv_own, seco_stream_t stream);

/* SpaCO sampling (Alg. 2 line 4 P:329 "Randomly select t distinct indices") and
 * scales (cap P:415), on the host, integer-only PRNG (splitmix64, state =
 * seed).  Writes the selected 0-based chunk indices strictly descending into
 * idx_out (capacity k), their count into *n_out, the relay scale gamma into
 * *relay_scale_out and the loss seed scale s into *seed_scale_out:
 *   SPACO_PAPER:     t distinct (partial Fisher-Yates), gamma = min(k/t, cap), s = 1
 *   SPACO_HT:        t distinct,                        gamma = (k-1)/(t-1), s = k/t
 *   SPACO_BERNOULLI: i kept iff floor(u*k/2^64) < t,    gamma = s = k/t
 * cap <= 0 disables the cap (applies to gamma in every mode).  Ratios are
 * computed in double and rounded once to float.  Errors: SECO_ERR_ARG for null
 * outputs, k < 1, t < 1, t > k, or SPACO_HT with t < 2. */
seco_status spaco_sample_and_scale(int32_t k, int32_t t, uint64_t seed, float cap, spaco_mode mode,
                                   int32_t* idx_out, int32_t* n_out,
                                   float* relay_scale_out, float* seed_scale_out);

/* ---- LoRA gradient accumulation ----------------------------------
 * For one LoRA-adapted projection Y = X W + (X A) B (LoRA on q, k, v, o of every
 * layer) and the cotangent dY of one chunk's rows:
 *   u = dY B^T   -> u_out [rows][rank] float32 (the caller forms dX = dY W^T + u A^T)
 *   dA += X^T u        [n_in][rank]   float32 accumulator
 *   dB += (X A)^T dY   [rank][n_out]  float32 accumulator
 * The accumulators are caller-owned (zeroed by the caller once per step) and sum the
 * chunks of a step in fp32; a layer's pair is final after its last chunk -- the
 * moment its all-reduce bucket can be sent (paper_2505_16710_b200/parallel.py).
 * Layouts: X [rows][n_in], dY [rows][n_out] row-major, row strides ldx, ldy in
 * elements (>= n_in, n_out); A [n_in][rank] and B [rank][n_out] dense, all of
 * `dtype` (SECO_BF16 or SECO_FP32_DEBUG).  n_in, n_out, ldx, ldy must be multiples
 * of one 16-B vector (8 bf16 / 4 fp32 elements) and x, dy, a, b, da, db 16-B aligned.
 * Summation order: bf16 with n_in, n_out multiples of 64 (128 at rank 16) up to 4096
 * runs one fused kernel whose per-cluster partial sums reach dA / dB by TMA reduce-add
 * (order of the clusters unfixed: results may differ in the last bits between calls);
 * flags = SECO_FLAG_DETERMINISTIC adds them in a fixed order instead (one more
 * launch).  Every other shape / dtype uses fixed-order kernels in either mode.
 * Errors: SECO_ERR_ARG (null pointer, non-positive size, short or misaligned stride,
 * workspace too small, unknown dtype), SECO_ERR_UNSUPPORTED (rank not in
 * {1, 2, 4, 8, 16}). */
typedef struct {
  int32_t rows, n_in, n_out, rank;
  seco_dtype dtype;
  int64_t ldx, ldy;
  int32_t flags;            /* SECO_FLAG_DETERMINISTIC or 0 */
} seco_lora_shape;

/* Bytes of device workspace seco_lora_grad needs. */
size_t seco_lora_workspace_size(const seco_lora_shape* shape);

seco_status seco_lora_grad(const seco_lora_shape* shape, const void* x, const void* dy, const void* a,
                           const void* b, float* da, float* db, float* u_out, void* ws, size_t ws_bytes,
                           seco_stream_t stream);

/* Static string for a status code (never NULL). */
const char* seco_status_string(seco_status status);

/* Human-readable description of the most recent error on the calling thread. */
const char* seco_last_error(void);

/* Number of kernel launches the most recent successful chunk call on the
 * calling thread enqueued (for launch accounting in the benchmark). */
int32_t seco_last_launch_count(void);

/* Diagnostics (host only, no GPU needed): the work list seco_chunk_backward would
 * launch for chunk j of a bf16 problem with `chunk` rows per chunk, hkv kv-heads,
 * G q-heads per kv-head and `num_sms` SMs (non-deterministic mode).  Writes
 * out4 = {n0, n1, f1, f2}: CTAs [0, n0) take whole 128-key units, the next n1 units
 * are split into f1 query-range pieces each, the rest into f2 pieces.
 * Returns the grid size. */
int32_t seco_debug_bwd_schedule(int32_t chunk, int32_t j, int32_t hkv, int32_t G, int32_t num_sms,
                                int32_t* out4);

/* Debug / test hook: the work plan seco_chunk_forward(shape, j) uses with a workspace of
 * seco_workspace_size(shape) bytes on a GPU with num_sms SMs (<= 0: this library's 148),
 * host only, bf16 shapes.  out5 = {CTA-pair kernel (0/1), work units, whole units n_full,
 * key-range pieces per split unit (1: no split), in-kernel merge (1) or combine kernel (0)}.
 * Returns the grid size in CTAs, -1 for an invalid shape. */
int32_t seco_debug_fwd_schedule(const seco_shape* shape, int32_t j, int32_t num_sms, int32_t* out5);

/* Bounds-check builds (libseco_check.so, compiled with -DSECO_CHECK=1; the stand-in for
 * compute-sanitizer, which this GPU pool does not offer).  Every kernel asserts its shared-
 * and tensor-memory operand ranges, mbarrier alignment, TMA box coordinates and global store
 * indices; a failed assertion is recorded, not trapped.
 *   seco_debug_check_enabled()   1 in a check build, 0 otherwise (host only).
 *   seco_debug_check_word()      (failed-check count << 32) | id of the first failed check
 *                                since the last read, then clears it; synchronises the device
 *                                (cudaMemcpyFromSymbol); always 0 in a normal build.
 *   seco_debug_check_selftest()  enqueues one kernel whose check fails (id 999) in a check
 *                                build, a no-op kernel otherwise. */
int32_t seco_debug_check_enabled(void);
uint64_t seco_debug_check_word(void);
seco_status seco_debug_check_selftest(seco_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SECO_H_ */
