"""Python binding with the C-ABI names (include/seco.h).  Torch tensors are used
only as device memory; each call forwards pointers, sizes and the current CUDA
stream to libseco.so.  No arithmetic happens here."""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import LoraShape, SecoShape, check, load

_DTYPES = {torch.bfloat16: _lib.SECO_BF16, torch.float32: _lib.SECO_FP32_DEBUG}


def make_shape(q_full: torch.Tensor, k_cache: torch.Tensor, chunk: int, softmax_scale: float = 0.0,
               deterministic: bool = False, prev_independent: bool = False) -> SecoShape:
    """Shape record for Q [hq][S][d] (full sequence) and a KV cache [hkv][S][d].
    deterministic: bit-reproducible backward (SECO_FLAG_DETERMINISTIC).
    prev_independent: SECO_FLAG_PREV_INDEPENDENT (the caller's promise that the kernel before
    each forward on the stream neither writes its inputs nor reads its outputs)."""
    if q_full.dtype not in _DTYPES or k_cache.dtype != q_full.dtype:
        raise TypeError("q / k_cache must both be bf16 (tensor-core path) or float32 (debug path)")
    hq, S, d = q_full.shape
    hkv = k_cache.shape[0]
    if q_full.stride(2) != 1 or k_cache.stride(2) != 1:
        raise ValueError("innermost (head) dimension must be contiguous")
    if S % chunk:
        raise ValueError("sequence length must be a multiple of the chunk size")
    return SecoShape(hq, hkv, d, chunk, S // chunk, float(softmax_scale), _DTYPES[q_full.dtype],
                     q_full.stride(0), q_full.stride(1), k_cache.stride(0), k_cache.stride(1),
                     (_lib.SECO_FLAG_DETERMINISTIC if deterministic else 0)
                     | (_lib.SECO_FLAG_PREV_INDEPENDENT if prev_independent else 0))


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _p(t):
    """Device pointer of a CUDA tensor (NULL for None).  A host tensor is refused here: the
    library takes device pointers and would only fault at the next synchronisation."""
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_cuda:
        raise ValueError("libseco takes CUDA tensors (got a tensor on %s)" % t.device)
    return ctypes.c_void_p(t.data_ptr())


def chunk_view(t: torch.Tensor, shape: SecoShape, j: int) -> torch.Tensor:
    """Rows of chunk j of a [h][S][d] (or [h][S]) tensor (a view, no copy)."""
    return t.narrow(1, j * shape.chunk, shape.chunk)


def seco_workspace_size(shape: SecoShape) -> int:
    return int(load().seco_workspace_size(ctypes.byref(shape)))


def seco_chunk_forward(shape: SecoShape, j: int, q_j, k_cache, v_cache, o_j, lse_j, ws=None, stream=None):
    """Chunk forward of chunk j (Eq. 1).  q_j / o_j: chunk views with the
    strides recorded in `shape`; lse_j: dense [hq][c] float32."""
    lib = load()
    wsb = ws.numel() * ws.element_size() if ws is not None else 0
    check(lib.seco_chunk_forward(ctypes.byref(shape), j, _p(q_j), _p(k_cache), _p(v_cache), _p(o_j), _p(lse_j),
                                 _p(ws), wsb, _stream(stream)), "seco_chunk_forward")


def seco_chunk_backward(shape: SecoShape, j: int, q_j, k_cache, v_cache, o_j, do_j, lse_j, relay_scale: float,
                        grad_scale: float, dkv, dq_j, dk_own=None, dv_own=None, ws=None, stream=None):
    """Chunk-local backward of chunk j with relay (Alg. 2 line 6)."""
    lib = load()
    wsb = ws.numel() * ws.element_size() if ws is not None else 0
    check(lib.seco_chunk_backward(ctypes.byref(shape), j, _p(q_j), _p(k_cache), _p(v_cache), _p(o_j), _p(do_j),
                                  _p(lse_j), float(relay_scale), float(grad_scale), _p(dkv), _p(dq_j),
                                  _p(dk_own), _p(dv_own), _p(ws), wsb, _stream(stream)), "seco_chunk_backward")


def spaco_chunk_skip(shape: SecoShape, j: int, dkv, dq_j, dk_own=None, dv_own=None, stream=None):
    """SpaCO chunk j outside the sample (Alg. 2 line 5; reading Z11): dQ_j = 0, own dK/dV = 0,
    its checkpoint-gradient slot in dkv dropped (zeroed)."""
    lib = load()
    check(lib.spaco_chunk_skip(ctypes.byref(shape), j, _p(dkv), _p(dq_j), _p(dk_own), _p(dv_own), _stream(stream)),
          "spaco_chunk_skip")


def spaco_sample_and_scale(k: int, t: int, seed: int, cap: float = 2.0, mode: int = _lib.SPACO_PAPER):
    """(I descending, relay gamma, seed scale s) from the host sampler (Alg. 2 line 4)."""
    lib = load()
    idx = (ctypes.c_int32 * k)()
    n = ctypes.c_int32()
    g = ctypes.c_float()
    s = ctypes.c_float()
    check(lib.spaco_sample_and_scale(k, t, ctypes.c_uint64(seed & ((1 << 64) - 1)), float(cap), mode, idx,
                                     ctypes.byref(n), ctypes.byref(g), ctypes.byref(s)), "spaco_sample_and_scale")
    return [int(idx[i]) for i in range(n.value)], float(g.value), float(s.value)


def last_launch_count() -> int:
    return int(load().seco_last_launch_count())


def lora_shape(x, dy, rank: int, deterministic: bool = False) -> LoraShape:
    """Shape record for X [rows][n_in], dY [rows][n_out] (row-major, unit inner stride).
    deterministic: fixed summation order (SECO_FLAG_DETERMINISTIC, include/seco.h)."""
    if x.dtype not in _DTYPES or dy.dtype != x.dtype:
        raise TypeError("x / dy must both be bf16 or float32")
    if x.stride(1) != 1 or dy.stride(1) != 1 or x.shape[0] != dy.shape[0]:
        raise ValueError("x, dy: [rows][n] with contiguous rows and equal row counts")
    return LoraShape(x.shape[0], x.shape[1], dy.shape[1], rank, _DTYPES[x.dtype], x.stride(0), dy.stride(0),
                     _lib.SECO_FLAG_DETERMINISTIC if deterministic else 0)


def seco_lora_workspace_size(shape: LoraShape) -> int:
    return int(load().seco_lora_workspace_size(ctypes.byref(shape)))


def seco_lora_grad(shape: LoraShape, x, dy, a, b, da, db, u_out, ws, stream=None):
    """dA += X^T (dY B^T), dB += (X A)^T dY (fp32), u_out = dY B^T."""
    lib = load()
    wsb = ws.numel() * ws.element_size()
    check(lib.seco_lora_grad(ctypes.byref(shape), _p(x), _p(dy), _p(a), _p(b), _p(da), _p(db), _p(u_out), _p(ws),
                             wsb, _stream(stream)), "seco_lora_grad")
