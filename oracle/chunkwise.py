"""O5 SeCO step (Algorithm 1) and O6 SpaCO step (Algorithm 2) for one attention
layer, written in the paper's order.  TEST INFRASTRUCTURE ONLY.

The KV cache chunks m'_i are the K/V rows of chunk i (Appendix C.1
``update_kv_cache``).  Their accumulated gradients m'_i.grad live in
the checkpoint-gradient buffer ``B`` ([Hkv][S][d] for K and for V), exactly the
``requires_grad`` leaves of P:546-549.  The relay "m_i.grad <- m'_i.grad"
(Alg. 1 line 3) / "m_i.grad <- (k/t) m'_i.grad" (Alg. 2 line 6)
is ``grad_hook(grad, base, scaler) = grad + base * scaler``: the
total gradient of chunk i's own K/V = local contribution + scaler * B[i].

Chunks are given as a list of sizes (ragged last chunk allowed, reading Z15).
"""
from __future__ import annotations

import numpy as np

from .attention import chunk_bwd, chunk_fwd


def chunk_bounds(sizes):
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(int)
    return [(int(s), int(s + n)) for s, n in zip(starts, sizes)]


def stage1(q, k, v, sizes, scale=None, dtype=np.float64):
    """Alg. 1 / Alg. 2 lines 1-3: inference-mode forward of
    every chunk in ascending order.  Returns (O [Hq][S][d], LSE [Hq][S])."""
    hq, s, d = q.shape
    o = np.zeros((hq, s, d), dtype)
    lse = np.zeros((hq, s), dtype)
    for (a, b) in chunk_bounds(sizes):
        o[:, a:b], lse[:, a:b] = chunk_fwd(q[:, a:b], k, v, a, scale, dtype)
    return o, lse


def sparse_stage2(q, k, v, do, sizes, selected, relay_scale=1.0, seed_scale=1.0,
                  scale=None, dtype=np.float64):
    """Stage 2 over the chunk indices in ``selected`` (processed in descending
    order, reading Z10).  For each selected chunk i (Alg. 2 lines 5-8):
      1. rebuild J_i, m_i  (chunk forward; the backward recomputes P from it)
      2. relay  m_i.grad <- relay_scale * m'_i.grad
      3. backprop(J_i): seed_scale * dO_i through chunk i, depositing into the
         checkpoint grads of every earlier chunk.
    Non-selected chunks get zero dQ/dK/dV and their B[i] is dropped (Z11).
    Returns dict(dq, dk, dv, B_k, B_v) -- dk/dv are the gradients of each chunk's
    own K/V (what flows on to the projections), B_* the final checkpoint grads."""
    q, k, v, do = (np.asarray(a, dtype) for a in (q, k, v, do))
    bounds = chunk_bounds(sizes)
    B_k = np.zeros_like(k)
    B_v = np.zeros_like(v)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for i in sorted(set(int(x) for x in selected), reverse=True):
        a, b = bounds[i]
        # 1. rebuild (J_i, m_i) -- chunk_bwd recomputes the forward internally
        dq_i, dk_src, dv_src = chunk_bwd(q[:, a:b], k, v, seed_scale * do[:, a:b], a, scale, dtype)
        # 2. relay: own-chunk total = local + scaler * m'_i.grad  (grad_hook)
        dk[:, a:b] = dk_src[:, a:b] + relay_scale * B_k[:, a:b]
        dv[:, a:b] = dv_src[:, a:b] + relay_scale * B_v[:, a:b]
        # 3. deposit into the preceding checkpoints m'_1..m'_{i-1}
        B_k[:, :a] += dk_src[:, :a]
        B_v[:, :a] += dv_src[:, :a]
        dq[:, a:b] = dq_i
    return dict(dq=dq, dk=dk, dv=dv, B_k=B_k, B_v=B_v)


def seco_step(q, k, v, do, sizes, scale=None, dtype=np.float64):
    """O5 -- Algorithm 1: stage 1 over all chunks, then stage 2 over
    k..1 with scaler 1.  Returns dict(o, lse, dq, dk, dv)."""
    o, lse = stage1(q, k, v, sizes, scale, dtype)
    g = sparse_stage2(q, k, v, do, sizes, range(len(sizes)), 1.0, 1.0, scale, dtype)
    return dict(o=o, lse=lse, dq=g["dq"], dk=g["dk"], dv=g["dv"])


def spaco_step(q, k, v, do, sizes, selected, relay_scale, seed_scale=1.0,
               scale=None, dtype=np.float64):
    """O6 -- Algorithm 2: stage 1 over all chunks ('preserves the
    integrity of forward propagation'), stage 2 only over the sampled set
    I with relay scaler gamma (the compensation factor, capped per P:415)
    and loss seed scale s (reading Z8; s = 1 is Alg. 2 literally)."""
    o, lse = stage1(q, k, v, sizes, scale, dtype)
    g = sparse_stage2(q, k, v, do, sizes, selected, relay_scale, seed_scale, scale, dtype)
    return dict(o=o, lse=lse, dq=g["dq"], dk=g["dk"], dv=g["dv"])
