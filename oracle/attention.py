"""O1-O4: causal GQA attention, its vector-Jacobian product, and the chunk-local
forward / backward of SeCO.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation: q-heads Hq, kv-heads Hkv, G = Hq/Hkv, head dim d,
softmax scale sigma = 1/sqrt(d) (reading Z2), q-head h reads kv-head
g = h // G (reading Z3, LLaMA ``repeat_kv``), query at absolute position p sees
keys at positions q <= p (reading Z1: bottom-right causal alignment of a chunk
against its cache).  LSE is the natural-log log-sum-exp of the scaled logits
(reading Z4).

Layouts: Q, dO, O are [Hq][rows][d]; K, V (the KV cache, the paper's m) are
[Hkv][S][d]; LSE is [Hq][rows].
"""
from __future__ import annotations

import math

import numpy as np


def _scale(d: int, scale):
    return 1.0 / math.sqrt(d) if (scale is None or scale <= 0) else float(scale)


def _probs(qh, kg, q_pos, k_len, scale):
    """Scaled, causally masked logits -> (P, LSE) for one head.

    logits[r, c] = scale * <Q[r], K[c]> for key position c <= q_pos[r]; rows
    with no visible key cannot occur (position p always sees key p).
    P = exp(logits - LSE), LSE = log sum_c exp(logits)  (textbook softmax).
    """
    logits = scale * (qh @ kg[:k_len].T)
    visible = np.arange(k_len)[None, :] <= q_pos[:, None]
    logits = np.where(visible, logits, -np.inf)
    m = logits.max(axis=1, keepdims=True)
    lse = m[:, 0] + np.log(np.exp(logits - m).sum(axis=1))
    p = np.exp(logits - lse[:, None])
    return p, lse


def full_attn_fwd(q, k, v, scale=None, dtype=np.float64):
    """O1 -- full-sequence causal GQA attention (the 'naive parallel' forward that
    Eq. (1), decomposes chunk by chunk).  Returns (O [Hq][S][d], LSE [Hq][S])."""
    q, k, v = (np.asarray(a, dtype) for a in (q, k, v))
    hq, s, d = q.shape
    g_size = hq // k.shape[0]
    sc = _scale(d, scale)
    o = np.zeros((hq, s, d), dtype)
    lse = np.zeros((hq, s), dtype)
    pos = np.arange(s)
    for h in range(hq):
        g = h // g_size
        p, lse[h] = _probs(q[h], k[g], pos, s, sc)
        o[h] = p @ v[g]
    return o, lse


def full_attn_bwd(q, k, v, do, scale=None, dtype=np.float64):
    """O2 -- VJP of O1 with cotangent dO (the gradient naive parallel training
    computes).  Textbook softmax-attention backward:
      D = rowsum(dO o O); dP = dO V^T; dS = P o (dP - D)
      dQ = scale dS K ; dK = scale sum_{h in g} dS^T Q ; dV = sum_{h in g} P^T dO
    Returns (dQ [Hq][S][d], dK [Hkv][S][d], dV [Hkv][S][d])."""
    q, k, v, do = (np.asarray(a, dtype) for a in (q, k, v, do))
    hq, s, d = q.shape
    g_size = hq // k.shape[0]
    sc = _scale(d, scale)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    pos = np.arange(s)
    for h in range(hq):
        g = h // g_size
        p, _ = _probs(q[h], k[g], pos, s, sc)
        o = p @ v[g]
        D = (do[h] * o).sum(axis=1)
        dp = do[h] @ v[g].T
        ds = p * (dp - D[:, None])
        dq[h] = sc * (ds @ k[g])
        dk[g] += sc * (ds.T @ q[h])
        dv[g] += p.T @ do[h]
    return dq, dk, dv


def chunk_fwd(q_j, k_cache, v_cache, start, scale=None, dtype=np.float64):
    """O3 -- forward of chunk j, Eq. (1) P:106 / Alg. 1 line 2 P:196: the chunk's
    queries (absolute positions start .. start+n-1) attend to every cached key
    of earlier chunks (m_1..m_{j-1}) plus their own chunk causally (reading Z1).
    q_j [Hq][n][d]; k_cache/v_cache [Hkv][>= start+n][d].
    Returns (O_j [Hq][n][d], LSE_j [Hq][n])."""
    q_j, kc, vc = (np.asarray(a, dtype) for a in (q_j, k_cache, v_cache))
    hq, n, d = q_j.shape
    g_size = hq // kc.shape[0]
    sc = _scale(d, scale)
    end = start + n
    pos = start + np.arange(n)
    o = np.zeros((hq, n, d), dtype)
    lse = np.zeros((hq, n), dtype)
    for h in range(hq):
        g = h // g_size
        p, lse[h] = _probs(q_j[h], kc[g], pos, end, sc)
        o[h] = p @ vc[g][:end]
    return o, lse


def chunk_bwd(q_j, k_cache, v_cache, do_j, start, scale=None, dtype=np.float64):
    """O4 -- chunk-local backpropagation of chunk j (Alg. 1 line 4 'backprop(J_i)',
    P:201; §4.1 step 3 P:164: 'accumulate gradients for model parameters and
    preceding checkpoints m'_1..m'_{j-1}').  Given the cotangent dO_j of the
    chunk's output, returns
      dQ_j            [Hq][n][d]      (complete: queries live only in chunk j)
      dK_src, dV_src  [Hkv][end][d]   gradient w.r.t. every key/value the chunk
                                      read, i.e. blocks dK^(j->i) for all i <= j
    The caller splits dK_src into the own block (i = j) and the deposits into
    earlier checkpoints (i < j)."""
    q_j, kc, vc, do_j = (np.asarray(a, dtype) for a in (q_j, k_cache, v_cache, do_j))
    hq, n, d = q_j.shape
    hkv = kc.shape[0]
    g_size = hq // hkv
    sc = _scale(d, scale)
    end = start + n
    pos = start + np.arange(n)
    dq = np.zeros_like(q_j)
    dk = np.zeros((hkv, end, d), dtype)
    dv = np.zeros((hkv, end, d), dtype)
    for h in range(hq):
        g = h // g_size
        p, _ = _probs(q_j[h], kc[g], pos, end, sc)
        o = p @ vc[g][:end]
        D = (do_j[h] * o).sum(axis=1)
        dp = do_j[h] @ vc[g][:end].T
        ds = p * (dp - D[:, None])
        dq[h] = sc * (ds @ kc[g][:end])
        dk[g] += sc * (ds.T @ q_j[h])
        dv[g] += p.T @ do_j[h]
    return dq, dk, dv
