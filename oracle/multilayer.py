"""O9: an L-layer attention stack with RoPE and LoRA-adapted projections, its loss and its
exact (full-sequence) gradients -- the plain definition that SeCO reaches across layers
(Eq. 2 P:111-113 and the multi-hop chains of Eq. 3: the KV cache
of chunk i in layer l feeds chunk j > i in layer l, whose output feeds layer l+1's cache of
chunk j, ...).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Model (reading Z18): LLaMA-shaped attention blocks without the per-token
RMSNorm / MLP (they touch no KV cache, so they do not change SeCO's chunk / relay
structure):
    W'_p = W_p + A_p B_p                   p in {q, k, v, o}    (LoRA, scale 1)
    Q = rope(x W'_q), K = rope(x W'_k), V = x W'_v               per head, positions 0..S-1
    x <- x + attn(Q, K, V) W'_o                                  (O1: causal GQA softmax)
after L blocks the loss is J = sum_p <x_L[p], G[p]> for a fixed cotangent G, so
dJ/dx_L = G; per chunk, J_j = sum over the chunk's rows.
RoPE: rotate-half (HF LLaMA) with inv_freq_i = base^(-2i/d), i < d/2.

Layouts: x, G [S][Hd]; per layer the projection weights are [in][out] (x @ W).
"""
from __future__ import annotations

import numpy as np

from .attention import full_attn_bwd, full_attn_fwd

PROJ = ("q", "k", "v", "o")


def rope_angles(pos, d, base=10000.0):
    """[S][d/2] angles p * base^(-2i/d)."""
    half = d // 2
    inv = base ** (-np.arange(half, dtype=np.float64) * 2.0 / d)
    return np.asarray(pos, np.float64)[:, None] * inv[None, :]


def rope(x, pos, base=10000.0):
    """x [S][H][d] -> rotated: (x1, x2) -> (x1 cos - x2 sin, x2 cos + x1 sin)."""
    d = x.shape[-1]
    ang = rope_angles(pos, d, base)[:, None, :]
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope_bwd(g, pos, base=10000.0):
    """VJP of rope (the transpose of the rotation = rotation by -angle)."""
    d = g.shape[-1]
    ang = rope_angles(pos, d, base)[:, None, :]
    c, s = np.cos(ang), np.sin(ang)
    g1, g2 = g[..., : d // 2], g[..., d // 2:]
    return np.concatenate([g1 * c + g2 * s, g2 * c - g1 * s], axis=-1)


def merged(p, name):
    """W'_name = W + A B."""
    return p["W" + name] + p["A" + name] @ p["B" + name]


def stack_forward(x0, layers, hq, hkv, d, base=10000.0, keep=False):
    """Run the L blocks on the full sequence.  Returns x_L (and per-layer saved tensors)."""
    x = np.asarray(x0, np.float64)
    S = x.shape[0]
    pos = np.arange(S)
    saved = []
    for p in layers:
        q = (x @ merged(p, "q")).reshape(S, hq, d)
        k = (x @ merged(p, "k")).reshape(S, hkv, d)
        v = (x @ merged(p, "v")).reshape(S, hkv, d)
        qr, kr = rope(q, pos, base), rope(k, pos, base)
        o, _ = full_attn_fwd(qr.transpose(1, 0, 2), kr.transpose(1, 0, 2), v.transpose(1, 0, 2))
        o2 = o.transpose(1, 0, 2).reshape(S, hq * d)
        if keep:
            saved.append(dict(x=x, qr=qr, kr=kr, v=v, o2=o2))
        x = x + o2 @ merged(p, "o")
    return (x, saved) if keep else x


def stack_loss(x0, layers, G, hq, hkv, d, base=10000.0):
    """J = sum <x_L, G>."""
    return float((stack_forward(x0, layers, hq, hkv, d, base) * G).sum())


def stack_grads(x0, layers, G, hq, hkv, d, base=10000.0):
    """Exact gradients of J: (list of {A_p, B_p, W_p grads} per layer, dJ/dx0).
    Reverse-mode through the residual, the projections, RoPE and O2 (full_attn_bwd)."""
    xL, saved = stack_forward(x0, layers, hq, hkv, d, base, keep=True)
    S = xL.shape[0]
    pos = np.arange(S)
    dx = np.asarray(G, np.float64).copy()
    grads = [None] * len(layers)
    for li in reversed(range(len(layers))):
        p, sv = layers[li], saved[li]
        g = {}
        dy = dx                                             # residual: x_{l+1} = x_l + y
        dWo = sv["o2"].T @ dy
        do2 = dy @ merged(p, "o").T
        do = do2.reshape(S, hq, d).transpose(1, 0, 2)
        dqr, dkr, dv = full_attn_bwd(sv["qr"].transpose(1, 0, 2), sv["kr"].transpose(1, 0, 2),
                                     sv["v"].transpose(1, 0, 2), do)
        dq = rope_bwd(dqr.transpose(1, 0, 2), pos, base).reshape(S, hq * d)
        dk = rope_bwd(dkr.transpose(1, 0, 2), pos, base).reshape(S, hkv * d)
        dv2 = dv.transpose(1, 0, 2).reshape(S, hkv * d)
        x = sv["x"]
        dW = {"q": x.T @ dq, "k": x.T @ dk, "v": x.T @ dv2, "o": dWo}
        dx = dx + dq @ merged(p, "q").T + dk @ merged(p, "k").T + dv2 @ merged(p, "v").T
        for n in PROJ:
            g["W" + n] = dW[n]
            g["A" + n] = dW[n] @ p["B" + n].T             # W' = W + A B
            g["B" + n] = p["A" + n].T @ dW[n]
        grads[li] = g
    return grads, dx


def lora_grads(x, dy, A, B):
    """the LoRA gradients of one projection Y = X W + (X A) B (LoRA) for the
    cotangent dY, through the merged-weight gradient dW' = X^T dY of O9 (stack_grads):
    dA = dW' B^T, dB = A^T dW'; also u = dY B^T (what dX = dY W^T + u A^T needs).
    Returns (dA [n_in][r], dB [r][n_out], u [rows][r])."""
    x, dy, A, B = (np.asarray(a, np.float64) for a in (x, dy, A, B))
    dW = x.T @ dy
    return dW @ B.T, A.T @ dW, dy @ B.T
