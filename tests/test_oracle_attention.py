"""Pins for oracle O1-O4 (oracle/attention.py) against things other than itself:
torch's own CPU attention kernels in fp64 (an independent implementation),
central finite differences, closed-form special cases and invariants."""
import math

import numpy as np
import pytest
import torch

from oracle import attention as A
from synth import make_inputs

TINY = dict(hq=2, hkv=1, seq=64, d=16)      # BASELINE.json configs[0]
GQA = dict(hq=4, hkv=2, seq=96, d=32)


def _torch_ref(q, k, v, do):
    """torch CPU fp64: SDPA (is_causal) + autograd, and the CPU flash kernel's LSE."""
    G = q.shape[0] // k.shape[0]
    tq = torch.tensor(q, dtype=torch.float64, requires_grad=True)
    tk = torch.tensor(k, dtype=torch.float64, requires_grad=True)
    tv = torch.tensor(v, dtype=torch.float64, requires_grad=True)
    kk = tk.repeat_interleave(G, dim=0)
    vv = tv.repeat_interleave(G, dim=0)
    o = torch.nn.functional.scaled_dot_product_attention(tq[None], kk[None], vv[None], is_causal=True)[0]
    o.backward(torch.tensor(do, dtype=torch.float64))
    with torch.no_grad():
        _, lse = torch.ops.aten._scaled_dot_product_flash_attention_for_cpu(
            tq[None].detach(), kk[None].detach(), vv[None].detach(), 0.0, True)[:2]
    return (o.detach().numpy(), lse[0].numpy(), tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy())


@pytest.mark.parametrize("cfg", [TINY, GQA])
def test_full_matches_torch_fp64(cfg):
    x = make_inputs(**cfg, seed=1, bf16=False)
    o, lse = A.full_attn_fwd(x.q, x.k, x.v)
    dq, dk, dv = A.full_attn_bwd(x.q, x.k, x.v, x.do)
    to, tlse, tdq, tdk, tdv = _torch_ref(x.q, x.k, x.v, x.do)
    for a, b in ((o, to), (lse, tlse), (dq, tdq), (dk, tdk), (dv, tdv)):
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())


def test_finite_differences_tiny():
    """Brute force: directional derivative of L = <dO, O(Q,K,V)> by central differences."""
    x = make_inputs(**TINY, seed=2, bf16=False)
    q, k, v, do = (a.astype(np.float64) for a in (x.q, x.k, x.v, x.do))
    dq, dk, dv = A.full_attn_bwd(q, k, v, do)
    rng = np.random.default_rng(7)
    eps = 1e-6

    def L(q_, k_, v_):
        return float((A.full_attn_fwd(q_, k_, v_)[0] * do).sum())

    for which, grad in (("q", dq), ("k", dk), ("v", dv)):
        dirn = rng.standard_normal(grad.shape)
        args_p = dict(q_=q, k_=k, v_=v)
        args_m = dict(q_=q, k_=k, v_=v)
        args_p[which + "_"] = args_p[which + "_"] + eps * dirn
        args_m[which + "_"] = args_m[which + "_"] - eps * dirn
        fd = (L(**args_p) - L(**args_m)) / (2 * eps)
        an = float((grad * dirn).sum())
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (which, fd, an)


def test_first_row_is_single_key_softmax():
    """Row p=0 sees one key: O = V[g,0], LSE = scale*<Q,K0>."""
    x = make_inputs(**GQA, seed=3, bf16=False)
    o, lse = A.full_attn_fwd(x.q, x.k, x.v)
    G = 2
    for h in range(4):
        g = h // G
        assert np.allclose(o[h, 0], x.v[g, 0], atol=1e-12, rtol=0)
        assert abs(lse[h, 0] - (x.q[h, 0].astype(np.float64) @ x.k[g, 0]) / math.sqrt(32)) < 1e-12


def test_zero_keys_give_prefix_mean():
    """K = 0: all logits 0, so O[p] = mean(V[0..p]) and LSE[p] = log(p+1)."""
    x = make_inputs(**GQA, seed=4, bf16=False)
    k0 = np.zeros_like(x.k)
    o, lse = A.full_attn_fwd(x.q, k0, x.v)
    S = x.q.shape[1]
    cum = np.cumsum(x.v.astype(np.float64), axis=1) / np.arange(1, S + 1)[None, :, None]
    for h in range(4):
        assert np.allclose(o[h], cum[h // 2], atol=1e-12, rtol=0)
        assert np.allclose(lse[h], np.log(np.arange(1, S + 1)), atol=1e-12, rtol=0)


def test_softmax_rows_sum_to_one():
    """V = 1 => O = sum_q P = 1 for every row (check (c) of the north star)."""
    x = make_inputs(**GQA, seed=5, bf16=False)
    o, _ = A.full_attn_fwd(x.q, x.k, np.ones_like(x.v))
    assert np.abs(o - 1.0).max() < 1e-13


def test_dk_columns_sum_to_zero():
    """Rows of dS sum to 0 (sum_q P (dP - D) = D - D), hence sum_q dK[g,q] = 0."""
    x = make_inputs(**GQA, seed=6, bf16=False)
    _, dk, _ = A.full_attn_bwd(x.q, x.k, x.v, x.do)
    assert np.abs(dk.sum(axis=1)).max() < 1e-11 * np.abs(dk).max() * dk.shape[1]


def test_causality():
    """Perturbing K/V at positions > p leaves O[p], LSE[p] unchanged."""
    x = make_inputs(**TINY, seed=7, bf16=False)
    o, lse = A.full_attn_fwd(x.q, x.k, x.v)
    p = 37
    k2, v2 = x.k.copy(), x.v.copy()
    k2[:, p + 1:] += 5.0
    v2[:, p + 1:] -= 3.0
    o2, lse2 = A.full_attn_fwd(x.q, k2, v2)
    assert np.array_equal(o[:, :p + 1], o2[:, :p + 1])
    assert np.array_equal(lse[:, :p + 1], lse2[:, :p + 1])
    assert not np.allclose(o[:, p + 1:], o2[:, p + 1:])


def test_chunk_fwd_rows_equal_full_rows():
    """O3 on chunk j = rows [jc,(j+1)c) of O1; includes a ragged chunk."""
    x = make_inputs(**GQA, seed=8, bf16=False)
    o, lse = A.full_attn_fwd(x.q, x.k, x.v)
    for a, b in ((0, 32), (32, 64), (64, 96), (40, 59)):
        oj, lj = A.chunk_fwd(x.q[:, a:b], x.k, x.v, a)
        assert np.abs(oj - o[:, a:b]).max() < 1e-13
        assert np.abs(lj - lse[:, a:b]).max() < 1e-13


def test_lse_merge_identity():
    """LSE_j = logaddexp(LSE over cache slots < j, LSE over the own slot)."""
    x = make_inputs(**GQA, seed=9, bf16=False)
    a, b = 64, 96
    _, lj = A.chunk_fwd(x.q[:, a:b], x.k, x.v, a)
    sc = 1 / math.sqrt(32)
    for h in range(4):
        g = h // 2
        lg = sc * (x.q[h, a:b].astype(np.float64) @ x.k[g, :b].astype(np.float64).T)
        prev = np.log(np.exp(lg[:, :a]).sum(1))
        own = np.array([np.log(np.exp(lg[r, a:a + r + 1]).sum()) for r in range(b - a)])
        assert np.abs(np.logaddexp(prev, own) - lj[h]).max() < 1e-12


def test_chunk_bwd_last_chunk_block_structure():
    """O4 for the last chunk: dQ rows equal the full dQ computed with dO zero outside the chunk."""
    x = make_inputs(**GQA, seed=10, bf16=False)
    a, b = 64, 96
    do_masked = np.zeros_like(x.do)
    do_masked[:, a:b] = x.do[:, a:b]
    dq_f, dk_f, dv_f = A.full_attn_bwd(x.q, x.k, x.v, do_masked)
    dq, dk, dv = A.chunk_bwd(x.q[:, a:b], x.k, x.v, x.do[:, a:b], a)
    assert np.abs(dq - dq_f[:, a:b]).max() < 1e-12
    assert np.abs(dk - dk_f[:, :b]).max() < 1e-12
    assert np.abs(dv - dv_f[:, :b]).max() < 1e-12
    assert np.abs(dq_f[:, :a]).max() == 0.0
