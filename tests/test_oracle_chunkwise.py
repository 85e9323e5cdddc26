"""Pins for O5/O6 (oracle/chunkwise.py): SeCO reaches the full-sequence gradient
exactly (App. D P:526 '>12 decimal places'), degenerate cases."""
import numpy as np
import pytest

from oracle import attention as A
from oracle import chunkwise as C
from synth import make_inputs


def _maxrel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("cfg,sizes", [
    (dict(hq=2, hkv=1, seq=64, d=16), [16, 16, 16, 16]),        # configs[0] tiny, k=4
    (dict(hq=4, hkv=2, seq=96, d=32), [32, 32, 32]),
    (dict(hq=4, hkv=1, seq=80, d=16), [24, 24, 24, 8]),          # ragged last chunk (Z15)
    (dict(hq=2, hkv=2, seq=60, d=8), [7, 13, 1, 20, 19]),        # irregular, a 1-token chunk
])
def test_seco_equals_full(cfg, sizes):
    x = make_inputs(**cfg, seed=11, bf16=False)
    o_f, lse_f = A.full_attn_fwd(x.q, x.k, x.v)
    dq_f, dk_f, dv_f = A.full_attn_bwd(x.q, x.k, x.v, x.do)
    r = C.seco_step(x.q, x.k, x.v, x.do, sizes)
    for a, b in ((r["o"], o_f), (r["lse"], lse_f), (r["dq"], dq_f), (r["dk"], dk_f), (r["dv"], dv_f)):
        assert _maxrel(a, b) < 1e-12


def test_single_chunk_is_full():
    x = make_inputs(hq=2, hkv=1, seq=64, d=16, seed=12, bf16=False)
    r = C.seco_step(x.q, x.k, x.v, x.do, [64])
    dq_f, dk_f, dv_f = A.full_attn_bwd(x.q, x.k, x.v, x.do)
    assert _maxrel(r["dq"], dq_f) < 1e-14 and _maxrel(r["dk"], dk_f) < 1e-14


def test_spaco_all_chunks_gamma1_is_seco():
    """Alg. 2 with t = k: gamma = k/t = 1, I = all -> identical to Alg. 1."""
    x = make_inputs(hq=2, hkv=1, seq=64, d=16, seed=13, bf16=False)
    sizes = [16] * 4
    a = C.seco_step(x.q, x.k, x.v, x.do, sizes)
    b = C.spaco_step(x.q, x.k, x.v, x.do, sizes, [3, 2, 1, 0], 1.0)
    for key in ("dq", "dk", "dv"):
        assert np.array_equal(a[key], b[key])


def test_spaco_nonselected_chunks_are_zero_and_relay_scales():
    x = make_inputs(hq=2, hkv=1, seq=64, d=16, seed=14, bf16=False)
    sizes = [16] * 4
    r1 = C.spaco_step(x.q, x.k, x.v, x.do, sizes, [3, 1], 1.0)
    r2 = C.spaco_step(x.q, x.k, x.v, x.do, sizes, [3, 1], 2.0)
    # chunks 0 and 2 not selected: no gradient at all
    for r in (r1, r2):
        assert np.abs(r["dq"][:, :16]).max() == 0 and np.abs(r["dk"][:, 32:48]).max() == 0
    # chunk 1's own K grad = local + gamma * (deposit from chunk 3): linear in gamma
    loc = 2 * r1["dk"][:, 16:32] - r2["dk"][:, 16:32]
    dep = r2["dk"][:, 16:32] - r1["dk"][:, 16:32]
    _, dk3, _ = A.chunk_bwd(x.q[:, 48:64], x.k, x.v, x.do[:, 48:64], 48)
    _, dk1, _ = A.chunk_bwd(x.q[:, 16:32], x.k, x.v, x.do[:, 16:32], 16)
    assert np.abs(dep - dk3[:, 16:32]).max() < 1e-12
    assert np.abs(loc - dk1[:, 16:32]).max() < 1e-12
    # chunk 3 (the last) has nothing relayed into it
    assert np.array_equal(r1["dk"][:, 48:], r2["dk"][:, 48:])
