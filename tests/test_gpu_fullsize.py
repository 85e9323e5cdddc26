"""Parity at the benchmark's full size (BASELINE configs[2] = cfg3: 32 q / 8 kv heads,
d=128, seq 32768, chunk 2048) in the launch configuration bench.py times (the same
ChunkedAttention step through the C ABI).  The oracle cannot afford the whole
sequence, so it checks
  * sampled rows one by one: O, LSE and dQ of a query row depend only on that row
    (oracle chunk_fwd / chunk_bwd on a one-row "chunk" at its absolute position);
  * dK, dV of keys in the last chunk: only the last chunk's rows see them
    (oracle chunk_bwd of the last chunk for one kv-head group);
  * properties that hold at any size: sum over keys of dK is 0 (rows of dS sum to
    0) and sum over keys of dV equals the sum of dO over the group's rows (rows of P
    sum to 1)."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import sampler as OS
from tests.gpu_util import BF16_TOL, err, host, upload
from synth import make_inputs

pytestmark = pytest.mark.gpu

HQ, HKV, D, S, C = 32, 8, 128, 32768, 2048
G = HQ // HKV


@pytest.fixture(scope="module")
def cfg3():
    x = make_inputs(HQ, HKV, S, D, seed=0)
    q, k, v, do = upload(x, torch.bfloat16)
    from paper_2505_16710_b200.step import ChunkedAttention
    layer = ChunkedAttention(HQ, HKV, D, S, C, dtype=torch.bfloat16)
    return x, (q, k, v, do), layer


ROWS = [(0, 0), (5, 2047), (13, 2048), (22, 7 * 2048 + 1000), (31, 15 * 2048 + 3), (17, S - 1), (8, 9 * 2048 + 2047)]


def _row_ref(x, h, p):
    g = h // G
    qr, dor = x.q[h:h + 1, p:p + 1], x.do[h:h + 1, p:p + 1]
    o, lse = OA.chunk_fwd(qr, x.k[g:g + 1], x.v[g:g + 1], p)
    dq, _, _ = OA.chunk_bwd(qr, x.k[g:g + 1], x.v[g:g + 1], dor, p)
    return o[0, 0], lse[0, 0], dq[0, 0]


def test_cfg3_seco_sampled_rows_and_invariants(cfg3):
    x, (q, k, v, do), layer = cfg3
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    o_g, dq_g = host(layer.o), host(layer.dq)
    lse_g = host(layer.lse_full())
    o_r, l_r, dq_r, o_s, l_s, dq_s = [], [], [], [], [], []
    for h, p in ROWS:
        a, b, c = _row_ref(x, h, p)
        o_r.append(a); l_r.append(b); dq_r.append(c)
        o_s.append(o_g[h, p]); l_s.append(lse_g[h, p]); dq_s.append(dq_g[h, p])
    assert err(np.array(o_s), np.array(o_r)) <= BF16_TOL
    assert err(np.array(l_s), np.array(l_r)) <= BF16_TOL
    assert err(np.array(dq_s), np.array(dq_r)) <= BF16_TOL
    # keys of the last chunk, kv-head group 5: exact from the last chunk's rows
    g = 5
    a0 = S - C
    _, dk_src, dv_src = OA.chunk_bwd(x.q[g * G:(g + 1) * G, a0:], x.k[g:g + 1], x.v[g:g + 1],
                                     x.do[g * G:(g + 1) * G, a0:], a0)
    dk_g = host(layer.dk[g, a0:])
    dv_g = host(layer.dv[g, a0:])
    assert err(dk_g, dk_src[0, a0:]) <= BF16_TOL
    assert err(dv_g, dv_src[0, a0:]) <= BF16_TOL
    # any-size properties over the whole sequence, every kv head
    dk_all = layer.dk.double().sum(dim=1).cpu().numpy()                  # [hkv][d], exactly 0
    dk_abs = layer.dk.double().abs().sum(dim=1).cpu().numpy()
    assert np.abs(dk_all).max() <= BF16_TOL * dk_abs.max()
    dv_sum = layer.dv.double().sum(dim=1).cpu().numpy()
    do_sum = x.do.astype(np.float64).reshape(HKV, G, S, D).sum(axis=(1, 2))
    assert err(dv_sum, do_sum) <= BF16_TOL


def test_cfg3_spaco_sampled_rows(cfg3):
    x, (q, k, v, do), layer = cfg3
    r = layer.spaco_step(q, k, v, do, 4, 0, cap=2.0, mode=OS.PAPER)
    torch.cuda.synchronize()
    assert r.selected == OS.sample_indices(16, 4, 0, OS.PAPER)
    dq_g = host(layer.dq)
    for h, p in ROWS:
        j = p // C
        if j in r.selected:
            _, _, ref = _row_ref(x, h, p)
            assert err(dq_g[h, p], r.seed_scale * ref) <= BF16_TOL
        else:
            assert np.abs(dq_g[h, p]).max() == 0.0


def test_memory_ledger_step_allocates_nothing():
    """a SeCO / SpaCO step allocates no device memory beyond the
    buffers set up once, and the per-call working set (workspace + chunk views) does not grow
    with the number of chunks k; only the O(S) checkpoint-sized buffers do."""
    from paper_2505_16710_b200.step import ChunkedAttention
    hq, hkv, d, c = 8, 2, 128, 256
    ledgers = {}
    for k in (2, 4, 8):
        x = make_inputs(hq, hkv, k * c, d, seed=k)
        q, kc, vc, do = upload(x, torch.bfloat16)
        layer = ChunkedAttention(hq, hkv, d, k * c, c, dtype=torch.bfloat16)
        layer.seco_step(q, kc, vc, do)           # warm (tensor maps, attributes)
        torch.cuda.synchronize()
        before = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        layer.seco_step(q, kc, vc, do)
        layer.spaco_step(q, kc, vc, do, t=1, seed=3)
        torch.cuda.synchronize()
        assert torch.cuda.max_memory_allocated() == before
        ledgers[k] = layer.memory_ledger()
    per_call = {k: (v["per_call_chunk_bytes"], v["per_call_workspace_bytes"]) for k, v in ledgers.items()}
    assert len(set(per_call.values())) == 1
    assert ledgers[8]["dkv_fp32_bytes"] == 4 * ledgers[2]["dkv_fp32_bytes"]
    assert ledgers[8]["kv_cache_bytes"] == 4 * ledgers[2]["kv_cache_bytes"]


def test_cfg4_rank_shape_seco_sampled_rows_tail_keys_and_invariants():
    """One rank of BASELINE cfg4 head-sharded over 8 GPUs (4 q heads / 1 kv
    head, d=128, seq 131072, chunk 4096), the per-rank launch configuration `bench.py --gpus
    8` times: a sub-wave forward grid (split-KV, row a9) and 4096-row chunks.  Sampled rows
    one by one; dK / dV of the last 8 keys, which only the last 8 query rows see (exact from
    those rows alone); and the any-size sums over every key."""
    from paper_2505_16710_b200.step import ChunkedAttention
    hq, hkv, d, s, c = 4, 1, 128, 131072, 4096
    x = make_inputs(hq, hkv, s, d, seed=4)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = ChunkedAttention(hq, hkv, d, s, c, dtype=torch.bfloat16)
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    o_g, dq_g, lse_g = host(layer.o), host(layer.dq), host(layer.lse_full())
    rows = [(0, 0), (1, 4095), (2, 4096), (3, 77 * 1000 + 5), (0, s - 4096), (1, s - 1), (3, 31 * 4096 + 4095)]
    got, ref = {"o": [], "lse": [], "dq": []}, {"o": [], "lse": [], "dq": []}
    for h, p in rows:
        qr, dor = x.q[h:h + 1, p:p + 1], x.do[h:h + 1, p:p + 1]
        o, lse = OA.chunk_fwd(qr, x.k, x.v, p)
        dq, _, _ = OA.chunk_bwd(qr, x.k, x.v, dor, p)
        ref["o"].append(o[0, 0]); ref["lse"].append(lse[0, 0]); ref["dq"].append(dq[0, 0])
        got["o"].append(o_g[h, p]); got["lse"].append(lse_g[h, p]); got["dq"].append(dq_g[h, p])
    for key in got:
        assert err(np.array(got[key]), np.array(ref[key])) <= BF16_TOL, key
    r = 8
    _, dk_src, dv_src = OA.chunk_bwd(x.q[:, s - r:], x.k, x.v, x.do[:, s - r:], s - r)
    assert err(host(layer.dk[0, s - r:]), dk_src[0, s - r:]) <= BF16_TOL
    assert err(host(layer.dv[0, s - r:]), dv_src[0, s - r:]) <= BF16_TOL
    dk_sum = layer.dk.double().sum(dim=1).cpu().numpy()
    assert np.abs(dk_sum).max() <= BF16_TOL * layer.dk.double().abs().sum(dim=1).max().item()
    do_sum = x.do.astype(np.float64).sum(axis=(0, 1))[None]
    assert err(layer.dv.double().sum(dim=1).cpu().numpy(), do_sum) <= BF16_TOL


def _whole_units(c, k, hkv, G):
    """Number of (call, CTA) work items that take a whole 128-key unit (n0 of the backward work
    list) over a step's chunk calls, on this GPU's SM count."""
    import ctypes
    from paper_2505_16710_b200 import _lib
    lib = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = (ctypes.c_int32 * 4)()
    return sum((lib.seco_debug_bwd_schedule(c, j, hkv, G, sms, out), out[0])[1] for j in range(k))


def _group_ref(x, groups, c, selected=None, gamma=1.0, s=1.0):
    """Oracle SeCO / SpaCO step of the given kv-head groups (their G q-heads each)."""
    from oracle import chunkwise as OC
    qh = [h for g in groups for h in range(g * G_OF(x), (g + 1) * G_OF(x))]
    sub = (x.q[qh], x.k[groups], x.v[groups], x.do[qh])
    k = x.q.shape[1] // c
    if selected is None:
        return qh, OC.seco_step(*sub, [c] * k)
    return qh, OC.spaco_step(*sub, [c] * k, selected, gamma, s)


def G_OF(x):
    return x.q.shape[0] // x.k.shape[0]


def _compare_groups(layer, ref, qh, groups, what):
    got = {"o": host(layer.o[qh]), "lse": host(layer.lse_full()[qh]), "dq": host(layer.dq[qh]),
           "dk": host(layer.dk[groups]), "dv": host(layer.dv[groups])}
    for name, g in got.items():
        e = err(g, ref[name])
        assert e <= BF16_TOL, (what, name, e)


def test_cfg2_full_size_elementwise_two_groups():
    """BASELINE configs[1] (cfg2: 32 q / 8 kv heads, d = 128, 8K tokens, 1K chunks) through the C
    ABI with every head, then O, LSE, dQ, dK and dV of two whole kv-head groups compared element
    by element with the oracle (the paper's own check compares every gradient element, App. D
    P:526).  At this size the backward work list runs whole 128-key units (one CTA owns a
    cache-slot tile for all of its query tiles, depositing into earlier checkpoints),
    which the small parity shapes never schedule."""
    from paper_2505_16710_b200.step import ChunkedAttention
    hq, hkv, d, s, c = 32, 8, 128, 8192, 1024
    assert _whole_units(c, s // c, hkv, hq // hkv) > 0
    x = make_inputs(hq, hkv, s, d, seed=21)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = ChunkedAttention(hq, hkv, d, s, c, dtype=torch.bfloat16)
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    groups = [2, 7]
    qh, ref = _group_ref(x, groups, c)
    _compare_groups(layer, ref, qh, groups, "cfg2 seco")
    # SpaCO (PAPER mode, t = 3 of 8, cap 2): sampled chunks element-wise, skipped ones zero
    r = layer.spaco_step(q, k, v, do, 3, 7, cap=2.0, mode=OS.PAPER)
    torch.cuda.synchronize()
    qh, ref = _group_ref(x, groups, c, r.selected, r.relay_scale, r.seed_scale)
    _compare_groups(layer, ref, qh, groups, ("cfg2 spaco", r.selected))


def test_cfg3_one_group_every_key(cfg3):
    """The bench configuration itself (cfg3, 32K tokens, 2K chunks, every head), one kv-head
    group compared element by element over the whole sequence: O, LSE, dQ of its 4 q heads and
    dK, dV of every one of its 32768 keys (fp64 oracle, ~5 TFLOP on the host)."""
    x, (q, k, v, do), layer = cfg3
    assert _whole_units(C, S // C, HKV, G) > 0
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    groups = [3]
    qh, ref = _group_ref(x, groups, C)
    _compare_groups(layer, ref, qh, groups, "cfg3 seco group 3")
