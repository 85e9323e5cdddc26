"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Tolerances from BASELINE.json north_star: bf16 <= 2e-2, fp32
debug <= 1e-4 (max relative error, reading Z13); sampling indices bit-exact."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import chunkwise as OC
from oracle import sampler as OS
from tests.gpu_util import BF16_TOL, FP32_TOL, err, host, inputs, upload

pytestmark = pytest.mark.gpu


def _layer(hq, hkv, d, seq, c, dtype, own=False):
    from paper_2505_16710_b200.step import ChunkedAttention
    return ChunkedAttention(hq, hkv, d, seq, c, dtype=dtype, own_copies=own)


def _check_step(layer, ref, tol, selected=None, what=""):
    o = host(layer.o)
    lse = host(layer.lse_full())
    assert err(o, ref["o"]) <= tol, (what, "o", err(o, ref["o"]))
    assert err(lse, ref["lse"]) <= tol, (what, "lse", err(lse, ref["lse"]))
    dk, dv = layer.own_grads()
    for name, gpu in (("dq", host(layer.dq)), ("dk", host(dk)), ("dv", host(dv))):
        e = err(gpu, ref[name])
        assert e <= tol, (what, name, e)
    if layer.own is not None:
        # dk_own / dv_own (row a7): the element-type copy of slot 0 -- the step's last stage-2
        # call is chunk 0's backward (or skip) -- against the oracle, and bit-equal to the
        # round-to-nearest-even conversion of the fp32 slot the library also returns
        c = layer.chunk
        for t, name in ((0, "dk"), (1, "dv")):
            own = layer.own[t]
            e = err(host(own), ref[name][:, :c])
            assert e <= tol, (what, name + "_own", e)
            assert torch.equal(own, layer.dkv[t, :, :c].to(own.dtype)), (what, name + "_own conversion")
    if selected is not None:
        # chunks outside the sample (reading Z11): exactly zero, written by spaco_chunk_skip
        c = layer.chunk
        for j in range(layer.k):
            if j not in selected:
                assert float(layer.dq[:, j * c:(j + 1) * c].abs().max()) == 0.0, (what, j, "dq")
                assert float(layer.dkv[:, :, j * c:(j + 1) * c].abs().max()) == 0.0, (what, j, "dkv")


# ------------------------------------------------------------------ fp32 debug build
FP32_CASES = [
    dict(hq=2, hkv=1, seq=64, d=16, c=16),        # BASELINE configs[0] (tiny)
    dict(hq=4, hkv=1, seq=1024, d=64, c=256),     # one head group at 1K
    dict(hq=6, hkv=2, seq=96, d=20, c=32),        # odd G, odd d
    dict(hq=2, hkv=1, seq=48, d=16, c=48),        # k = 1
]


@pytest.mark.parametrize("cfg", FP32_CASES)
def test_fp32_seco_step(cfg):
    x = inputs(cfg["hq"], cfg["hkv"], cfg["seq"], cfg["d"], seed=1, dtype=torch.float32)
    q, k, v, do = upload(x, torch.float32)
    layer = _layer(cfg["hq"], cfg["hkv"], cfg["d"], cfg["seq"], cfg["c"], torch.float32, own=True)
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [cfg["c"]] * (cfg["seq"] // cfg["c"]))
    _check_step(layer, ref, FP32_TOL, what=str(cfg))
    # own-slot copy of the last processed chunk (j = 0) equals dkv slot 0
    assert np.array_equal(host(layer.own[0]), host(layer.dk[:, :cfg["c"]]))


@pytest.mark.parametrize("mode,t", [(OS.PAPER, 2), (OS.PAPER, 3), (OS.HT, 2), (OS.BERNOULLI, 2)])
def test_fp32_spaco_step(mode, t):
    hq, hkv, seq, d, c = 2, 1, 64, 16, 16
    x = inputs(hq, hkv, seq, d, seed=2, dtype=torch.float32)
    q, k, v, do = upload(x, torch.float32)
    layer = _layer(hq, hkv, d, seq, c, torch.float32, own=True)
    for seed in (0, 1, 5):
        r = layer.spaco_step(q, k, v, do, t, seed, cap=0.0, mode=mode)
        torch.cuda.synchronize()
        idx, g, s = OS.sample_and_scale(4, t, seed, 0.0, mode)
        assert r.selected == idx and np.float32(r.relay_scale) == np.float32(g)
        ref = OC.spaco_step(x.q, x.k, x.v, x.do, [c] * 4, idx, g, s)
        _check_step(layer, ref, FP32_TOL, selected=idx, what=(mode, t, seed))


# ------------------------------------------------------------------ bf16 tensor cores
BF16_CASES = [
    dict(hq=8, hkv=2, seq=512, d=128, c=128),     # 4 chunks, NH=2 pairs, 1 tile per chunk
    dict(hq=4, hkv=1, seq=1024, d=128, c=256),    # several tiles per chunk, G=4
    dict(hq=3, hkv=1, seq=768, d=128, c=384),     # odd G -> one head per CTA (NH=1), 3 tiles / chunk
    dict(hq=2, hkv=2, seq=512, d=128, c=256),     # MHA (G=1)
    dict(hq=8, hkv=2, seq=512, d=64, c=128),      # d = 64 (zero-padded 128-wide tiles)
    dict(hq=3, hkv=1, seq=768, d=64, c=384),      # d = 64, NH=1
    dict(hq=16, hkv=2, seq=640, d=128, c=128),    # G = 8, 5 chunks of the minimum size
    dict(hq=6, hkv=3, seq=1536, d=128, c=768),    # odd kv-head count, 6 query tiles per chunk
    dict(hq=4, hkv=1, seq=384, d=128, c=384),     # k = 1: one chunk, SeCO = plain full attention
    # ragged chunks (c % 128 != 0): the last query tile of every chunk is partial, chunk starts
    # and key tiles are misaligned, so the causal diagonal straddles two key tiles
    dict(hq=4, hkv=1, seq=600, d=128, c=200),     # 128 + 72 rows per chunk, G=4 (NH=2)
    dict(hq=3, hkv=1, seq=600, d=64, c=300),      # NH=1, d = 64, 128 + 128 + 44 rows
    dict(hq=8, hkv=2, seq=400, d=128, c=100),     # chunk shorter than one tile, 4 chunks
    dict(hq=2, hkv=2, seq=520, d=128, c=520),     # k = 1, MHA, 4 tiles + 8 rows
    dict(hq=6, hkv=3, seq=999, d=128, c=333),     # odd G and kv heads, 3 chunks of 333
    dict(hq=4, hkv=1, seq=512, d=96, c=256),      # d = 96 (zero-padded to the 128-wide tiles)
    dict(hq=8, hkv=2, seq=600, d=32, c=200),      # d = 32, ragged chunks
    dict(hq=2, hkv=1, seq=5, d=128, c=1),         # degenerate: 1-token chunks (every row its own chunk)
    dict(hq=4, hkv=2, seq=21, d=64, c=7),         # 7-token chunks, d = 64
]


@pytest.mark.parametrize("cfg", BF16_CASES)
@pytest.mark.parametrize("peaky", [False, True])
def test_bf16_seco_step(cfg, peaky):
    x = inputs(cfg["hq"], cfg["hkv"], cfg["seq"], cfg["d"], seed=3, peaky=peaky)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = _layer(cfg["hq"], cfg["hkv"], cfg["d"], cfg["seq"], cfg["c"], torch.bfloat16, own=True)
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [cfg["c"]] * (cfg["seq"] // cfg["c"]))
    _check_step(layer, ref, BF16_TOL, what=(cfg, peaky))


def test_bf16_forward_deterministic():
    """Stage-2 rebuild must reproduce stage 1 bit for bit (checkpoint reconstruction)."""
    x = inputs(8, 2, 1024, 128, seed=4)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = _layer(8, 2, 128, 1024, 256, torch.bfloat16)
    layer.forward_chunk(q, k, v, 3)
    o1, l1 = layer.o[:, 768:].clone(), layer.lse[3].clone()
    layer.o.zero_()
    layer.forward_chunk(q, k, v, 3)
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int16), layer.o[:, 768:].view(torch.int16))
    assert torch.equal(l1.view(torch.int32), layer.lse[3].view(torch.int32))


@pytest.mark.parametrize("t,seed,c", [(2, 0, 256), (1, 3, 256), (4, 1, 256), (2, 4, 250), (3, 6, 250)])
def test_bf16_spaco_step(t, seed, c):
    hq, hkv, d = 8, 2, 128
    seq = 4 * c                                    # c = 250: ragged chunks (skip kernel rows, relay)
    x = inputs(hq, hkv, seq, d, seed=5)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = _layer(hq, hkv, d, seq, c, torch.bfloat16, own=True)
    r = layer.spaco_step(q, k, v, do, t, seed, cap=2.0, mode=OS.PAPER)
    torch.cuda.synchronize()
    idx, g, s = OS.sample_and_scale(4, t, seed, 2.0, OS.PAPER)
    assert r.selected == idx
    ref = OC.spaco_step(x.q, x.k, x.v, x.do, [c] * 4, idx, g, s)
    _check_step(layer, ref, BF16_TOL, selected=idx, what=(t, seed))


def test_bf16_chunk_calls_compose():
    """Single backward calls with relay / grad scale: dkv semantics of include/seco.h."""
    hq, hkv, seq, d, c = 4, 1, 512, 128, 128
    x = inputs(hq, hkv, seq, d, seed=6)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = _layer(hq, hkv, d, seq, c, torch.bfloat16)
    from paper_2505_16710_b200 import ops
    # pre-load a fake relayed gradient B in slot 2, then run chunk 2's backward
    layer.dkv.zero_()
    base = torch.randn(2, hkv, c, d, device="cuda")
    layer.dkv[:, :, 2 * c:3 * c] = base
    layer.forward_chunk(q, k, v, 2)
    layer.backward_chunk(q, k, v, do, 2, relay_scale=1.5, grad_scale=0.5)
    torch.cuda.synchronize()
    dq_ref, dk_src, dv_src = OA.chunk_bwd(x.q[:, 2 * c:3 * c], x.k, x.v, x.do[:, 2 * c:3 * c], 2 * c)
    own_k = 1.5 * host(base[0]) + 0.5 * dk_src[:, 2 * c:]
    own_v = 1.5 * host(base[1]) + 0.5 * dv_src[:, 2 * c:]
    assert err(host(layer.dq[:, 2 * c:3 * c]), 0.5 * dq_ref) <= BF16_TOL
    assert err(host(layer.dk[:, 2 * c:3 * c]), own_k) <= BF16_TOL
    assert err(host(layer.dv[:, 2 * c:3 * c]), own_v) <= BF16_TOL
    assert err(host(layer.dk[:, :2 * c]), 0.5 * dk_src[:, :2 * c]) <= BF16_TOL
    assert err(host(layer.dv[:, :2 * c]), 0.5 * dv_src[:, :2 * c]) <= BF16_TOL
    assert float(layer.dkv[:, :, 3 * c:].abs().max()) == 0.0


@pytest.mark.parametrize("j,d,c", [(2, 128, 1024), (3, 128, 1024), (3, 64, 1024), (3, 128, 1000), (2, 64, 1000)])
def test_bf16_forward_split_kv(j, d, c):
    """Long chunks: the forward splits each query tile's key range and merges partials (a9);
    c = 1000 is ragged (the partials keep 1024 rows per head, the last 24 never stored)."""
    hq, hkv, seq = 8, 2, 4 * c                      # 32 units < 148 SMs: the forward splits
    x = inputs(hq, hkv, seq, d, seed=7, peaky=(j == 3))
    q, k, v, do = upload(x, torch.bfloat16)
    layer = _layer(hq, hkv, d, seq, c, torch.bfloat16)
    layer.forward_chunk(q, k, v, j)
    launches = __import__("paper_2505_16710_b200").ops.last_launch_count()
    torch.cuda.synchronize()
    assert launches == 2       # split-KV kernel + combine (a sub-wave grid)
    o_ref, lse_ref = OA.chunk_fwd(x.q[:, j * c:(j + 1) * c], x.k, x.v, j * c)
    assert err(host(layer.o[:, j * c:(j + 1) * c]), o_ref) <= BF16_TOL
    assert err(host(layer.lse[j]), lse_ref) <= 1e-4
    # rebuild reproduces the split result bit for bit
    o1 = layer.o[:, j * c:(j + 1) * c].clone()
    layer.forward_chunk(q, k, v, j)
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int16), layer.o[:, j * c:(j + 1) * c].view(torch.int16))


def test_bf16_strided_sequence_major_layout():
    """The ABI takes arbitrary head/row strides: Q, O, dO, dQ as [S][Hq][d] (projection output
    layout) and the KV cache as [S][Hkv][d], passed as strided views -- same results."""
    from paper_2505_16710_b200 import ops
    hq, hkv, seq, d, c = 8, 2, 512, 128, 128
    x = inputs(hq, hkv, seq, d, seed=8)
    q, k, v, do = upload(x, torch.bfloat16)
    qs, dos = q.transpose(0, 1).contiguous(), do.transpose(0, 1).contiguous()    # [S][H][d]
    ks, vs = k.transpose(0, 1).contiguous(), v.transpose(0, 1).contiguous()
    qv, dov, kv_, vv = qs.transpose(0, 1), dos.transpose(0, 1), ks.transpose(0, 1), vs.transpose(0, 1)
    shape = ops.make_shape(qv, kv_, c)
    assert shape.q_row_stride == hq * d and shape.q_head_stride == d
    o = torch.empty(seq, hq, d, dtype=torch.bfloat16, device="cuda").transpose(0, 1)
    dq = torch.zeros(seq, hq, d, dtype=torch.bfloat16, device="cuda").transpose(0, 1)
    lse = torch.empty(seq // c, hq, c, dtype=torch.float32, device="cuda")
    dkv = torch.zeros(2, hkv, seq, d, dtype=torch.float32, device="cuda")
    ws = torch.empty(ops.seco_workspace_size(shape) // 4, dtype=torch.float32, device="cuda")
    k_chunks = seq // c
    for j in range(k_chunks):
        ops.seco_chunk_forward(shape, j, ops.chunk_view(qv, shape, j), kv_, vv, ops.chunk_view(o, shape, j), lse[j], ws)
    for j in reversed(range(k_chunks)):
        ops.seco_chunk_forward(shape, j, ops.chunk_view(qv, shape, j), kv_, vv, ops.chunk_view(o, shape, j), lse[j], ws)
        ops.seco_chunk_backward(shape, j, ops.chunk_view(qv, shape, j), kv_, vv, ops.chunk_view(o, shape, j),
                                ops.chunk_view(dov, shape, j), lse[j], 1.0, 1.0, dkv, ops.chunk_view(dq, shape, j),
                                None, None, ws)
    torch.cuda.synchronize()
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * k_chunks)
    assert err(host(o), ref["o"]) <= BF16_TOL
    assert err(host(dq), ref["dq"]) <= BF16_TOL
    assert err(host(dkv[0]), ref["dk"]) <= BF16_TOL
    assert err(host(dkv[1]), ref["dv"]) <= BF16_TOL


@pytest.mark.parametrize("hq,hkv,seq,c", [(8, 2, 2048, 512), (4, 1, 1024, 128), (4, 1, 1000, 250)])
def test_bf16_deterministic_mode_bit_reproducible(hq, hkv, seq, c):
    """SECO_FLAG_DETERMINISTIC: two SeCO steps and two SpaCO
    steps on the same inputs give bit-identical O, dQ and dKV, and stay within the bf16
    tolerance of the oracle.  These shapes use Q-split and many key tiles per query tile in
    the default mode, so both ordering mechanisms are exercised."""
    from paper_2505_16710_b200.step import ChunkedAttention
    x = inputs(hq, hkv, seq, 128, seed=11)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = ChunkedAttention(hq, hkv, 128, seq, c, dtype=torch.bfloat16, deterministic=True)
    outs = []
    for _ in range(2):
        layer.seco_step(q, k, v, do)
        torch.cuda.synchronize()
        outs.append((layer.o.clone(), layer.dq.clone(), layer.dkv.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a.view(torch.int32),
                           b.view(torch.int16) if b.dtype == torch.bfloat16 else b.view(torch.int32))
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    assert err(host(layer.dq), ref["dq"]) <= BF16_TOL
    assert err(host(layer.dkv[0]), ref["dk"]) <= BF16_TOL
    assert err(host(layer.dkv[1]), ref["dv"]) <= BF16_TOL
    sp = []
    for _ in range(2):
        layer.spaco_step(q, k, v, do, t=max(1, seq // c // 2), seed=5)
        torch.cuda.synchronize()
        sp.append((layer.dq.clone(), layer.dkv.clone()))
    assert torch.equal(sp[0][0].view(torch.int16), sp[1][0].view(torch.int16))
    assert torch.equal(sp[0][1].view(torch.int32), sp[1][1].view(torch.int32))


def test_bf16_two_layers_on_two_streams():
    """Reentrancy (include/seco.h): two independent layers stepped concurrently on two CUDA
    streams, each with its own workspace, give bit-identical results to the same steps run
    one after the other -- the only shared library state is the tensor-map cache; the split
    forward's counters live in each caller's workspace."""
    from paper_2505_16710_b200.step import ChunkedAttention
    shapes = [(8, 2, 4096, 128, 1024), (4, 1, 2000, 128, 250)]     # split-KV forward; ragged chunks
    xs = [inputs(hq, hkv, seq, d, seed=20 + n) for n, (hq, hkv, seq, d, c) in enumerate(shapes)]
    ups = [upload(x, torch.bfloat16) for x in xs]
    layers = [ChunkedAttention(hq, hkv, d, seq, c) for (hq, hkv, seq, d, c) in shapes]
    for L, (q, k, v, do) in zip(layers, ups):
        L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    ref = [(L.o.clone(), L.dq.clone(), L.dkv.clone()) for L in layers]
    streams = [torch.cuda.Stream() for _ in layers]
    for _ in range(3):
        for L in layers:
            L.o.zero_(); L.dq.zero_()
        torch.cuda.synchronize()
        for L, (q, k, v, do), st in zip(layers, ups, streams):
            L.seco_step(q, k, v, do, stream=st)
        torch.cuda.synchronize()
        for L, (o, dq, dkv) in zip(layers, ref):
            assert torch.equal(L.o.view(torch.int16), o.view(torch.int16))
            assert torch.equal(L.dq.view(torch.int16), dq.view(torch.int16)) or \
                err(host(L.dq), host(dq)) <= 1e-2                   # dQ reduce-adds: any order
            assert err(host(L.dkv), host(dkv)) <= 1e-2


def test_bf16_chunked_attention_sequence_major_layout():
    """ChunkedAttention(layout="shd"): sequence-major storage (the bench's end-to-end path)
    gives the same step as the oracle."""
    from paper_2505_16710_b200.step import ChunkedAttention
    hq, hkv, seq, d, c = 8, 2, 1024, 128, 256
    x = inputs(hq, hkv, seq, d, seed=12)
    q, k, v, do = (t.transpose(0, 1).contiguous().transpose(0, 1) for t in upload(x, torch.bfloat16))
    layer = ChunkedAttention(hq, hkv, d, seq, c, layout="shd")
    layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    assert err(host(layer.o), ref["o"]) <= BF16_TOL
    assert err(host(layer.dq), ref["dq"]) <= BF16_TOL
    assert err(host(layer.dkv[0]), ref["dk"]) <= BF16_TOL
    assert err(host(layer.dkv[1]), ref["dv"]) <= BF16_TOL
    with pytest.raises(ValueError):
        layer.seco_step(*upload(x, torch.bfloat16))          # head-major inputs: wrong strides


def test_bf16_backward_v1_subprocess():
    """The v1 backward (SECO_BWD_V2=0: dV dK dQ^T(i) -> R0 then S^T(i+1), dQ staged in the dead
    Q / dO buffers; still the deterministic-mode kernel) matches the oracle too.  The
    switch is read once per process, so the check runs in a child process."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import chunkwise as OC
from tests.gpu_util import BF16_TOL, err, host, inputs, upload
from paper_2505_16710_b200.step import ChunkedAttention
for (hq, hkv, seq, c) in ((8, 2, 512, 128), (4, 1, 1024, 256), (3, 1, 768, 384), (4, 1, 600, 200)):
    x = inputs(hq, hkv, seq, 128, seed=5, peaky=True)
    q, k, v, do = upload(x, torch.bfloat16)
    L = ChunkedAttention(hq, hkv, 128, seq, c, dtype=torch.bfloat16)
    L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    dk, dv = L.own_grads()
    for name, gpu in (("dq", host(L.dq)), ("dk", host(dk)), ("dv", host(dv))):
        e = err(gpu, ref[name])
        assert e <= BF16_TOL, (hq, hkv, seq, c, name, e)
print("v1 ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, SECO_BWD_V2="0"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "v1 ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_bf16_forward_waits_for_producer_kernel():
    """The unsplit forward is a programmatic-dependent launch.  Without
    SECO_FLAG_PREV_INDEPENDENT it must wait for its predecessor before the first load: a torch
    copy kernel that writes the K / V cache right before the call is always seen.  With the flag
    (stage-1 chains, forward after forward) the results are bit-identical to the plain call."""
    from paper_2505_16710_b200 import ops
    hq, hkv, seq, d, c = 8, 2, 8192, 128, 2048
    x = inputs(hq, hkv, seq, d, seed=13)
    q, k, v, do = upload(x, torch.bfloat16)
    layer = _layer(hq, hkv, d, seq, c, torch.bfloat16)
    kc, vc = torch.zeros_like(k), torch.zeros_like(v)
    big_k = k.repeat(8, 1, 1)                     # a longer producer kernel (8x the cache)
    sink = torch.empty_like(big_k)
    j = 3
    o_ref, lse_ref = OA.chunk_fwd(x.q[:, j * c:(j + 1) * c], x.k, x.v, j * c)
    qj, oj = ops.chunk_view(q, layer.shape, j), ops.chunk_view(layer.o, layer.shape, j)
    for rep in range(4):
        kc.zero_()
        vc.zero_()
        torch.cuda.synchronize()
        sink.copy_(big_k)                         # keeps the GPU busy
        kc.copy_(k)                               # the producer the forward must wait for
        vc.copy_(v)
        ops.seco_chunk_forward(layer.shape, j, qj, kc, vc, oj, layer.lse[j], None)   # ws=None: unsplit, PDL
        torch.cuda.synchronize()
        assert err(host(oj), o_ref) <= BF16_TOL, rep
        assert err(host(layer.lse[j]), lse_ref) <= 1e-4, rep
    # stage 1 with chained launches == stage 1 with plain launches, bit for bit
    outs = []
    for chained in (False, True):
        layer.o.zero_()
        for jj in range(seq // c):
            ops.seco_chunk_forward(layer.shape_chain if (chained and jj > 0) else layer.shape, jj,
                                   ops.chunk_view(q, layer.shape, jj), k, v,
                                   ops.chunk_view(layer.o, layer.shape, jj), layer.lse[jj], None)
        torch.cuda.synchronize()
        outs.append((layer.o.clone(), layer.lse.clone()))
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1].view(torch.int32), outs[1][1].view(torch.int32))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_spaco_expectation_through_the_kernels(dtype):
    """North-star check (b) on the GPU path: averaging the C-ABI SpaCO step over EVERY sampled set
    with its probability reproduces the oracle's exact expectation (O7): unbiased
    (= the SeCO gradient) under independent Bernoulli(rho) inclusion with s = gamma = 1/rho
    (reading Z7), and the closed-form biased factors t/k, t(t-1)/(k(k-1)) under Alg. 2's
    literal t-of-k sampling."""
    import itertools
    from oracle import expectation as OE
    hq, hkv, seq = 4, 1, 512
    d, c = (16, 128) if dtype == torch.float32 else (128, 128)
    k = seq // c
    x = inputs(hq, hkv, seq, d, seed=17, dtype=dtype)
    q, kk, v, do = upload(x, dtype)
    layer = _layer(hq, hkv, d, seq, c, dtype)
    tol = FP32_TOL if dtype == torch.float32 else BF16_TOL
    parts = OE.decompose(x.q, x.k, x.v, x.do, [c] * k)
    # Bernoulli(1/2), s = gamma = 2: the weighted mean over all 2^k sets is the SeCO gradient
    rho = 0.5
    acc = {n: 0.0 for n in ("dq", "dk", "dv")}
    for n in range(k + 1):
        for sel in itertools.combinations(range(k), n):
            layer.step(q, kk, v, do, list(sel), 1 / rho, 1 / rho)
            w = rho ** n * (1 - rho) ** (k - n)
            acc["dq"] = acc["dq"] + w * layer.dq.double()
            acc["dk"] = acc["dk"] + w * layer.dkv[0].double()
            acc["dv"] = acc["dv"] + w * layer.dkv[1].double()
    torch.cuda.synchronize()
    ref = OE.closed_form_bernoulli(parts, rho, 1 / rho, 1 / rho)
    seco = OC.seco_step(x.q, x.k, x.v, x.do, [c] * k)
    for n in ("dq", "dk", "dv"):
        assert err(acc[n].cpu().numpy(), ref[n]) <= tol, ("bernoulli", n)
        assert err(acc[n].cpu().numpy(), seco[n]) <= tol, ("bernoulli = seco", n)
    # t-of-k (PAPER mode, no cap): uniform mean over the C(k, t) sets = the biased closed form
    t, gamma = 2, k / 2
    acc = {n: 0.0 for n in ("dq", "dk", "dv")}
    sets = list(itertools.combinations(range(k), t))
    for sel in sets:
        layer.step(q, kk, v, do, list(sel), gamma, 1.0)
        acc["dq"] = acc["dq"] + layer.dq.double() / len(sets)
        acc["dk"] = acc["dk"] + layer.dkv[0].double() / len(sets)
        acc["dv"] = acc["dv"] + layer.dkv[1].double() / len(sets)
    torch.cuda.synchronize()
    ref = OE.closed_form_t_of_k(parts, k, t, gamma, 1.0)
    for n in ("dq", "dk", "dv"):
        assert err(acc[n].cpu().numpy(), ref[n]) <= tol, ("t-of-k", n)


@pytest.mark.parametrize("pair", ["1", "0"])
def test_bf16_forward_pair_switch_subprocess(pair):
    """The CTA-pair forward (seco_fwd2_sm100_kernel: cta_group::2 over the 4 q-heads of a kv group,
    half of every K / V tile per CTA) is the default only on full-wave grids (cfg3);
    SECO_FWD_PAIR=1 forces it on the small parity shapes here (split-KV, d = 64, ragged ranks of
    units), SECO_FWD_PAIR=0 forces the unpaired kernel.  O, LSE and the whole step against the
    oracle; the stage-2 rebuild reproduces stage 1 bit for bit.  Read once per process: child."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import chunkwise as OC
from tests.gpu_util import BF16_TOL, err, host, inputs, upload
from paper_2505_16710_b200.step import ChunkedAttention
for (hq, hkv, seq, c, d) in ((8, 2, 1024, 256, 128), (16, 4, 2048, 512, 128), (8, 2, 1024, 256, 64),
                             (4, 1, 4096, 1024, 128), (8, 2, 1000, 250, 128)):
    x = inputs(hq, hkv, seq, d, seed=7, peaky=True)
    q, k, v, do = upload(x, torch.bfloat16)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=torch.bfloat16)
    for j in range(seq // c):
        L.forward_chunk(q, k, v, j)
    torch.cuda.synchronize()
    o1, lse1 = L.o.clone(), L.lse.clone()
    L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    assert torch.equal(o1, L.o) and torch.equal(lse1, L.lse), (hq, hkv, seq, c, d, "rebuild not bitwise")
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    dk, dv = L.own_grads()
    for name, gpu in (("o", host(L.o)), ("dq", host(L.dq)), ("dk", host(dk)), ("dv", host(dv))):
        e = err(gpu, ref[name])
        assert e <= BF16_TOL, (hq, hkv, seq, c, d, name, e)
    lse = L.lse_full().cpu().numpy()
    assert np.abs(lse - ref["lse"]).max() <= 1e-3, (hq, hkv, seq, c, d, "lse")
print("pair switch ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, SECO_FWD_PAIR=pair),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "pair switch ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("pair,nsplit", [("0", ""), ("1", ""), ("0", "2"), ("1", "4")])
def test_bf16_forward_dp_split_tail_subprocess(pair, nsplit):
    """The DP + split-tail forward (multi-wave grids): whole units first, then the
    remaining units cut into key-range pieces whose last piece merges in-kernel (counter per
    CTA-unit, bulk-copied parts).  SECO_FWD_SLOTS=5 pretends 5 work slots so the small parity
    shapes here are multi-wave grids; SECO_FWD_NSPLIT forces the split factor.  O, LSE and the
    whole step against the oracle; the stage-2 rebuild reproduces stage 1 bit for bit; one
    library launch per split forward (no combine kernel).  Read once per process: child."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import chunkwise as OC
from tests.gpu_util import BF16_TOL, err, host, inputs, upload
from paper_2505_16710_b200 import ops
from paper_2505_16710_b200.step import ChunkedAttention
for (hq, hkv, seq, c, d) in ((8, 2, 4096, 1024, 128), (4, 1, 8192, 2048, 128), (8, 2, 4096, 1024, 64),
                             (8, 2, 4000, 1000, 128)):
    x = inputs(hq, hkv, seq, d, seed=11, peaky=True)
    q, k, v, do = upload(x, torch.bfloat16)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=torch.bfloat16)
    for j in range(seq // c):
        L.forward_chunk(q, k, v, j)
        n = ops.last_launch_count()
        assert n == 1, (hq, hkv, seq, c, d, j, n)
    torch.cuda.synchronize()
    o1, lse1 = L.o.clone(), L.lse.clone()
    L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    assert torch.equal(o1, L.o) and torch.equal(lse1, L.lse), (hq, hkv, seq, c, d, "rebuild not bitwise")
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    dk, dv = L.own_grads()
    for name, gpu in (("o", host(L.o)), ("dq", host(L.dq)), ("dk", host(dk)), ("dv", host(dv))):
        e = err(gpu, ref[name])
        assert e <= BF16_TOL, (hq, hkv, seq, c, d, name, e)
    lse = L.lse_full().cpu().numpy()
    assert np.abs(lse - ref["lse"]).max() <= 1e-3, (hq, hkv, seq, c, d, "lse")
print("dp split tail ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SECO_FWD_PAIR=pair, SECO_FWD_SLOTS="5")
    if nsplit:
        env["SECO_FWD_NSPLIT"] = nsplit
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "dp split tail ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_bf16_backward_pair_subprocess():
    """The CTA-pair backward (SECO_BWD_PAIR=1: seco_bwd3_sm100_kernel, clusters of two adjacent key
    tiles, S^T / dP^T / dV / dK as cta_group::2 MMAs with half of every B operand per CTA, dQ^T per
    CTA; an A/B path) against the oracle on small shapes (d = 64 included), in a child
    process because the switch is read once per process."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, ".")
from oracle import chunkwise as OC
from tests.gpu_util import BF16_TOL, err, host, inputs, upload
from paper_2505_16710_b200.step import ChunkedAttention
for (hq, hkv, seq, c, d) in ((8, 2, 512, 256, 128), (8, 2, 1024, 256, 128), (4, 1, 2048, 512, 128),
                             (8, 2, 1024, 256, 64)):
    x = inputs(hq, hkv, seq, d, seed=5, peaky=True)
    q, k, v, do = upload(x, torch.bfloat16)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=torch.bfloat16)
    L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    dk, dv = L.own_grads()
    for name, gpu in (("dq", host(L.dq)), ("dk", host(dk)), ("dv", host(dv))):
        e = err(gpu, ref[name])
        assert e <= BF16_TOL, (hq, hkv, seq, c, d, name, e)
print("pair bwd ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, SECO_BWD_PAIR="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "pair bwd ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
