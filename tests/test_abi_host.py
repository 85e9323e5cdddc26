"""CPU-side checks of the C ABI (no GPU needed): libseco.so loads and exports every
symbol include/seco.h declares; the host sampler agrees bit for bit with the
oracle's independent implementation; argument validation rejects bad calls
before any CUDA work; FLOP accounting matches brute-force pair counting."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import sampler as OS
from paper_2505_16710_b200 import _lib, flops
from paper_2505_16710_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def _declared_functions():
    with open(os.path.join(ROOT, "include", "seco.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(seco_\w+|spaco_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    declared = _declared_functions()
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_status_strings(lib):
    for code, name in enumerate(["SECO_OK", "SECO_ERR_ARG", "SECO_ERR_UNSUPPORTED", "SECO_ERR_CUDA"]):
        assert lib.seco_status_string(code).decode() == name


def _c_sample(k, t, seed, cap, mode):
    from paper_2505_16710_b200 import ops
    return ops.spaco_sample_and_scale(k, t, seed, cap, mode)


@pytest.mark.parametrize("mode", [_lib.SPACO_PAPER, _lib.SPACO_HT, _lib.SPACO_BERNOULLI])
def test_sampler_bit_exact_vs_oracle(lib, mode):
    rng = np.random.default_rng(0)
    for _ in range(300):
        k = int(rng.integers(2, 70))
        t = int(rng.integers(2 if mode == _lib.SPACO_HT else 1, k + 1))
        seed = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        cap = float(rng.choice([0.0, 2.0, 1.5]))
        idx, g, s = _c_sample(k, t, seed, cap, mode)
        oidx, og, os_ = OS.sample_and_scale(k, t, seed, cap, mode)
        assert idx == oidx
        assert np.float32(g) == np.float32(og) and np.float32(s) == np.float32(os_)


def test_sampler_kats_golden(lib):
    path = os.path.join(ROOT, "tests", "golden", "sampler_kats.txt")
    with open(path) as f:
        lines = f.readlines()
    for ln in lines:
        if not ln.strip() or ln.startswith("#"):
            continue
        mode, k, t, seed, want = ln.split()
        m = _lib.SPACO_PAPER if mode == "T_OF_K" else _lib.SPACO_BERNOULLI
        idx, _, _ = _c_sample(int(k), int(t), int(seed), 0.0, m)
        assert idx == [int(x) for x in want.split(",")]


def test_sampler_errors(lib):
    from paper_2505_16710_b200 import ops
    for k, t, mode in ((4, 0, 0), (4, 5, 0), (4, 1, _lib.SPACO_HT), (0, 0, 0), (4, 2, 7)):
        with pytest.raises(_lib.SecoError):
            ops.spaco_sample_and_scale(k, t, 0, 2.0, mode)


def _shape(**kw):
    d = dict(hq=32, hkv=8, d=128, chunk=256, num_chunks=4, softmax_scale=0.0, dtype=0,
             q_head_stride=1024 * 128, q_row_stride=128, kv_head_stride=1024 * 128, kv_row_stride=128, flags=0)
    d.update(kw)
    return _lib.SecoShape(*[d[f] for f, _ in _lib.SecoShape._fields_])


@pytest.mark.parametrize("kw,j,code", [
    (dict(), -1, _lib.SECO_ERR_ARG),
    (dict(), 4, _lib.SECO_ERR_ARG),
    (dict(hkv=5), 0, _lib.SECO_ERR_ARG),
    (dict(chunk=0), 0, _lib.SECO_ERR_ARG),                                   # empty chunk
    (dict(num_chunks=0), 0, _lib.SECO_ERR_ARG),                              # empty sequence
    (dict(hq=0), 0, _lib.SECO_ERR_ARG),                                      # no heads
    (dict(d=0), 0, _lib.SECO_ERR_ARG),                                       # empty head dim
    (dict(d=80, q_row_stride=80, kv_row_stride=80, q_head_stride=1024 * 80, kv_head_stride=1024 * 80), 0,
     _lib.SECO_ERR_UNSUPPORTED),                                              # bf16 needs d % 32 == 0
    (dict(q_row_stride=100), 0, _lib.SECO_ERR_ARG),
    (dict(dtype=1, d=300, q_row_stride=300, kv_row_stride=300, q_head_stride=1024 * 300,
          kv_head_stride=1024 * 300), 0, _lib.SECO_ERR_UNSUPPORTED),
    (dict(dtype=5), 0, _lib.SECO_ERR_ARG),
    (dict(q_head_stride=128 * 128), 0, _lib.SECO_ERR_ARG),                  # heads overlap rows
    (dict(q_head_stride=128, q_row_stride=16 * 128), 0, _lib.SECO_ERR_ARG),  # interleaved, too few heads/row
    (dict(kv_head_stride=256 * 128), 0, _lib.SECO_ERR_ARG),                 # cache heads overlap
    (dict(flags=4), 0, _lib.SECO_ERR_ARG),                                   # unknown flag bit
])
def test_argument_validation(lib, kw, j, code):
    s = _shape(**kw)
    dummy = ctypes.c_void_p(1 << 20)  # never dereferenced: validation happens before any launch
    r = lib.seco_chunk_forward(ctypes.byref(s), j, dummy, dummy, dummy, dummy, dummy, None, 0, None)
    assert r == code, lib.seco_last_error()
    r = lib.seco_chunk_backward(ctypes.byref(s), j, dummy, dummy, dummy, dummy, dummy, dummy, 1.0, 1.0,
                                dummy, dummy, None, None, dummy, 1 << 30, None)
    assert r == code, lib.seco_last_error()
    r = lib.spaco_chunk_skip(ctypes.byref(s), j, dummy, dummy, None, None, None)
    assert r == code, lib.seco_last_error()


def test_null_pointers_rejected(lib):
    s = _shape()
    r = lib.seco_chunk_forward(ctypes.byref(s), 0, None, None, None, None, None, None, 0, None)
    assert r == _lib.SECO_ERR_ARG
    dummy = ctypes.c_void_p(1 << 20)
    r = lib.seco_chunk_backward(ctypes.byref(s), 0, dummy, dummy, dummy, dummy, dummy, dummy, 1.0, 1.0,
                                dummy, dummy, None, None, dummy, 16, None)   # workspace too small
    assert r == _lib.SECO_ERR_ARG
    assert lib.spaco_chunk_skip(ctypes.byref(s), 0, None, dummy, None, None, None) == _lib.SECO_ERR_ARG
    assert lib.spaco_chunk_skip(ctypes.byref(s), 0, dummy, None, None, None, None) == _lib.SECO_ERR_ARG
    misaligned = ctypes.c_void_p((1 << 20) + 4)
    assert lib.spaco_chunk_skip(ctypes.byref(s), 0, misaligned, dummy, None, None, None) == _lib.SECO_ERR_ARG


def test_workspace_size(lib):
    s = _shape()
    assert lib.seco_workspace_size(ctypes.byref(s)) >= 4 * (32 * 256 * 128 + 32 * 256)


def test_flops_pairs_brute_force():
    for c, k in ((16, 4), (7, 5), (128, 3)):
        S = c * k
        tot = 0
        for j in range(k):
            brute = sum(1 for p in range(j * c, (j + 1) * c) for q in range(S) if q <= p)
            assert flops.pairs(c, j) == brute
            tot += brute
        assert tot == S * (S + 1) // 2
    # SeCO = 4.5 F ; SpaCO with all chunks = SeCO
    hq, d, S, c = 32, 128, 32768, 2048
    F = flops.total_fwd(hq, d, S)
    assert abs(flops.seco_step_flops(hq, d, S, c) / F - 4.5) < 1e-12
    assert abs(F - 8.796e12) / 8.796e12 < 1e-3     # cfg3 F = 8.796 TF
    assert flops.spaco_step_flops(hq, d, S, c, range(16)) == flops.seco_step_flops(hq, d, S, c)


def test_workspace_independent_of_sequence_length(lib):
    """SeCO's memory claim at this level ('reduces the memory requirements for
    storing forward activations by a factor of k'): the per-call working set of the chunk
    kernels depends on the chunk size c, not on the number of chunks k."""
    sizes = set()
    for k in (1, 4, 16, 64):
        s = _shape(num_chunks=k, q_head_stride=k * 256 * 128, kv_head_stride=k * 256 * 128)
        sizes.add(lib.seco_workspace_size(ctypes.byref(s)))
    assert len(sizes) == 1
    s2 = _shape(chunk=512, q_head_stride=4 * 512 * 128, kv_head_stride=4 * 512 * 128)
    assert lib.seco_workspace_size(ctypes.byref(s2)) == 2 * sizes.pop()


@pytest.mark.parametrize("kw,code", [
    (dict(rank=3), _lib.SECO_ERR_UNSUPPORTED),
    (dict(rows=0), _lib.SECO_ERR_ARG),
    (dict(ldx=10), _lib.SECO_ERR_ARG),
    (dict(dtype=7), _lib.SECO_ERR_ARG),
])
def test_lora_argument_validation(lib, kw, code):
    d = dict(rows=64, n_in=32, n_out=48, rank=8, dtype=0, ldx=32, ldy=48, flags=0)
    d.update(kw)
    s = _lib.LoraShape(*[d[f] for f, _ in _lib.LoraShape._fields_])
    dummy = ctypes.c_void_p(1 << 20)
    r = lib.seco_lora_grad(ctypes.byref(s), dummy, dummy, dummy, dummy, dummy, dummy, dummy, dummy, 1 << 30, None)
    assert r == code


def _bwd_work_list(lib, c, j, hkv, G, sms):
    """Decode the backward work list exactly as seco_bwd_sm100_kernel does (blockIdx ->
    unit U, piece of f) and return, per unit, the query-iteration ranges of its pieces."""
    out = (ctypes.c_int32 * 4)()
    grid = lib.seco_debug_bwd_schedule(c, j, hkv, G, sms, out)
    n0, n1, f1, f2 = list(out)
    nqt, ntiles = -(-c // 128), -(-(j + 1) * c // 128)        # ceil: ragged chunks (c % 128 != 0)
    ranges = {}
    for bid in range(grid):
        if bid < n0:
            U, piece, f = bid, 0, 1
        elif bid < n0 + n1 * f1:
            r = bid - n0
            U, piece, f = n0 + r // f1, r % f1, f1
        else:
            r = bid - n0 - n1 * f1
            U, piece, f = n0 + n1 + r // f2, r % f2, f2
        u = U // hkv
        rel = u * 128 - j * c
        n_all = G * (nqt - (rel // 128 if rel > 0 else 0))
        ranges.setdefault(U, []).append((piece * n_all // f, (piece + 1) * n_all // f, n_all))
    return grid, ntiles * hkv, ranges


@pytest.mark.parametrize("c,k,hkv,G", [(2048, 16, 8, 4), (1024, 8, 8, 4), (4096, 32, 1, 4), (1024, 16, 2, 4),
                                       (256, 5, 3, 2), (128, 4, 1, 1),
                                       (200, 3, 2, 2), (1000, 4, 8, 4), (100, 4, 1, 4)])   # ragged chunks
def test_bwd_work_list_covers_every_block_once(lib, c, k, hkv, G):
    """The balanced backward work list (whole units, then f1- / f2-way query splits for the
    last wave): every (key tile, kv head) unit appears, its pieces tile [0, n_all) exactly,
    and units come in ascending key-tile order (longest work first)."""
    for j in sorted({0, 1, k // 2, k - 1}):
        grid, n_units, ranges = _bwd_work_list(lib, c, j, hkv, G, 148)
        assert sorted(ranges) == list(range(n_units))
        for U, rs in ranges.items():
            n_all = rs[0][2]
            assert rs[0][0] == 0 and rs[-1][1] == n_all
            for (a0, a1, _), (b0, b1, _) in zip(rs, rs[1:]):
                assert a1 == b0 and a0 <= a1
        assert grid >= n_units


def test_normal_build_has_no_checks(lib):
    """The product libseco.so is not the bounds-checked build (tests/test_gpu_check.py runs that)."""
    assert lib.seco_debug_check_enabled() == 0


def test_binding_refuses_host_tensors():
    """The binding passes device pointers only: a host tensor is refused before the library
    is called (it would otherwise fault on the device at the next synchronisation)."""
    import torch
    from paper_2505_16710_b200 import ops
    q = torch.zeros(2, 256, 128, dtype=torch.bfloat16)
    k = torch.zeros(1, 256, 128, dtype=torch.bfloat16)
    shape = ops.make_shape(q, k, 128)
    lse = torch.zeros(2, 128)
    with pytest.raises(ValueError, match="CUDA tensors"):
        ops.seco_chunk_forward(shape, 0, q[:, :128], k, k, q[:, :128], lse)


def _fwd_plan(lib, hq, hkv, c, k, j, sms=0):
    s = _shape(hq=hq, hkv=hkv, chunk=c, num_chunks=k, q_head_stride=k * c * 128, kv_head_stride=k * c * 128)
    out = (ctypes.c_int32 * 5)()
    grid = lib.seco_debug_fwd_schedule(ctypes.byref(s), j, sms, out)
    return grid, dict(zip(("pair", "units", "n_full", "nsplit", "merge"), list(out)))


def test_forward_split_plan_policy(lib):
    """The forward's work plan (seco_debug_fwd_schedule, host only): cfg3 runs the
    CTA-pair kernel on 128 pair-units, whole for j < 10 and DP + split tail from j = 10 (74
    whole units, then 4 key-range pieces of the other 54, merged in-kernel); the 8-rank per-rank
    shape (4 q / 1 kv heads) is a sub-wave grid, split into pieces merged by the combine kernel;
    chunk 0 never splits; every plan's grid covers its work items exactly."""
    for j in range(16):
        grid, p = _fwd_plan(lib, 32, 8, 2048, 16, j)
        assert p["pair"] == 1 and p["units"] == 128
        if j < 10:
            assert p["nsplit"] == 1 and p["n_full"] == 128 and p["merge"] == 0 and grid == 256
        else:
            assert p == dict(pair=1, units=128, n_full=74, nsplit=4, merge=1)
            assert grid == 2 * (74 + 54 * 4)
    for j in range(16):
        grid, p = _fwd_plan(lib, 4, 1, 2048, 16, j)
        assert p["pair"] == 0 and p["units"] == 32 and p["n_full"] in (0, 32)
        if j == 0:
            assert p["nsplit"] == 1 and grid == 32
        else:
            assert p["nsplit"] > 1 and p["merge"] == 0 and p["n_full"] == 0 and grid == 32 * p["nsplit"]
            assert (j * 2048 // 128 + 1) >= 8 * p["nsplit"]          # >= 8 K/V tiles per piece
    # ragged chunks: ceil(c / 128) query tiles per chunk
    grid, p = _fwd_plan(lib, 8, 2, 1000, 4, 3)
    assert p["units"] == 8 * 4 and p["n_full"] == 0 and grid == 32 * p["nsplit"]
    # a pretended 5-SM GPU: multi-wave grids at small shapes take the DP + tail form
    grid, p = _fwd_plan(lib, 8, 2, 1024, 4, 3, sms=5)
    assert p["merge"] == 1 and p["n_full"] == 30 and grid == p["n_full"] + (p["units"] - p["n_full"]) * p["nsplit"]
    assert lib.seco_debug_fwd_schedule(ctypes.byref(_shape()), 9, 0, (ctypes.c_int32 * 5)()) == -1   # j out of range
