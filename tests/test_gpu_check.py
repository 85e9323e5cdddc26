"""Bounds-checked build (libseco_check.so, -DSECO_CHECK=1; the stand-in for compute-sanitizer,
which this GPU pool does not offer -- SURVEY §5).  Every kernel asserts its shared- and
tensor-memory operand ranges, tensor-memory lanes per warp, mbarrier alignment, TMA box
coordinates and global store indices (paper_2505_16710_b200/csrc/common.cuh).  The parity
workloads below run through the check build in a child process (the library variant is chosen
when the binding loads); every call must leave the check word at 0 and still match the oracle.
A self-test kernel with one failing check proves that failures are reported."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import chunkwise as OC
from oracle import sampler as OS
from tests.gpu_util import BF16_TOL, FP32_TOL, err, host, inputs, upload
from paper_2505_16710_b200 import _lib, ops
from paper_2505_16710_b200.step import ChunkedAttention
lib = _lib.load()
assert lib.seco_debug_check_enabled() == 1, "not the check build"
lib.seco_debug_check_word()                               # clear
lib.seco_debug_check_selftest(None)
w = lib.seco_debug_check_word()
assert (w & 0xFFFFFFFF) == 999 and (w >> 32) == 1, hex(w)
assert lib.seco_debug_check_word() == 0                  # read clears

def clean(what):
    w = lib.seco_debug_check_word()
    assert w == 0, (what, "check id", w & 0xFFFFFFFF, "count", w >> 32)

cases = [(8, 2, 512, 128, 128, False), (3, 1, 768, 128, 384, False), (8, 2, 512, 64, 128, False),
         (6, 3, 1536, 128, 768, False), (8, 2, 4096, 128, 1024, False), (4, 1, 1024, 128, 256, True),
         (4, 1, 600, 128, 200, False), (8, 2, 4000, 128, 1000, False), (4, 1, 1000, 128, 250, True),
         (4, 1, 512, 96, 256, False), (8, 2, 600, 32, 200, False)]
for hq, hkv, seq, d, c, det in cases:
    x = inputs(hq, hkv, seq, d, seed=9, peaky=True)
    q, k, v, do = upload(x, torch.bfloat16)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=torch.bfloat16, own_copies=True, deterministic=det)
    L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    clean((hq, hkv, seq, d, c, det))
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    for name, got in (("o", L.o), ("dq", L.dq), ("dk", L.dk), ("dv", L.dv)):
        assert err(host(got), ref[name]) <= BF16_TOL, (hq, hkv, seq, d, c, name)
    r = L.spaco_step(q, k, v, do, max(1, seq // c // 2), 3, cap=2.0, mode=OS.BERNOULLI)
    torch.cuda.synchronize()
    clean(("spaco", hq, hkv, seq, d, c))
# fp32 debug path
x = inputs(6, 2, 96, 20, seed=2, dtype=torch.float32)
q, k, v, do = upload(x, torch.float32)
L = ChunkedAttention(6, 2, 20, 96, 32, dtype=torch.float32, own_copies=True)
L.seco_step(q, k, v, do)
torch.cuda.synchronize()
clean("fp32")
ref = OC.seco_step(x.q, x.k, x.v, x.do, [32] * 3)
assert err(host(L.dq), ref["dq"]) <= FP32_TOL
# LoRA gradients: tensor-core and CUDA-core kernels
for rows, n_in, n_out, r, dt in ((2048, 4096, 1024, 8, torch.bfloat16), (300, 1024, 512, 16, torch.bfloat16),
                                 (129, 72, 40, 4, torch.float32)):
    xx = torch.randn(rows, n_in, device="cuda").to(dt)
    dy = torch.randn(rows, n_out, device="cuda").to(dt)
    a = torch.randn(n_in, r, device="cuda").to(dt)
    b = torch.randn(r, n_out, device="cuda").to(dt)
    da = torch.zeros(n_in, r, device="cuda"); db = torch.zeros(r, n_out, device="cuda")
    u = torch.empty(rows, r, device="cuda")
    sh = ops.lora_shape(xx, dy, r)
    ws = torch.empty(ops.seco_lora_workspace_size(sh) // 4, device="cuda")
    ops.seco_lora_grad(sh, xx, dy, a, b, da, db, u, ws)
    torch.cuda.synchronize()
    clean(("lora", rows, n_in, n_out, r))
print("check build clean")
'''


@pytest.mark.parametrize("extra", [{"SECO_BWD_V2": "1"}, {"SECO_BWD_V2": "0"},
                                   # the DP + split-tail forward (5 pretended work slots) and its
                                   # in-kernel merge, CTA-pair and single-CTA forward
                                   {"SECO_FWD_SLOTS": "5", "SECO_FWD_PAIR": "1"},
                                   {"SECO_FWD_SLOTS": "5", "SECO_FWD_PAIR": "0"}])
def test_check_build_reports_nothing_on_parity_workloads(extra):
    lib = os.path.join(ROOT, "paper_2505_16710_b200", "libseco_check.so")
    assert os.path.exists(lib), "build it with python -m paper_2505_16710_b200.build --check (__graft_entry__.build)"
    env = dict(os.environ, SECO_LIB_VARIANT="libseco_check.so", **extra)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "check build clean" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
