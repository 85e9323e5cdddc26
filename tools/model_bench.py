"""Step time of the L-layer RoPE + LoRA stack (paper_2505_16710_b200/model.py) at a LLaMA-3-8B
layer shape (hidden 4096, 32 q / 8 kv heads, d = 128, LoRA r = 8 on q, k, v, o) for SeCO and
SpaCO (PAPER mode, t of k, cap 2), with synthetic random-init weights.  Reports ms per step,
tokens/s and the share of the step spent in libseco.so attention calls (CUDA events around
them on the launching stream).
usage: python tools/model_bench.py [L] [seq] [chunk] [t]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2505_16710_b200 import model as M
from paper_2505_16710_b200 import ops

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
C = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
T = int(sys.argv[4]) if len(sys.argv) > 4 else 4
HD, HQ, HKV, D, R = 4096, 32, 8, 128, 8

torch.manual_seed(0)
dev = torch.device("cuda")
dims = {"q": (HD, HQ * D), "k": (HD, HKV * D), "v": (HD, HKV * D), "o": (HQ * D, HD)}
layers = []
for _ in range(L):
    p = {}
    for n, (i, o) in dims.items():
        p["W" + n] = torch.randn(i, o, device=dev) / i ** 0.5
        p["A" + n] = torch.randn(i, R, device=dev) / i ** 0.5
        p["B" + n] = torch.randn(R, o, device=dev) / R ** 0.5 * 0.1
    layers.append(p)
stack = M.ChunkedLoRAStack(layers, HQ, HKV, D, S, C, dtype=torch.bfloat16)
del layers
x0 = torch.randn(S, HD, device=dev).bfloat16()
G = torch.randn(S, HD, device=dev)

# attention-call timing: wrap the two ops with events on the current stream
att_events = []
_fwd, _bwd = ops.seco_chunk_forward, ops.seco_chunk_backward


def _timed(fn):
    def w(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*a, **k)
        e1.record()
        att_events.append((e0, e1))
    return w


M.ops.seco_chunk_forward = _timed(_fwd)
M.ops.seco_chunk_backward = _timed(_bwd)

k = S // C
idx, gamma, s = ops.spaco_sample_and_scale(k, T, 0, 2.0)
out = {"layers": L, "seq": S, "chunk": C, "hidden": HD, "lora_rank": R, "data": "synthetic, random init"}
for name, sel, g, sc in (("seco", None, 1.0, 1.0), (f"spaco_t{T}", idx, gamma, s)):
    for _ in range(2):
        stack.step(x0, G, sel, g, sc)
    torch.cuda.synchronize()
    att_events.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 3
    e0.record()
    for _ in range(steps):
        stack.step(x0, G, sel, g, sc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    att = sum(a.elapsed_time(b) for a, b in att_events) / steps
    out[name] = {"ms_per_step": ms, "tokens_per_s": S / (ms * 1e-3), "attention_ms": att,
                 "attention_share": att / ms, "selected": sel}
print(json.dumps(out))
