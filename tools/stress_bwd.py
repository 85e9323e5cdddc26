"""Stress check of the default backward (v2): repeat SeCO steps on a few shapes and compare every
repeat with the oracle (a sporadic race would show as an occasional mismatch).
usage: python tools/stress_bwd.py [repeats]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from oracle import chunkwise as OC
from tests.gpu_util import BF16_TOL, err, host, inputs, upload
from paper_2505_16710_b200.step import ChunkedAttention

R = int(sys.argv[1]) if len(sys.argv) > 1 else 30
worst = 0.0
for (hq, hkv, seq, c, d) in ((8, 2, 1024, 256, 128), (16, 2, 640, 128, 128), (6, 3, 1536, 768, 64)):
    x = inputs(hq, hkv, seq, d, seed=11, peaky=True)
    q, k, v, do = upload(x, torch.bfloat16)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=torch.bfloat16)
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    for r in range(R):
        L.seco_step(q, k, v, do)
        torch.cuda.synchronize()
        dk, dv = L.own_grads()
        for name, gpu in (("dq", host(L.dq)), ("dk", host(dk)), ("dv", host(dv))):
            e = err(gpu, ref[name])
            worst = max(worst, e)
            assert e <= BF16_TOL, (hq, hkv, seq, c, d, r, name, e)
    print(f"shape {(hq, hkv, seq, c, d)}: {R} repeats ok", flush=True)
print(f"worst relative error {worst:.3e} (tolerance {BF16_TOL})")
