"""Plain SeCO step timing (default cfg3; argv[1] = cfg2 / cfg5 / cfg4p8 = one rank of cfg4 at 8 ranks) (no per-call events): CUDA events around R steps only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200.step import ChunkedAttention
from paper_2505_16710_b200.flops import seco_step_flops
CFG = {"cfg3": (32, 8, 128, 32768, 2048), "cfg2": (32, 8, 128, 8192, 1024), "cfg5": (32, 8, 128, 16384, 1024),
       "cfg4p8": (4, 1, 128, 131072, 4096), "cfg3p8": (4, 1, 128, 32768, 2048), "cfg3p4": (8, 2, 128, 32768, 2048)}
hq, hkv, d, S, c = CFG[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
q, do = (torch.randn(hq, S, d, device="cuda").bfloat16() for _ in range(2))
k, v = (torch.randn(hkv, S, d, device="cuda").bfloat16() for _ in range(2))
L = ChunkedAttention(hq, hkv, d, S, c)
for _ in range(3):
    L.seco_step(q, k, v, do)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = {8192: 100, 16384: 30, 32768: 10 if hq >= 16 else 40}.get(S, 2)
e0.record()
for _ in range(R):
    L.seco_step(q, k, v, do)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
print(f"{os.environ.get('SECO_LIB_VARIANT', 'libseco.so')}: {ms:.2f} ms/step, {seco_step_flops(hq, d, S, c) / ms / 1e9:.1f} TFLOP/s")
