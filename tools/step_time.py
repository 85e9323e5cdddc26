"""Plain SeCO step timing at cfg3 (no per-call events): CUDA events around R steps only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200.step import ChunkedAttention
from paper_2505_16710_b200.flops import seco_step_flops
hq, hkv, d, S, c = 32, 8, 128, 32768, 2048
q, do = (torch.randn(hq, S, d, device="cuda").bfloat16() for _ in range(2))
k, v = (torch.randn(hkv, S, d, device="cuda").bfloat16() for _ in range(2))
L = ChunkedAttention(hq, hkv, d, S, c)
for _ in range(3):
    L.seco_step(q, k, v, do)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 10
e0.record()
for _ in range(R):
    L.seco_step(q, k, v, do)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
print(f"{os.environ.get('SECO_LIB_VARIANT', 'libseco.so')}: {ms:.2f} ms/step, {seco_step_flops(hq, d, S, c) / ms / 1e9:.1f} TFLOP/s")
