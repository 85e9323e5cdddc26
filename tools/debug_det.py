"""Debug helper: run the deterministic-mode chunk calls one by one with a sync after each."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200.step import ChunkedAttention
hq, hkv, seq, c = [int(x) for x in sys.argv[1:5]]
q = torch.randn(hq, seq, 128, device="cuda").bfloat16()
k = torch.randn(hkv, seq, 128, device="cuda").bfloat16()
v = torch.randn(hkv, seq, 128, device="cuda").bfloat16()
do = torch.randn(hq, seq, 128, device="cuda").bfloat16()
L = ChunkedAttention(hq, hkv, 128, seq, c, deterministic=True)
L.dkv.zero_()
for j in reversed(range(seq // c)):
    L.forward_chunk(q, k, v, j); torch.cuda.synchronize(); print("fwd", j, flush=True)
    L.backward_chunk(q, k, v, do, j); torch.cuda.synchronize(); print("bwd", j, flush=True)
print("ok")
