"""Per-rank step time of head-sharded cfg3: N ranks each own Hkv/N kv heads and
their q heads.  Runs the per-rank shape on one GPU and compares with the N = 1 step / N
(the scaling efficiency the driver will see, up to NCCL barrier costs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200.step import ChunkedAttention

def step_ms(hq, hkv, S=32768, c=2048, d=128, reps=5):
    q, do = (torch.randn(hq, S, d, device="cuda").bfloat16() for _ in range(2))
    k, v = (torch.randn(hkv, S, d, device="cuda").bfloat16() for _ in range(2))
    L = ChunkedAttention(hq, hkv, d, S, c)
    for _ in range(2):
        L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.seco_step(q, k, v, do)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

t1 = step_ms(32, 8)
print(f"N=1: {t1:.2f} ms")
for n in (2, 4, 8):
    tn = step_ms(32 // n, 8 // n)
    print(f"N={n}: per-rank {tn:.2f} ms, ideal {t1 / n:.2f} ms, efficiency {t1 / n / tn:.2f}")
