"""SeCO step time, eager vs captured in a CUDA graph (ChunkedAttention.step replayed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200.step import ChunkedAttention
from paper_2505_16710_b200.flops import seco_step_flops
for (S, c) in ((8192, 1024), (32768, 2048)):
    hq, hkv, d = 32, 8, 128
    q, do = (torch.randn(hq, S, d, device="cuda").bfloat16() for _ in range(2))
    k, v = (torch.randn(hkv, S, d, device="cuda").bfloat16() for _ in range(2))
    L = ChunkedAttention(hq, hkv, d, S, c)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            L.seco_step(q, k, v, do, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        L.seco_step(q, k, v, do, stream=s)
    torch.cuda.synchronize()
    fl = seco_step_flops(hq, d, S, c)
    for name, fn in (("eager", lambda: L.seco_step(q, k, v, do)), ("graph", g.replay)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"S={S} c={c} {name}: {ms:.3f} ms/step, {fl / ms / 1e9:.1f} TFLOP/s")
