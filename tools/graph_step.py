"""SeCO step time, eager vs captured in a CUDA graph (ChunkedAttention.step replayed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200.step import ChunkedAttention
from paper_2505_16710_b200.flops import seco_step_flops
SHAPES = {"cfg2": (32, 8, 8192, 1024), "cfg3": (32, 8, 32768, 2048), "cfg5": (32, 8, 16384, 1024),
          "cfg3p8": (4, 1, 32768, 2048), "cfg3p4": (8, 2, 32768, 2048)}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg2", "cfg3"]
for nm in names:
    hq, hkv, S, c = SHAPES[nm]
    d = 128
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
    R = 10 if (hq >= 16 and S >= 32768) else 50
    for name, fn in (("eager", lambda: L.seco_step(q, k, v, do)), ("graph", g.replay),
                     ("eager", lambda: L.seco_step(q, k, v, do)), ("graph", g.replay)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(R):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        print(f"{nm} hq={hq} S={S} c={c} {name}: {ms:.3f} ms/step, {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
