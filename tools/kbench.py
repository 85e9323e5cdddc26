"""Per-chunk kernel timing at the bench shape: CUDA events around R back-to-back calls
of seco_chunk_forward(j) / seco_chunk_backward(j), for selected j.  Prints TFLOP/s
(algorithmic) per call type and j.  Library variant via SECO_LIB_VARIANT.
usage: python tools/kbench.py [cfg3|cfg2] [j,j,...] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_16710_b200 import flops as FL
from paper_2505_16710_b200.step import ChunkedAttention

CFG = {"cfg3": (32, 8, 128, 32768, 2048), "cfg2": (32, 8, 128, 8192, 1024), "cfg3p8": (4, 1, 128, 32768, 2048)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
hq, hkv, d, S, c = CFG[name]
k = S // c
js = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 3, 7, 11, 15]
R = int(sys.argv[3]) if len(sys.argv) > 3 else 10
try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

    def _sm_mhz():
        return pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM)
except Exception:                            # no NVML: report 0
    def _sm_mhz():
        return 0
torch.manual_seed(0)
q = torch.randn(hq, S, d, device="cuda").bfloat16()
kc = torch.randn(hkv, S, d, device="cuda").bfloat16()
vc = torch.randn(hkv, S, d, device="cuda").bfloat16()
do = torch.randn(hq, S, d, device="cuda").bfloat16()
L = ChunkedAttention(hq, hkv, d, S, c)
L.dkv.zero_()
for j in range(k):
    L.forward_chunk(q, kc, vc, j)
torch.cuda.synchronize()
tot_f = tot_b = 0.0
for j in js:
    for kind in ("fwd", "bwd"):
        for _ in range(2):
            (L.forward_chunk(q, kc, vc, j) if kind == "fwd" else L.backward_chunk(q, kc, vc, do, j))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(R):
            (L.forward_chunk(q, kc, vc, j) if kind == "fwd" else L.backward_chunk(q, kc, vc, do, j))
        e1.record()
        mhz = _sm_mhz()                     # sampled while the queued calls still run
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        fl = FL.fwd_flops(hq, d, c, j) if kind == "fwd" else FL.bwd_flops(hq, d, c, j)
        print(f"{name} j={j:2d} {kind}: {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s  sm {mhz} MHz"
              f"  {fl / ms / 1e9 / max(mhz, 1) * 1e3:6.1f} TFLOP/s per GHz", flush=True)
