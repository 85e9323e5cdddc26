"""clock64 timeline of the experimental backward v2 (seco_bwd2_sm100_kernel, SECO_BWD_V2=1; needs
libseco_trace.so from `python -m paper_2505_16710_b200.build --trace`).  One chunk backward at cfg3;
per iteration i, event times in SM cycles relative to the compute warps seeing s_full(i).
usage: SECO_BWD_V2=1 SECO_LIB_VARIANT=libseco_trace.so python tools/trace_bwd2.py [j]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SECO_LIB_VARIANT", "libseco_trace.so")
os.environ.setdefault("SECO_BWD_V2", "1")
import numpy as np
import torch

from paper_2505_16710_b200 import _lib
from paper_2505_16710_b200.step import ChunkedAttention

j = int(sys.argv[1]) if len(sys.argv) > 1 else 15
hq, hkv, d, S, c = 32, 8, 128, 32768, 2048
torch.manual_seed(0)
q, do = (torch.randn(hq, S, d, device="cuda").bfloat16() for _ in range(2))
k, v = (torch.randn(hkv, S, d, device="cuda").bfloat16() for _ in range(2))
L = ChunkedAttention(hq, hkv, d, S, c)
L.dkv.zero_()
for rep in range(3):
    L.forward_chunk(q, k, v, j)
    L.backward_chunk(q, k, v, do, j)
torch.cuda.synchronize()
lib = _lib.load()
lib.seco_debug_trace_ptr.restype = ctypes.c_void_p
ptr = lib.seco_debug_trace_ptr()
CT, SL, IT = 4, 20, 128
host = np.zeros((CT, SL, IT), dtype=np.uint64)
cudart = ctypes.CDLL("libcudart.so.12")
cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
assert cudart.cudaMemcpy(host.ctypes.data, ptr, host.nbytes, 2) == 0
t = host.astype(np.int64)
names = {0: "Q(i) ld", 1: "dO(i) ld", 2: "S(i+1) iss", 3: "MMA ds(i)", 4: "dQ(i) iss", 5: "MMA dqE(i)",
         6: "dP(i+1) iss", 7: "dV(i+1) iss", 8: "A start", 9: "A end(p_rdy)", 10: "B start(dp)",
         11: "B end WG0", 12: "B end WG1", 13: "drain dqF", 14: "drain dqE", 15: "drain staged",
         16: "red c0", 17: "red c3"}
for cta in range(2):
    n = int((t[cta, 8] > 0).sum())
    per = np.diff(t[cta, 8, :n])
    print(f"CTA {cta}: {n} iterations, mean period (A start -> A start) {per.mean():.0f} cycles, "
          f"median {np.median(per):.0f}")
    print("   i  " + " ".join(f"{names[s]:>12s}" for s in sorted(names)))
    for i in range(2, min(n - 1, 10)):
        b = t[cta, 8, i]
        print(f"  {i:3d} " + " ".join(f"{(t[cta, s, i] - b) if t[cta, s, i] else 0:12d}" for s in sorted(names)))
