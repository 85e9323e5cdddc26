"""Per-role clock64 timeline of seco_fwd_sm100_kernel (libseco_trace.so).  For CTA 0 prints per
KV step t, relative to the step's first event:
  Pb      MMA saw p_full(b)            Sb   MMA issued S_b(t+1)
  sf_b    softmax b saw s_full(t)      ld_b  row max done      ex_b  exp+STTM done
  kv      MMA saw V_t in smem          Pbb  MMA saw p_half(b,1)   h_b  softmax b arrived p_half(b,0)
usage: SECO_LIB_VARIANT=libseco_trace.so python tools/trace_fwd.py [j]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SECO_LIB_VARIANT", "libseco_trace.so")
import numpy as np
import torch
from paper_2505_16710_b200 import _lib
from paper_2505_16710_b200.step import ChunkedAttention
j = int(sys.argv[1]) if len(sys.argv) > 1 else 15
hq, hkv, d, S, c = 32, 8, 128, 32768, 2048
q = torch.randn(hq, S, d, device="cuda").bfloat16()
k = torch.randn(hkv, S, d, device="cuda").bfloat16()
v = torch.randn(hkv, S, d, device="cuda").bfloat16()
L = ChunkedAttention(hq, hkv, d, S, c)
for _ in range(3):
    L.forward_chunk(q, k, v, j)
torch.cuda.synchronize()
lib = _lib.load()
lib.seco_debug_fwd_trace_ptr.restype = ctypes.c_void_p
CT, SL, IT = 2, 24, 256
host = np.zeros((CT, SL, IT), dtype=np.uint64)
cudart = ctypes.CDLL("libcudart.so.12")
cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
assert cudart.cudaMemcpy(host.ctypes.data, lib.seco_debug_fwd_trace_ptr(), host.nbytes, 2) == 0
t = host.astype(np.int64)[0]
n = int((t[4] > 0).sum())
print("steps", n)
names = ["P0", "P1", "S0", "S1", "sf0", "sf1", "ld0", "ld1", "ex0", "ex1", "kv", "Pb0", "h0", "h1", "Pb1"]
for i in list(range(1, 8)) + list(range(n // 2, n // 2 + 4)):
    base = t[4, i]
    print(f"t={i:3d} " + " ".join(f"{nm}={t[s, i] - base:6d}" for s, nm in enumerate(names) if t[s, i]))
per = np.diff(t[4, :n])
print("mean period sf0->sf0:", per[5:].mean(), "cycles")
print("softmax0 s_full->exp done:", (t[8, 5:n] - t[4, 5:n]).mean(), " max-part:", (t[6, 5:n] - t[4, 5:n]).mean())
print("softmax1 s_full->exp done:", (t[9, 5:n] - t[5, 5:n]).mean())
print("MMA: P0 seen after ex0 by", (t[0, 5:n] - t[8, 5:n]).mean(), "; S0 issued after P0 by", (t[2, 5:n-1] - t[0, 5:n-1]).mean())
print("sf0(t+1) after S0(t) issue:", (t[4, 6:n] - t[2, 5:n-1]).mean())

print("MMA warp detail relative to sf0(t): loopend(t-1), kv(t), pre-P0(t), P0(t); producer K_t+?, V_t+? issue")
for i in range(5, 12):
    print("  t=%d" % i, int(t[15, i-1]-t[4, i]), int(t[10, i]-t[4, i]), int(t[18, i]-t[4, i]), int(t[0, i]-t[4, i]),
          "| prod K%d/V%d issued at" % (i, i), int(t[16, i]-t[4, i]), int(t[17, i]-t[4, i]))
