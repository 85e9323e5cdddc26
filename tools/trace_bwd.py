"""Per-role clock64 timeline of seco_bwd_sm100_kernel (needs libseco_trace.so, built with
`python -m paper_2505_16710_b200.build --trace`).  Runs one chunk backward at the bench
shape and prints, for the first traced CTAs, per-iteration intervals in SM cycles:
  period   MMA: ds_ready(i) -> ds_ready(i+1)
  s_lat    MMA got ds_ready(i-1) (issues S/dP(i)) -> compute sees s_full(i)
  comp     compute: s_full(i) -> arrive ds_ready(i)   (WG0; WG1 in brackets)
  dqwait   MMA: q_full(i+1) ok -> dq_empty(i) ok      (includes dV/dK issue)
  drain    drain: dq_full(i) -> bulk reduce issued
usage: SECO_LIB_VARIANT=libseco_trace.so python tools/trace_bwd.py [j] [cfg]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SECO_LIB_VARIANT", "libseco_trace.so")
import numpy as np
import torch

from paper_2505_16710_b200 import _lib
from paper_2505_16710_b200.step import ChunkedAttention

j = int(sys.argv[1]) if len(sys.argv) > 1 else 15
hq, hkv, d, S, c = 32, 8, 128, 32768, 2048
torch.manual_seed(0)
q = torch.randn(hq, S, d, device="cuda").bfloat16()
k = torch.randn(hkv, S, d, device="cuda").bfloat16()
v = torch.randn(hkv, S, d, device="cuda").bfloat16()
do = torch.randn(hq, S, d, device="cuda").bfloat16()
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
rc = cudart.cudaMemcpy(host.ctypes.data, ptr, host.nbytes, 2)
assert rc == 0, ("cudaMemcpy", rc)
t = host.astype(np.int64)
for cta in range(2):
    n = int((t[cta, 1] > 0).sum())
    print(f"CTA {cta}: {n} iterations")
    for i in range(1, min(n, 12)):
        period = t[cta, 1, i] - t[cta, 1, i - 1]
        kvq = t[cta, 2, i] - t[cta, 1, i]          # dV dK dQ^T issue (blocking issue)
        dqw = t[cta, 3, i] - t[cta, 2, i] if t[cta, 3, i] else 0     # dP(i+1) issue + wait dq_empty
        s_lat = t[cta, 5, i] - t[cta, 4, i - 1]     # S(i) issued -> compute sees s_full
        comp = t[cta, 6, i] - t[cta, 5, i]
        drain = t[cta, 8, i] - t[cta, 7, i]
        print(f"  i={i:3d} period={period:6d} issue_kvq={kvq:6d} dP+dqwait={dqw:6d} s_lat={s_lat:6d} "
              f"comp={comp:6d} drain={drain:6d}")
    for i in range(2, 6):
        b = t[cta, 5, i]
        print(f"    compute detail i={i}: r0_ld={t[cta,10,i]-b} r0_math={t[cta,11,i]-b} r1_ld={t[cta,12,i]-b} "
              f"r1_math={t[cta,13,i]-b} arrive={t[cta,6,i]-b}")
    print("    timeline rel. to compute s_full(i): ds0 MMAseen_ds0 ds1 MMAseen_ds1 dQcommit dPissued "
          "dq_full_seen dq_empty_arr MMAseen_dq_empty S_issued s_full(i+1)")
    for i in range(2, 8):
        b = t[cta, 5, i]
        ds0 = t[cta, 13, i] if False else 0
        vals = [t[cta, 11, i], t[cta, 1, i], t[cta, 6, i], t[cta, 16, i], t[cta, 2, i], t[cta, 17, i],
                t[cta, 14, i], t[cta, 15, i], t[cta, 3, i], t[cta, 4, i], t[cta, 5, i + 1]]
        print("     i=%d " % i + " ".join("%6d" % (x - b) for x in vals))
    print("    drain rel. to s_full(i): stg1(i-1)->reduce issued, dO half read(i-1), -, Q half read(i-1)")
    for i in range(2, 8):
        b = t[cta, 5, i]
        print("     i=%d %6d %6d %6d %6d | dO(i+1) load issued %6d, Q(i+1) issued %6d, dP(i+1) issued %6d" % (
            i, t[cta, 7, i - 1] - b, t[cta, 18, i - 1] - b, 0, t[cta, 8, i - 1] - b,
            t[cta, 19, i + 1] - b, t[cta, 0, i + 1] - b, t[cta, 17, i] - b))
    per = np.diff(t[cta, 1, :n])
    print(f"  mean period {per.mean():.0f} cycles over {n} iterations (128 query rows each); MMA ideal 2560")
