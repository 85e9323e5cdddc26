"""Per-phase clock64 trace of lora_fused_kernel (CTA 0) from the SECO_LORA_TRACE build:
    SECO_VARIANT=ltrace SECO_DEFINES=-DSECO_LORA_TRACE=1 python -m paper_2505_16710_b200.build
    SECO_LIB_VARIANT=libseco_ltrace.so python tools/trace_lora.py [rows n_in n_out r]
Points per block: 0 full-wait done, 1 pass 1 MMAs, 2 warp partials synced, 3 CTA partial published,
4 cluster ready, 5 t/u summed, 6 pass 2 done; 7 producer issue; 8 warp sum done, 9 CTA sync."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_16710_b200 import _lib, ops  # noqa: E402

rows, n_in, n_out, r = (int(a) for a in sys.argv[1:5]) if len(sys.argv) > 4 else (2048, 4096, 4096, 8)
x = torch.randn(rows, n_in, device="cuda").bfloat16()
dy = torch.randn(rows, n_out, device="cuda").bfloat16()
a = torch.randn(n_in, r, device="cuda").bfloat16()
b = torch.randn(r, n_out, device="cuda").bfloat16()
da = torch.zeros(n_in, r, device="cuda")
db = torch.zeros(r, n_out, device="cuda")
u = torch.empty(rows, r, device="cuda")
sh = ops.lora_shape(x, dy, r)
ws = torch.empty(ops.seco_lora_workspace_size(sh) // 4, device="cuda")
flush = torch.ones(64 << 20, device="cuda")
for _ in range(3):
    ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
flush.mul_(1.0)
ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 384)()
_lib.load().seco_debug_lora_trace(buf, 384)
t = [[buf[i * 12 + p] for p in range(12)] for i in range(32)]
base = t[0][10]
print(f"kernel entry {t[0][10] - base}, fragments loaded {t[1][10] - base}, loop done {t[0][11] - base}, "
      f"flag published {t[1][11] - base}, all flags seen {t[2][11] - base}, reduced {t[3][11] - base}")
print("blk  prod_issue  full  pass1  wsync  publish  ready  summed  pass2  wsum  csync (cycles from first event)")
for i, row in enumerate(t):
    if not row[0]:
        break
    print(f"{i:3d} " + " ".join(f"{(v - base) if v else -1:7d}" for v in [row[7]] + row[:7] + row[8:10]))
