"""Time seco_lora_grad alone at a LLaMA-3-8B projection shape (rows = chunk 2048, 4096 -> 4096,
r = 8, bf16) and report its HBM throughput against the bytes it must move (X, dY read twice,
u written)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200 import ops
rows, n_in, n_out, r = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (2048, 4096, 4096, 8)))
x = torch.randn(rows, n_in, device="cuda").bfloat16()
dy = torch.randn(rows, n_out, device="cuda").bfloat16()
a = torch.randn(n_in, r, device="cuda").bfloat16()
b = torch.randn(r, n_out, device="cuda").bfloat16()
da = torch.zeros(n_in, r, device="cuda"); db = torch.zeros(r, n_out, device="cuda")
u = torch.empty(rows, r, device="cuda")
sh = ops.lora_shape(x, dy, r)
ws = torch.empty(ops.seco_lora_workspace_size(sh) // 4, device="cuda")
for _ in range(5):
    ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
e0.record()
for _ in range(n):
    ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / n * 1e3
need = 2 * rows * (n_in + n_out) * 2        # X and dY, each read twice
print(f"lora_grad rows={rows} {n_in}->{n_out} r={r}: {us:.1f} us, {need / us / 1e3:.0f} GB/s of X/dY reads")
