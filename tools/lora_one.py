"""One shape of seco_lora_grad, R calls (for ncu launch lists of the LoRA kernels).
usage: python tools/lora_one.py [rows n_in n_out r reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_16710_b200 import ops  # noqa: E402

rows, n_in, n_out, r, reps = (int(a) for a in sys.argv[1:6]) if len(sys.argv) > 5 else (2048, 4096, 4096, 8, 3)
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
for _ in range(reps):
    flush.mul_(1.0)
    ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
torch.cuda.synchronize()
