"""Time seco_lora_grad alone at LLaMA-3-8B projection shapes (rows = one 2048-row chunk, r = 8,
bf16) and report its HBM throughput against the algorithmic bytes (X and dY read once, u
written, dA / dB read-modify-written).

    python tools/lora_bench.py [rows n_in n_out r]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_16710_b200 import ops  # noqa: E402

shapes = [tuple(int(a) for a in sys.argv[1:5])] if len(sys.argv) > 4 else \
    [(2048, 4096, 4096, 8), (2048, 4096, 1024, 8), (4096, 4096, 4096, 8), (2048, 4096, 4096, 16)]
# L2 flush between launches by READING 256 MB (> L2): a memset would leave L2 full of dirty lines
# whose write-back the next kernel pays for (~20 us), a read leaves clean lines
flush = torch.ones(256 * 1024 * 1024 // 4, device="cuda")
sink = torch.empty(1, device="cuda")
for (rows, n_in, n_out, r), det in [(sh_, dt_) for sh_ in shapes for dt_ in (False, True)]:
    x = torch.randn(rows, n_in, device="cuda").bfloat16()
    dy = torch.randn(rows, n_out, device="cuda").bfloat16()
    a = torch.randn(n_in, r, device="cuda").bfloat16()
    b = torch.randn(r, n_out, device="cuda").bfloat16()
    da = torch.zeros(n_in, r, device="cuda")
    db = torch.zeros(r, n_out, device="cuda")
    u = torch.empty(rows, r, device="cuda")
    sh = ops.lora_shape(x, dy, r, deterministic=det)
    ws = torch.empty(ops.seco_lora_workspace_size(sh) // 4, device="cuda")
    for _ in range(5):
        ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
    torch.cuda.synchronize()
    n = 30
    ts = []
    for _ in range(n):
        sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    alg = rows * (n_in + n_out) * 2 + rows * r * 4 + 2 * (n_in + n_out) * r * 4
    print(f"lora_grad rows={rows} {n_in}->{n_out} r={r}{' det' if det else ''}: median {us:.1f} us (min {ts[0]:.1f}), "
          f"{alg / 1e6:.1f} MB algorithmic -> {alg / us / 1e3:.0f} GB/s "
          f"({100 * alg / us / 1e3 / 6547.8:.0f}% of 6547.8 measured HBM), launches {ops.last_launch_count()}")
