"""Small end-to-end run of every libseco.so entry point for compute-sanitizer (memcheck):
bf16 SeCO + SpaCO steps (d = 128 and 64, split-KV forward, deterministic mode), the fp32
debug path, and the LoRA gradient kernel.  No checks -- the sanitizer reports."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_16710_b200 import ops
from paper_2505_16710_b200.step import ChunkedAttention
torch.manual_seed(0)
for hq, hkv, seq, d, c, det, dt in ((8, 2, 1024, 128, 256, False, torch.bfloat16),
                                   (4, 1, 2048, 64, 512, True, torch.bfloat16),
                                   (8, 2, 4096, 128, 1024, False, torch.bfloat16),
                                   (4, 2, 96, 20, 32, False, torch.float32)):
    q = torch.randn(hq, seq, d, device="cuda").to(dt)
    k = torch.randn(hkv, seq, d, device="cuda").to(dt)
    v = torch.randn(hkv, seq, d, device="cuda").to(dt)
    do = torch.randn(hq, seq, d, device="cuda").to(dt)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=dt, own_copies=True, deterministic=det)
    L.seco_step(q, k, v, do)
    L.spaco_step(q, k, v, do, t=max(1, seq // c // 2), seed=1)
    torch.cuda.synchronize()
    print("ok", hq, hkv, seq, d, c, det, dt, flush=True)
for dt in (torch.bfloat16, torch.float32):
    x = torch.randn(300, 264, device="cuda").to(dt)[:, :256]
    dy = torch.randn(300, 128, device="cuda").to(dt)
    a = torch.randn(256, 8, device="cuda").to(dt)
    b = torch.randn(8, 128, device="cuda").to(dt)
    da, db = torch.zeros(256, 8, device="cuda"), torch.zeros(8, 128, device="cuda")
    u = torch.empty(300, 8, device="cuda")
    sh = ops.lora_shape(x, dy, 8)
    ws = torch.empty(ops.seco_lora_workspace_size(sh) // 4, device="cuda")
    ops.seco_lora_grad(sh, x, dy, a, b, da, db, u, ws)
    torch.cuda.synchronize()
    print("ok lora", dt, flush=True)
