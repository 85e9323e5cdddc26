"""Context only: one FA4 (library) forward at the cfg3 j=15 chunk-call shape, for ncu comparison
captures against seco_fwd_sm100_kernel.  usage: python tools/fa4_one.py [j] [reps]"""
import sys

import torch
from vllm.vllm_flash_attn.cute.interface import flash_attn_func

j = int(sys.argv[1]) if len(sys.argv) > 1 else 15
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hq, hkv, d, c = 32, 8, 128, 2048
q = torch.randn(1, c, hq, d, device="cuda", dtype=torch.bfloat16)
k = torch.randn(1, c * (j + 1), hkv, d, device="cuda", dtype=torch.bfloat16)
v = torch.randn(1, c * (j + 1), hkv, d, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    flash_attn_func(q, k, v, causal=True)
torch.cuda.synchronize()
