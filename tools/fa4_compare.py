"""Context measurement, not product: the image's FlashAttention-4 (vllm_flash_attn.cute, a
library) timed on the same chunk-call shapes as tools/kbench.py, so the per-call TFLOP/s of
libseco.so can be read against a state-of-the-art Blackwell attention kernel on the same box.

Shape of chunk call j at cfg3: queries = chunk j (c rows, Hq heads), keys = slots 0..j
(c(j+1) rows, Hkv heads), bottom-right-aligned causal mask (FlashAttention's convention for
seqlen_q < seqlen_k is exactly the chunk-wise mask of P:106, Eq. 1).  FLOPs are the same
algorithmic counts paper_2505_16710_b200.flops uses (4 d Hq Pairs fwd, 10 d Hq Pairs bwd).

usage: python tools/fa4_compare.py [j,j,...] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_16710_b200 import flops as FL

hq, hkv, d, S, c = 32, 8, 128, 32768, 2048
js = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 3, 7, 15]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 10

from vllm.vllm_flash_attn.cute.interface import flash_attn_func  # noqa: E402

torch.manual_seed(0)
for j in js:
    sk = c * (j + 1)
    q = torch.randn(1, c, hq, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    k = torch.randn(1, sk, hkv, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    v = torch.randn(1, sk, hkv, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    do = torch.randn(1, c, hq, d, device="cuda", dtype=torch.bfloat16)

    def fwd():
        with torch.no_grad():
            return flash_attn_func(q, k, v, causal=True)

    def fwdbwd():
        o = flash_attn_func(q, k, v, causal=True)
        if isinstance(o, tuple):
            o = o[0]
        torch.autograd.backward(o, do)

    res = {}
    for name, fn in (("fwd", fwd), ("fwd+bwd", fwdbwd)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(R):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / R
    ff, fb = FL.fwd_flops(hq, d, c, j), FL.bwd_flops(hq, d, c, j)
    tb = res["fwd+bwd"] - res["fwd"]
    print(f"FA4 cfg3 j={j:2d} fwd: {res['fwd'] * 1e3:8.1f} us {ff / res['fwd'] / 1e9:7.1f} TFLOP/s   "
          f"bwd (fwd+bwd - fwd): {tb * 1e3:8.1f} us {fb / tb / 1e9:7.1f} TFLOP/s", flush=True)
