"""Stage-2 schedule experiment at cfg3: the rebuild forward of chunk j-1 does not depend on
chunk j's backward (it reads only the checkpoints), so it can run on a second stream and
fill the backward's last partial wave.  Times R SeCO steps per schedule.
usage: python tools/overlap_time.py [cfg3|cfg2|cfg5] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_16710_b200.flops import seco_step_flops
from paper_2505_16710_b200.step import ChunkedAttention

CFG = {"cfg3": (32, 8, 128, 32768, 2048), "cfg2": (32, 8, 128, 8192, 1024), "cfg5": (32, 8, 128, 16384, 1024)}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 10
hq, hkv, d, S, c = CFG[name]
k = S // c
torch.manual_seed(0)
q, do = (torch.randn(hq, S, d, device="cuda").bfloat16() for _ in range(2))
kc, vc = (torch.randn(hkv, S, d, device="cuda").bfloat16() for _ in range(2))
L = ChunkedAttention(hq, hkv, d, S, c)
ws_f = torch.empty_like(L.ws)
main = torch.cuda.current_stream()


def serial():
    L.dkv.zero_()
    for j in range(k):
        L.forward_chunk(q, kc, vc, j)
    for j in reversed(range(k)):
        L.forward_chunk(q, kc, vc, j)
        L.backward_chunk(q, kc, vc, do, j)


def overlapped(side, ahead, mstream=None):
    """Backwards on `mstream` (default: the current stream), rebuild forwards on `side`;
    ahead = how many backwards the side stream may run ahead of (None: unbounded)."""
    m = mstream or main
    if m is not main:
        m.wait_stream(main)
    with torch.cuda.stream(m):
        L.dkv.zero_()
        for j in range(k):
            L.forward_chunk(q, kc, vc, j)
        e1 = torch.cuda.Event()
        e1.record(m)
        side.wait_event(e1)
        ev_f, ev_b = {}, {}
        order = list(reversed(range(k)))
        ws0 = L.ws
        for n, j in enumerate(order):
            if ahead is not None and n - ahead >= 1:
                side.wait_event(ev_b[order[n - ahead - 1]])
            L.ws = ws_f
            L.forward_chunk(q, kc, vc, j, stream=side)
            L.ws = ws0
            ev_f[j] = torch.cuda.Event()
            ev_f[j].record(side)
            m.wait_event(ev_f[j])
            L.backward_chunk(q, kc, vc, do, j)
            ev_b[j] = torch.cuda.Event()
            ev_b[j].record(m)
    if m is not main:
        main.wait_stream(m)


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(R):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R


lo, hi = torch.cuda.Stream.priority_range()     # lo = least urgent (0), hi = most urgent
print("priority range", lo, hi)
variants = [("serial", serial)]
side0 = torch.cuda.Stream(priority=lo)
mhi = torch.cuda.Stream(priority=hi)
for ahead in (0, 1, 2, None):
    variants.append((f"same-prio ahead={ahead}", lambda ahead=ahead: overlapped(side0, ahead)))
    variants.append((f"bwd-high ahead={ahead}", lambda ahead=ahead: overlapped(side0, ahead, mhi)))
fl = seco_step_flops(hq, d, S, c)
ref = None
for rnd in range(2):
    for nm, fn in variants:
        ms = timeit(fn)
        if nm == "serial":
            ref = ms
        print(f"{name} round {rnd} {nm:24s}: {ms:8.3f} ms/step  {fl / ms / 1e9:7.1f} TFLOP/s  ({ref / ms:5.3f}x)",
              flush=True)
# parity of the overlapped schedule against the serial one (bitwise: same kernels, same order per buffer)
serial()
torch.cuda.synchronize()
dq0, dkv0 = L.dq.clone(), L.dkv.clone()
overlapped(side0, 1, mhi)
torch.cuda.synchronize()
print("dq max diff", (L.dq.float() - dq0.float()).abs().max().item(), "dkv max diff",
      (L.dkv - dkv0).abs().max().item())
