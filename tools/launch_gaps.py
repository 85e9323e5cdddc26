"""Launch-overhead evidence (PAPER §4.2 names "frequent kernel launches for small-scale tensor
operations" as SeCO's second overhead): one SeCO step under torch.profiler (CUPTI
kernel records with device timestamps; nsys is not installed in this image), then the gaps
between consecutive kernels on the stream -- the device idle time the launches leave.

    python tools/launch_gaps.py [config ...]      configs: cfg3, cfg3r8 (one rank of cfg3 over 8
                                                  GPUs: 4 q / 1 kv heads), cfg4r8, cfg2
"""
import json
import os
import statistics
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2505_16710_b200.step import ChunkedAttention  # noqa: E402
from synth import make_inputs  # noqa: E402

SHAPES = {"cfg3": (32, 8, 128, 32768, 2048), "cfg3r8": (4, 1, 128, 32768, 2048),
          "cfg4r8": (4, 1, 128, 131072, 4096), "cfg2": (32, 8, 128, 8192, 1024)}


def short(name):
    for key in ("seco_fwd_sm100", "seco_fwd2_sm100", "seco_bwd2_sm100", "seco_bwd_sm100", "bwd_prep", "bwd_final", "fwd_combine",
                "chunk_skip"):
        if key in name:
            return key
    return "other:" + name[:40]


def run(cfg):
    hq, hkv, d, s, c = SHAPES[cfg]
    x = make_inputs(hq, hkv, s, d, seed=0)
    q, k, v, do = (torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).cuda()
                   for b in (x.q_bits, x.k_bits, x.v_bits, x.do_bits))
    layer = ChunkedAttention(hq, hkv, d, s, c)
    for _ in range(3):
        layer.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        layer.seco_step(q, k, v, do)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
    span = ks[-1]["ts"] + ks[-1]["dur"] - ks[0]["ts"]
    busy = sum(e["dur"] for e in ks)
    gaps = [max(0.0, b["ts"] - (a["ts"] + a["dur"])) for a, b in zip(ks, ks[1:])]
    print(f"== {cfg}: hq={hq} hkv={hkv} d={d} S={s} c={c}: {len(ks)} kernels in one SeCO step")
    print(f"   span {span:.1f} us, kernels busy {busy:.1f} us, gaps {sum(gaps):.1f} us "
          f"({100 * sum(gaps) / span:.2f}% of the step); gap median {statistics.median(gaps):.2f} us, "
          f"max {max(gaps):.2f} us (overlapping PDL launches count as 0)")
    if os.environ.get("GAPS_DETAIL"):                # every launch: kernel, duration, gap before it
        for e, gp in zip(ks, [0.0] + gaps):
            print(f"     {short(e['name']):18s} {e['dur']:9.1f} us  gap before {gp:6.2f} us")
    by = {}
    for e, gp in zip(ks, [0.0] + gaps):
        n = short(e["name"])
        by.setdefault(n, []).append((e["dur"], gp))
    for n, lst in sorted(by.items(), key=lambda kv: -sum(t for t, _ in kv[1])):
        durs = [t for t, _ in lst]
        print(f"   {n:18s} n={len(lst):3d} total {sum(durs):9.1f} us  mean {statistics.mean(durs):8.1f} us  "
              f"min {min(durs):7.1f}  gap before: mean {statistics.mean(g for _, g in lst):5.2f} us")


if __name__ == "__main__":
    for cfg in (sys.argv[1:] or ["cfg3", "cfg3r8", "cfg4r8"]):
        run(cfg)
