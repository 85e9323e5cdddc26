#!/usr/bin/env python
"""Benchmark of the SeCO / SpaCO chunked-attention hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--mode seco|spaco]
                    [--t 4] [--shard heads|batch] [--impl ours|reference]

One step = one pass of the whole hot path over one sequence:
stage 1 (chunk forward, j = 0..k-1) then stage 2 (for j = k-1..0 in the sampled set:
rebuild forward + chunk backward with relay), all through the C ABI of libseco.so on
one CUDA stream.  Metric (BASELINE.json): algorithmic TFLOP/s of the step (SeCO =
4.5 F, F = 2 d Hq S (S+1); SpaCO = F + 3.5 sum_{j in I} fwd_j), plus tokens/s.

Multi-GPU (torchrun, one process per GPU, NCCL): `--shard heads` gives rank r the
kv-head group slice [r Hkv/N, (r+1) Hkv/N) and the matching q heads (no collective
on the attention path; total work fixed -> "strong"); `--shard batch` gives every
rank its own sequence ("weak").  Time = max over ranks of the CUDA-event time.

`--impl reference` times the CPU oracle (oracle/, fp64 NumPy) on the host cores on a
bounded sample of the same workload (the reference arm; rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chunked attn fwd+bwd TFLOP/s & tokens/s, Llama-3-8B shape, 32K ctx"
CONFIGS = {
    # BASELINE.json configs[1..4]; configs[0] (tiny) is a parity case only
    "cfg2": dict(hq=32, hkv=8, d=128, seq=8192, chunk=1024),
    "cfg3": dict(hq=32, hkv=8, d=128, seq=32768, chunk=2048),
    "cfg4": dict(hq=32, hkv=8, d=128, seq=131072, chunk=4096),
    "cfg5": dict(hq=32, hkv=8, d=128, seq=16384, chunk=1024),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="seco", choices=["seco", "spaco"])
    ap.add_argument("--t", type=int, default=4, help="SpaCO budget (sampled chunks)")
    ap.add_argument("--cap", type=float, default=2.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--shard", default="heads", choices=["heads", "batch"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--allreduce", action="store_true",
                    help="batch mode: all_reduce a LLaMA3-8B LoRA r=8 fp32 gradient bucket (27.3 MB) each step")
    ap.add_argument("--deterministic", action="store_true",
                    help="SECO_FLAG_DETERMINISTIC: bit-reproducible backward (ordered dQ reduction)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run this many steps, no timing output")
    ap.add_argument("--oracle-gflop", type=float, default=0.0,
                    help="oracle sample size in GFLOP (default: 150 per reference-arm step, 1000 for cpu_baseline)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample_shape(cfg, target_flops):
    """The bounded oracle sample: whole kv-head groups (G q-heads + their kv head) over the
    first n chunks of the sequence, the largest such sample whose algorithmic SeCO-step FLOPs
    stay within target_flops (chunks first, then more groups once the whole sequence fits)."""
    from paper_2505_16710_b200.flops import seco_step_flops
    G, c, d, k = cfg["hq"] // cfg["hkv"], cfg["chunk"], cfg["d"], cfg["seq"] // cfg["chunk"]
    n = 1
    while n < k and seco_step_flops(G, d, (n + 1) * c, c) <= target_flops:
        n += 1
    groups = 1
    while groups < cfg["hkv"] and seco_step_flops(G * (groups + 1), d, n * c, c) <= target_flops:
        groups += 1
    return groups, n


def cpu_oracle_sample(cfg, target_flops=1.0e12):
    """Time the oracle (fp64 NumPy, as it stands) on a bounded sample of the workload
    (oracle_sample_shape: <= 1 TFLOP, ~15 s on the 16 host cores of the GPU box, for the cpu_baseline key).
    Returns (TFLOP/s, seconds, description, threads)."""
    from oracle import chunkwise as OC
    from synth import make_inputs
    from paper_2505_16710_b200.flops import seco_step_flops
    c, d = cfg["chunk"], cfg["d"]
    G = cfg["hq"] // cfg["hkv"]
    groups, n = oracle_sample_shape(cfg, target_flops)
    seq = n * c
    x = make_inputs(G * groups, groups, seq, d, seed=0)
    fl = seco_step_flops(G * groups, d, seq, c)
    t0 = time.perf_counter()
    OC.seco_step(x.q, x.k, x.v, x.do, [c] * n)
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    desc = (f"oracle.chunkwise.seco_step fp64 on {groups} kv-head group(s) ({G * groups} q-heads, {groups} "
            f"kv-head(s)), first {seq} tokens ({n} chunks of {c}), d={d}: {fl / 1e9:.1f} GFLOP algorithmic "
            f"(same FLOP model as the GPU arm)")
    return fl / dt / 1e12, dt, desc, threads


def config_block(args, cfg, world, sel=None, gamma=None):
    """The `config` object of the JSON line -- identical for both arms."""
    from paper_2505_16710_b200.parallel import LORA_PARAMS_LLAMA3_8B_R8
    hq, hkv, d, seq, c = cfg["hq"], cfg["hkv"], cfg["d"], cfg["seq"], cfg["chunk"]
    k = seq // c
    n_seq = world if (args.shard == "batch" or world == 1) else 1
    return {"workload": f"{args.config}: Llama-3-8B attention shape, seq {seq}, chunk {c}, {args.mode}"
                        + (f" t={args.t} of {k} (I={sel}, gamma={gamma})" if sel is not None else ""),
            "hq": hq, "hkv": hkv, "d": d, "seq_len": seq, "chunk": c, "num_chunks": k,
            "mode": args.mode, "sequences_per_step": n_seq, "deterministic": args.deterministic,
            "parallelism": f"{args.shard}{world}" if world > 1 else "single",
            "allreduce_bytes_per_step": (LORA_PARAMS_LLAMA3_8B_R8 * 4 if args.allreduce else 0),
            "l2_policy": "inputs larger than L2 (Q,dO 256 MiB, K,V 64 MiB each, dKV 256 MiB per rank)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    # each step a smaller bounded sample (~0.15 TFLOP, a few seconds) so that the whole
    # --steps K --warmup W run ends within a few minutes
    target = args.oracle_gflop * 1e9 if args.oracle_gflop > 0 else 0.15e12
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, target)
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        v, dt, desc, threads = cpu_oracle_sample(cfg, target)
        vals.append(v)
        t_all += dt
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
            "higher_is_better": True, "scaling": "strong" if (args.shard == "heads" and world > 1) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, cfg, world),
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    from synth import make_inputs
    from paper_2505_16710_b200.step import ChunkedAttention
    from paper_2505_16710_b200 import ops, flops as FL

    # SECO_BENCH_SHARED_GPU=1 is a plumbing check only (never a measurement): every rank uses
    # cuda:0 and gloo carries the barrier / max-over-ranks, so the N > 1 code path can be
    # exercised on a one-GPU box (ranks share nothing on the data path).
    shared = os.environ.get("SECO_BENCH_SHARED_GPU") == "1"
    gpu_index = 0 if shared else local_rank
    torch.cuda.set_device(gpu_index)
    dev = torch.device("cuda", gpu_index)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    coll_dev = torch.device("cpu") if shared else dev
    cfg = dict(CONFIGS[args.config])
    hq, hkv, d, seq, c = cfg["hq"], cfg["hkv"], cfg["d"], cfg["seq"], cfg["chunk"]
    from paper_2505_16710_b200.parallel import (LORA_PARAMS_LLAMA3_8B_R8, allreduce_grad_bucket, head_shard,
                                                max_over_ranks)
    if args.shard == "heads" and world > 1:
        shard = head_shard(hq, hkv, world, rank)      # no collective on the data path
        hq_r, hkv_r = shard.hq, shard.hkv
    else:
        hq_r, hkv_r = hq, hkv
    k = seq // c

    # inputs: seeded on the host (synth), pinned, then resident in HBM for the device timing
    x = make_inputs(hq_r, hkv_r, seq, d, seed=args.seed + 1000 * rank)
    pinned = []
    for bits in (x.q_bits, x.k_bits, x.v_bits, x.do_bits):
        t = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).pin_memory()
        pinned.append(t)
    del x
    q, kc, vc, do = (t.to(dev, non_blocking=True) for t in pinned)
    layer = ChunkedAttention(hq_r, hkv_r, d, seq, c, dtype=torch.bfloat16, device=dev,
                             deterministic=args.deterministic)
    stream = torch.cuda.current_stream()

    def sampled():
        if args.mode == "seco":
            return None, 1.0, 1.0
        return ops.spaco_sample_and_scale(k, args.t, args.seed, args.cap, ops._lib.SPACO_PAPER)

    sel, gamma, sscale = sampled()
    bucket = torch.zeros(LORA_PARAMS_LLAMA3_8B_R8, dtype=torch.float32, device=dev) if args.allreduce else None

    if args.profile_steps:
        for _ in range(args.profile_steps):
            layer.step(q, kc, vc, do, sel, gamma, sscale)
        torch.cuda.synchronize()
        return

    # ---------------------------------------------------------------- warm-up
    for _ in range(max(args.warmup, 0)):
        layer.step(q, kc, vc, do, sel, gamma, sscale)
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed (device-resident inputs)
    # The headline: exactly K steps between two events on the launching stream, nothing else
    # recorded inside.  The per-kernel attribution (fwd / bwd CUDA-event times per call, for
    # `kernels` and `roofline`) comes from a second, separate set of K steps below.
    order = [("f", j) for j in range(k)]
    stage2 = list(range(k))[::-1] if sel is None else sorted(sel, reverse=True)
    for j in stage2:
        order += [("f", j), ("b", j)]

    def one_step(events=None):
        n_launch = 0
        layer.dkv.zero_()
        if sel is not None:
            layer.dq.zero_()
        for n, (kind, j) in enumerate(order):
            if events is not None:
                events[2 * n].record(stream)
            if kind == "f":
                n_launch += layer.forward_chunk(q, kc, vc, j)
            else:
                n_launch += layer.backward_chunk(q, kc, vc, do, j, gamma, sscale)
            if events is not None:
                events[2 * n + 1].record(stream)
        if bucket is not None:
            allreduce_grad_bucket(bucket)
        return n_launch

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    mem_before = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    clk = ClockSampler(gpu_index)
    with clk:
        t_start.record(stream)
        for s in range(args.steps):
            launches += one_step()
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_local = t_start.elapsed_time(t_end)
    memory = dict(layer.memory_ledger())
    memory["allocated_during_timed_steps_bytes"] = torch.cuda.max_memory_allocated(dev) - mem_before
    # attribution pass (not part of the headline)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * len(order))] for _ in range(args.steps)]
    a_start, a_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_start.record(stream)
    for s in range(args.steps):
        one_step(ev[s])
    a_end.record(stream)
    torch.cuda.synchronize()
    ms_attr = a_start.elapsed_time(a_end)
    t_f = t_b = 0.0
    for s in range(args.steps):
        for n, (kind, j) in enumerate(order):
            dt = ev[s][2 * n].elapsed_time(ev[s][2 * n + 1])
            if kind == "f":
                t_f += dt
            else:
                t_b += dt
    ms = max_over_ranks(ms_local, coll_dev)
    ms_per_step = ms / args.steps

    step_flops_rank = FL.seco_step_flops(hq_r, d, seq, c) if sel is None else \
        FL.spaco_step_flops(hq_r, d, seq, c, sel)
    n_seq = world if (args.shard == "batch" or world == 1) else 1
    total_flops = step_flops_rank * world          # all ranks' work per step
    tokens = seq * n_seq
    value = total_flops / (ms_per_step * 1e-3) / 1e12
    # dominant kernel: algorithmic flops per launch / average launch time (this rank)
    fwd_fl = sum(FL.fwd_flops(hq_r, d, c, j) for kind, j in order if kind == "f") * args.steps
    bwd_fl = sum(FL.bwd_flops(hq_r, d, c, j) for kind, j in order if kind == "b") * args.steps
    kern = {"fwd": {"tflops": fwd_fl / (t_f * 1e-3) / 1e12 if t_f else None, "ms_per_step": t_f / args.steps,
                    "share_of_step": t_f / ms_attr},
            "bwd": {"tflops": bwd_fl / (t_b * 1e-3) / 1e12 if t_b else None, "ms_per_step": t_b / args.steps,
                    "share_of_step": t_b / ms_attr},
            "note": "per-call CUDA events from a separate attribution pass of K steps (not the timed one)"}
    dom = "bwd" if t_b >= t_f else "fwd"
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, peak_src = peaks["bf16_tflops_sustained"], "MEASURED_PEAKS.json bf16_tflops_sustained"
        peak_burst = peaks["bf16_tflops"]
    except Exception:
        peak, peak_src, peak_burst = 1400.0, "fallback B200_PROFILING.md sustained ~1.4 PF", 1590.0
    traffic = None
    traffic_launch = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        traffic = tr.get(dom, {}).get(args.config)
        traffic_launch = tr.get(dom, {}).get(args.config + "_launch")
    except Exception:
        pass
    achieved = kern[dom]["tflops"]
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "kernel": f"seco_chunk_{'backward' if dom == 'bwd' else 'forward'} "
                          f"({('bwd_prep + seco_bwd_sm100_kernel + bwd_final' if args.deterministic else 'bwd_prep + seco_bwd2_sm100_kernel + bwd_final') if dom == 'bwd' else 'seco_fwd_sm100_kernel'})",
                "peak_source": peak_src, "frac_of_burst_peak": achieved / peak_burst if achieved else None,
                "traffic_note": f"DRAM bytes of the {traffic_launch} launch from ncu --set full "
                                "(profiles/roofline_traffic.json); achieved averages all launches"}

    # ---------------------------------------------------------------- end to end (host buffers)
    # Every step: H2D of that step's Q, K, V, dO from pinned host memory, the step, D2H of its
    # dQ and dKV -- pipelined at chunk granularity.  Host and device tensors are sequence-major
    # ([S][h][d], the layout a projection produces; the ABI takes its strides), so a chunk is
    # one contiguous block: K/V/Q of chunk j are copied in stage-1 order and the forward of
    # chunk j waits only for them; dO arrives in stage-2 (descending) order; dQ_j and dKV slot
    # j (final once chunk j's backward is done) go back while the earlier chunks compute.
    # Copies run on two copy streams (both PCIe directions) and also overlap the neighbouring
    # steps; two device buffer sets alternate so a step never reads inputs or writes outputs
    # still in flight.
    e2e = None
    if not args.no_e2e:
        del layer
        host = [t.transpose(0, 1).contiguous().pin_memory() for t in pinned]      # [S][h][d]
        sets = [tuple(torch.empty(t.shape, dtype=t.dtype, device=dev) for t in host) for _ in range(2)]
        layers = [ChunkedAttention(hq_r, hkv_r, d, seq, c, dtype=torch.bfloat16, device=dev,
                                   deterministic=args.deterministic, layout="shd") for _ in range(2)]
        out_dq = [torch.empty(seq, hq_r, d, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        out_dkv = [torch.empty(layers[0].dkv.shape, dtype=layers[0].dkv.dtype).pin_memory() for _ in range(2)]
        h2d = sum(t.numel() * t.element_size() for t in host)
        d2h = out_dq[0].numel() * out_dq[0].element_size() + out_dkv[0].numel() * out_dkv[0].element_size()
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        done = [None, None]      # compute-finished event of the last step that used set b
        drained = [None, None]   # D2H-finished event of the last step that used set b
        stage2 = list(range(k))[::-1] if sel is None else sorted(sel, reverse=True)
        rest = [j for j in range(k) if j not in stage2]

        def rows(t, j):
            return t[j * c:(j + 1) * c]

        def d2h_chunk(b, j):
            rows(out_dq[b], j).copy_(rows(layers[b].dq.transpose(0, 1), j), non_blocking=True)
            for tt in range(2):
                for gg in range(hkv_r):
                    out_dkv[b][tt, gg, j * c:(j + 1) * c].copy_(layers[b].dkv[tt, gg, j * c:(j + 1) * c],
                                                               non_blocking=True)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(s_in)
        stream.wait_event(e0)
        s_out.wait_event(e0)
        for st_i in range(args.steps):
            b = st_i % 2
            qd, kd, vd, dod = sets[b]
            lay = layers[b]
            ev_qkv, ev_do = [torch.cuda.Event() for _ in range(k)], [torch.cuda.Event() for _ in range(k)]
            with torch.cuda.stream(s_in):
                if done[b] is not None:
                    s_in.wait_event(done[b])
                for j in range(k):                       # stage-1 order
                    for dst, src in ((kd, host[1]), (vd, host[2]), (qd, host[0])):
                        rows(dst, j).copy_(rows(src, j), non_blocking=True)
                    ev_qkv[j].record(s_in)
                for j in reversed(range(k)):             # stage-2 order
                    rows(dod, j).copy_(rows(host[3], j), non_blocking=True)
                    ev_do[j].record(s_in)
            if drained[b] is not None:
                stream.wait_event(drained[b])
            qv, kv, vv, dov = (t.transpose(0, 1) for t in (qd, kd, vd, dod))
            lay.dkv.zero_()
            if sel is not None:
                lay.dq.zero_()
            for j in range(k):                           # stage 1
                stream.wait_event(ev_qkv[j])
                lay.forward_chunk(qv, kv, vv, j)
            ev_out = {}
            for j in stage2:                             # stage 2, descending
                stream.wait_event(ev_do[j])
                lay.forward_chunk(qv, kv, vv, j)
                lay.backward_chunk(qv, kv, vv, dov, j, gamma, sscale)
                ev_out[j] = torch.cuda.Event()
                ev_out[j].record(stream)
            done[b] = torch.cuda.Event()
            done[b].record(stream)
            with torch.cuda.stream(s_out):
                for j in stage2:
                    s_out.wait_event(ev_out[j])
                    d2h_chunk(b, j)
                s_out.wait_event(done[b])
                for j in rest:                           # SpaCO: chunks outside the sample
                    d2h_chunk(b, j)
                drained[b] = torch.cuda.Event()
                drained[b].record(s_out)
        s_in.wait_event(drained[(args.steps - 1) % 2])
        if args.steps > 1:
            s_in.wait_event(drained[args.steps % 2])
        e1.record(s_in)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1), coll_dev)
        e2e = {"value": total_flops / (ems / args.steps * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": ems / args.steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "pinned host Q,K,V,dO ([S][h][d]) -> device per chunk in the order the step consumes "
                       "them (copy stream); SeCO/SpaCO chunk calls via the C ABI, each waiting only for its "
                       "chunk's inputs; dQ_j, dKV slot j -> pinned host as soon as chunk j's backward is "
                       "done (copy stream); steps double-buffered"}
        del sets, layers

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, desc, threads = cpu_oracle_sample(cfg, args.oracle_gflop * 1e9 if args.oracle_gflop > 0 else 1.0e12)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": desc,
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if (args.shard == "heads" and world > 1) else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config_block(args, cfg, world, sel, gamma),
            "tokens_per_s": tokens / (ms_per_step * 1e-3),
            "step_tflop": total_flops / 1e12,
            "roofline": roofline, "kernels": kern, "memory": memory,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
