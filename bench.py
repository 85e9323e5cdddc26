#!/usr/bin/env python
"""Benchmark of the SeCO / SpaCO chunked-attention hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--mode seco|spaco]
                    [--t 4] [--sampler paper|ht|bernoulli] [--dtype bf16|fp32dbg]
                    [--shard heads|batch] [--allreduce] [--impl ours|reference]

One step = one pass of the whole hot path over one sequence:
stage 1 (chunk forward, j = 0..k-1) then stage 2 (for j = k-1..0: rebuild forward + chunk
backward with relay if j is in the sampled set, else the SpaCO skip), all through the C ABI
of libseco.so on one CUDA stream (ChunkedAttention.plan / run).  Metric (BASELINE.json):
algorithmic TFLOP/s of the step (SeCO = 4.5 F, F = 2 d Hq S (S+1); SpaCO = F + 3.5
sum_{j in I} fwd_j, on the realised I), plus tokens/s.

Multi-GPU, one process per GPU (NCCL): `--gpus N` without a torchrun environment re-launches
this script under `torch.distributed.run` with N local ranks.  `--shard heads` gives rank r the
kv-head groups [r Hkv/N, (r+1) Hkv/N) and their q heads (no collective on the attention path;
total work fixed -> "strong"); `--shard batch` gives every rank its own sequence ("weak"), with
`--allreduce` adding the LoRA-gradient all_reduce of BASELINE configs[4].  Time = max over
ranks of the CUDA-event time.  `--dry-run` exercises the same N-rank plumbing on CPU (gloo,
no kernels; tests/test_bench_host.py).

`--impl reference` times the CPU oracle (oracle/, NumPy) on the host cores on a bounded
sample of the same workload (the reference arm; rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chunked attn fwd+bwd TFLOP/s & tokens/s, Llama-3-8B shape, 32K ctx"
CONFIGS = {
    # BASELINE.json configs[0..4]; configs[0] (tiny, fp32) runs only with --dtype fp32dbg
    "cfg1": dict(hq=2, hkv=1, d=16, seq=64, chunk=16),
    "cfg2": dict(hq=32, hkv=8, d=128, seq=8192, chunk=1024),
    "cfg3": dict(hq=32, hkv=8, d=128, seq=32768, chunk=2048),
    "cfg4": dict(hq=32, hkv=8, d=128, seq=131072, chunk=4096),
    "cfg5": dict(hq=32, hkv=8, d=128, seq=16384, chunk=1024),
}
SAMPLERS = {"paper": 0, "ht": 1, "bernoulli": 2}     # spaco_mode of include/seco.h


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="seco", choices=["seco", "spaco"])
    ap.add_argument("--t", type=int, default=4, help="SpaCO budget (sampled chunks)")
    ap.add_argument("--cap", type=float, default=2.0)
    ap.add_argument("--sampler", default="paper", choices=sorted(SAMPLERS),
                    help="SpaCO sampling mode (reading Z7): paper = Alg. 2 literally, ht / bernoulli = unbiased")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32dbg"],
                    help="bf16 tensor-core path, or the SIMT fp32 debug build (SECO_FP32_DEBUG)")
    ap.add_argument("--shard", default="heads", choices=["heads", "batch"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--allreduce", action="store_true",
                    help="batch mode: all_reduce a LLaMA3-8B LoRA r=8 fp32 gradient bucket (27.3 MB) each step")
    ap.add_argument("--deterministic", action="store_true",
                    help="SECO_FLAG_DETERMINISTIC: bit-reproducible backward (ordered dQ reduction)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nvtx", action="store_true", help="NVTX range per chunk call in the attribution pass")
    ap.add_argument("--dry-run", action="store_true", help="N-rank plumbing only (gloo, CPU, no kernels)")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run this many steps, no timing output")
    ap.add_argument("--oracle-gflop", type=float, default=0.0,
                    help="reference arm: oracle sample size per step in GFLOP (default: sized by a time budget)")
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------- N ranks
def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: run this script as N local ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1).  Returns the exit
    code, or None when this process is already a rank (or N = 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


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
def step_flops(cfg, hq, seq, sel):
    from paper_2505_16710_b200.flops import seco_step_flops, spaco_step_flops
    if sel is None:
        return seco_step_flops(hq, cfg["d"], seq, cfg["chunk"])
    return spaco_step_flops(hq, cfg["d"], seq, cfg["chunk"], sel)


def oracle_sample_shape(cfg, target_flops, sel=None):
    """A bounded prefix sample: one kv-head group (G q-heads + their kv head) over the first n
    chunks of the sequence, the largest n whose algorithmic step FLOPs stay within
    target_flops (at least 1 chunk).  SpaCO samples keep the chunks of I below n."""
    G, c, k = cfg["hq"] // cfg["hkv"], cfg["chunk"], cfg["seq"] // cfg["chunk"]

    def fl(n):
        return step_flops(cfg, G, n * c, None if sel is None else [j for j in sel if j < n])
    n = 1
    while n < k and fl(n + 1) <= target_flops:
        n += 1
    return 1, n


def cpu_oracle_run(cfg, n_chunks, sel=None, gamma=1.0, sscale=1.0, dtype="float32"):
    """Run the oracle (NumPy, as it stands: oracle.chunkwise.seco_step / spaco_step) on one
    kv-head group over the first n_chunks chunks.  Returns (seconds, algorithmic FLOPs of the
    sample, description, BLAS threads)."""
    import numpy as np
    from oracle import chunkwise as OC
    from synth import make_inputs
    c, d, G = cfg["chunk"], cfg["d"], cfg["hq"] // cfg["hkv"]
    seq = n_chunks * c
    x = make_inputs(G, 1, seq, d, seed=0)
    sub = None if sel is None else [j for j in sel if j < n_chunks]
    fl = step_flops(cfg, G, seq, sub)
    dt_np = np.float32 if dtype == "float32" else np.float64
    t0 = time.perf_counter()
    if sub is None:
        OC.seco_step(x.q, x.k, x.v, x.do, [c] * n_chunks, dtype=dt_np)
    else:
        OC.spaco_step(x.q, x.k, x.v, x.do, [c] * n_chunks, sub, gamma, sscale, dtype=dt_np)
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    whole = n_chunks == cfg["seq"] // c
    desc = (f"oracle.chunkwise.{'seco' if sub is None else 'spaco'}_step NumPy {dtype} on 1 kv-head group "
            f"({G} q-heads, 1 kv head), {'the whole sequence' if whole else f'the first {seq} tokens'} "
            f"({n_chunks} chunks of {c}), d={d}: {fl / 1e9:.1f} GFLOP algorithmic (same FLOP model as the "
            f"GPU arm); value = that rate"
            + (f", i.e. the whole workload extrapolated from 1 of {cfg['hkv']} independent head groups "
               f"(work scales exactly: head groups share nothing)" if whole else
               " (a prefix of 1 of the head groups; sized to the run's time budget)"))
    return dt, fl, desc, threads


def config_block(args, cfg, world, sel=None, gamma=None):
    """The `config` object of the JSON line -- identical for both arms."""
    from paper_2505_16710_b200.parallel import LORA_PARAMS_LLAMA3_8B_R8
    hq, hkv, d, seq, c = cfg["hq"], cfg["hkv"], cfg["d"], cfg["seq"], cfg["chunk"]
    k = seq // c
    n_seq = world if (args.shard == "batch" or world == 1) else 1
    return {"workload": f"{args.config}: Llama-3-8B attention shape, seq {seq}, chunk {c}, {args.mode}"
                        + (f" t={args.t} of {k}, sampler {args.sampler} (I={sel}, gamma={gamma})"
                           if sel is not None else ""),
            "hq": hq, "hkv": hkv, "d": d, "seq_len": seq, "chunk": c, "num_chunks": k,
            "mode": args.mode, "sampler": args.sampler if args.mode == "spaco" else None,
            "sequences_per_step": n_seq, "deterministic": args.deterministic,
            "parallelism": f"{args.shard}{world}" if world > 1 else "single",
            "allreduce_bytes_per_step": (LORA_PARAMS_LLAMA3_8B_R8 * 4 if args.allreduce else 0),
            "l2_policy": "inputs larger than L2 (Q,dO 256 MiB, K,V 64 MiB each, dKV 256 MiB per rank at cfg3)"}


def host_sample(args, cfg):
    """SpaCO sample of the run (the C-ABI sampler; pure host code, no GPU needed)."""
    if args.mode == "seco":
        return None, 1.0, 1.0
    from paper_2505_16710_b200 import ops
    k = cfg["seq"] // cfg["chunk"]
    return ops.spaco_sample_and_scale(k, args.t, args.seed, args.cap, SAMPLERS[args.sampler])


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle as it stands, on the host cores.  Each step is the
    same bounded sample (a prefix of one kv-head group), sized so the whole --steps K --warmup W
    run stays within ~3 minutes (calibrated on one 1-chunk run); the rate is the step's
    algorithmic FLOPs over its time."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    sel, gamma, sscale = host_sample(args, cfg)
    if args.oracle_gflop > 0:
        target = args.oracle_gflop * 1e9
    else:
        dt1, fl1, _, _ = cpu_oracle_run(cfg, 1)              # calibration (not timed)
        rate = fl1 / max(dt1, 1e-6)
        target = rate * 180.0 / max(args.steps + args.warmup, 1)
    _, n = oracle_sample_shape(cfg, target, sel)
    for _ in range(args.warmup):
        cpu_oracle_run(cfg, n, sel, gamma, sscale)
    secs, fl, desc, threads = [], 0.0, "", 1
    for _ in range(args.steps):
        dt, fl, desc, threads = cpu_oracle_run(cfg, n, sel, gamma, sscale)
        secs.append(dt)
    value = fl / statistics.median(secs) / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
            "ms_per_step_median": 1e3 * statistics.median(secs), "ms_per_step_min": 1e3 * min(secs),
            "higher_is_better": True, "scaling": "strong" if (args.shard == "heads" and world > 1) else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(args, cfg, world, sel, gamma),
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- dry run
def run_dry(args, rank, world):
    """The N-rank code path without kernels: shard assignment, barrier, max-over-ranks timing
    and the rank-0 JSON line (tests/test_bench_host.py runs it with --gpus 2 on CPU)."""
    import torch.distributed as dist
    from paper_2505_16710_b200.parallel import head_shard, max_over_ranks
    if world > 1:
        dist.init_process_group("gloo")
    cfg = CONFIGS[args.config]
    if args.shard == "heads" and world > 1:
        s = head_shard(cfg["hq"], cfg["hkv"], world, rank)
        shard = {"q_heads": list(s.q_heads), "kv_heads": list(s.kv_heads)}
        hq_r = s.hq
    else:
        shard = {"q_heads": [0, cfg["hq"]], "kv_heads": [0, cfg["hkv"]]}
        hq_r = cfg["hq"]
    if world > 1:
        dist.barrier()
    ms = max_over_ranks(10.0 + rank)          # stand-in per-rank time: the max is rank N-1's
    shards = [None] * world
    if world > 1:
        dist.all_gather_object(shards, shard)
        dist.barrier()
    else:
        shards = [shard]
    if rank == 0:
        sel, gamma, _ = host_sample(args, cfg)
        print(json.dumps({"dry_run": True, "n_gpus": world, "ms_max_over_ranks": ms, "shards": shards,
                          "step_tflop_per_rank": step_flops(cfg, hq_r, cfg["seq"], sel) / 1e12,
                          "config": config_block(args, cfg, world, sel, gamma)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- our arm
def alg_bytes_bwd(hq, hkv, d, c, j):
    """Algorithmic DRAM bytes of one chunk-backward call j (bf16 inputs, fp32 dKV): read Q_j,
    dO_j, O_j and K/V slots 0..j, write dQ_j, read-modify-write dKV slots 0..j, plus LSE / D."""
    return 2 * (4 * hq * c * d + 2 * hkv * (j + 1) * c * d) + 4 * 2 * 2 * hkv * (j + 1) * c * d + 3 * 4 * hq * c


def alg_bytes_fwd(hq, hkv, d, c, j):
    """Read Q_j and K/V slots 0..j, write O_j and LSE_j."""
    return 2 * (2 * hq * c * d + 2 * hkv * (j + 1) * c * d) + 4 * hq * c


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.dry_run:
        return run_dry(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    from synth import make_inputs
    from paper_2505_16710_b200.step import ChunkedAttention
    from paper_2505_16710_b200 import flops as FL

    fp32 = args.dtype == "fp32dbg"
    tdt = torch.float32 if fp32 else torch.bfloat16
    # SECO_BENCH_SHARED_GPU=1 is a plumbing check only (never a measurement): every rank uses
    # cuda:0 and gloo carries the barrier / max-over-ranks, so the N > 1 code path can be
    # exercised on a one-GPU box (ranks share nothing on the data path).
    shared = os.environ.get("SECO_BENCH_SHARED_GPU") == "1"
    if world > 1 and not shared and torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks need {world} GPUs, found {torch.cuda.device_count()}")
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
    x = make_inputs(hq_r, hkv_r, seq, d, seed=args.seed + 1000 * rank, bf16=not fp32)
    pinned = []
    for arr, bits in ((x.q, x.q_bits), (x.k, x.k_bits), (x.v, x.v_bits), (x.do, x.do_bits)):
        t = torch.from_numpy(np.ascontiguousarray(arr, np.float32)) if fp32 else \
            torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16)
        pinned.append(t.pin_memory())
    del x
    q, kc, vc, do = (t.to(dev, non_blocking=True) for t in pinned)
    layer = ChunkedAttention(hq_r, hkv_r, d, seq, c, dtype=tdt, device=dev, deterministic=args.deterministic)
    stream = torch.cuda.current_stream()

    sel, gamma, sscale = host_sample(args, cfg)
    order = layer.plan(sel)
    bucket = torch.zeros(LORA_PARAMS_LLAMA3_8B_R8, dtype=torch.float32, device=dev) if args.allreduce else None

    def one_step(events=None, nvtx=False):
        n = layer.run(order, q, kc, vc, do, gamma, sscale, events=events, nvtx=nvtx)
        if bucket is not None:
            allreduce_grad_bucket(bucket)
        return n

    if args.profile_steps:
        for _ in range(args.profile_steps):
            one_step(nvtx=args.nvtx)
        torch.cuda.synchronize()
        return

    # ---------------------------------------------------------------- warm-up
    for _ in range(max(args.warmup, 0)):
        one_step()
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed (device-resident inputs)
    # The headline: exactly K steps on the launching stream with one event between consecutive
    # steps (per-step times for the median / min; nothing else recorded inside).  The per-call
    # attribution (fwd / bwd CUDA-event times, for `kernels` and `roofline`) comes from a
    # second, separate set of K steps below.
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    mem_before = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    clk = ClockSampler(gpu_index)
    with clk:
        marks[0].record(stream)
        for s in range(args.steps):
            launches += one_step()
            marks[s + 1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_local = marks[0].elapsed_time(marks[-1])
    per_step_local = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    memory = dict(layer.memory_ledger())
    memory["allocated_during_timed_steps_bytes"] = torch.cuda.max_memory_allocated(dev) - mem_before
    # attribution pass (not part of the headline)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
          for _ in range(args.steps)]
    a_start, a_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_start.record(stream)
    for s in range(args.steps):
        one_step(ev[s], nvtx=args.nvtx)
    a_end.record(stream)
    torch.cuda.synchronize()
    ms_attr = a_start.elapsed_time(a_end)
    t_kind = {"f": 0.0, "b": 0.0, "z": 0.0}
    t_j15 = {"f": [], "b": []}
    for s in range(args.steps):
        for n, op in enumerate(order):
            dt = ev[s][n][0].elapsed_time(ev[s][n][1])
            t_kind[op[0]] += dt
            if op[0] in t_j15 and op[1] == k - 1:
                t_j15[op[0]].append(dt)
    ms = max_over_ranks(ms_local, coll_dev)
    ms_per_step = ms / args.steps
    # median / min over steps of the slowest rank's per-step times (max over ranks per step)
    per_step = [max_over_ranks(v, coll_dev) for v in per_step_local]

    step_flops_rank = FL.seco_step_flops(hq_r, d, seq, c) if sel is None else \
        FL.spaco_step_flops(hq_r, d, seq, c, sel)
    n_seq = world if (args.shard == "batch" or world == 1) else 1
    total_flops = step_flops_rank * world          # all ranks' work per step
    tokens = seq * n_seq
    value = total_flops / (ms_per_step * 1e-3) / 1e12
    # dominant kernel: algorithmic flops per launch / average launch time (this rank)
    fwd_fl = sum(FL.fwd_flops(hq_r, d, c, op[1]) for op in order if op[0] == "f") * args.steps
    bwd_fl = sum(FL.bwd_flops(hq_r, d, c, op[1]) for op in order if op[0] == "b") * args.steps
    kern = {"fwd": {"tflops": fwd_fl / (t_kind["f"] * 1e-3) / 1e12 if t_kind["f"] else None,
                    "ms_per_step": t_kind["f"] / args.steps, "share_of_step": t_kind["f"] / ms_attr},
            "bwd": {"tflops": bwd_fl / (t_kind["b"] * 1e-3) / 1e12 if t_kind["b"] else None,
                    "ms_per_step": t_kind["b"] / args.steps, "share_of_step": t_kind["b"] / ms_attr},
            "skip": {"ms_per_step": t_kind["z"] / args.steps, "share_of_step": t_kind["z"] / ms_attr},
            "note": "per-call CUDA events on the launching stream from a separate attribution pass of K steps"}
    for kk, name in (("f", "fwd"), ("b", "bwd")):
        if t_j15[kk]:
            fl1 = (FL.fwd_flops if kk == "f" else FL.bwd_flops)(hq_r, d, c, k - 1)
            kern[name][f"tflops_j{k - 1}"] = fl1 / (statistics.median(t_j15[kk]) * 1e-3) / 1e12
    dom = "bwd" if t_kind["b"] >= t_kind["f"] else "fwd"
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_burst, peak_sus = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
        peak_src = "MEASURED_PEAKS.json bf16_tflops (burst; sustained beside it)"
    except Exception:
        peak_burst, peak_sus = 1590.0, 1400.0
        peak_src = "fallback B200_PROFILING.md (1.59 PF burst, ~1.4 PF sustained)"
    achieved = kern[dom]["tflops"]
    if fp32:
        # SIMT FFMA debug kernels: 148 SMs x 128 fp32 lanes x 2 flop x 1.965 GHz
        roofline = {"bound": "alu", "achieved": achieved, "peak": 74.4, "unit": "TFLOP/s",
                    "frac": achieved / 74.4 if achieved else None, "traffic": None, "alg_bytes": None,
                    "kernel": "fp32 debug kernels (SECO_FP32_DEBUG)",
                    "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md unit counts)"}
    else:
        traffic = traffic_launch = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
            traffic = tr.get(dom, {}).get(args.config)
            traffic_launch = tr.get(dom, {}).get(args.config + "_launch")
        except Exception:
            pass
        jt = k - 1
        ab = (alg_bytes_bwd if dom == "bwd" else alg_bytes_fwd)(hq_r, hkv_r, d, c, jt)
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                    "frac": achieved / peak_burst if achieved else None,
                    "peak_sustained": peak_sus, "frac_of_sustained": achieved / peak_sus if achieved else None,
                    "traffic": traffic, "alg_bytes": ab,
                    "kernel": f"seco_chunk_{'backward' if dom == 'bwd' else 'forward'} "
                              + ("(bwd_prep + seco_bwd" + ("" if args.deterministic else "2")
                                 + "_sm100_kernel + bwd_final)" if dom == "bwd" else "(seco_fwd_sm100_kernel)"),
                    "peak_source": peak_src,
                    "traffic_note": f"traffic = DRAM bytes of the {traffic_launch} launch from ncu --set full "
                                    f"(profiles/roofline_traffic.json); alg_bytes = algorithmic bytes of the same "
                                    f"launch (j={jt}); achieved averages all launches of the step"}

    # ---------------------------------------------------------------- end to end (host buffers)
    # Every step: H2D of that step's Q, K, V, dO from pinned host memory, the step, D2H of its
    # dQ and dKV -- pipelined at chunk granularity.  Host and device tensors are sequence-major
    # ([S][h][d], the layout a projection produces; the ABI takes its strides), so a chunk is
    # one contiguous block: K/V/Q of chunk j are copied in stage-1 order and the forward of
    # chunk j waits only for them; dO arrives in stage-2 (descending) order; dQ_j and dKV slot
    # j (final once chunk j's backward or skip is done) go back while the earlier chunks
    # compute, dKV slot j as one 2-D copy (2 Hkv rows of c d floats).  Copies run on two copy
    # streams (both PCIe directions) and also overlap the neighbouring steps; two device buffer
    # sets alternate so a step never reads inputs or writes outputs still in flight.
    e2e = None
    if not args.no_e2e:
        from cuda.bindings import runtime as cudart
        del layer
        host = [t.transpose(0, 1).contiguous().pin_memory() for t in pinned]      # [S][h][d]
        sets = [tuple(torch.empty(t.shape, dtype=t.dtype, device=dev) for t in host) for _ in range(2)]
        layers = [ChunkedAttention(hq_r, hkv_r, d, seq, c, dtype=tdt, device=dev,
                                   deterministic=args.deterministic, layout="shd") for _ in range(2)]
        out_dq = [torch.empty(seq, hq_r, d, dtype=tdt).pin_memory() for _ in range(2)]
        out_dkv = [torch.empty(layers[0].dkv.shape, dtype=layers[0].dkv.dtype).pin_memory() for _ in range(2)]
        need_do = {op[1] for op in order if op[0] == "b"}      # chunks whose backward reads dO_j
        h2d = sum(t.numel() * t.element_size() for t in host[:3]) + \
            host[3].numel() * host[3].element_size() * len(need_do) // k
        d2h = out_dq[0].numel() * out_dq[0].element_size() + out_dkv[0].numel() * out_dkv[0].element_size()
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        done = [None, None]      # compute-finished event of the last step that used set b
        drained = [None, None]   # D2H-finished event of the last step that used set b
        stage2 = [op[1] for op in order if op[0] in "bz"]        # descending: every chunk, sampled or skipped
        slot_bytes = c * d * 4
        pitch = seq * d * 4

        def rows(t, j):
            return t[j * c:(j + 1) * c]

        def d2h_chunk(b, j):
            rows(out_dq[b], j).copy_(rows(layers[b].dq.transpose(0, 1), j), non_blocking=True)
            err, = cudart.cudaMemcpy2DAsync(out_dkv[b].data_ptr() + j * slot_bytes, pitch,
                                            layers[b].dkv.data_ptr() + j * slot_bytes, pitch, slot_bytes,
                                            2 * hkv_r, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost,
                                            s_out.cuda_stream)
            if err != cudart.cudaError_t.cudaSuccess:
                raise RuntimeError(f"cudaMemcpy2DAsync: {err}")

        def e2e_steps(n_steps, step0):
            """Enqueue n_steps pipelined end-to-end steps; returns the D2H-drained event of each."""
            ends = []
            for st_i in range(step0, step0 + n_steps):
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
                    for j in reversed(range(k)):             # stage-2 order; SpaCO: sampled chunks
                        if j in need_do:                     # only (a skipped chunk's dO is never read)
                            rows(dod, j).copy_(rows(host[3], j), non_blocking=True)
                        ev_do[j].record(s_in)
                if drained[b] is not None:
                    stream.wait_event(drained[b])
                qv, kv, vv, dov = (t.transpose(0, 1) for t in (qd, kd, vd, dod))
                lay.dkv.zero_()
                ev_out = {}
                for n_op, op in enumerate(order):
                    j = op[1]
                    if op[0] == "f":
                        if n_op < k:                         # stage 1: chunk j's K, V, Q have arrived
                            stream.wait_event(ev_qkv[j])
                        lay.forward_chunk(qv, kv, vv, j, chained=op[2])
                    elif op[0] == "b":
                        stream.wait_event(ev_do[j])
                        lay.backward_chunk(qv, kv, vv, dov, j, gamma, sscale)
                    else:
                        lay.skip_chunk(j)
                    if op[0] in "bz":
                        ev_out[j] = torch.cuda.Event()
                        ev_out[j].record(stream)
                done[b] = torch.cuda.Event()
                done[b].record(stream)
                with torch.cuda.stream(s_out):
                    for j in stage2:
                        s_out.wait_event(ev_out[j])
                        d2h_chunk(b, j)
                    drained[b] = torch.cuda.Event(enable_timing=True)
                    drained[b].record(s_out)
                ends.append(drained[b])
            return ends

        # untimed warm-up steps of the same pipeline (first-call costs of the copy paths)
        e2e_steps(max(args.warmup, 1), 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(s_in)
        stream.wait_event(e0)
        s_out.wait_event(e0)
        ends = e2e_steps(args.steps, max(args.warmup, 1))
        for ev in ends[-2:]:
            s_in.wait_event(ev)
        e1.record(s_in)
        torch.cuda.synchronize()
        # per-step completion intervals (D2H drained -> D2H drained), first one from e0
        e2e_per_step = [e0.elapsed_time(ends[0])] + [ends[i - 1].elapsed_time(ends[i]) for i in range(1, len(ends))]
        e2e_per_step = [max_over_ranks(v, coll_dev) for v in e2e_per_step]
        ems = max_over_ranks(e0.elapsed_time(e1), coll_dev)
        e2e = {"value": total_flops / (ems / args.steps * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": ems / args.steps, "ms_per_step_median": statistics.median(e2e_per_step),
               "ms_per_step_min": min(e2e_per_step), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "pinned host Q,K,V,dO ([S][h][d]) -> device per chunk in the order the step consumes "
                       "them (copy stream; SpaCO: dO only for the sampled chunks); SeCO/SpaCO chunk calls via the C "
                       "ABI, each waiting only for its "
                       "chunk's inputs; dQ_j, dKV slot j -> pinned host as soon as chunk j's backward (or "
                       "skip) is done (copy stream, dKV slot as one 2-D copy); steps double-buffered; W untimed "
                       "warm-up steps of the same pipeline first; per-step times = intervals between "
                       "consecutive steps' D2H completions"}
        del sets, layers

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the whole workload of one kv-head group (1 of Hkv independent groups), NumPy fp32
        dt, fl, desc, threads = cpu_oracle_run(cfg, k, sel, gamma, sscale)
        cpu = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": desc,
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ms_per_step_median": statistics.median(per_step), "ms_per_step_min": min(per_step),
            "higher_is_better": True,
            "scaling": "strong" if (args.shard == "heads" and world > 1) else "weak",
            "vs_baseline": None, "dtype": "f32" if fp32 else "bf16", "data": "synthetic",
            "config": config_block(args, cfg, world, sel, gamma),
            "tokens_per_s": tokens / (ms_per_step * 1e-3),
            "step_tflop": total_flops / 1e12,
            "value_at_median_step": total_flops / (statistics.median(per_step) * 1e-3) / 1e12,
            "roofline": roofline, "kernels": kern, "memory": memory,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
