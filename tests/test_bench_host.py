"""bench.py host-side contract (no GPU): the reference arm's JSON line and the bounded
oracle sample sizing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2505_16710_b200.flops import seco_step_flops  # noqa: E402


def test_oracle_sample_shape_is_bounded_and_maximal():
    for name, cfg in bench.CONFIGS.items():
        G, c, d = cfg["hq"] // cfg["hkv"], cfg["chunk"], cfg["d"]
        k = cfg["seq"] // c
        for target in (5e9, 0.15e12, 1e12):
            groups, n = bench.oracle_sample_shape(cfg, target)
            assert 1 <= n <= k and 1 <= groups <= cfg["hkv"]
            fl = seco_step_flops(G * groups, d, n * c, c)
            assert fl <= target or (n == 1 and groups == 1)
            if n < k:                      # one more chunk would exceed the budget
                assert seco_step_flops(G, d, (n + 1) * c, c) > target


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg2",
                          "--steps", "1", "--warmup", "0", "--oracle-gflop", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "TFLOP/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("cfg2")


def test_bench_gpus_n_spawns_n_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 local ranks
    (torch.distributed.run); --dry-run takes the same N-rank path on CPU (gloo): head shards,
    barrier, max-over-ranks time, one JSON line from rank 0."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--config", "cfg3", "--mode", "spaco", "--sampler", "bernoulli"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["dry_run"] and line["n_gpus"] == 2
    assert line["shards"] == [{"q_heads": [0, 16], "kv_heads": [0, 4]}, {"q_heads": [16, 32], "kv_heads": [4, 8]}]
    assert line["ms_max_over_ranks"] == 11.0          # rank 1's stand-in time: the max is taken
    assert line["config"]["parallelism"] == "heads2" and line["config"]["sampler"] == "bernoulli"
