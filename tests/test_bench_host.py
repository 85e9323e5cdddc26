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
