"""A/B step timing of environment settings for the same library (alternating processes).
usage: python tools/ab_step_env.py cfg3 "SECO_BWD_V2=0" "SECO_BWD_V2=1" [rounds]"""
import os
import subprocess
import sys

cfg, envs = sys.argv[1], sys.argv[2:4]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {e: [] for e in envs}
for r in range(rounds):
    for e in envs:
        env = dict(os.environ)
        for kv in e.split():
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "step_time.py"), cfg], env=env,
                             capture_output=True, text=True)
        line = (out.stdout.strip().splitlines() or ["?"])[-1]
        print(f"round {r} {e}: {line}", flush=True)
        try:
            res[e].append(float(line.split("ms/step")[0].split(":")[-1]))
        except ValueError:
            pass
for e, ts in res.items():
    if ts:
        ts = sorted(ts)
        print(f"{cfg} {e}: median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f} ms  ({len(ts)} runs)")
