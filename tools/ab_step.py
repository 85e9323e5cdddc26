"""A/B step timing of library variants (SECO_LIB_VARIANT .so files in the package dir),
alternated in separate processes so the power-capped clock state is shared fairly.
usage: python tools/ab_step.py cfg3 libseco_base.so,libseco.so [rounds] [ENV=VAL ...per variant via 'lib.so:ENV=VAL']"""
import os
import subprocess
import sys

cfg = sys.argv[1]
variants = sys.argv[2].split(",")
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        lib, *envs = v.split(":")
        env = dict(os.environ, SECO_LIB_VARIANT=lib)
        for e in envs:
            k, val = e.split("=")
            env[k] = val
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "step_time.py"), cfg], env=env,
                             capture_output=True, text=True)
        line = (out.stdout.strip().splitlines() or ["?"])[-1]
        if out.returncode:
            line += " ERR " + out.stderr[-500:]
        print(f"round {r} {v}: {line}", flush=True)
        try:
            res[v].append(float(line.split("ms/step")[0].split(":")[-1]))
        except ValueError:
            pass
for v, ts in res.items():
    if ts:
        ts = sorted(ts)
        print(f"{cfg} {v}: median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f} ms  ({len(ts)} runs)")
