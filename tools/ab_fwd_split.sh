set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "forward or split or pair or rebuild" 2>&1 | tail -5
for r in 1 2; do for v in 1 0 2 3 4; do echo "== nsplit=$v round $r"; SECO_FWD_NSPLIT=$v python tools/kbench.py cfg3 3,7,11,15 10 2>&1 | grep fwd; done; done
