# Forward split-KV A/B (DP + split tail): forward parity subset, then per-call times
# at cfg3 for forced split factors (1 = never split, 0 = the cost model) and cfg3p8 (sub-wave).
# usage: bash tools/ab_fwd_split.sh  (on the GPU box, e.g. via gpurun)
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "forward or split or pair or rebuild" 2>&1 | tail -5
for r in 1 2; do for v in 1 0 2 3 4; do echo "== nsplit=$v round $r"; SECO_FWD_NSPLIT=$v python tools/kbench.py cfg3 3,7,11,15 10 2>&1 | grep fwd; done; done
for v in 1 0; do echo "== cfg3p8 nsplit=$v"; SECO_FWD_NSPLIT=$v python tools/kbench.py cfg3p8 1,3,7,15 10 2>&1 | grep fwd; done
