# Backward v2 (SECO_BWD_V2=1) vs v1: parity on the bf16 GPU tests, then per-call and step timing.
export CUDA_LAUNCH_BLOCKING=0
SECO_BWD_V2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16_seco_step or chunk_calls or spaco" 2>&1 | tail -15
echo "parity rc=$?"
for r in 1 2; do
  for v in 0 1; do echo "== v2=$v $r"; SECO_BWD_V2=$v timeout 300 python tools/kbench.py cfg3 3,7,15 10 | grep bwd; done
done
