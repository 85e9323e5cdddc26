# Backward v2 (SECO_BWD_V2=1) variants vs v1: parity on the bf16 GPU tests, then per-call timing.
# usage: bash tools/ab_bwd2.sh [variant.so ...]   (each run with SECO_BWD_V2=1; libseco.so with 0 = v1)
for lib in "$@"; do
  SECO_LIB_VARIANT=$lib SECO_BWD_V2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16_seco_step or chunk_calls or spaco" 2>&1 | tail -2
  echo "parity $lib rc=$?"
done
for r in 1 2; do
  echo "== v1 $r"; SECO_BWD_V2=0 timeout 300 python tools/kbench.py cfg3 3,7,15 10 | grep bwd
  for lib in "$@"; do echo "== $lib $r"; SECO_LIB_VARIANT=$lib SECO_BWD_V2=1 timeout 300 python tools/kbench.py cfg3 3,7,15 10 | grep bwd; done
done
