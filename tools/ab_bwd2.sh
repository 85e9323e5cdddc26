# Backward v2 (SECO_BWD_V2=1) vs v1: parity (bf16 GPU tests under v2), per-call timing alternated,
# and the v2 clock64 trace (libseco_trace.so).
SECO_BWD_V2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "bf16_seco_step or chunk_calls or spaco or strided" 2>&1 | tail -3
echo "parity rc=$?"
for r in 1 2; do
  for v in 0 1; do echo "== v2=$v $r"; SECO_BWD_V2=$v timeout 300 python tools/kbench.py cfg3 3,7,15 10 | grep bwd; done
done
SECO_BWD_V2=1 SECO_LIB_VARIANT=libseco_trace.so timeout 300 python tools/trace_bwd2.py 15 | head -14
