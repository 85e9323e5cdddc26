# Parity (bf16 GPU tests) and A/B timing of a library variant against libseco.so, alternated.
# usage: bash tools/ab_variant.sh libseco_<name>.so [cfg] [js]
V=$1; CFG=${2:-cfg3}; JS=${3:-3,7,15}
SECO_LIB_VARIANT=$V timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k bf16 > gpurun_out/par_$V.log 2>&1; echo "parity $V rc=$?"
for r in 1 2; do for v in libseco.so $V; do echo "== $v $r"; SECO_LIB_VARIANT=$v python tools/kbench.py $CFG $JS 20; done; done
python tools/ab_step.py $CFG libseco.so,$V 3
