# A/B per-call timing: libseco.so vs a variant library, alternated (usage: bash tools/ab_lib_kbench.sh libseco_x.so [cfg] [js])
V=$1; CFG=${2:-cfg3}; JS=${3:-3,7,15}
for r in 1 2; do
  echo "== libseco.so $r"; python tools/kbench.py $CFG $JS 10 | grep -E "fwd|bwd"
  echo "== $V $r"; SECO_LIB_VARIANT=$V python tools/kbench.py $CFG $JS 10 | grep -E "fwd|bwd"
done
