# A/B per-call forward/backward timing of two library variants, alternated (usage: bash tools/ab_kbench.sh libA.so libB.so cfg js reps)
for r in 1 2; do
  for lib in $1 $2; do
    echo "== $lib round $r"; SECO_LIB_VARIANT=$lib python tools/kbench.py $3 $4 $5
  done
done
