#!/bin/bash
# A/B of environment-variable variants (KP_FLAT_MAX, KP_PROP_GRID, KP_SEL_GRID, ...)
# on the same library, two rounds each, with ab_perf.py:
#   bash scripts/ab_env.sh TAG "SCENES" "ENV=a" "ENV=b ENV2=c" ...   (under gpurun)
set -u
TAG=$1; SCENES=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in 1 2; do
k=0
for v in "$@"; do
  echo "== variant $k [$v] (round $r)" >> $OUT/ab.log
  env $v timeout 300 python scripts/ab_perf.py $SCENES >> $OUT/ab.log 2>&1
  k=$((k+1))
done
done
echo done
