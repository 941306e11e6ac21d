#!/bin/bash
# ncu full captures of steady-state kernels (each run first without ncu)
set -u
TAG=${1:-x}
OUT=gpurun_out
mkdir -p $OUT
for spec in "forest_di6 40" "building_quad12 30"; do
  set -- $spec
  python scripts/prof_run.py $1 $2 > $OUT/plain_${1}_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s $(( $2 - 3 )) -c 1 \
     -o $OUT/prop_${1}_$TAG -f python scripts/prof_run.py $1 $2 > $OUT/ncu_prop_${1}_$TAG.log 2>&1
done
python scripts/prof_run.py forest_di6 40 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 74 -c 2 \
   -o $OUT/sel_forest_di6_$TAG -f python scripts/prof_run.py forest_di6 40 > $OUT/ncu_sel_$TAG.log 2>&1
echo done
