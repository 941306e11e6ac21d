#!/bin/bash
# ncu --set full captures of k_propagate: headline iteration + saturated sweep (each run first without ncu)
set -u
TAG=${1:-x}
OUT=gpurun_out
mkdir -p $OUT
python scripts/prof_run.py forest_di6 40 > $OUT/plain_it_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 37 -c 1 \
   -o $OUT/prop_it_$TAG -f python scripts/prof_run.py forest_di6 40 > $OUT/ncu_it_$TAG.log 2>&1
python scripts/prof_sweep.py forest_di6 20 > $OUT/plain_sw_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 2 -c 1 \
   -o $OUT/prop_sw_$TAG -f python scripts/prof_sweep.py forest_di6 20 > $OUT/ncu_sw_$TAG.log 2>&1
echo done
