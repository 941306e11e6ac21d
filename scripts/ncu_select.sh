#!/bin/bash
# ncu full capture of select_reduce / select_scatter at forest_di6 iteration 15
set -u
OUT=gpurun_out/sel15
mkdir -p $OUT
python scripts/prof_run.py forest_di6 16 > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 28 -c 2 \
   -o $OUT/sel15 -f python scripts/prof_run.py forest_di6 16 > $OUT/ncu.log 2>&1
echo done
