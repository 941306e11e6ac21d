#!/bin/bash
# ncu capture of a single-warp propagate (latency anatomy): bash scripts/ncu_small.sh TAG [LOG2_ITEMS]
set -u
TAG=${1:-x}; K=${2:-5}
OUT=gpurun_out
mkdir -p $OUT
python scripts/prof_sweep.py forest_di6 $K > $OUT/plain_small_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 2 -c 1 \
   --warp-sampling-interval 0 -o $OUT/small_$TAG -f python scripts/prof_sweep.py forest_di6 $K > $OUT/ncu_small_$TAG.log 2>&1
echo done
