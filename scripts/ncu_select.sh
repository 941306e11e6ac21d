#!/bin/bash
# ncu full captures of select_reduce / select_scatter at a large steady-state iteration
# usage: bash scripts/ncu_select.sh TAG [SCENE ITERS]
set -u
TAG=${1:-x}; SCENE=${2:-forest_di6}; IT=${3:-40}
OUT=gpurun_out
mkdir -p $OUT
python scripts/prof_run.py $SCENE $IT > $OUT/plain_sel_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s $(( 2 * IT - 6 )) -c 2 \
   -o $OUT/sel_$TAG -f python scripts/prof_run.py $SCENE $IT > $OUT/ncu_sel_$TAG.log 2>&1
echo done
