#!/bin/bash
# in-graph trace summaries for each library variant: bash scripts/ab_trace.sh DIR SCENES...
D=$1; shift
L=paper_2602_02846_b200/lib/libkinoplan_b200.so
cp $L /tmp/lib_cur.so
for f in $D/lib_*.so; do
  cp $f $L
  for s in "$@"; do
    echo "== $(basename $f .so) $s"
    python scripts/trace_gpu.py $s 2>&1 | grep -E "^mean|iterations"
  done
done
cp /tmp/lib_cur.so $L
