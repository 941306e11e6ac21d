#!/bin/bash
# latency probe for each library variant: bash scripts/ab_latency.sh DIR
D=$1; shift
L=paper_2602_02846_b200/lib/libkinoplan_b200.so
cp $L /tmp/lib_cur.so
for f in $D/lib_*.so; do
  cp $f $L
  echo "== $(basename $f .so)"
  python scripts/latency_probe.py
done
cp /tmp/lib_cur.so $L
