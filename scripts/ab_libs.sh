#!/bin/bash
# A/B builds of the library: bash scripts/ab_libs.sh DIR SCENES...  (DIR holds lib_<name>.so variants)
D=$1; shift
L=paper_2602_02846_b200/lib/libkinoplan_b200.so
cp $L /tmp/lib_cur.so
for r in 1 2; do
  for f in $D/lib_*.so; do
    cp $f $L
    echo "== $(basename $f .so) (round $r)"
    python scripts/ab_perf.py "$@"
  done
done
cp /tmp/lib_cur.so $L
