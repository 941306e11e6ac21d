#!/bin/bash
# A/B of library builds abtmp/lib_*.so with parity tests on each build first:
# bash scripts/ab_libs3.sh TAG SCENES...   (two perf rounds, builds interleaved)
set -u
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
L=paper_2602_02846_b200/lib/libkinoplan_b200.so; cp $L /tmp/lib_cur.so
for f in abtmp/lib_*.so; do
  cp $f $L; n=$(basename $f .so)
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/parity_$n.log 2>&1; echo "parity $n rc=$?" >> $OUT/ab.log
done
for r in 1 2; do
for f in abtmp/lib_*.so; do
  cp $f $L; n=$(basename $f .so)
  echo "== $n (round $r)" >> $OUT/ab.log
  timeout 300 python scripts/ab_perf.py "$@" >> $OUT/ab.log 2>&1
done
done
cp /tmp/lib_cur.so $L
echo done
