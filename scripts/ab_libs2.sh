#!/bin/bash
# A/B of library builds abtmp/lib_*.so (two rounds: ab_perf + a forest trace;
# parity tests on the current library first): bash scripts/ab_libs2.sh TAG SCENES...
set -u
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/parity.log 2>&1; echo "parity rc=$?" >> $OUT/parity.log
L=paper_2602_02846_b200/lib/libkinoplan_b200.so; cp $L /tmp/lib_cur.so
for r in 1 2; do
for f in abtmp/lib_*.so; do
  cp $f $L; n=$(basename $f .so)
  echo "== $n (round $r)" >> $OUT/ab.log
  timeout 300 python scripts/ab_perf.py "$@" >> $OUT/ab.log 2>&1
  [ $r = 1 ] && timeout 120 python scripts/trace_gpu.py forest_di6 > $OUT/trace_$n.txt 2>&1
done
done
cp /tmp/lib_cur.so $L
echo done
