set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
L=paper_2602_02846_b200/lib/libkinoplan_b200.so; cp $L /tmp/lib_cur.so
for r in 1 2; do
for f in abtmp/lib_*.so; do
  cp $f $L; n=$(basename $f .so)
  echo "== $n (round $r)" >> $OUT/ab.log
  timeout 300 python scripts/ab_perf.py forest_di6 narrow_dubins6 >> $OUT/ab.log 2>&1
  timeout 300 python scripts/wall_probe.py forest_di6 >> $OUT/ab.log 2>&1
done
done
cp /tmp/lib_cur.so $L
echo done
