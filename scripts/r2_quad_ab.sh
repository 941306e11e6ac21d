set -u
TAG=${1:-x}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "quad or dubins or building or narrow" > $OUT/parity.log 2>&1; echo "parity rc=$?" >> $OUT/parity.log
L=paper_2602_02846_b200/lib/libkinoplan_b200.so; cp $L /tmp/lib_cur.so
for f in abtmp/lib_*.so; do
  cp $f $L
  echo "== $(basename $f .so)" >> $OUT/ab.log
  for k in 20 22; do timeout 120 python scripts/prof_sweep.py building_quad12 $k >> $OUT/ab.log 2>&1; done
  timeout 120 python scripts/prof_sweep.py narrow_dubins6 22 >> $OUT/ab.log 2>&1
  timeout 300 python scripts/ab_perf.py building_quad12 narrow_dubins6 forest_di6 >> $OUT/ab.log 2>&1
done
cp /tmp/lib_cur.so $L
echo done
if [ -n "${NCU_LIB:-}" ]; then
  cp abtmp/$NCU_LIB $L
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 2 -c 1 \
     -o $OUT/prop_sw_quad -f python scripts/prof_sweep.py building_quad12 22 > $OUT/ncu_sw.log 2>&1
  cp /tmp/lib_cur.so $L
fi
