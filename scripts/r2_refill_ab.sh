set -u
TAG=${1:-x}; OUT=gpurun_out/$TAG; mkdir -p $OUT
L=paper_2602_02846_b200/lib/libkinoplan_b200.so; cp $L /tmp/lib_cur.so
cp abtmp/lib_new.so $L
KP_REFILL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/parity_refill.log 2>&1; echo "rc=$?" >> $OUT/parity_refill.log
for v in "head:" "new:KP_REFILL=0" "new:KP_REFILL=1" "new:KP_REFILL=1 KP_FLAT_MAX=0"; do
  lib=${v%%:*}; envs=${v#*:}
  cp abtmp/lib_$lib.so $L
  echo "== $lib $envs" >> $OUT/ab.log
  env $envs timeout 120 python scripts/prof_sweep.py building_quad12 22 >> $OUT/ab.log 2>&1
  env $envs timeout 120 python scripts/prof_sweep.py narrow_dubins6 22 >> $OUT/ab.log 2>&1
  env $envs timeout 300 python scripts/ab_perf.py building_quad12 narrow_dubins6 forest_di6 >> $OUT/ab.log 2>&1
  env $envs timeout 120 python scripts/trace_gpu.py building_quad12 0.2 > $OUT/trace_quad_${lib}_$(echo $envs | tr ' =' '__').txt 2>&1
done
cp /tmp/lib_cur.so $L
echo done
