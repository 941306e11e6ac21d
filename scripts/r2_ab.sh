# A/B of env-selectable variants + parity tests: bash scripts/r2_ab.sh TAG ["ENV=a ENV=b" ...]
# each extra argument is a set of environment assignments for one variant ("" = default)
set -u
TAG=${1:-x}; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/parity.log 2>&1; echo "parity rc=$?" >> $OUT/parity.log
k=0
for v in "${@:-}"; do
  echo "variant $k: $v" > $OUT/ab_$k.log
  env $v timeout 300 python scripts/ab_perf.py forest_di6 narrow6d zigzag6d building6d >> $OUT/ab_$k.log 2>&1
  env $v timeout 120 python scripts/trace_gpu.py forest_di6 > $OUT/trace_$k.txt 2>&1
  k=$((k+1))
done
if [ -d abtmp ]; then timeout 600 bash scripts/ab_libs.sh abtmp forest_di6 narrow6d > $OUT/ab_libs.log 2>&1; fi
echo done
