# A/B of environment variants on given scenes: bash scripts/r2_env_ab.sh TAG "SCENES" "ENV..." ...
set -u
TAG=$1; SCENES=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in 1 2; do
k=0
for v in "$@"; do
  echo "== variant $k [$v] (round $r)" >> $OUT/ab.log
  env $v timeout 300 python scripts/ab_perf.py $SCENES >> $OUT/ab.log 2>&1
  k=$((k+1))
done
done
echo done
