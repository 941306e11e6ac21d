set -u
TAG=${1:-x}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python scripts/prof_run.py forest_di6 40 > $OUT/plain_it.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 37 -c 1 \
   -o $OUT/prop_it -f python scripts/prof_run.py forest_di6 40 > $OUT/ncu_it.log 2>&1
echo done
