set -u
TAG=${1:-x}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python scripts/prof_run.py forest_di6 40 > $OUT/plain_it.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 37 -c 1 \
   -o $OUT/sel_it -f python scripts/prof_run.py forest_di6 40 > $OUT/ncu_sel.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_select -c 60 --csv \
   --log-file $OUT/sel_launches.csv python scripts/prof_run.py forest_di6 40 > $OUT/ncu_sel2.log 2>&1
echo done
