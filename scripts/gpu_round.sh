#!/bin/bash
# One GPU session: tests, smoke, peaks, bench, ncu launch list + full capture.
# Usage (under gpurun): bash scripts/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
./tools/fp32_peak > $OUT/fp32_peak_$TAG.json 2> $OUT/fp32_peak_$TAG.err
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
#timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
PCMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --iters 60"
timeout 300 $PCMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_$TAG.csv $PCMD > $OUT/ncu_launch_$TAG.log 2>&1
timeout 300 $PCMD > $OUT/plain2_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 40 -c 2 -o $OUT/prof_prop_$TAG -f $PCMD > $OUT/ncu_full_$TAG.log 2>&1
timeout 300 $PCMD > $OUT/plain3_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_select -s 40 -c 4 -o $OUT/prof_sel_$TAG -f $PCMD > $OUT/ncu_sel_$TAG.log 2>&1
echo done
