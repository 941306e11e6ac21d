#!/bin/bash
# One GPU session: peaks, tests, smoke, bench (+reference arm), ncu launch list + full captures.
# Usage (under gpurun): bash scripts/gpu_round.sh TAG
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
./tools/fp32_peak > $OUT/fp32_peak.json 2> $OUT/fp32_peak.err
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
for cfg in narrow_dubins6 building_quad12; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for cfg in building_quad12 narrow_dubins6 forest_di6; do
  timeout 600 python bench.py --sweep --config $cfg --steps 5 --warmup 3 > $OUT/sweep_$cfg.json 2> $OUT/sweep_$cfg.err
done
timeout 600 python bench.py --batch 64 --lanes 8 > $OUT/bench_batch.json 2> $OUT/bench_batch.err
python scripts/trace_gpu.py forest_di6 > $OUT/trace_forest_di6.txt 2>&1
python scripts/trace_gpu.py building_quad12 1.0 > $OUT/trace_building_quad12.txt 2>&1
python scripts/trace_gpu.py narrow_dubins6 > $OUT/trace_narrow_dubins6.txt 2>&1
# launch list of the bench command itself (first 400 launches: the warm-up queries; same command first without ncu)
BCMD="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --dist-seeds 0"
timeout 600 $BCMD > $OUT/plain_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv $BCMD > $OUT/ncu_bench.log 2>&1
# launch list of a fixed-iteration query (the same command first without ncu)
PCMD="python scripts/prof_run.py forest_di6 60"
timeout 300 $PCMD > $OUT/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_forest_di6.csv $PCMD > $OUT/ncu_launch.log 2>&1
# full captures of the steady-state kernels
for spec in "forest_di6 40" "building_quad12 30" "narrow_dubins6 40"; do
  set -- $spec
  timeout 300 python scripts/prof_run.py $1 $2 > $OUT/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s $(( $2 - 3 )) -c 1 \
     -o $OUT/prop_$1 -f python scripts/prof_run.py $1 $2 > $OUT/ncu_prop_$1.log 2>&1
done
# the saturated Quad12 propagate (BASELINE config 5 at 2^22 items)
timeout 300 python scripts/prof_sweep.py building_quad12 22 > $OUT/plain_sweep.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 2 -c 1 \
   -o $OUT/prop_sweep_building_quad12 -f python scripts/prof_sweep.py building_quad12 22 > $OUT/ncu_sweep.log 2>&1
timeout 300 python scripts/prof_sweep.py narrow_dubins6 22 > $OUT/plain_sweep_dubins.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 2 -c 1 \
   -o $OUT/prop_sweep_narrow_dubins6 -f python scripts/prof_sweep.py narrow_dubins6 22 > $OUT/ncu_sweep_dubins.log 2>&1
timeout 300 python scripts/prof_run.py forest_di6 40 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 74 -c 2 \
   -o $OUT/sel_forest_di6 -f python scripts/prof_run.py forest_di6 40 > $OUT/ncu_sel.log 2>&1
echo done
