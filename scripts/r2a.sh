set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
python bench.py --sweep --config building_quad12 --steps 5 --warmup 3 > $OUT/sweep_quad.json 2> $OUT/sweep_quad.err
python bench.py --sweep --config narrow_dubins6 --steps 5 --warmup 3 > $OUT/sweep_dubins.json 2> $OUT/sweep_dubins.err
python scripts/prof_sweep.py building_quad12 22 > $OUT/plain_sw.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 2 -c 1 \
   -o $OUT/prop_sw_quad -f python scripts/prof_sweep.py building_quad12 22 > $OUT/ncu_sw.log 2>&1
echo done
