# The paper-table view: kinoplan bench, 25 trials x 100 ms on the four headline scenes (run under gpurun).
set -e
mkdir -p gpurun_out/trials
for sc in forest_di6 narrow_dubins6 building_quad12 zigzag2d; do
  paper_2602_02846_b200/bin/kinoplan bench --scenario paper_2602_02846_b200/scenarios/$sc.json --out gpurun_out/trials/$sc --trials 25 --time-limit-ms 100 > gpurun_out/trials/$sc.log 2>&1
done
ls gpurun_out/trials
