"""Host wall clock of kp_reset_query and of a stop-at-first-solution kp_solve beside the device time to first solution: python scripts/wall_split.py"""
import statistics, sys, time
sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios
s = scenarios.load("forest_di6")
x0 = s["problem"]["x_init"]
with Planner(s, seed=0) as g:
    g.set_stop_at_first_solution(True)
    for sd in range(3):
        g.reset(sd, x_init=x0); g.solve(1.0, 0)
    tr, ts, td, tt = [], [], [], []
    for sd in range(40):
        t0 = time.perf_counter()
        g.reset(sd, x_init=x0)
        t1 = time.perf_counter()
        r = g.solve(1.0, 0)
        t2 = time.perf_counter()
        tr.append((t1 - t0) * 1e3); ts.append((t2 - t1) * 1e3); td.append(r["first_solution_s"] * 1e3)
    print("reset %.3f ms, solve %.3f ms, device ttfs %.3f ms" % (statistics.median(tr), statistics.median(ts), statistics.median(td)))
