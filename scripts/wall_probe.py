"""Host wall clock of stop-at-first-solution solves and of 100 ms queries
(C-ABI, includes launch / tail overheads): python scripts/wall_probe.py SCENE"""
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

scene = sys.argv[1] if len(sys.argv) > 1 else "forest_di6"
s = scenarios.load(scene)
with Planner(s, seed=0) as g:
    g.set_stop_at_first_solution(True)
    walls, dev = [], []
    for sd in range(12):
        g.reset(sd)
        t = time.perf_counter()
        r = g.solve(1.0, 0)
        w = time.perf_counter() - t
        if sd >= 2:
            walls.append(w * 1e3)
            dev.append(r["first_solution_s"] * 1e3)
    g.set_stop_at_first_solution(False)
    q = []
    for sd in range(5):
        g.reset(100 + sd)
        t = time.perf_counter()
        r = g.solve(0.1, 0)
        q.append((time.perf_counter() - t) * 1e3)
print(f"{scene}: stop-first wall {statistics.median(walls):.3f} ms (device ttfs {statistics.median(dev):.3f}), "
      f"100 ms query wall {statistics.median(q):.2f} ms")
