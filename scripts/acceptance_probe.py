"""Probe the bundled scenes on the GPU: success / first / final cost over a
few seeds at two budgets (sizing the acceptance tests)."""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2602_02846_b200 import planner, scenarios  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(scenarios.BUILDERS)
budgets = [float(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0.1, 1.0]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16
for name in names:
    s = scenarios.load(name)
    for b in budgets:
        t0 = time.time()
        bp = planner.BatchPlanner(s, lanes=8)
        res, wall = bp.solve(range(n), budget_s=b)
        bp.close()
        ok = [r for r in res if r["found"]]
        row = {"scene": name, "budget_s": b, "n": n, "success": len(ok),
               "ttfs_ms_med": statistics.median([r["first_solution_s"] * 1e3 for r in ok]) if ok else None,
               "first_med": statistics.median([r["first_solution_cost"] for r in ok]) if ok else None,
               "final_med": statistics.median([r["best_cost"] for r in ok]) if ok else None,
               "iters_med": statistics.median([r["iterations"] for r in res]),
               "props_med": statistics.median([r["propagations_attempted"] for r in res]),
               "cap_ex": sum(bool(r["capacity_exhausted"]) for r in res),
               "nodes_med": statistics.median([r["node_count"] for r in res]),
               "wall_s": round(time.time() - t0, 2)}
        print(json.dumps(row), flush=True)
