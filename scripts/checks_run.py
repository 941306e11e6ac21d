"""Short planner runs touching every kernel (for the `make checks` build): python scripts/checks_run.py [ITERS]
Every kernel of the library is exercised: reset, propagate/select/scatter (graph
path and profiled launches), debug propagate, path extraction + re-integration,
sweep, batch engine."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2602_02846_b200 import BatchPlanner, Planner, scenarios  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for name in ("forest_di6", "narrow_dubins6", "building_quad12", "zigzag2d"):
    s = scenarios.load(name, capacity=1 << 16, max_slots=1 << 21)
    with Planner(s, seed=3) as g:
        r = g.solve(0.0, it)
        g.set_profiling(True)
        g.solve(0.0, 2)
        g.set_profiling(False)
        if r["found"]:
            g.path()
            g.trajectory()
        nd = g.nodes()
        k = min(64, len(nd["acc"]))
        g.debug_propagate(nd["state"][:k], nd["acc"][:k], np.arange(k), np.zeros(k), 1)
        g.sweep(64, launches=1)
        print(name, "ok", r["iterations"], r["node_count"], r["found"], flush=True)
b = BatchPlanner(scenarios.load("forest_di6", capacity=1 << 16, max_slots=1 << 21), lanes=2)
res, _ = b.solve([1, 2, 3], budget_s=0.0, max_iterations=it)
b.close()
print("batch ok", [r["iterations"] for r in res])
