"""Work counters of a profiled solve: python scripts/prof_counters.py SCENE [BUDGET_S]"""
import sys
sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

scene = sys.argv[1]
b = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
with Planner(scenarios.load(scene), seed=0) as g:
    g.set_profiling(True)
    r = g.solve(budget_s=b)
    p = g.profile()
it = r["iterations"]
print(scene, "iterations", it, "nodes", r["node_count"], "committed", r["nodes_committed"])
for k in ("items", "rk4_steps", "interp_points", "box_tests", "live_scanned", "ancestor_hops", "slots_scanned",
          "admitted_checked"):
    print(f"  {k:18s} {p[k]:14d}  per-iteration {p[k] / it:12.1f}")
print("  hops per live", p["ancestor_hops"] / max(1, p["live_scanned"]))
print("  t_prop/sel/scat per it (us)", *(round(p[k] / it * 1e6, 1) for k in ("t_propagate_s", "t_select_s", "t_scatter_s")))
