"""Prune-pass work of one query: live nodes scanned, ancestor hops, items
(python scripts/prune_stats.py SCENE [BUDGET_S])."""
import sys

sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

scene = sys.argv[1] if len(sys.argv) > 1 else "forest_di6"
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
with Planner(scenarios.load(scene), seed=1000) as g:
    g.reset(1000)
    p0 = g.profile()
    r = g.solve(budget)
    p1 = g.profile()
    d = {k: p1[k] - p0[k] for k in p1 if isinstance(p1[k], (int, float))}
    it = r["iterations"]
    print(scene, "iterations", it, "items/it %.0f" % (d["items"] / it), "live/it %.0f" % (d["live_scanned"] / it),
          "hops/it %.0f" % (d["ancestor_hops"] / it), "frontier/it %.0f" % (d["items"] / it / 32))
