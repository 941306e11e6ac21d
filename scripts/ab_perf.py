"""Quick A/B perf probe: sweep throughput + 100 ms query rate + TTFS.
python scripts/ab_perf.py SCENE [SCENE...]   (env KP_ENV_MODE=cells for the cell-list broad phase)"""
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

mode = os.environ.get("KP_ENV_MODE", "slab")
for scene in sys.argv[1:]:
    s = scenarios.load(scene, capacity=1 << 22, max_slots=1 << 23)
    lam = s["planner"]["lambda"]
    with Planner(s, seed=1) as g:
        g.sweep((1 << 20) // lam, launches=2)
        ms, pr = g.sweep((1 << 20) // lam, launches=10)
    s = scenarios.load(scene)
    rates, ttfs = [], []
    with Planner(s, seed=0) as g:
        for seed in range(6):
            g.reset(seed)
            r = g.solve(budget_s=0.1)
            if seed:
                rates.append(r["propagations_attempted"] / r["elapsed_s"])
                if r["found"]:
                    ttfs.append(r["first_solution_s"] * 1e3)
    print(f"{scene:16s} {mode:5s} sweep {(1 << 20) / ms / 1e6:6.2f} G items/s  query {statistics.median(rates) / 1e9:5.2f} G/s"
          f"  ttfs {statistics.median(ttfs) if ttfs else float('nan'):6.2f} ms  steps/item {pr['rk4_steps'] / pr['items']:.2f}"
          f" box {pr['box_tests'] / pr['items']:.2f} look {pr.get('slab_lookups', 0) / pr['items']:.2f}", flush=True)
