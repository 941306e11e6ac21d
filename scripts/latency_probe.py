"""Propagate-kernel latency at tiny sizes (synthetic frontier), with and without obstacles."""
import sys
sys.path.insert(0, '.')
from paper_2602_02846_b200 import Planner, scenarios

for scene in ("forest_di6", "building_quad12"):
    for obst in (True, False):
        s = scenarios.load(scene)
        if not obst:
            s["problem"]["environment"]["obstacles"] = []
        with Planner(s, seed=1) as g:
            g.sweep(4, launches=3)
            row = []
            for n in (1, 4, 32, 256, 1024, 4096):
                ms, one = g.sweep(n, launches=20)
                row.append(f"n={n * 32}: {ms * 1e3:6.1f}us steps/item={one['rk4_steps'] / one['items']:.1f}")
            print(scene, "obstacles" if obst else "empty", " | ".join(row))
