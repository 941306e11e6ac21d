"""Propagate sweep for ncu captures: python scripts/prof_sweep.py SCENE LOG2_ITEMS [LAUNCHES]"""
import sys
sys.path.insert(0, '.')
from paper_2602_02846_b200 import Planner, scenarios

scene, k = sys.argv[1], int(sys.argv[2])
launches = int(sys.argv[3]) if len(sys.argv) > 3 else 3
s = scenarios.load(scene, capacity=1 << 22, max_slots=1 << 23)
lam = s["planner"].get("lambda", 32)
with Planner(s, seed=1) as g:
    ms, pr = g.sweep((1 << k) // lam, launches=launches)
    print(scene, k, f"{ms:.4f} ms/launch", f"{(1 << k) / ms / 1e6:.3f} G items/s")
