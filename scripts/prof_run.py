"""Fixed-iteration planner run for ncu captures: python scripts/prof_run.py SCENE ITERS [SEED]"""
import sys
sys.path.insert(0, '.')
from paper_2602_02846_b200 import Planner, scenarios

scene, iters = sys.argv[1], int(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
with Planner(scenarios.load(scene), seed=seed) as g:
    r = g.solve(0.0, iters)
    print(scene, {k: r[k] for k in ('iterations', 'propagations_attempted', 'node_count', 'found', 'best_cost')})
