"""Per-iteration device trace of one query (graph mode, no profiler)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2602_02846_b200 import Planner, scenarios

scene = sys.argv[1] if len(sys.argv) > 1 else 'forest_di6'
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
s = scenarios.load(scene)
with Planner(s, seed=1000) as g:
    for w in range(3):
        g.reset(50 + w); g.solve(budget)
    g.reset(1000)
    r = g.solve(budget)
    tr = g.trace()
    t = tr['t_ns'].astype(np.float64) / 1e3
    d = np.diff(np.concatenate([[0.0], t]))
    print(scene, 'iterations', r['iterations'], 'first sol it', r['first_solution_iteration'], 'ttfs_ms', r['first_solution_s'] * 1e3)
    print('it  dt_us  items  live  frontier  nodes  committed')
    for k in list(range(0, min(40, len(tr)))) + list(range(40, len(tr), max(1, len(tr) // 30))):
        e = tr[k]
        print(f"{e['iteration']:5d} {d[k]:7.1f} {e['items']:8d} {e['live']:7d} {e['frontier']:7d} {e['nodes']:8d} {e['committed']:6d}")
    big = tr['items'] > 100000
    print('mean dt_us small(<2k items): %.1f' % d[tr['items'] < 2000].mean(), ' large(>100k): %.1f' % (d[big].mean() if big.any() else -1))
