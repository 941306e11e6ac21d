"""Per-iteration device trace of one query (graph mode, no profiler): time per
iteration split into propagate / select_reduce / select_scatter / gaps.
Since the early iteration boundary (select_scatter's block 0 writes it right
after its tile prefix), `scat` is block 0's entry -> boundary and the `gap`
after it includes the rest of the scatter's tile writes."""
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
    t_end = tr['t_ns'].astype(np.float64) / 1e3
    t_prev = np.concatenate([[0.0], t_end[:-1]])
    tp, ts, tse, tsc = (tr[k].astype(np.float64) / 1e3 for k in ('t_prop', 't_sel', 't_sel_end', 't_scat'))
    prop, sel, gap2, scat, gap1 = ts - tp, tse - ts, tsc - tse, t_end - tsc, tp - t_prev
    print(scene, 'iterations', r['iterations'], 'first sol it', r['first_solution_iteration'],
          'ttfs_ms %.3f' % (r['first_solution_s'] * 1e3))
    print('  it  total   gap  prop   sel  gap  scat    items   live frontier')
    rows = list(range(0, min(30, len(tr)))) + list(range(30, len(tr), max(1, len(tr) // 20)))
    for k in rows:
        e = tr[k]
        print(f"{e['iteration']:4d} {t_end[k]-t_prev[k]:6.1f} {gap1[k]:5.1f} {prop[k]:5.1f} {sel[k]:5.1f} {gap2[k]:4.1f} "
              f"{scat[k]:5.1f} {e['items']:8d} {e['live']:6d} {e['frontier']:6d}")
    for name, m in (('small(<2k items)', tr['items'] < 2000), ('large(>100k)', tr['items'] > 100000)):
        if m.any():
            print(f"mean {name}: total {np.mean((t_end-t_prev)[m]):.1f}  gap {gap1[m].mean():.1f}  prop {prop[m].mean():.1f}  "
                  f"sel {sel[m].mean():.1f}  gap2 {gap2[m].mean():.1f}  scat {scat[m].mean():.1f}")
