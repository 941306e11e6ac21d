import sys, time
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np
from paper_2602_02846_b200 import Planner, scenarios
import kpo
s = scenarios.load('forest_di6')
with Planner(s, seed=0) as g:
    t=time.time(); r=g.solve(budget_s=0.0, max_iterations=10); print('gpu 10 it', time.time()-t, r)
    o = kpo.Oracle(s, kpo.MIRROR32, seed=0, workers=8); ro=o.run(0.0, 10, 0); print('cpu', ro)
    ng, no = g.nodes(), o.nodes()
    print(ng['state'][:3], no['state'][:3])
for sc in ['forest_di6','narrow_dubins6','building_quad12']:
    s = scenarios.load(sc, stop_at_first_solution=True)
    with Planner(s, seed=0) as g:
        for i in range(3):
            g.reset(i); t=time.time(); r=g.solve(budget_s=5.0); w=time.time()-t
            print(sc, i, 'wall %.2f ms'%(w*1e3), {k:r[k] for k in ['found','best_cost','first_solution_s','first_solution_iteration','iterations','propagations_attempted','node_count','elapsed_s']})
