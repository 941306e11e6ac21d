"""Where do invalid items stop?  Histogram of executed RK4 steps for invalid vs
valid items of a real frontier (debug propagate on the tree after N iterations).
python scripts/exit_hist.py SCENE [ITERS]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

scene = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s = scenarios.load(scene)
with Planner(s, seed=0) as g:
    g.solve(0.0, iters)
    nd = g.nodes()
    live = np.nonzero(nd["status"] != 2)[0]
    rng = np.random.default_rng(0)
    ids = rng.choice(live, size=min(len(live), 20000), replace=True)
    br = rng.integers(0, 32, size=len(ids))
    out = g.debug_propagate(nd["state"][ids], nd["acc"][ids], ids, br, iters + 1)
valid = out["valid"].astype(bool)
steps = out["steps"]
S = np.ceil(out["dt"] / s["planner"]["ode_step"]).astype(int)
print(scene, "items", len(ids), "valid frac %.3f" % valid.mean())
inv = ~valid
print("invalid: executed steps quantiles", np.quantile(steps[inv], [0.1, 0.25, 0.5, 0.75, 0.9]), "of S", np.quantile(S[inv], [0.5]))
print("invalid: fraction stopping within 1/2/3/5 steps", [round(float((steps[inv] <= k).mean()), 3) for k in (1, 2, 3, 5)])
print("lane-step waste if groups ran full S: %.3f" % (1 - steps.sum() / S.sum()))
