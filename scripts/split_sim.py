"""Warp-step model of the two-pass (split) rollout: for a real frontier
(tree after ITERS iterations) and a sweep-like frontier (positions uniform in
free space, other dims as x_init), debug-propagate items and count warp-steps
(per 32-slot group: the max executed steps) for one pass vs a first pass of K
steps + compacted survivors.  python scripts/split_sim.py SCENE [ITERS]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

scene = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s = scenarios.load(scene)
env = s["problem"]["environment"]
ws = np.array(env["workspace_bounds"], float)


def free(p):
    ok = np.ones(len(p), bool)
    for o in env.get("obstacles", []):
        if o["type"] == "box":
            lo, hi = np.array(o["min"]), np.array(o["max"])
            ok &= ~np.all((p >= lo) & (p <= hi), axis=1)
        else:
            c = np.array(o["center"])
            ok &= ((p - c) ** 2).sum(1) > o["radius"] ** 2
    return ok


def model(steps, S, valid, K, chunk=1024):
    one = two = 0
    for c0 in range(0, len(S), chunk):
        st, SS, va = steps[c0:c0 + chunk], S[c0:c0 + chunk], valid[c0:c0 + chunk]
        o = np.argsort(-SS, kind="stable")
        st, SS, va = st[o], SS[o], va[o]
        for g in range(0, len(st), 32):
            one += st[g:g + 32].max()
            two += np.minimum(st[g:g + 32], K).max()
        surv = (st > K) | ((st == K) & (SS > K) & va)  # still running after K steps
        rem = st[surv] - K
        for g in range(0, len(rem), 32):
            two += rem[g:g + 32].max()
    return one, two


rng = np.random.default_rng(0)
with Planner(s, seed=0) as g:
    g.solve(0.0, iters)
    nd = g.nodes()
    live = np.nonzero(nd["status"] != 2)[0]
    ids = rng.choice(live, size=min(len(live), 20480), replace=True)
    br = rng.integers(0, 32, size=len(ids))
    real = g.debug_propagate(nd["state"][ids], nd["acc"][ids], ids, br, iters + 1)
    n = len(ids)
    x0 = np.array(s["problem"]["start"], np.float32) if "start" in s["problem"] else nd["state"][0]
    pts = []
    while sum(len(p) for p in pts) < n:
        p = ws[:, 0] + rng.random((4 * n, len(ws))) * (ws[:, 1] - ws[:, 0])
        pts.append(p[free(p)])
    pos = np.concatenate(pts)[:n]
    st = np.tile(nd["state"][0], (n, 1))
    st[:, :len(ws)] = pos
    sweep = g.debug_propagate(st, np.zeros(n, np.float32), np.arange(n), rng.integers(0, 32, size=n), 1)
h = s["planner"]["ode_step"]
for name, out in (("real", real), ("sweep", sweep)):
    steps = out["steps"].astype(int)
    S = np.maximum(1, np.ceil(out["dt"] / h)).astype(int)
    valid = out["valid"].astype(bool)
    print(f"{scene} {name}: valid {valid.mean():.3f}, lane-steps {steps.sum()}, full-S lane-steps {S.sum()}")
    for K in (2, 4, 6, 8, 10):
        one, two = model(steps, S, valid, K)
        print(f"  K={K:2d}: warp-steps one pass {one}, split {two} ({two / one:.3f}), lane use {steps.sum() / (32 * one):.3f} -> {steps.sum() / (32 * two):.3f}")
