"""End-to-end distributional parity over 100 seeds (BASELINE.json north_star:
"time-to-first-solution, success rate and cost-versus-time curves must match
distributionally over >= 100 seeds").

GPU: the fp32 device planner with the reference's own SplitMix64 streams
(rng.hpp:44-57).  CPU: the fp64 reference-faithful restatement (oracle
Faithful64).  The two trajectories diverge chaotically (fp32 vs fp64), so the
comparison is of distributions: time-to-first-solution measured in iterations
(wall time is hardware-bound), success rate, first-solution cost
and the cost-versus-iteration curve.  Both planners are deterministic, so the
test is reproducible.  Two-sample KS and Mann-Whitney with alpha = 1e-3.
"""
import math
import os

import numpy as np
import pytest
from scipy import stats

import kpo
from paper_2602_02846_b200 import Planner, scenarios

pytestmark = pytest.mark.gpu
SEEDS = range(100)


def _summ(timeline, iters, marks):
    first_it = timeline[0]["iteration"] if timeline else math.inf
    first_cost = timeline[0]["cost"] if timeline else math.inf
    curve = []
    for m in marks:
        c = [e["cost"] for e in timeline if e["iteration"] <= m]
        curve.append(c[-1] if c else math.inf)
    return first_it, first_cost, curve


def _collect(scene, iters, marks):
    s = scenarios.load(scene, rng="splitmix")
    g_rows, c_rows = [], []
    with Planner(s, seed=0) as g:
        for sd in SEEDS:
            g.reset(sd)
            g.solve(0.0, iters)
            g_rows.append(_summ(g.timeline(), iters, marks))
    workers = os.cpu_count() or 1
    for sd in SEEDS:
        o = kpo.Oracle(s, kpo.FAITHFUL64, seed=sd, workers=workers)
        o.run(0.0, iters, 0)
        c_rows.append(_summ(o.timeline(), iters, marks))
        o.close()
    return g_rows, c_rows


def _check(g_rows, c_rows, marks):
    g_first = np.array([r[0] for r in g_rows], float)
    c_first = np.array([r[0] for r in c_rows], float)
    g_ok, c_ok = np.isfinite(g_first), np.isfinite(c_first)
    # success rate: two-proportion agreement (Fisher exact)
    table = [[g_ok.sum(), (~g_ok).sum()], [c_ok.sum(), (~c_ok).sum()]]
    assert stats.fisher_exact(table)[1] > 1e-3, table
    # time to first solution in iterations (successful runs)
    assert stats.mannwhitneyu(g_first[g_ok], c_first[c_ok]).pvalue > 1e-3
    # first-solution cost
    g_fc = np.array([r[1] for r in g_rows])[g_ok]
    c_fc = np.array([r[1] for r in c_rows])[c_ok]
    assert stats.ks_2samp(g_fc, c_fc).pvalue > 1e-3
    # cost-versus-iteration curve at each mark (runs with a solution by then)
    for k, m in enumerate(marks):
        gc = np.array([r[2][k] for r in g_rows])
        cc = np.array([r[2][k] for r in c_rows])
        gc, cc = gc[np.isfinite(gc)], cc[np.isfinite(cc)]
        if len(gc) >= 20 and len(cc) >= 20:
            assert stats.ks_2samp(gc, cc).pvalue > 1e-3, (m, np.median(gc), np.median(cc))
            # medians within 2 % (the curves overlay)
            assert abs(np.median(gc) - np.median(cc)) <= 0.02 * np.median(cc)
    return g_ok.mean(), c_ok.mean()


@pytest.mark.parametrize("scene,iters,marks", [("forest_di6", 30, (20, 25, 30)),
                                               ("narrow_dubins6", 30, (22, 26, 30))])
def test_distribution_matches_fp64_reference_planner(scene, iters, marks):
    g_rows, c_rows = _collect(scene, iters, marks)
    g_succ, c_succ = _check(g_rows, c_rows, marks)
    assert g_succ >= 0.9 and c_succ >= 0.9
