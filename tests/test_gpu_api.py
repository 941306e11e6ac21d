"""Solution output (§8f #1) and API behaviour on the GPU."""
import math

import numpy as np
import pytest

import kpo
from paper_2602_02846_b200 import Planner, plan, scenarios
from paper_2602_02846_b200.planner import InvalidProblemError

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scene", ["forest_di6", "narrow_dubins6", "building_quad12", "zigzag2d"])
def test_path_and_reintegrated_trajectory(scene):
    s = scenarios.load(scene, stop_at_first_solution=True)
    with Planner(s, seed=3) as g:
        r = g.solve(budget_s=2.0)
        assert r["found"]
        p = g.path()
        nodes = g.nodes()
        k = len(p["acc"])
        assert p["acc"][0] == 0.0 and np.all(np.diff(p["acc"]) > 0)  # monotone
        assert np.float32(p["acc"][-1]) == np.float32(r["best_cost"])
        # chain follows parent links and carries the stored node records
        leaf = r["best_leaf"]
        chain = [leaf]
        while nodes["parent"][chain[-1]] >= 0:
            chain.append(int(nodes["parent"][chain[-1]]))
        chain = chain[::-1]
        assert len(chain) == k
        np.testing.assert_array_equal(p["states"], nodes["state"][chain].astype(np.float64))
        t = g.trajectory()
        # fp32 running sum of re-integrated segment costs == stored acc, bit-exact
        run = np.float32(0.0)
        for c in t["segment_costs"]:
            run = np.float32(run + np.float32(c))
        assert run == np.float32(r["best_cost"])
        # every node state appears as the last sample of its segment
        n_samp = t["samples"].shape[0]
        assert n_samp > k
        np.testing.assert_array_equal(t["samples"][0], p["states"][0])
        np.testing.assert_array_equal(t["samples"][-1], p["states"][-1])
        # the re-integrated samples are valid states of the problem (oracle checker)
        o = kpo.Oracle(s, kpo.MIRROR32)
        assert o.is_segment_valid(t["samples"])


def test_plan_entry_point_and_errors():
    s = scenarios.load("forest_di6")
    r = plan(s, seed=9, budget_s=0.05)
    assert r["found"] and r["path"]["states"].shape[1] == 6 and len(r["timeline"]) >= 1
    tl = r["timeline"]
    assert all(a["cost"] > b["cost"] for a, b in zip(tl, tl[1:]))
    bad = scenarios.load("forest_di6")
    ob = bad["problem"]["environment"]["obstacles"][0]
    with Planner(bad) as g:
        with pytest.raises(InvalidProblemError):
            g.reset(1, x_init=[(ob["min"][0] + ob["max"][0]) / 2, (ob["min"][1] + ob["max"][1]) / 2, 5, 0, 0, 0])


def test_budget_respected_and_trace():
    s = scenarios.load("forest_di6")
    with Planner(s, seed=2) as g:
        r = g.solve(budget_s=0.02)
        assert 0.02 <= r["elapsed_s"] < 0.025  # stops at the first boundary past the budget
        tr = g.trace()
        assert len(tr) == r["iterations"] and np.all(np.diff(tr["t_ns"].astype(np.int64)) > 0)
        assert int(tr["items"].sum()) == r["propagations_attempted"]
        prof = g.profile()
        assert prof["items"] == r["propagations_attempted"] and prof["rk4_steps"] > prof["items"]


def test_batch_engine_matches_single_planner():
    """Concurrent lanes are independent replicas: with an iteration budget each
    query's result is identical to the same seed solved alone."""
    from paper_2602_02846_b200 import BatchPlanner

    s = scenarios.load("forest_di6", capacity=1 << 18, max_slots=1 << 21)
    seeds = [11, 12, 13, 14, 15, 16, 17]
    with BatchPlanner(s, lanes=3) as b:
        res, wall = b.solve(seeds, budget_s=0.0, max_iterations=12)
    assert wall > 0 and len(res) == len(seeds)
    with Planner(s) as g:
        for sd, r in zip(seeds, res):
            g.reset(sd)
            one = g.solve(0.0, 12)
            for k in ("best_cost", "best_leaf", "node_count", "propagations_attempted", "propagations_valid",
                      "iterations", "nodes_pruned_terminal"):
                assert r[k] == one[k], (sd, k, r[k], one[k])


def test_stop_at_first_solution_then_sweep_and_replay():
    """Stop-at-first-solution ends the solve at the first iteration boundary
    with a solution (the next propagate takes that decision, after the
    boundary's goal commits); the same seed run for exactly that many
    iterations reproduces it, and the planner still sweeps afterwards (the
    stop test must not end a sweep launch)."""
    s = scenarios.load("forest_di6", capacity=1 << 18, max_slots=1 << 21)
    with Planner(s, seed=3) as g:
        g.set_stop_at_first_solution(True)
        a = g.solve(5.0, 0)
        assert a["found"] and a["iterations"] == a["first_solution_iteration"]
        tl_a = g.timeline()
        assert len(tl_a) == 1 and tl_a[0]["iteration"] == a["iterations"]
        g.set_stop_at_first_solution(False)
        g.reset(3)
        b = g.solve(0.0, a["iterations"])
        assert b["best_cost"] == a["best_cost"] and b["best_leaf"] == a["best_leaf"]
        assert b["node_count"] == a["node_count"] and b["first_solution_iteration"] == a["iterations"]
        assert [(e["iteration"], e["cost"], e["leaf"]) for e in g.timeline()] == [(e["iteration"], e["cost"], e["leaf"]) for e in tl_a]
        g.set_stop_at_first_solution(True)
        g.reset(3)
        g.solve(5.0, 0)
        ms, prof = g.sweep(1024, launches=1)
        assert prof["items"] == 1024 * s["planner"]["lambda"] and prof["rk4_steps"] > prof["items"]
