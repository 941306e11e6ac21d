"""SPEC.md examples, properties and acceptance criteria against the oracle
restatement (the reference ships no tests; SURVEY.md §4 lists the intent).
CPU only; sized to run in a few seconds each."""
import math

import numpy as np
import pytest

import kpo
from paper_2602_02846_b200 import scenarios


def _di6(**pl):
    s = scenarios.load("forest_di6", **pl)
    s["problem"]["environment"]["obstacles"] = []
    return s


# ------------------------------------------------------------- integrator --
def test_rk4_exact_on_double_integrator():
    o = kpo.Oracle(_di6(), kpo.FAITHFUL64)
    s = o.propagate_ode([0, 0, 0, 1, 0, 0], [0, 0, 0], 1.0, 0.1)
    assert len(s) == 11
    np.testing.assert_allclose(s[-1], [1, 0, 0, 1, 0, 0], atol=1e-12)
    s = o.propagate_ode([0] * 6, [1, 0, 0], 1.0, 0.1)
    np.testing.assert_allclose(s[-1], [0.5, 0, 0, 1, 0, 0], atol=1e-12)


def test_samples0_bit_exact_and_last_step_shortened():
    o = kpo.Oracle(_di6(), kpo.MIRROR32)
    x = np.array([0.3, 0.1, 0.7, 0.2, -0.4, 0.9], np.float32).astype(float)
    s = o.propagate_ode(x, [0.5, -0.25, 1.0], 0.3, 0.07)
    assert np.array_equal(s[0], x)
    assert len(s) == 1 + math.ceil(np.float32(0.3) / np.float32(0.07))


def test_time_reversal_double_integrator():
    o = kpo.Oracle(_di6(), kpo.FAITHFUL64)
    x0 = np.array([1.0, 2.0, 3.0, 0.5, -0.2, 0.1])
    u = np.array([0.3, -0.6, 0.2])
    x1 = o.propagate_ode(x0, u, 0.8, 0.02)[-1]
    back = x1.copy()
    back[3:] = -back[3:]
    x2 = o.propagate_ode(back, u, 0.8, 0.02)[-1]
    np.testing.assert_allclose(x2[:3], x0[:3], atol=1e-9)


def test_dubins_rk4_order():  # SPEC.md:163, acceptance 9
    s = scenarios.load("narrow_dubins6")
    o = kpo.Oracle(s, kpo.FAITHFUL64)
    x0 = np.array([2.0, 2.0, 2.5, 0.3, 0.1, 1.5])
    u = np.array([0.8, 0.05, 0.2])
    dt = 0.5
    ref = o.propagate_ode(x0, u, dt, dt / 4000)[-1]
    e1 = np.max(np.abs(o.propagate_ode(x0, u, dt, dt / 20)[-1] - ref))
    e2 = np.max(np.abs(o.propagate_ode(x0, u, dt, dt / 40)[-1] - ref))
    assert e1 / e2 >= 12.0, (e1, e2)


def _quad_f(x, u, p):
    m, g, ix, iy, iz = p
    ph, th, ps = x[6:9]
    a = u[0] / m
    f = np.zeros(12)
    f[0:3] = x[3:6]
    f[3] = a * (math.cos(ph) * math.sin(th) * math.cos(ps) + math.sin(ph) * math.sin(ps))
    f[4] = a * (math.cos(ph) * math.sin(th) * math.sin(ps) - math.sin(ph) * math.cos(ps))
    f[5] = a * math.cos(ph) * math.cos(th) - g
    w = x[10] * math.sin(ph) + x[11] * math.cos(ph)
    f[6] = x[9] + w * math.tan(th)
    f[7] = x[10] * math.cos(ph) - x[11] * math.sin(ph)
    f[8] = w / math.cos(th)
    f[9] = ((iy - iz) * x[10] * x[11] + u[1]) / ix
    f[10] = ((iz - ix) * x[9] * x[11] + u[2]) / iy
    f[11] = ((ix - iy) * x[9] * x[10] + u[3]) / iz
    return f


def test_quadcopter_hover_vs_fine_euler():
    s = scenarios.load("building_quad12")
    o = kpo.Oracle(s, kpo.FAITHFUL64)
    x0 = np.array([5.0, 5.0, 2.0, 0, 0, 0, 0.02, -0.01, 0.1, 0.01, 0.02, -0.01])
    u = np.array([9.81, 0.01, -0.02, 0.005])
    rk = o.propagate_ode(x0, u, 0.5, 0.01)[-1]
    p = (1.0, 9.81, 1.0, 1.0, 2.0)
    x = x0.copy()
    h = 1e-5
    for _ in range(50000):
        x = x + h * _quad_f(x, u, p)
    np.testing.assert_allclose(rk, x, atol=1e-4)
    # the oracle's derivative is the same model the independent script integrates
    np.testing.assert_allclose(o.derivative(x0, u), _quad_f(x0, u, p), atol=1e-12)


# --------------------------------------------------------------- sampling --
@pytest.mark.parametrize("rng", ["philox", "splitmix"])
def test_sampling_statistics_and_range(rng):  # SPEC.md:147-160, acceptance 10
    s = _di6(rng=rng, t_prop=2.0)
    s["problem"]["control_bounds"] = [[0, 1], [0, 1], [-2, 2]]
    s["problem"]["state_bounds"][3:] = [[-2, 2]] * 3
    o = kpo.Oracle(s, kpo.FAITHFUL64 if rng == "splitmix" else kpo.MIRROR32, seed=17)
    k = 100_000
    ps = np.tile(np.array([5, 5, 5, 0, 0, 0], float), (k, 1))
    ids = np.arange(k, dtype=np.uint32) // 32
    brs = np.arange(k, dtype=np.uint32) % 32
    r = o.propagate_items(ps, np.zeros(k), ids, brs, 0)
    u, dt = r["control"], r["dt"]
    sigma = math.sqrt(1 / 12 / k)
    assert abs(u[:, 0].mean() - 0.5) < 3 * sigma and abs(u[:, 1].mean() - 0.5) < 3 * sigma
    assert abs(u[:, 2].mean()) < 3 * 4 * sigma
    assert 0.49 <= u[:, 0].mean() <= 0.51
    assert np.all(dt > 0) and np.all(dt <= 2.0)
    assert 0.99 <= dt.mean() <= 1.01
    r2 = o.propagate_items(ps[:100], np.zeros(100), ids[:100], brs[:100], 0)
    assert np.array_equal(r2["control"], u[:100]) and np.array_equal(r2["dt"], dt[:100])


def test_degenerate_control_bounds():
    s = _di6()
    s["problem"]["control_bounds"] = [[0.5, 0.5], [-1, -1], [0, 0]]
    for pol in (kpo.MIRROR32, kpo.FAITHFUL64):
        for rng in ("philox", "splitmix"):
            s["planner"]["rng"] = rng
            o = kpo.Oracle(s, pol)
            r = o.propagate_items(np.tile([5, 5, 5, 0, 0, 0], (50, 1)), np.zeros(50), np.arange(50), np.zeros(50), 0)
            assert np.all(r["control"] == [0.5, -1.0, 0.0])


# ------------------------------------------------------------- validity ---
def test_state_validity_examples():
    s = _di6()
    s["problem"]["environment"]["obstacles"] = [{"type": "box", "min": [4, 4, 4], "max": [6, 6, 6]}]
    o = kpo.Oracle(s, kpo.FAITHFUL64)
    assert not o.is_state_valid([5, 5, 5, 0, 0, 0])
    assert not o.is_state_valid([4, 5, 5, 0, 0, 0])  # boundary contact is collision
    assert o.is_state_valid([3.99, 5, 5, 0, 0, 0])
    assert not o.is_state_valid([1, 1, 1, 2 + 1e-9, 0, 0])
    e = kpo.Oracle(_di6(), kpo.FAITHFUL64)
    assert e.is_state_valid([5, 5, 5, 0, 0, 0])


def test_interpolation_catches_thin_box():
    s = _di6(collision_step=0.05)
    s["problem"]["environment"]["obstacles"] = [{"type": "box", "min": [5.0, 0, 0], "max": [5.02, 10, 10]}]
    o = kpo.Oracle(s, kpo.FAITHFUL64)
    assert not o.is_segment_valid([[4.9, 5, 5, 1, 0, 0], [5.1, 5, 5, 1, 0, 0]])
    assert o.is_segment_valid([[4.8, 5, 5, 1, 0, 0], [4.9, 5, 5, 1, 0, 0]])


def test_monotone_refinement_and_containment():
    rng = np.random.default_rng(3)
    for trial in range(200):
        box_lo = rng.uniform(2, 7, 3)
        box_hi = box_lo + rng.uniform(0.01, 0.3, 3)
        a = rng.uniform(0, 10, 3)
        b = np.clip(a + rng.normal(0, 1.0, 3), 0, 10)
        seg = [np.r_[a, 0, 0, 0], np.r_[b, 0, 0, 0]]
        verdicts = []
        for c in (0.4, 0.2, 0.1, 0.05, 0.025):
            s = _di6(collision_step=c)
            s["problem"]["environment"]["obstacles"] = [{"type": "box", "min": list(box_lo), "max": list(box_hi)}]
            verdicts.append(kpo.Oracle(s, kpo.FAITHFUL64).is_segment_valid(seg))
        for coarse, fine in zip(verdicts, verdicts[1:]):
            assert coarse or not fine  # invalid at c  =>  invalid at every c' <= c
        if verdicts[-1]:
            s = _di6(collision_step=0.025)
            mid = (box_lo + box_hi) / 2
            s["problem"]["environment"]["obstacles"] = [
                {"type": "box", "min": list((box_lo + mid) / 2), "max": list((box_hi + mid) / 2)}]
            assert kpo.Oracle(s, kpo.FAITHFUL64).is_segment_valid(seg)


# ------------------------------------------------------------------ grid ---
def test_grid_examples():
    s = scenarios.load("free2d")
    s["decomposition"] = {"dims": [0, 1], "cells": [2, 2]}
    s["problem"]["state_bounds"][:2] = [[0, 1], [0, 1]]
    s["problem"]["environment"]["workspace_bounds"] = [[0, 1], [0, 1]]
    s["problem"]["x_init"] = [0.1, 0.1, 0, 0]
    s["problem"]["goal"]["center"] = [0.9, 0.9]
    s["problem"]["goal"]["radius"] = 0.05
    o = kpo.Oracle(s, kpo.FAITHFUL64)
    cells, side, nr = o.grid()
    assert nr == 4 and list(cells[:2]) == [2, 2] and list(side[:2]) == [0.5, 0.5]
    assert math.isclose(math.hypot(*side[:2]), 0.5 * math.sqrt(2), rel_tol=1e-12)
    assert o.region_index([0.25, 0.25, 0, 0]) == 0
    assert o.region_index([0.75, 0.25, 0, 0]) == 1
    assert o.region_index([1.0, 1.0, 0, 0]) == 3


def test_grid_delta_and_too_fine():  # SPEC.md:270-275, errors.hpp:26
    s = scenarios.load("free2d")
    s["problem"]["state_bounds"][0] = [0, 10]
    s["decomposition"] = {"dims": [0], "delta": 1.0}
    cells, side, nr = kpo.Oracle(s, kpo.FAITHFUL64).grid()
    assert nr == 10 and side[0] == 1.0
    s["decomposition"] = {"dims": [0, 1], "delta": 1e-5}
    with pytest.raises(kpo.OracleError) as e:
        kpo.Oracle(s, kpo.FAITHFUL64)
    assert e.value.code == 4


def test_forest_grid_is_27000_regions():
    assert kpo.Oracle(scenarios.load("forest_di6"), kpo.MIRROR32).grid()[2] == 27000
    assert kpo.Oracle(scenarios.load("narrow_dubins6"), kpo.MIRROR32).grid()[2] == 52000
    assert kpo.Oracle(scenarios.load("building_quad12"), kpo.MIRROR32).grid()[2] == 100000


def test_try_update_examples_and_stress():  # SPEC.md:293-305, acceptance 2
    t, out = kpo.atomic_min_stress(1, [0, 0, 0, 0], [5.0, 7.0, 5.0, 2.0], 1)
    assert list(out) == [0, 2, 1, 0] and t[0] == 2.0
    rng = np.random.default_rng(0)
    n = 1_000_000
    regions = rng.integers(0, 1000, n).astype(np.uint32)
    costs = rng.random(n) * 1000
    table, _ = kpo.atomic_min_stress(1000, regions, costs, 8)
    want = np.full(1000, np.inf)
    np.minimum.at(want, regions, costs)
    assert np.array_equal(table, want)
    t, _ = kpo.atomic_min_stress(1, np.zeros(1000), np.arange(1000, 0, -1.0), 8)
    assert t[0] == 1.0


def test_encoding_order_isomorphism():
    rng = np.random.default_rng(1)
    a = (rng.random(100000) * 10.0 ** rng.integers(-30, 30, 100000)).astype(np.float32)
    b = (rng.random(100000) * 10.0 ** rng.integers(-30, 30, 100000)).astype(np.float32)
    assert np.array_equal(a < b, a.view(np.uint32) < b.view(np.uint32))
    assert np.all(np.float32(np.inf).view(np.uint32) >= a.view(np.uint32))


# ---------------------------------------------------------------- planner --
def test_free2d_lower_bound():
    o = kpo.Oracle(scenarios.load("free2d"), kpo.FAITHFUL64, seed=1, workers=4)
    r = o.run(budget_s=0, max_iterations=40, stop_first=0)
    assert r["found"] and r["best_cost"] >= 5 - 0.5


def test_infeasible_goal_enclosed():
    s = scenarios.load("free2d")
    c = s["problem"]["goal"]["center"]
    s["problem"]["environment"]["obstacles"] = [
        {"type": "box", "min": [c[0] - 1, c[1] - 1], "max": [c[0] + 1, c[1] - 0.8]},
        {"type": "box", "min": [c[0] - 1, c[1] + 0.8], "max": [c[0] + 1, c[1] + 1]},
        {"type": "box", "min": [c[0] - 1, c[1] - 1], "max": [c[0] - 0.8, c[1] + 1]},
        {"type": "box", "min": [c[0] + 0.8, c[1] - 1], "max": [c[0] + 1, c[1] + 1]},
    ]
    r = kpo.Oracle(s, kpo.FAITHFUL64, workers=4).run(0, 60, 0)
    assert not r["found"] and r["best_cost"] == math.inf and r["best_leaf"] == -1


def test_invalid_start_is_invalid_problem():
    s = scenarios.load("forest_di6")
    ob = s["problem"]["environment"]["obstacles"][0]
    s["problem"]["x_init"][:3] = [(a + b) / 2 for a, b in zip(ob["min"], ob["max"])]
    with pytest.raises(kpo.OracleError) as e:
        kpo.Oracle(s)
    assert e.value.code == 2


def test_config_errors():
    for key, val in [("lambda", 0), ("i_max", 0), ("capacity", 0), ("t_prop", 0.0), ("ode_step", 2.0)]:
        s = scenarios.load("free2d", **{key: val})
        with pytest.raises(kpo.OracleError) as e:
            kpo.Oracle(s)
        assert e.value.code == 3, key


def _invariants(o, prev_status=None):
    n = o.nodes()
    t = o.table()
    k = len(n["acc"])
    assert np.all(n["parent"][1:] < np.arange(1, k)) and n["parent"][0] == -1  # tree well-formed
    assert np.all(n["acc"] >= t[n["region"]])  # region dominance
    assert np.all(n["acc"][1:] >= n["acc"][n["parent"][1:]])  # monotone costs
    if prev_status is not None:
        m = len(prev_status)
        was_t = prev_status == 2
        assert np.all(n["status"][:m][was_t] == 2)  # Terminal absorbing
    return n


@pytest.mark.parametrize("scene,pol", [("zigzag2d", kpo.MIRROR32), ("forest_di6", kpo.FAITHFUL64),
                                       ("narrow_dubins6", kpo.MIRROR32)])
def test_invariant_suite(scene, pol):  # acceptance 1 (scaled)
    o = kpo.Oracle(scenarios.load(scene), pol, seed=4, workers=8)
    prev = None
    last_best = math.inf
    for it in range(12):
        r = o.run(0, 1, 0)
        n = _invariants(o, prev)
        prev = n["status"]
        assert r["best_cost"] <= last_best
        last_best = r["best_cost"]
    tl = o.timeline()
    assert all(a["cost"] > b["cost"] for a, b in zip(tl, tl[1:]))  # strictly decreasing
    assert r["propagations_admitted"] <= r["propagations_valid"] <= r["propagations_attempted"]


def test_additivity_of_stored_costs():  # SPEC.md:430, acceptance 1(d)
    s = scenarios.load("forest_di6")
    o = kpo.Oracle(s, kpo.FAITHFUL64, seed=2, workers=8)
    o.run(0, 6, 0)
    n = o.nodes()
    rng = np.random.default_rng(0)
    for i in rng.choice(np.arange(1, len(n["acc"])), 30, replace=False):
        p = n["parent"][i]
        smp = o.propagate_ode(n["state"][p], n["control"][i], n["dt"][i], 0.02)
        np.testing.assert_array_equal(smp[-1], n["state"][i])
        seg = kpo.segment_cost(smp, 3, 0, n["dt"][i])
        assert abs(n["acc"][p] + seg - n["acc"][i]) <= 1e-9 * max(1.0, n["acc"][i])


def test_determinism_and_worker_independence():  # SPEC.md:429, acceptance 3
    s = scenarios.load("zigzag2d")
    a = kpo.Oracle(s, kpo.MIRROR32, seed=7, workers=1)
    ra = a.run(0, 25, 0)
    b = kpo.Oracle(s, kpo.MIRROR32, seed=7, workers=1)
    rb = b.run(0, 25, 0)
    c = kpo.Oracle(s, kpo.MIRROR32, seed=7, workers=8)
    rc = c.run(0, 25, 0)
    for k in ("best_cost", "best_leaf", "node_count", "propagations_valid", "nodes_pruned_terminal"):
        assert ra[k] == rb[k] == rc[k], k
    na, nc = a.nodes(), c.nodes()
    assert np.array_equal(na["state"], nc["state"]) and np.array_equal(na["status"], nc["status"])
