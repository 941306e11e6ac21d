"""GPU vs oracle parity through the C-ABI.

Bar (BASELINE.json north_star): validity verdicts, region indices, control /
duration draws, accumulated-cost bits and final states are bit-exact against
the fp32 restatement (oracle Mirror32) on identical inputs; whole planner runs
are bit-identical to the restatement's workers=1 serial run (node store,
region table, best solution, timeline, stats except the race-dependent
`propagations_admitted`).  Against the fp64 reference-faithful planner the
propagated states agree within 1e-5 relative (fp32 tolerance, north_star).
"""
import numpy as np
import pytest

import kpo
from paper_2602_02846_b200 import Planner, scenarios

pytestmark = pytest.mark.gpu

SCENES = ["forest_di6", "narrow_dubins6", "building_quad12", "zigzag2d", "free2d"]


def _random_parents(s, k, rng):
    """Valid parent states (the planner only ever expands stored, valid nodes;
    samples[0] is not re-checked on the device), uniform in the state bounds."""
    lo = np.array([b[0] for b in s["problem"]["state_bounds"]], float)
    hi = np.array([b[1] for b in s["problem"]["state_bounds"]], float)
    o = kpo.Oracle(s, kpo.MIRROR32)
    out = [np.asarray(s["problem"]["x_init"], np.float32)]
    while len(out) < k:
        x = (lo + (hi - lo) * rng.random(len(lo))).astype(np.float32)
        if o.is_state_valid(x.astype(np.float64)):
            out.append(x)
    return np.stack(out)


@pytest.mark.parametrize("scene", SCENES)
@pytest.mark.parametrize("rng_kind", ["philox", "splitmix"])
def test_work_item_parity_bit_exact(scene, rng_kind):
    s = scenarios.load(scene, rng=rng_kind, max_slots=1 << 16, capacity=1 << 14)
    rng = np.random.default_rng(7)
    k = 4096
    ps = _random_parents(s, k, rng)
    pacc = (rng.random(k) * 10).astype(np.float32)
    ids = rng.integers(0, 1 << 20, k).astype(np.uint32)
    brs = rng.integers(0, 32, k).astype(np.uint32)
    with Planner(s, seed=1234) as g:
        d = g.debug_propagate(ps, pacc, ids, brs, iteration=3)
    o = kpo.Oracle(s, kpo.MIRROR32, seed=1234).propagate_items(ps.astype(np.float64), pacc.astype(np.float64),
                                                                 ids, brs, 3)
    np.testing.assert_array_equal(d["control"].astype(np.float64), o["control"])
    np.testing.assert_array_equal(d["dt"].astype(np.float64), o["dt"])
    gv, ov = d["valid"] == 1, o["valid"] == 1
    np.testing.assert_array_equal(gv, ov)
    assert gv.sum() > 0
    np.testing.assert_array_equal(d["region"][gv], o["region"][ov])
    np.testing.assert_array_equal(d["acc"][gv].astype(np.float64), o["acc"][ov])
    np.testing.assert_array_equal(d["state"][gv].astype(np.float64), o["state"][ov])
    np.testing.assert_array_equal(d["goal"][gv], o["goal"][ov])
    np.testing.assert_array_equal(d["steps"][gv], o["steps"][ov])


@pytest.mark.parametrize("scene", ["forest_di6", "narrow_dubins6", "building_quad12"])
def test_work_item_states_within_1e5_of_fp64(scene):
    """fp32 device vs the fp64 reference-faithful restatement on identical
    (u, dt): final states within 1e-5 relative (north_star tolerance)."""
    s = scenarios.load(scene, rng="splitmix", max_slots=1 << 16, capacity=1 << 14)
    rng = np.random.default_rng(11)
    k = 2048
    ps = _random_parents(s, k, rng)
    pacc = np.zeros(k, np.float32)
    ids = rng.integers(0, 1 << 20, k).astype(np.uint32)
    brs = rng.integers(0, 32, k).astype(np.uint32)
    with Planner(s, seed=99) as g:
        d = g.debug_propagate(ps, pacc, ids, brs, iteration=0)
    o = kpo.Oracle(s, kpo.FAITHFUL64, seed=99)
    h = float(s["planner"]["ode_step"])
    worst = 0.0
    checked = 0
    for i in range(0, k, 7):
        if d["valid"][i] != 1:
            continue
        ref = o.propagate_ode(ps[i].astype(np.float64), d["control"][i].astype(np.float64),
                              float(d["dt"][i]), h)[-1]
        got = d["state"][i].astype(np.float64)
        scale = np.maximum(np.abs(ref), 1.0)
        worst = max(worst, float(np.max(np.abs(got - ref) / scale)))
        checked += 1
    assert checked > 20
    assert worst < 1e-5, worst


def _compare_runs(g: Planner, o: "kpo.Oracle", rg: dict, ro: dict):
    for key in ("found", "best_cost", "best_leaf", "iterations", "propagations_attempted", "propagations_valid",
                "nodes_committed", "nodes_pruned_terminal", "nodes_deactivated", "nodes_reactivated",
                "candidates_dropped_capacity", "node_count", "capacity_exhausted", "first_solution_iteration",
                "best_found_iteration", "timeline_len"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rg["propagations_admitted"] >= rg["nodes_committed"]
    ng, no = g.nodes(), o.nodes()
    for f in ("state", "control", "dt", "acc"):
        np.testing.assert_array_equal(ng[f].astype(np.float64), no[f], err_msg=f)
    np.testing.assert_array_equal(ng["parent"].astype(np.int64), no["parent"])
    np.testing.assert_array_equal(ng["region"], no["region"])
    np.testing.assert_array_equal(ng["status"], no["status"])
    np.testing.assert_array_equal(ng["icount"].astype(np.uint32), np.minimum(no["icount"], 255))
    tg = g.region_table().view(np.float32).astype(np.float64)
    np.testing.assert_array_equal(tg, o.table())
    lg, lo = g.timeline(), o.timeline()
    assert [(e["iteration"], e["cost"], e["leaf"]) for e in lg] == [(e["iteration"], e["cost"], e["leaf"]) for e in lo]


@pytest.mark.parametrize("scene,iters", [("forest_di6", 14), ("narrow_dubins6", 10), ("building_quad12", 6),
                                          ("zigzag2d", 40), ("free2d", 30)])
@pytest.mark.parametrize("rng_kind", ["philox", "splitmix"])
def test_whole_run_bit_identical(scene, iters, rng_kind):
    s = scenarios.load(scene, rng=rng_kind)
    with Planner(s, seed=5) as g:
        rg = g.solve(budget_s=0.0, max_iterations=iters)
        o = kpo.Oracle(s, kpo.MIRROR32, seed=5, workers=8)
        ro = o.run(budget_s=0.0, max_iterations=iters, stop_first=0)
        _compare_runs(g, o, rg, ro)


def test_whole_run_deactivate_and_capacity():
    s = scenarios.load("forest_di6", deactivate_after_expansion=True, capacity=3000)
    with Planner(s, seed=3) as g:
        rg = g.solve(budget_s=0.0, max_iterations=12)
        o = kpo.Oracle(s, kpo.MIRROR32, seed=3, workers=8)
        ro = o.run(budget_s=0.0, max_iterations=12, stop_first=0)
        assert rg["capacity_exhausted"] == 1
        _compare_runs(g, o, rg, ro)


def test_solve_continues_and_reset_repeats():
    s = scenarios.load("forest_di6")
    with Planner(s, seed=21) as g:
        a = g.solve(budget_s=0.0, max_iterations=6)
        b = g.solve(budget_s=0.0, max_iterations=6)
        assert b["iterations"] == 12
        g.reset(21)
        c = g.solve(budget_s=0.0, max_iterations=12)
        assert c["node_count"] == b["node_count"] and c["best_cost"] == b["best_cost"]
        assert a["iterations"] == 6


def test_control_duration_cost_whole_run():
    """CostKind::ControlDuration (cost.hpp:15, :50-51): segment cost = dt."""
    s = scenarios.load("forest_di6")
    s["problem"]["cost"] = "control_duration"
    with Planner(s, seed=8) as g:
        rg = g.solve(budget_s=0.0, max_iterations=12)
        o = kpo.Oracle(s, kpo.MIRROR32, seed=8, workers=8)
        ro = o.run(budget_s=0.0, max_iterations=12, stop_first=0)
        _compare_runs(g, o, rg, ro)


@pytest.mark.parametrize("obstacles", [[], [{"type": "sphere", "center": [5, 5, 5], "radius": 2.0},
                                            {"type": "sphere", "center": [2, 8, 3], "radius": 1.0}]])
def test_empty_and_sphere_environments(obstacles):
    s = scenarios.load("forest_di6")
    s["problem"]["environment"]["obstacles"] = obstacles
    with Planner(s, seed=4) as g:
        rg = g.solve(budget_s=0.0, max_iterations=10)
        o = kpo.Oracle(s, kpo.MIRROR32, seed=4, workers=8)
        ro = o.run(budget_s=0.0, max_iterations=10, stop_first=0)
        _compare_runs(g, o, rg, ro)


def test_new_start_state_query():
    s = scenarios.load("forest_di6")
    start = [5.2, 0.7, 2.0, 0.5, 0.0, -0.25]
    with Planner(s) as g:
        g.reset(6, x_init=start)
        rg = g.solve(budget_s=0.0, max_iterations=10)
        s2 = scenarios.load("forest_di6")
        s2["problem"]["x_init"] = start
        o = kpo.Oracle(s2, kpo.MIRROR32, seed=6, workers=8)
        ro = o.run(budget_s=0.0, max_iterations=10, stop_first=0)
        _compare_runs(g, o, rg, ro)


def test_slot_overflow_fails_loudly():
    from paper_2602_02846_b200.planner import KinoplanError

    s = scenarios.load("forest_di6", max_slots=4096)
    with Planner(s, seed=1) as g:
        with pytest.raises(KinoplanError, match="max_slots"):
            g.solve(budget_s=0.0, max_iterations=20)


@pytest.mark.parametrize("scene,iters", [("forest_di6", 10), ("narrow_dubins6", 8), ("building_quad12", 5),
                                          ("zigzag2d", 30)])
def test_whole_run_bit_identical_multi_group(scene, iters, monkeypatch):
    """A small propagate grid (test hook KP_PROP_GRID) makes every warp run
    several item groups (and the quadcopter's rollouts split into two passes
    with compaction in between); results stay bit-identical."""
    monkeypatch.setenv("KP_PROP_GRID", "12")
    s = scenarios.load(scene)
    with Planner(s, seed=9) as g:
        rg = g.solve(budget_s=0.0, max_iterations=iters)
    monkeypatch.delenv("KP_PROP_GRID")
    with Planner(s, seed=9) as g2:
        rg2 = g2.solve(budget_s=0.0, max_iterations=iters)
        o = kpo.Oracle(s, kpo.MIRROR32, seed=9, workers=8)
        ro = o.run(budget_s=0.0, max_iterations=iters, stop_first=0)
        _compare_runs(g2, o, rg2, ro)
    for k in ("best_cost", "node_count", "propagations_valid", "nodes_committed", "timeline_len"):
        assert rg[k] == ro[k], (k, rg[k], ro[k])


@pytest.mark.parametrize("scene,iters", [("forest_di6", 150), ("narrow_dubins6", 100), ("building_quad12", 40)])
def test_whole_run_bit_identical_steady_state(scene, iters):
    """Longer runs: past the growth phase into the steady state (sparse select
    layout, multi-group propagate chunks, capacity pressure on the frontier)."""
    s = scenarios.load(scene)
    with Planner(s, seed=13) as g:
        rg = g.solve(budget_s=0.0, max_iterations=iters)
        o = kpo.Oracle(s, kpo.MIRROR32, seed=13, workers=16)
        ro = o.run(budget_s=0.0, max_iterations=iters, stop_first=0)
        _compare_runs(g, o, rg, ro)


@pytest.mark.parametrize("mode", ["sample_parallel", "step_sorted"])
@pytest.mark.parametrize("scene,iters", [("forest_di6", 24), ("zigzag2d", 40), ("building6d", 20)])
def test_whole_run_bit_identical_propagate_paths(scene, iters, mode, monkeypatch):
    """The double integrator's propagate paths (kp_kernels.cu flat_phase, the
    sample-parallel path for one-wave launches,
    the step-sorted path for larger ones) each reproduce the restatement on
    their own: forced for every launch size here."""
    if mode == "step_sorted":
        monkeypatch.setenv("KP_FLAT", "0")
    else:
        monkeypatch.setenv("KP_FLAT_MAX", str(1 << 30))
    s = scenarios.load(scene)
    with Planner(s, seed=21) as g:
        rg = g.solve(budget_s=0.0, max_iterations=iters)
    for k in ("KP_FLAT_MAX", "KP_FLAT"):
        monkeypatch.delenv(k, raising=False)
    o = kpo.Oracle(s, kpo.MIRROR32, seed=21, workers=8)
    ro = o.run(budget_s=0.0, max_iterations=iters, stop_first=0)
    for k in ("best_cost", "node_count", "propagations_valid", "nodes_committed", "timeline_len"):
        assert rg[k] == ro[k], (k, rg[k], ro[k])


@pytest.mark.parametrize("t_prop,h,lam", [(0.02, 0.02, 32), (2.0, 0.02, 4), (0.5, 0.02, 1), (0.5, 0.02, 5)])
@pytest.mark.parametrize("mode", ["sample_parallel", "step_sorted"])
def test_whole_run_bit_identical_rollout_lengths(t_prop, h, lam, mode, monkeypatch):
    """Rollout-length extremes on the double integrator's propagate paths: one
    sample per rollout (t_prop = h), up to 101 samples (past the step-count
    sort's 64 buckets), lambda = 1 and lambda = 5 (not a power of two: slot ->
    frontier position by division)."""
    if mode == "step_sorted":
        monkeypatch.setenv("KP_FLAT", "0")
    else:
        monkeypatch.setenv("KP_FLAT_MAX", str(1 << 30))
    s = scenarios.load("forest_di6", t_prop=t_prop, ode_step=h, collision_step=0.05, **{"lambda": lam})
    iters = 12
    with Planner(s, seed=3) as g:
        rg = g.solve(budget_s=0.0, max_iterations=iters)
    for k in ("KP_FLAT_MAX", "KP_FLAT"):
        monkeypatch.delenv(k, raising=False)
    o = kpo.Oracle(s, kpo.MIRROR32, seed=3, workers=8)
    ro = o.run(budget_s=0.0, max_iterations=iters, stop_first=0)
    for k in ("best_cost", "node_count", "propagations_valid", "nodes_committed", "timeline_len"):
        assert rg[k] == ro[k], (k, rg[k], ro[k])


def test_quadcopter_split_long_rollouts(monkeypatch):
    """Quadcopter split rollouts (first pass of 8 steps, parked survivors) with
    rollouts of up to 51 steps and several groups per warp (small grid)."""
    monkeypatch.setenv("KP_PROP_GRID", "12")
    s = scenarios.load("building_quad12", t_prop=1.0, **{"lambda": 8})
    iters = 10
    with Planner(s, seed=4) as g:
        rg = g.solve(budget_s=0.0, max_iterations=iters)
    monkeypatch.delenv("KP_PROP_GRID")
    o = kpo.Oracle(s, kpo.MIRROR32, seed=4, workers=16)
    ro = o.run(budget_s=0.0, max_iterations=iters, stop_first=0)
    for k in ("best_cost", "node_count", "propagations_valid", "nodes_committed", "timeline_len"):
        assert rg[k] == ro[k], (k, rg[k], ro[k])


def _item_parity(s, ps, seed, it=5):
    """debug_propagate on the device vs the Mirror32 restatement, bit-exact."""
    k = ps.shape[0]
    rng = np.random.default_rng(seed)
    pacc = (rng.random(k) * 5).astype(np.float32)
    ids = rng.integers(0, 1 << 20, k).astype(np.uint32)
    brs = rng.integers(0, 32, k).astype(np.uint32)
    with Planner(s, seed=seed) as g:
        d = g.debug_propagate(ps, pacc, ids, brs, iteration=it)
    o = kpo.Oracle(s, kpo.MIRROR32, seed=seed).propagate_items(ps.astype(np.float64), pacc.astype(np.float64),
                                                                ids, brs, it)
    gv, ov = d["valid"] == 1, o["valid"] == 1
    np.testing.assert_array_equal(d["valid"], o["valid"])
    np.testing.assert_array_equal(d["state"][gv].astype(np.float64), o["state"][ov])
    np.testing.assert_array_equal(d["acc"][gv].astype(np.float64), o["acc"][ov])
    np.testing.assert_array_equal(d["region"][gv], o["region"][ov])
    np.testing.assert_array_equal(d["steps"][gv], o["steps"][ov])
    return gv


def test_velocity_bounds_checked_once_per_item():
    """Double integrator: the device checks the velocity bounds once per item,
    at the last sample (kp_math.cuh vel_ok_at_end; v(t) = fma(u, t, v0) is
    monotone), the restatement at every sample.  Parents on, just inside and
    a few ulps inside the velocity bounds, controls pushing both ways: the
    verdicts (and every valid item's bits) must be the same."""
    s = scenarios.load("forest_di6", max_slots=1 << 16, capacity=1 << 14)
    rng = np.random.default_rng(3)
    base = _random_parents(s, 512, rng)
    hi = np.array([b[1] for b in s["problem"]["state_bounds"]], np.float32)
    lo = np.array([b[0] for b in s["problem"]["state_bounds"]], np.float32)
    rows = []
    for r, x in enumerate(base):
        x = x.copy()
        d = 3 + r % 3
        edge = [hi[d], lo[d], np.nextafter(hi[d], np.float32(0)), np.nextafter(lo[d], np.float32(0)),
                hi[d] - np.float32(1e-3), lo[d] + np.float32(1e-3)][r % 6]
        x[d] = edge
        rows.append(x)
    ps = np.stack(rows).astype(np.float32)
    gv = _item_parity(s, ps, seed=17)
    assert 0 < gv.sum() < len(gv)  # both verdicts occur


def test_small_angle_sincos_fast_path_boundary():
    """Quadcopter roll / pitch sincos: the device skips the range reduction when
    |x * 2/pi| < 1/2 (bit-identical by construction).  Roll / pitch bounds
    widened to +-1.2 rad and parents placed around pi/4 (the fast-path edge),
    so stage angles fall on both sides of it: bit-exact against the
    restatement's general recipe."""
    s = scenarios.load("building_quad12", max_slots=1 << 16, capacity=1 << 14)
    for d in (6, 7):
        s["problem"]["state_bounds"][d] = [-1.2, 1.2]
    rng = np.random.default_rng(5)
    ps = _random_parents(s, 1024, rng)
    edge = np.float32(np.pi / 4)
    for r in range(len(ps)):
        ps[r, 6 + r % 2] = np.float32(edge + (r % 7 - 3) * 1e-4) * (1 if r % 3 else -1)
    _item_parity(s, ps, seed=23)


def test_angle_wrap_all_angles_at_once():
    """One wrap test for all of a model's angles (max |a| >= pi): headings on
    and around +-pi, so single steps cross the wrap; bit-exact against the
    restatement's per-angle wrap_angle."""
    for scene, d in (("narrow_dubins6", 3), ("building_quad12", 8)):
        s = scenarios.load(scene, max_slots=1 << 16, capacity=1 << 14)
        rng = np.random.default_rng(9)
        ps = _random_parents(s, 1024, rng)
        pi = np.float32(np.pi)
        for r in range(len(ps)):
            ps[r, d] = [pi, -np.nextafter(pi, np.float32(0)), np.float32(3.1), np.float32(-3.1)][r % 4]
        _item_parity(s, ps, seed=29)


def _oracle_table(s, seed, states, lam, n_regions, workers=8):
    """Per-region minimum of the accumulated-cost bits over the valid items of
    one propagate launch over the frontier `states` (iteration 0, parent cost
    0, items node-major: node k, branch b), from the oracle's fp32
    restatement, in threads (ctypes releases the GIL), one oracle per chunk."""
    from concurrent.futures import ThreadPoolExecutor

    n = states.shape[0]
    step = max(1, (n + 4 * workers - 1) // (4 * workers))

    def part(lo):
        hi = min(n, lo + step)
        k = (hi - lo) * lam
        ids = np.repeat(np.arange(lo, hi, dtype=np.uint32), lam)
        brs = np.tile(np.arange(lam, dtype=np.uint32), hi - lo)
        ps = np.repeat(states[lo:hi].astype(np.float64), lam, axis=0)
        r = kpo.Oracle(s, kpo.MIRROR32, seed=seed).propagate_items(ps, np.zeros(k), ids, brs, 0)
        v = r["valid"] == 1
        t = np.full(n_regions, 0x7F800000, np.uint32)
        np.minimum.at(t, r["region"][v], r["acc"][v].astype(np.float32).view(np.uint32))
        return t, int(v.sum())

    with ThreadPoolExecutor(workers) as ex:
        parts = list(ex.map(part, range(0, n, step)))
    return np.minimum.reduce([p[0] for p in parts]), sum(p[1] for p in parts)


@pytest.mark.parametrize("scene,k", [("building_quad12", 22), ("forest_di6", 22), ("narrow_dubins6", 20)])
def test_sweep_full_size_region_table(scene, k):
    """BASELINE config 5 at its full size: one propagate launch over 2^k work
    items of a synthetic frontier (step-sorted path, many chunks per block).
    The region table it leaves is the per-region minimum of the valid items'
    accumulated costs — order-independent, so it must equal the oracle's over
    every item, bit for bit."""
    s = scenarios.load(scene, capacity=1 << 22, max_slots=1 << 23)
    lam = int(s["planner"]["lambda"])
    n = (1 << k) // lam
    with Planner(s, seed=5) as g:
        g.sweep(n, launches=1)
        states = g.nodes()["state"]
        table = g.region_table()
    assert states.shape[0] == n
    want, n_valid = _oracle_table(s, 5, states, lam, table.shape[0])
    assert n_valid > 0
    assert (want != 0x7F800000).sum() > 100
    np.testing.assert_array_equal(table, want)
