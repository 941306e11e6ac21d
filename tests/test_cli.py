"""The bench module and CLI on CPU: scenario parsing with
field-path schema errors, summary medians (lower-middle rule, NaN when no
trial succeeds), CSV / SVG emitters, byte-identical re-emission.  Everything
here runs `kinoplan validate` / `kinoplan report`, which never touch a GPU;
planning runs are in test_gpu_cli.py."""
import csv
import json
import math
import os
import re
import subprocess

import pytest

from paper_2602_02846_b200 import scenarios

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2602_02846_b200", "bin", "kinoplan")
SCEN = os.path.join(ROOT, "paper_2602_02846_b200", "scenarios")


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", ROOT, "paper_2602_02846_b200/bin/kinoplan"], check=True)


def run(*args, check=True):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=60)
    if check:
        assert p.returncode == 0, (p.returncode, p.stdout, p.stderr)
    return p


def lower_median(v):
    v = sorted(v)
    return v[(len(v) - 1) // 2] if v else math.nan


# ---------------------------------------------------------------- scenarios
@pytest.mark.parametrize("name", sorted(scenarios.BUILDERS))
def test_validate_bundled_matches_python_loader(name):
    out = json.loads(run("validate", "--scenario", os.path.join(SCEN, name + ".json")).stdout)
    s = scenarios.load(name)
    pl = s["planner"]
    assert out["name"] == s["name"] and out["model"] == s["problem"]["model"]
    assert out["obstacles"] == len(s["problem"]["environment"].get("obstacles", []))
    assert out["decomposition_dims"] == len(s["decomposition"]["dims"])
    assert out["lambda"] == pl.get("lambda", 32) and out["i_max"] == pl.get("i_max", 5)
    assert out["t_prop"] == pl["t_prop"] and out["t_max_ms"] == pl.get("t_max_ms", 100)
    assert out["trials"] == s["trials"]["n"] and out["base_seed"] == s["trials"]["base_seed"]


def test_flags_override_scenario_values():
    f = os.path.join(SCEN, "forest_di6.json")
    out = json.loads(run("validate", "--scenario", f, "--seed", "18446744073709551615", "--workers", "4",
                         "--time-limit-ms", "250", "--max-iterations", "77", "--trials", "3").stdout)
    assert out["base_seed"] == 2**64 - 1 and out["workers"] == 4
    assert out["t_max_ms"] == 250 and out["max_iterations"] == 77 and out["trials"] == 3
    out = json.loads(run("validate", "--scenario", f, "--workers", "4", "--deterministic").stdout)
    assert out["workers"] == 1  # --deterministic forces workers = 1


def _mutated(tmp_path, fn):
    s = json.load(open(os.path.join(SCEN, "free2d.json")))
    fn(s)
    p = tmp_path / "s.json"
    p.write_text(json.dumps(s))
    return str(p)


@pytest.mark.parametrize("mutate,path", [
    (lambda s: s["problem"]["goal"].__setitem__("radius", -1), "scenario.problem.goal.radius"),
    (lambda s: s["problem"].pop("x_init"), "scenario.problem.x_init: missing"),
    (lambda s: s["problem"].__setitem__("x_init", [0, 0]), "scenario.problem.x_init"),
    (lambda s: s["problem"].__setitem__("model", "unicycle"), "scenario.problem.model"),
    (lambda s: s["decomposition"].__setitem__("delta", 0.5), "scenario.decomposition: exactly one"),
    (lambda s: s["problem"]["environment"].__setitem__("obstacles", [{"type": "cone"}]),
     "scenario.problem.environment.obstacles[0].type"),
    (lambda s: s["problem"]["environment"].__setitem__(
        "obstacles", [{"type": "box", "min": [1, 1], "max": [0, 2]}]), "scenario.problem.environment.obstacles[0]"),
    (lambda s: s["problem"]["state_bounds"].__setitem__(0, [1, 0]), "scenario.problem.state_bounds[0]: lo > hi"),
    (lambda s: s["planner"].__setitem__("lambda", "many"), "scenario.planner.lambda: expected a number"),
    (lambda s: s["planner"].__setitem__("rng", "mt19937"), "scenario.planner.rng"),
    (lambda s: s.pop("planner"), "scenario.planner: missing"),
])
def test_schema_errors_carry_field_path(tmp_path, mutate, path):
    p = run("validate", "--scenario", _mutated(tmp_path, mutate), check=False)
    assert p.returncode == 3 and path in p.stderr, p.stderr


def test_json_syntax_error_reports_position(tmp_path):
    p = tmp_path / "s.json"
    p.write_text('{\n "name": "x",\n "problem": [1, 2,,]\n}')
    r = run("validate", "--scenario", str(p), check=False)
    assert r.returncode == 3 and "line 3" in r.stderr


def test_usage_errors_exit_2():
    assert run("frobnicate", check=False).returncode == 2
    assert run("plan", check=False).returncode == 2
    assert run("bench", "--scenario", "x.json", check=False).returncode == 2  # --out required
    assert run("validate", "--scenario", "x", "--bogus", "1", check=False).returncode == 2


# ---------------------------------------------------------------- report emitters
def _records(tmp_path, trials, name="demo"):
    p = tmp_path / "in.records.json"
    p.write_text(json.dumps({"scenario": name, "trials": trials}))
    return str(p)


def _trial(seed, first=None, final=None, timeline=(), iters=10):
    return {"seed": seed, "success": final is not None, "first_solution": first, "final_solution": final,
            "iterations": iters, "first_iteration": 3 if first else 0, "cost_timeline": [list(e) for e in timeline]}


def _report(tmp_path, trials, name="demo"):
    out = tmp_path / "out"
    run("report", "--records", _records(tmp_path, trials, name), "--out", str(out))
    rows = list(csv.DictReader(open(out / f"{name}.csv")))
    summ = list(csv.DictReader(open(out / f"{name}.csv.summary.csv")))
    assert len(summ) == 1
    return out, rows, summ[0]


def test_median_of_three(tmp_path):
    tr = [_trial(k, (t, c), (t, c), [(t, c)]) for k, (t, c) in enumerate([(4.0, 9.0), (1.0, 2.0), (2.0, 5.0)])]
    _, rows, s = _report(tmp_path, tr)
    assert float(s["first_cost"]) == 5.0 and float(s["first_ms"]) == 2.0
    assert float(s["success_rate"]) == 100.0 and len(rows) == 3


def test_even_count_takes_lower_middle_and_skips_failures(tmp_path):
    tr = [_trial(0, (1, 8.0), (5, 7.0)), _trial(1, (2, 6.0), (6, 3.0)), _trial(2),
          _trial(3, (3, 4.0), (7, 2.0)), _trial(4, (4, 9.0), (8, 1.0))]
    _, rows, s = _report(tmp_path, tr)
    assert float(s["first_cost"]) == 6.0 and float(s["final_cost"]) == 2.0
    assert float(s["first_ms"]) == 2.0 and float(s["final_ms"]) == 6.0
    assert float(s["success_rate"]) == 80.0
    assert rows[2]["success"] == "0" and rows[2]["first_ms"] == "NaN"


def test_infeasible_gives_nan_medians(tmp_path):
    _, rows, s = _report(tmp_path, [_trial(0)])
    assert float(s["success_rate"]) == 0.0  # SPEC.md:487 "NaN & NaN & NaN"
    assert all(s[k] == "NaN" for k in ("first_ms", "first_cost", "final_ms", "final_cost"))


def test_zero_trials_header_only_and_one_trial_two_lines(tmp_path):
    out, rows, _ = _report(tmp_path, [])
    assert open(out / "demo.csv").read().count("\n") == 1 and rows == []
    out, rows, _ = _report(tmp_path, [_trial(0, (1.5, 2.5), (1.5, 2.5), [(1.5, 2.5)])], name="one")
    assert open(out / "one.csv").read().count("\n") == 2


def test_round_trip_precision_and_byte_identical_reemission(tmp_path):
    c = 12.700000000000001 + 1e-15
    tr = [_trial(7, (0.1 + 0.2, c), (1 / 3, c / 3), [(0.1 + 0.2, c), (1 / 3, c / 3)])]
    out, rows, s = _report(tmp_path, tr)
    assert float(rows[0]["first_ms"]) == 0.1 + 0.2 and float(rows[0]["final_cost"]) == c / 3
    a = [open(out / f).read() for f in ("demo.csv", "demo.csv.summary.csv", "demo.svg")]
    out2 = tmp_path / "again"
    run("report", "--records", str(tmp_path / "in.records.json"), "--out", str(out2))
    assert a == [open(out2 / f).read() for f in ("demo.csv", "demo.csv.summary.csv", "demo.svg")]


def test_summary_recomputable_from_trial_csv(tmp_path):
    import random
    rnd = random.Random(5)
    tr = []
    for k in range(41):
        if rnd.random() < 0.2:
            tr.append(_trial(k))
        else:
            t1, c1 = rnd.uniform(0.5, 3), rnd.uniform(12, 20)
            tr.append(_trial(k, (t1, c1), (t1 * 7, c1 * 0.9), [(t1, c1), (t1 * 7, c1 * 0.9)]))
    _, rows, s = _report(tmp_path, tr)
    ok = [r for r in rows if r["success"] == "1"]
    for col in ("first_ms", "first_cost", "final_ms", "final_cost"):
        assert float(s[col]) == lower_median([float(r[col]) for r in ok])  # exact agreement
    assert float(s["success_rate"]) == 100.0 * len(ok) / len(rows)


def _polylines(svg, cls):
    out = []
    for m in re.finditer(r'<polyline class="%s"[^>]*points="([^"]*)"' % cls, svg):
        out.append([tuple(map(float, p.split(","))) for p in m.group(1).split()])
    return out


def test_svg_single_trial_two_steps(tmp_path):
    out, _, _ = _report(tmp_path, [_trial(0, (10, 5.0), (100, 4.0), [(10, 5.0), (100, 4.0)])])
    svg = open(out / "demo.svg").read()
    assert svg.startswith("<svg") and "http" not in svg.replace('xmlns="http://www.w3.org/2000/svg"', "")
    (pts,) = _polylines(svg, "trial")
    assert len(pts) == 4
    ys = [p[1] for p in pts]
    assert ys[0] == ys[1] and ys[2] == ys[3] and ys[0] < ys[2]  # cost 5.0 drawn above cost 4.0
    xs = [p[0] for p in pts]
    assert xs == sorted(xs) and xs[1] == xs[2]
    # log axis: 10 ms and 100 ms are one decade apart; the decade ticks are evenly spaced
    ticks = [float(m) for m in re.findall(r'<line x1="([0-9.]+)" y1="440" x2="[0-9.]+" y2="445"', svg)]
    assert len(ticks) >= 2 and abs((ticks[1] - ticks[0]) - (xs[2] - xs[0])) < 0.01


def test_svg_curves_monotone_and_median_inside_envelope(tmp_path):
    import random
    rnd = random.Random(1)
    tr = []
    for k in range(50):
        t, c, tl = rnd.uniform(0.5, 2), rnd.uniform(15, 20), []
        for _ in range(rnd.randint(1, 6)):
            tl.append((t, c))
            t *= rnd.uniform(1.2, 3)
            c -= rnd.uniform(0.1, 1.5)
        tr.append(_trial(k, tl[0], tl[-1], tl))
    out, _, _ = _report(tmp_path, tr)
    svg = open(out / "demo.svg").read()
    curves = _polylines(svg, "trial")
    assert len(curves) == 50
    for pts in curves:  # cost non-increasing == SVG y non-decreasing
        ys = [p[1] for p in pts]
        assert all(a <= b for a, b in zip(ys, ys[1:]))
    (med,) = _polylines(svg, "median")
    for x, y in med[::2]:  # each step start: within the min/max envelope of trials that have a solution at x
        ys = []
        for pts in curves:
            if pts[0][0] <= x:
                ys.append(max(p[1] for p in pts if p[0] <= x))
        assert min(ys) <= y <= max(ys)


def test_svg_all_failed_is_annotated_empty_plot(tmp_path):
    out, _, _ = _report(tmp_path, [_trial(0), _trial(1)])
    svg = open(out / "demo.svg").read()
    assert 'class="empty"' in svg and "polyline" not in svg


def test_records_reject_success_without_final(tmp_path):
    t = _trial(0)
    t["success"] = True
    p = run("report", "--records", _records(tmp_path, [t]), "--out", str(tmp_path / "o"), check=False)
    assert p.returncode == 3 and "trials[0]" in p.stderr
