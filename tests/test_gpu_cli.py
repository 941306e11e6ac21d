"""`kinoplan plan|bench` on the GPU: the CLI's runs equal the
Python binding's runs bit-for-bit, trial k uses seed base_seed + k,
iteration-budgeted benches are reproducible (all columns except the
device-clock ones), worker concurrency does not change a record, and
infeasibility exits 0 with NaN medians."""
import csv
import json
import math
import os
import subprocess

import pytest

from paper_2602_02846_b200 import planner, scenarios

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2602_02846_b200", "bin", "kinoplan")
SCEN = os.path.join(ROOT, "paper_2602_02846_b200", "scenarios")
TIME_COLS = ("first_ms", "final_ms")


def run(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, (p.returncode, p.stdout, p.stderr)
    return p


def rows(path):
    return list(csv.DictReader(open(path)))


def untimed(rs):
    return [{k: v for k, v in r.items() if k not in TIME_COLS} for r in rs]


@pytest.mark.parametrize("name,iters", [("forest_di6", 40), ("narrow_dubins6", 30), ("zigzag2d", 60)])
def test_plan_matches_python_binding(tmp_path, name, iters):
    f = os.path.join(SCEN, name + ".json")
    out = tmp_path / "o"
    p = run("plan", "--scenario", f, "--seed", "11", "--time-limit-ms", "60000", "--max-iterations", str(iters),
            "--out", str(out))
    st = json.loads(p.stdout)
    assert st == json.loads(open(out / "stats.json").read())
    ref = planner.plan(scenarios.load(name), seed=11, budget_s=60.0, max_iterations=iters)
    assert st["iterations"] == ref["iterations"] == iters
    assert st["propagations_attempted"] == ref["propagations_attempted"]
    assert st["node_count"] == ref["node_count"]
    if ref["found"]:
        assert st["success"] and st["best_cost"] == ref["best_cost"]
        traj = rows(out / "trajectory.csv")
        assert len(traj) == len(ref["path"]["states"])
        assert [float(t["x0"]) for t in traj] == list(ref["path"]["states"][:, 0])
    else:
        assert not st["success"] and not os.path.exists(out / "trajectory.csv")


def test_bench_seeds_and_reproducibility(tmp_path):
    f = os.path.join(SCEN, "forest_di6.json")
    args = ["--scenario", f, "--trials", "4", "--seed", "100", "--time-limit-ms", "60000", "--max-iterations", "30"]
    run("bench", *args, "--out", str(tmp_path / "a"), "--deterministic")
    run("bench", *args, "--out", str(tmp_path / "b"), "--deterministic")
    a, b = rows(tmp_path / "a" / "forest_di6.csv"), rows(tmp_path / "b" / "forest_di6.csv")
    assert [r["seed"] for r in a] == ["100", "101", "102", "103"]  # seed = base_seed + k
    assert untimed(a) == untimed(b)
    assert all(r["iterations"] == "30" for r in a)
    # each trial equals an independent single run with its seed
    for r in a[:2]:
        ref = planner.plan(scenarios.load("forest_di6"), seed=int(r["seed"]), budget_s=60.0, max_iterations=30)
        assert (r["success"] == "1") == bool(ref["found"])
        if ref["found"]:
            assert float(r["final_cost"]) == ref["best_cost"]
            assert int(r["first_iteration"]) == ref["first_solution_iteration"]
    for ext in (".csv.summary.csv", ".svg", ".records.json"):
        assert os.path.getsize(tmp_path / "a" / ("forest_di6" + ext)) > 0


def test_bench_workers_do_not_change_records(tmp_path):
    f = os.path.join(SCEN, "narrow_dubins6.json")
    args = ["--scenario", f, "--trials", "6", "--time-limit-ms", "60000", "--max-iterations", "25"]
    run("bench", *args, "--workers", "1", "--out", str(tmp_path / "w1"))
    run("bench", *args, "--workers", "3", "--out", str(tmp_path / "w3"))
    assert untimed(rows(tmp_path / "w1" / "narrow_dubins6.csv")) == untimed(rows(tmp_path / "w3" / "narrow_dubins6.csv"))


def test_bench_free2d_fifty_trials_all_succeed(tmp_path):
    f = os.path.join(SCEN, "free2d.json")
    p = run("bench", "--scenario", f, "--trials", "50", "--time-limit-ms", "500", "--out", str(tmp_path))
    s = json.loads(p.stdout)
    assert s["trials"] == 50 and s["success_rate"] == 100.0
    summ = rows(tmp_path / "free2d.csv.summary.csv")[0]
    assert float(summ["success_rate"]) == 100.0 and float(summ["first_cost"]) > 0
    assert open(tmp_path / "free2d.svg").read().count('class="trial"') == 50


def test_infeasible_budget_exits_zero_with_nan(tmp_path):
    f = os.path.join(SCEN, "forest_di6.json")
    p = run("bench", "--scenario", f, "--trials", "2", "--max-iterations", "2", "--out", str(tmp_path))
    s = json.loads(p.stdout)
    assert s["success_rate"] == 0.0 and math.isnan(s["first_ms"])
    summ = rows(tmp_path / "forest_di6.csv.summary.csv")[0]
    assert summ["first_cost"] == "NaN" and summ["final_cost"] == "NaN"
    assert 'class="empty"' in open(tmp_path / "forest_di6.svg").read()
    p = run("plan", "--scenario", f, "--max-iterations", "2")
    assert json.loads(p.stdout)["success"] is False


def test_plan_invalid_start_is_an_error(tmp_path):
    s = json.load(open(os.path.join(SCEN, "forest_di6.json")))
    box = s["problem"]["environment"]["obstacles"][0]
    s["problem"]["x_init"][:3] = [(a + b) / 2 for a, b in zip(box["min"], box["max"])]  # inside a tree
    f = tmp_path / "bad.json"
    f.write_text(json.dumps(s))
    p = subprocess.run([CLI, "plan", "--scenario", str(f), "--max-iterations", "3"], capture_output=True, text=True,
                       timeout=120)
    assert p.returncode == 1 and "error" in p.stderr  # InvalidProblemError, not a schema error
