#!/usr/bin/env python
"""Benchmark of the B200 Kino-PAX+ planning iteration (BASELINE.json).

Metric: node propagations/sec (whole job), with the other two BASELINE metrics
(ms to first solution, solution cost at 100 ms) reported in the same line.

One step = one seeded query of the workload solved with a 100 ms budget
(BASELINE "cost at 100 ms"): fresh tree/grid (Alg. 1 init), then iterations
(propagate -> prune -> update) until the budget is spent.  Inputs (problem,
obstacles) are resident in HBM; L2 is flushed (256 MiB write) before every
step.  Timed with CUDA events on the planner's own stream; max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config forest_di6]
  python bench.py --impl reference ...   # the reference CPU planner arm

Multi-GPU (torchrun, one rank per GPU): replicas only — every rank solves its
own seeds (seed = base + rank * K + i); no collective on the data path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def _peaks():
    p = {"hbm_gbs": HBM_FALLBACK_GBS, "hbm_src": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        p["hbm_gbs"] = float(m["hbm_gbs"])
        p["hbm_src"] = "measured (MEASURED_PEAKS.json)"
        p["sm_max_mhz"] = float(m.get("sm_max_mhz", 1965.0))
    except Exception:
        pass
    # FP32 issue peak: 148 SMs x 128 lanes x clock (one FP32 lane-op per lane per cycle);
    # a measured FFMA-chain number is used when profiles/fp32_peak.json exists.
    p["fp32_lane_ops"] = 148 * 128 * p["sm_max_mhz"] * 1e6
    p["fp32_src"] = "nominal 148 SM x 128 lanes x sm_max_mhz"
    try:
        f = json.load(open(os.path.join(ROOT, "profiles", "fp32_peak.json")))
        p["fp32_lane_ops"] = float(f["ffma_lane_ops_per_s"])
        p["fp32_src"] = "measured FFMA chains (profiles/fp32_peak.json)"
    except Exception:
        pass
    return p


# Algorithmic FP32 lane-ops of the implemented recipe (FFMA, FADD, FMUL, FSETP,
# FMNMX, FRND, FDIV, FSQRT each = 1), per unit of device work counted by
# kp_profile.  Per RK4 step: 3N stage FMAs + 4N combine + 1 (h/2)
# + 2N bound compares + distance (7 in 3-D, 5 in 2-D) + 1 cost add + 4
# derivative evaluations (+2 per wrapped angle).  sincos recipe = 15.  The
# double integrator's samples are closed-form: t and t*t, then
# per position dim u/2 and two FMAs, per velocity dim one FMA; + bounds,
# distance and cost add as above.  The Dubins airplane's stages (round 2,
# DESIGN.md §4): 2 stage speeds, 4N accumulate + combine, one slope with two
# sincos at the step start and two rotated slopes (2 rotations x 4 + 4 each;
# stage 3 equals stage 2), plus per item the four rotation factors (4 sincos
# + 5).
_SINCOS = 15
OPS_PER_STEP = {
    "double_integrator_4d": 2 + 2 * 4 + 8 + 5 + 1,                               # 24
    "double_integrator_6d": 2 + 3 * 4 + 12 + 7 + 1,                              # 34
    "dubins_airplane_6d": 2 + 4 * 6 + 1 + 12 + 7 + 1 + 2 + (2 * _SINCOS + 4) + 2 * 12,   # 107
    "quadcopter_12d": 3 * 12 + 4 * 12 + 1 + 24 + 7 + 1 + 6 + 4 * (3 * _SINCOS + 26),   # 407
}
OPS_PER_ITEM = 35      # U conversions + control FMAs, S = ceil(dt/h), region index (3 dims), goal test, acc add
OPS_PER_ITEM_MODEL = {"dubins_airplane_6d": 4 * _SINCOS + 5}  # the Dubins rotation factors (step_ctx)
OPS_PER_BOX = 6        # six closed-interval compares
OPS_PER_SPHERE = 7     # 3 sub + mul + 2 fma + compare
OPS_PER_INTERP = 4     # j/k + 3 fma


def lane_ops(model, d):
    """Algorithmic FP32 lane-ops of the work counted in a kp_profile (delta) d."""
    return (d["rk4_steps"] * OPS_PER_STEP[model] + d["items"] * (OPS_PER_ITEM + OPS_PER_ITEM_MODEL.get(model, 0))
            + d["box_tests"] * OPS_PER_BOX + d["sphere_tests"] * OPS_PER_SPHERE + d["interp_points"] * OPS_PER_INTERP)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.stamps = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])
            self.stamps.append(time.time())

    def only_within(self, windows):
        """Keep the samples taken inside the given (t0, t1) wall-clock windows."""
        keep = [i for i, t in enumerate(self.stamps) if any(a <= t <= b for a, b in windows)]
        self.rows = [self.rows[i] for i in keep]
        self.stamps = [self.stamps[i] for i in keep]

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for name, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(name)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _init_ranks(ws: int, local: int):
    """One process per GPU (NCCL).  Returns (device index, reduce device): on
    a box with fewer GPUs than ranks (functional checks only: replicas never
    wait on each other) ranks share devices and reduce over gloo on the host."""
    import torch

    ngpu = max(1, torch.cuda.device_count())
    dev_idx = local % ngpu
    torch.cuda.set_device(dev_idx)
    if ws > 1:
        import torch.distributed as dist

        if ngpu >= ws:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
            return dev_idx, torch.device("cuda", dev_idx)
        dist.init_process_group("gloo")
        return dev_idx, torch.device("cpu")
    return dev_idx, torch.device("cuda", dev_idx)


def _cpu_model():
    """Host CPU model (the CPU baseline states its cores and model)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _median(xs):
    xs = [x for x in xs if x == x]
    return statistics.median(xs) if xs else None


def cpu_planner_run(scenario, seed, budget_s, workers, stop_first, max_iterations=0):
    """The reference CPU planner (fp64 restatement, oracle/, SplitMix64, worker pool)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import kpo

    s = json.loads(json.dumps(scenario))
    s["planner"]["rng"] = "splitmix"  # rng.hpp derive_stream, as the reference
    o = kpo.Oracle(s, kpo.FAITHFUL64, seed=seed, workers=workers)
    t = time.perf_counter()
    r = o.run(budget_s=budget_s, max_iterations=max_iterations, stop_first=1 if stop_first else 0)
    r["wall_s"] = time.perf_counter() - t
    return r


def query_config(args, scenario, ws):
    """`config` of the default (one query per step) workload, shared by both arms
    so the reference line names the same workload as ours."""
    return {"workload": f"{args.config}: one seeded query per step, {args.budget_ms:g} ms budget "
                        "(Alg. 1 until t_max), replicas across ranks",
            "budget_ms": args.budget_ms, "seeds_rank0": [args.seed_base, args.seed_base + args.steps - 1],
            "lambda": scenario["planner"]["lambda"], "capacity": scenario["planner"]["capacity"],
            "regions": _regions(scenario), "l2": "flushed before every step (256 MiB write)",
            "parallelism": f"replicas x{ws}"}


def run_reference(args, scenario):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    budget = args.budget_ms / 1000.0
    for i in range(args.warmup):
        cpu_planner_run(scenario, args.seed_base - 1 - i, budget, cores, False)
    props, wall, ttfs, costs, found = 0, 0.0, [], [], 0
    for i in range(args.steps):
        r = cpu_planner_run(scenario, args.seed_base + i, budget, cores, False)
        props += r["propagations_attempted"]
        wall += r["wall_s"]
        if r["found"]:
            found += 1
            ttfs.append(r["first_solution_s"] * 1e3)
            costs.append(r["best_cost"])
    value = props / wall
    line = {
        "impl": "reference", "metric": "node propagations/sec", "value": value, "unit": "propagations/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (pinned scene geometry, seeded queries)",
        "config": query_config(args, scenario, ws),
        "metrics": {"ms_to_first_solution_median": _median(ttfs), "solution_cost_at_budget_median": _median(costs),
                    "success_rate": found / args.steps, "node_propagations_per_sec": value},
        "cpu_baseline": {"value": value, "unit": "propagations/s", "cores": cores, "kind": "port",
                         "cpu_model": _cpu_model(),
                         "sample": f"{args.steps} queries x {args.budget_ms} ms budget, fp64 restatement "
                                   f"(oracle/kpo.hpp Faithful64, SplitMix64), {cores} worker threads"},
        "e2e": {"value": value, "unit": "propagations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_b200(args, scenario):
    import torch

    from paper_2602_02846_b200 import Planner, replicas

    ws, rank, local = _dist()
    local, red_dev = _init_ranks(ws, local)
    dev = torch.device("cuda", local)
    budget = args.budget_ms / 1000.0
    iters = args.iters
    if iters > 0:
        budget = 0.0
    planner = Planner(scenario, device=local, seed=args.seed_base)
    ext = torch.cuda.ExternalStream(planner.stream(), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    n = planner.n
    x_init = scenario["problem"]["x_init"]
    seeds = replicas.shard_seeds(args.seed_base, rank, ws, args.steps)

    clk = ClockSampler(local).__enter__()  # sampler up before the timed region (NVML init is slow)
    for i in range(args.warmup):
        with torch.cuda.stream(ext):
            flush.zero_()  # also loads torch's kernel before timing
        planner.reset(args.seed_base + 100000 + i)
        planner.solve(budget, iters)
    time.sleep(0.3)

    # ---- timed region (device) ----
    prof0 = planner.profile()
    results = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    n_rows0 = len(clk.rows)
    try:
        e0.record(ext)
        for sd in seeds:
            with torch.cuda.stream(ext):
                flush.zero_()
            planner.reset(sd)
            results.append(planner.solve(budget, iters))
        e1.record(ext)
        torch.cuda.synchronize()
    finally:
        clk.rows = clk.rows[n_rows0:]
        clk.__exit__(None, None, None)
    if ws > 1:
        torch.distributed.barrier()
    prof1 = planner.profile()
    dev_ms = e0.elapsed_time(e1)
    props = sum(r["propagations_attempted"] for r in results)
    dev_ms, props_total = replicas.reduce_job(dev_ms, props, world=ws, device=red_dev)
    results = replicas.gather_results(results, world=ws)
    value = props_total / (dev_ms / 1e3)

    # ---- end-to-end through the public C-ABI with host buffers ----
    e2e_props, t_e2e = 0, 0.0
    d2h_path = 0
    for sd in seeds:
        t0 = time.perf_counter()
        planner.reset(sd, x_init=x_init)          # H2D: start state (pinned staging), seed
        r = planner.solve(budget, iters)           # D2H: result/control block
        p = planner.path() if r["found"] else None  # D2H: root->leaf chain
        t_e2e += time.perf_counter() - t0
        e2e_props += r["propagations_attempted"]
        if p is not None:
            d2h_path += p["states"].nbytes // 2 + p["controls"].nbytes // 2 + 2 * 4 * len(p["durations"])
    planner.set_stop_at_first_solution(True)
    ttfs_wall = []
    for sd in seeds:
        t0 = time.perf_counter()
        planner.reset(sd, x_init=x_init)
        r = planner.solve(max(budget, 1.0), 0)
        ttfs_wall.append((time.perf_counter() - t0) * 1e3 if r["found"] else float("nan"))
    planner.set_stop_at_first_solution(False)
    t_e2e, e2e_total = replicas.reduce_job(t_e2e, e2e_props, world=ws, device=red_dev)

    # ---- per-kernel roofline pass (one query, per-launch CUDA events) ----
    roof = None
    if rank == 0:
        planner.set_profiling(True)
        pa = planner.profile()
        planner.reset(seeds[0])
        planner.solve(budget, iters)
        pb = planner.profile()
        planner.set_profiling(False)
        roof = roofline(scenario, pa, pb)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        # bounded sample (~10 s of CPU work): the first seeds of the timed run,
        # each query run for args.cpu_query_s seconds on every host core
        cores = os.cpu_count() or 1
        n_q = max(1, int(round(args.cpu_sample_s / args.cpu_query_s)))
        props, wall, ttfs, costs = 0, 0.0, [], []
        qs = seeds[:n_q]
        n_q = len(qs)
        for sd in qs:
            r = cpu_planner_run(scenario, sd, args.cpu_query_s, cores, False)
            props += r["propagations_attempted"]
            wall += r["wall_s"]
            if r["found"]:
                ttfs.append(r["first_solution_s"] * 1e3)
                costs.append(r["best_cost"])
        # deterministic mode (workers = 1) beside it: a shorter sample
        p1, w1 = 0, 0.0
        for sd in qs[:max(1, n_q // 2)]:
            r = cpu_planner_run(scenario, sd, args.cpu_query_s, 1, False)
            p1 += r["propagations_attempted"]
            w1 += r["wall_s"]
        cpu = {"value": props / wall, "unit": "propagations/s", "cores": cores, "kind": "port",
               "cpu_model": _cpu_model(),
               "sample": f"{args.config}, {n_q} queries (seeds {qs[0]}..{qs[-1]}) "
                         f"x {args.cpu_query_s:g} s budget each on {cores} threads, fp64 restatement "
                         "(oracle Faithful64, SplitMix64)",
               "wall_s": wall,
               "ms_to_first_solution_median": _median(ttfs), "solution_cost_at_budget_median": _median(costs),
               "success_rate": len(ttfs) / n_q,
               "single_thread": {"value": p1 / w1, "unit": "propagations/s", "cores": 1,
                                 "sample": f"{max(1, n_q // 2)} queries x {args.cpu_query_s:g} s, workers = 1"}}

    dist = None
    if rank == 0 and args.dist_seeds > 0:
        # BASELINE metrics as distributions over seeds 0..N-1:
        # time to first solution (stop-at-first queries) and cost at the budget
        tt, costs_d, found = [], [], 0
        planner.set_stop_at_first_solution(True)
        for sd in range(args.dist_seeds):
            planner.reset(sd, x_init=x_init)
            r = planner.solve(max(budget, 1.0), 0)
            if r["found"]:
                tt.append(r["first_solution_s"] * 1e3)
        planner.set_stop_at_first_solution(False)
        for sd in range(args.dist_seeds):
            planner.reset(sd, x_init=x_init)
            r = planner.solve(budget, iters)
            if r["found"]:
                found += 1
                costs_d.append(r["best_cost"])
        dist = {"seeds": [0, args.dist_seeds - 1],
                "ms_to_first_solution_median": _median(tt), "ms_to_first_solution_p25_p75": _quart(tt),
                "solution_cost_at_budget_median": _median(costs_d), "solution_cost_at_budget_p25_p75": _quart(costs_d),
                "success_rate": found / args.dist_seeds}

    extras = {}
    if rank == 0 and ws == 1 and not args.no_extras:
        extras = other_configs(args, budget)

    if rank == 0:
        ttfs = [r["first_solution_s"] * 1e3 for r in results if r["found"]]
        costs = [r["best_cost"] for r in results if r["found"]]
        launches = prof1["kernel_launches"] - prof0["kernel_launches"] + 2 * len(seeds)
        ctl_bytes = 328 + 256 * 24  # result block read back per query: KpCtl header + 256 timeline entries (kp_capi.cpp fetch_ctl)
        line = {
            "metric": "node propagations/sec", "value": value, "unit": "propagations/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / len(seeds),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (pinned scene geometry, seeded queries)",
            "config": query_config(args, scenario, ws),
            "metrics": {
                "ms_to_first_solution_median": _median(ttfs),
                "ms_to_first_solution_p25_p75": _quart(ttfs),
                "solution_cost_at_100ms_median": _median(costs) if abs(args.budget_ms - 100) < 1e-9 else None,
                "solution_cost_at_budget_median": _median(costs),
                "success_rate": len(ttfs) / len(results),
                "node_propagations_per_sec": value,
                "iterations_median": _median([r["iterations"] for r in results]),
                "capacity_exhausted_steps": sum(r["capacity_exhausted"] for r in results),
                "over_seeds": dist,
            },
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_total / t_e2e, "unit": "propagations/s",
                    "h2d_bytes_per_step": 4 * 12 + 8,
                    "d2h_bytes_per_step": int(ctl_bytes + d2h_path / max(1, len(seeds))),
                    "ms_to_first_solution_median_wall": _median(ttfs_wall),
                    "note": "host wall clock around kp_reset_query + kp_solve + kp_get_path per query"},
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "other_configs": extras,
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    planner.close()
    return 0


def other_configs(args, budget):
    """The other BASELINE configs, summarised in the headline line (each guarded):
    Dubins6/narrow and Quad12/building single queries (config 2, 3), a batch
    through the concurrent engine (config 4) and the Quad12 propagate sweep's
    saturated roofline (config 5)."""
    from paper_2602_02846_b200 import BatchPlanner, Planner, scenarios

    out = {}
    for cfg in ("narrow_dubins6", "building_quad12"):
        try:
            s = scenarios.load(cfg)
            b = budget if cfg != "building_quad12" else max(budget, 0.1)
            with Planner(s, seed=args.seed_base) as g:
                g.reset(1)
                g.solve(b)
                res, dev = [], 0.0
                for i in range(5):
                    g.reset(args.seed_base + i)
                    r = g.solve(b)
                    res.append(r)
                    dev += r["elapsed_s"]
                # time to first solution over seeds 0..N-1 (stop-at-first queries)
                dist = None
                if args.dist_seeds > 0:
                    g.set_stop_at_first_solution(True)
                    tt_d = []
                    for sd in range(args.dist_seeds):
                        g.reset(sd)
                        r = g.solve(max(b, 1.0))
                        if r["found"]:
                            tt_d.append(r["first_solution_s"] * 1e3)
                    g.set_stop_at_first_solution(False)
                    # and the cost at the budget over the same seeds (the
                    # SURVEY's cost-at-100-ms distribution)
                    costs_d = []
                    for sd in range(args.dist_seeds):
                        g.reset(sd)
                        r = g.solve(b)
                        if r["found"]:
                            costs_d.append(r["best_cost"])
                    dist = {"seeds": [0, args.dist_seeds - 1], "ms_to_first_solution_median": _median(tt_d),
                            "ms_to_first_solution_p25_p75": _quart(tt_d),
                            "success_rate_first": len(tt_d) / args.dist_seeds, "first_budget_s": max(b, 1.0),
                            "solution_cost_at_budget_median": _median(costs_d),
                            "solution_cost_at_budget_p25_p75": _quart(costs_d),
                            "success_rate": len(costs_d) / args.dist_seeds, "budget_s": b}
            tt = [r["first_solution_s"] * 1e3 for r in res if r["found"]]
            out[cfg] = {"budget_ms": b * 1e3, "queries": len(res), "success_rate": len(tt) / len(res),
                        "ms_to_first_solution_median": _median(tt),
                        "solution_cost_at_budget_median": _median([r["best_cost"] for r in res if r["found"]]),
                        "node_propagations_per_sec": sum(r["propagations_attempted"] for r in res) / dev,
                        "over_seeds": dist}
        except Exception as e:  # noqa: BLE001
            out[cfg] = {"error": str(e)[:200]}
    try:
        s = scenarios.load(args.config, capacity=1 << 19, max_slots=1 << 21)
        with BatchPlanner(s, lanes=8) as bp:
            bp.solve(range(900000, 900008), budget)
            res, wall = bp.solve(range(args.seed_base, args.seed_base + 64), budget)
        tt = [r["first_solution_s"] * 1e3 for r in res if r["found"]]
        out["batch_" + args.config] = {
            "queries": len(res), "lanes": 8, "budget_ms": budget * 1e3, "wall_s": wall,
            "queries_per_s": len(res) / wall,
            "node_propagations_per_sec": sum(r["propagations_attempted"] for r in res) / wall,
            "ms_to_first_solution_median": _median(tt), "success_rate": len(tt) / len(res)}
    except Exception as e:  # noqa: BLE001
        out["batch_" + args.config] = {"error": str(e)[:200]}
    # propagate throughput sweeps (config 5 on Quad12; the DI6 headline model
    # beside it shows the same kernel's saturated efficiency)
    pk = _peaks()
    for scene, model in (("building_quad12", "quadcopter_12d"), ("forest_di6", "double_integrator_6d")):
        try:
            s = scenarios.load(scene)
            s["planner"]["capacity"] = max(int(s["planner"]["capacity"]), (1 << 22) // 32)
            s["planner"]["max_slots"] = 1 << 22
            with Planner(s, seed=1) as g:
                g.sweep(1 << 10, launches=2)
                rows = []
                for k in (18, 20, 22):
                    ms, one = g.sweep((1 << k) // 32, launches=3)
                    ops = lane_ops(model, one)
                    rows.append({"k": k, "items_per_s": one["items"] / (ms * 1e-3),
                                 "frac": ops / (ms * 1e-3) / pk["fp32_lane_ops"]})
            mi = {"double_integrator_6d": 1, "quadcopter_12d": 3}[model]
            out["sweep_" + scene] = {"kernel": f"k_propagate<{mi}>", "bound": "fp32", "peak_src": pk["fp32_src"],
                                     "rows": rows, "best_frac": max(r["frac"] for r in rows)}
        except Exception as e:  # noqa: BLE001
            out["sweep_" + scene] = {"error": str(e)[:200]}
    return out


def _quart(xs):
    xs = sorted(x for x in xs if x == x)
    if len(xs) < 2:
        return None
    return [xs[len(xs) // 4], xs[(3 * len(xs)) // 4]]


def _regions(s):
    r = 1
    for c in s["decomposition"].get("cells", []):
        r *= c
    return r


def roofline(scenario, pa, pb):
    """Dominant kernel = propagate (FP32 issue-bound, no tensor-core work);
    select/scatter reported against HBM bandwidth."""
    pk = _peaks()
    model = scenario["problem"]["model"]
    d = {k: pb[k] - pa[k] for k in pb}
    ops = lane_ops(model, d)
    n_prop = max(1, d["n_propagate"])
    t_prop = d["t_propagate_s"] / n_prop
    ops_launch = ops / n_prop
    achieved = ops_launch / t_prop if t_prop > 0 else 0.0
    n = {"double_integrator_4d": 4, "double_integrator_6d": 6, "dubins_airplane_6d": 6, "quadcopter_12d": 12}[model]
    m = {"double_integrator_4d": 2, "double_integrator_6d": 3, "dubins_airplane_6d": 3, "quadcopter_12d": 4}[model]
    # select + scatter algorithmic bytes: live node prune, ancestor hops, slot scan, commits
    sel_bytes = (d["live_scanned"] * 15 + d["ancestor_hops"] * 16 + d["slots_scanned"] / 8 * 3
                 + d["admitted_checked"] * 12)
    n_sel = max(1, d["n_select"])
    t_sel = d["t_select_s"] / n_sel
    sel_gbs = sel_bytes / n_sel / t_sel / 1e9 if t_sel > 0 else 0.0
    t_total = d["t_propagate_s"] + d["t_select_s"] + d["t_scatter_s"]
    traffic, issue = None, None  # from the committed ncu --set full capture of a steady-state launch
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        cfg_name = scenario.get("name", "")
        mi = {'double_integrator_4d': 0, 'double_integrator_6d': 1, 'dubins_airplane_6d': 2, 'quadcopter_12d': 3}[model]
        ent = tr.get(cfg_name, {})
        rec = ent.get(f"k_propagate<{mi}>") or ent.get(f"kp::k_propagate<{mi}>") or {}
        traffic = rec.get("dram_bytes")
        if rec.get("issue_active_pct") is not None:
            # the resource the launch is actually bound by: instruction issue
            # (FP32 is a minority of the issued instructions; SIMT = active lanes / 32)
            issue = {"issue_active_frac": rec["issue_active_pct"] / 100.0,
                     "simt_lanes_per_inst": rec.get("simt"), "warp_inst_per_launch": rec.get("warp_inst"),
                     "fp32_share_of_thread_inst": rec.get("fp32_share"), "source": rec.get("source")}
    except Exception:
        pass
    return {
        "kernel": "k_propagate",
        "bound": "fp32",
        "achieved": achieved / 1e12, "peak": pk["fp32_lane_ops"] / 1e12, "unit": "T lane-op/s",
        "frac": achieved / pk["fp32_lane_ops"], "traffic": traffic,
        "traffic_note": "dram bytes/launch of a steady-state launch, profiles/ncu_traffic.json (working set is L2-resident)",
        "issue": issue,
        "peak_src": pk["fp32_src"],
        "ops_per_launch": ops_launch, "avg_launch_us": t_prop * 1e6, "launches": n_prop,
        # propagations per second of the propagate kernel alone (SURVEY.md §8d:
        # reported beside the whole-query rate; per-launch CUDA events, serialised)
        "items_per_s_kernel_only": d["items"] / d["t_propagate_s"] if d["t_propagate_s"] > 0 else None,
        "ops_convention": "FP32 lane-ops of the pinned recipe: FFMA, FADD, FMUL, FSETP, FMNMX, FDIV each = 1",
        "share_of_iteration_time": d["t_propagate_s"] / t_total if t_total else None,
        "select": {"kernel": "k_select_reduce", "bound": "latency (L2-resident dependent loads; HBM shown for scale)",
                   "achieved": sel_gbs, "peak": pk["hbm_gbs"],
                   "unit": "GB/s", "frac": sel_gbs / pk["hbm_gbs"], "avg_launch_us": t_sel * 1e6,
                   "peak_src": pk["hbm_src"],
                   "share_of_iteration_time": d["t_select_s"] / t_total if t_total else None},
        "scatter": {"kernel": "k_select_scatter", "avg_launch_us": d["t_scatter_s"] / max(1, d["n_scatter"]) * 1e6,
                    "share_of_iteration_time": d["t_scatter_s"] / t_total if t_total else None},
        "state_dims": n, "control_dims": m,
    }


def run_sweep(args, scenario):
    """BASELINE config 5: propagate throughput vs samples per iteration
    (2^14 .. 2^22) on a synthetic frontier, lambda = 32, M = 2^k / 32 nodes."""
    import torch

    from paper_2602_02846_b200 import Planner

    pk = _peaks()
    model = scenario["problem"]["model"]
    s = json.loads(json.dumps(scenario))
    s["planner"]["capacity"] = max(int(s["planner"].get("capacity", 0)), (1 << 22) // 32)
    s["planner"]["max_slots"] = 1 << 22
    rows = []
    windows = []  # clocks are kept from the timed launches only (the synthetic frontier is built on the host)
    with ClockSampler(0) as clk, Planner(s, device=0, seed=1) as g:
        g.sweep(1 << 10, launches=max(3, args.warmup))  # warm-up
        for k in range(14, 23):
            n = (1 << k) // int(s["planner"]["lambda"])
            ms_w, _ = g.sweep(n, launches=max(3, args.warmup))  # untimed launches at this size
            # at least ~0.25 s of launches per size, so the clock sampler sees the load
            launches = max(3, args.steps, int(250.0 / max(ms_w, 1e-3)))
            t0 = time.time()
            ms, one = g.sweep(n, launches=launches)
            windows.append((t0, time.time()))
            ops = lane_ops(model, one)
            rate = ops / (ms * 1e-3)
            rows.append({"k": k, "items": one["items"], "frontier_nodes": n, "ms_per_launch": ms,
                         "items_per_s": one["items"] / (ms * 1e-3), "rk4_steps": one["rk4_steps"],
                         "lane_ops_per_launch": ops, "achieved_T_lane_ops": rate / 1e12,
                         "frac": rate / pk["fp32_lane_ops"], "launches": launches})
    clk.only_within(windows)
    best = max(rows, key=lambda r: r["frac"])
    line = {"metric": "node propagations/sec (propagate kernel, synthetic frontier sweep)",
            "value": best["items_per_s"], "unit": "propagations/s", "n_gpus": 1, "steps": max(3, args.steps),
            "warmup": max(3, args.warmup), "higher_is_better": True, "dtype": "f32", "data": "synthetic frontier (positions uniform "
            "in free space, hover-ish), region table reset per launch",
            "config": {"workload": f"{args.config} propagate sweep 2^14..2^22 samples per launch", "lambda":
                       s["planner"]["lambda"]},
            "roofline": {"kernel": f"k_propagate<{model}>", "bound": "fp32", "achieved": best["achieved_T_lane_ops"],
                         "peak": pk["fp32_lane_ops"] / 1e12, "unit": "T lane-op/s", "frac": best["frac"],
                         "peak_src": pk["fp32_src"], "at_k": best["k"]},
            "sweep": rows, "clocks": clk.summary()}
    print(json.dumps(line))
    return 0


def run_batch(args, scenario):
    """BASELINE config 4: a batch of independent seeded queries per GPU through
    the concurrent batch engine (replicas; ranks take queries round-robin)."""
    import torch

    from paper_2602_02846_b200 import BatchPlanner, replicas

    ws, rank, local = _dist()
    local, red_dev = _init_ranks(ws, local)
    s = json.loads(json.dumps(scenario))
    s["planner"]["capacity"] = 1 << 19
    s["planner"]["max_slots"] = 1 << 21
    all_seeds = list(range(args.seed_base, args.seed_base + args.batch))
    mine = replicas.round_robin(all_seeds, rank, ws)
    budget = args.budget_ms / 1000.0
    with BatchPlanner(s, lanes=args.lanes, device=local) as b, ClockSampler(local) as clk:
        b.solve(list(range(900000, 900000 + args.lanes)), budget)  # warm-up: one query per lane
        if ws > 1:
            torch.distributed.barrier()
        res, wall = b.solve(mine, budget)
        if ws > 1:
            torch.distributed.barrier()
    props = sum(r["propagations_attempted"] for r in res)
    wall_max, props_total = replicas.reduce_job(wall * 1e3, props, world=ws, device=red_dev)
    res_all = replicas.gather_results(res, world=ws)
    if rank == 0:
        ttfs = [r["first_solution_s"] * 1e3 for r in res_all if r["found"]]
        costs = [r["best_cost"] for r in res_all if r["found"]]
        line = {
            "metric": "node propagations/sec", "value": props_total / (wall_max / 1e3), "unit": "propagations/s",
            "n_gpus": ws, "steps": len(all_seeds), "warmup": args.lanes, "ms_per_step": wall_max / max(1, len(mine)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (pinned scene geometry, seeded queries)",
            "config": {"workload": f"{args.config}: batch of {len(all_seeds)} independent seeded queries, "
                                   f"{args.budget_ms:g} ms budget each, {args.lanes} concurrent lanes per GPU",
                       "parallelism": f"replicas x{ws} (round-robin)", "lanes": args.lanes},
            "metrics": {"queries_per_s": len(all_seeds) / (wall_max / 1e3),
                        "ms_to_first_solution_median": _median(ttfs), "ms_to_first_solution_p25_p75": _quart(ttfs),
                        "solution_cost_at_budget_median": _median(costs), "success_rate": len(ttfs) / len(res_all),
                        "node_propagations_per_sec": props_total / (wall_max / 1e3)},
            "timing": "host wall clock around kp_batch_solve (max over ranks)",
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="forest_di6",
                    help="a bundled scenario name (paper_2602_02846_b200/scenarios/) or a scenario JSON path")
    ap.add_argument("--budget-ms", type=float, default=100.0)
    ap.add_argument("--iters", type=int, default=0, help="fixed iterations per step instead of a time budget "
                                                          "(profiling runs; not the headline workload)")
    ap.add_argument("--seed-base", type=int, default=1000)
    ap.add_argument("--cpu-sample-s", type=float, default=10.0, help="CPU baseline sample: total seconds")
    ap.add_argument("--dist-seeds", type=int, default=100,
                    help="seeds 0..N-1 for the TTFS / cost distributions (untimed; 0 = skip)")
    ap.add_argument("--cpu-query-s", type=float, default=2.5, help="CPU baseline sample: budget per query")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other-config summaries")
    ap.add_argument("--sweep", action="store_true", help="BASELINE config 5: propagate throughput sweep")
    ap.add_argument("--batch", type=int, default=0, help="BASELINE config 4: number of queries in the batch")
    ap.add_argument("--lanes", type=int, default=8, help="concurrent planner lanes per GPU (--batch; 8 measured best)")
    args = ap.parse_args()
    from paper_2602_02846_b200 import scenarios

    scenario = scenarios.load(args.config)
    if args.impl == "reference":
        return run_reference(args, scenario)
    if args.sweep:
        return run_sweep(args, scenario)
    if args.batch:
        return run_batch(args, scenario)
    return run_b200(args, scenario)


if __name__ == "__main__":
    sys.exit(main())
