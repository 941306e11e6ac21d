"""Python mirror of the reference planner API over the C-ABI.

Same names and error behaviour as the reference's `kinoplan` library
(errors.hpp:11-33, SPEC.md:370 `plan(problem, config)`), driving the sm_100a
library through include/kinoplan_b200.h.  There is no CPU path: constructing a
Planner without the built library or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import Descriptors, Result, TimelineEntry, load_library, ptr


class KinoplanError(RuntimeError):
    pass


class SchemaError(KinoplanError):            # errors.hpp:11
    pass


class InvalidProblemError(KinoplanError):    # errors.hpp:16
    pass


class ConfigError(KinoplanError):            # errors.hpp:21
    pass


class GridTooFineError(KinoplanError):       # errors.hpp:26
    pass


class InvalidSegmentError(KinoplanError):    # errors.hpp:31
    pass


class DeviceError(KinoplanError):            # CUDA / ABI failures (no reference counterpart)
    pass


_ERRORS = {
    _capi.KP_ERR_SCHEMA: SchemaError,
    _capi.KP_ERR_INVALID_PROBLEM: InvalidProblemError,
    _capi.KP_ERR_CONFIG: ConfigError,
    _capi.KP_ERR_GRID_TOO_FINE: GridTooFineError,
    _capi.KP_ERR_INVALID_SEGMENT: InvalidSegmentError,
}


def _raise(rc: int, msg: bytes | None):
    text = (msg or b"").decode(errors="replace")
    raise _ERRORS.get(rc, DeviceError)(f"[kp status {rc}] {text}")


class Planner:
    """One GPU planner instance (single owner)."""

    def __init__(self, scenario: dict, device: int = 0, seed: int | None = None):
        self._lib = load_library()
        self.scenario = scenario
        self.desc = Descriptors(scenario)
        if seed is not None:
            self.desc.config.seed = seed
        self.n, self.m = self.desc.n, self.desc.m
        h = C.c_void_p()
        rc = self._lib.kp_create(C.byref(self.desc.problem), C.byref(self.desc.config), device, C.byref(h))
        if rc:
            _raise(rc, self._lib.kp_last_error(None))
        self._h = h

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.kp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc):
        if rc:
            _raise(rc, self._lib.kp_last_error(self._h))

    def reset(self, seed: int, x_init=None):
        """New query: seed and (optionally) a new start state, copied host->device."""
        if x_init is None:
            self._check(self._lib.kp_reset(self._h, seed))
        else:
            self._x0 = np.ascontiguousarray(x_init, np.float64)
            self._check(self._lib.kp_reset_query(self._h, seed, ptr(self._x0)))

    def set_stop_at_first_solution(self, on: bool):
        self._check(self._lib.kp_set_stop_at_first_solution(self._h, 1 if on else 0))

    # -- solve -------------------------------------------------------------
    def solve(self, budget_s: float = -1.0, max_iterations: int = 0) -> dict:
        r = Result()
        self._check(self._lib.kp_solve(self._h, budget_s, max_iterations, C.byref(r)))
        return r.as_dict()

    def solve_batch(self, seeds, budget_s: float = -1.0, max_iterations: int = 0) -> list[dict]:
        seeds = list(seeds)
        arr = (C.c_uint64 * len(seeds))(*seeds)
        res = (Result * len(seeds))()
        self._check(self._lib.kp_solve_batch(self._h, arr, len(seeds), budget_s, max_iterations, res))
        return [r.as_dict() for r in res]

    def timeline(self) -> list[dict]:
        n = C.c_size_t()
        self._check(self._lib.kp_get_timeline(self._h, None, 0, C.byref(n)))
        buf = (TimelineEntry * max(1, n.value))()
        self._check(self._lib.kp_get_timeline(self._h, buf, n.value, C.byref(n)))
        return [{"iteration": e.iteration, "elapsed_s": e.elapsed_s, "cost": e.cost, "leaf": e.leaf}
                for e in buf[: n.value]]

    # -- introspection -----------------------------------------------------
    def nodes(self) -> dict:
        n = C.c_size_t()
        self._check(self._lib.kp_get_nodes(self._h, *([None] * 8), 0, C.byref(n)))
        k = n.value
        out = {
            "state": np.zeros((k, self.n), np.float32), "control": np.zeros((k, self.m), np.float32),
            "dt": np.zeros(k, np.float32), "acc": np.zeros(k, np.float32), "parent": np.zeros(k, np.int32),
            "region": np.zeros(k, np.uint32), "status": np.zeros(k, np.uint8), "icount": np.zeros(k, np.uint8),
        }
        self._check(self._lib.kp_get_nodes(self._h, ptr(out["state"]), ptr(out["control"]), ptr(out["dt"]),
                                           ptr(out["acc"]), ptr(out["parent"]), ptr(out["region"]),
                                           ptr(out["status"]), ptr(out["icount"]), k, C.byref(n)))
        return out

    def region_table(self) -> np.ndarray:
        n = C.c_size_t()
        self._check(self._lib.kp_get_region_table(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.uint32)
        self._check(self._lib.kp_get_region_table(self._h, ptr(out), n.value, C.byref(n)))
        return out

    def grid(self):
        cells = np.zeros(8, np.int32)
        side = np.zeros(8, np.float32)
        nr = C.c_uint64()
        self._check(self._lib.kp_get_grid(self._h, ptr(cells), ptr(side), C.byref(nr)))
        g = len(self.scenario["decomposition"]["dims"])
        return cells[:g], side[:g], nr.value

    def path(self, leaf: int = -1) -> dict:
        n = C.c_size_t()
        self._check(self._lib.kp_get_path(self._h, leaf, None, None, None, None, 0, C.byref(n)))
        k = n.value
        st, ct = np.zeros((k, self.n)), np.zeros((k, self.m))
        du, ac = np.zeros(k), np.zeros(k)
        self._check(self._lib.kp_get_path(self._h, leaf, ptr(st), ptr(ct), ptr(du), ptr(ac), k, C.byref(n)))
        return {"states": st, "controls": ct, "durations": du, "acc": ac}

    def trajectory(self, leaf: int = -1) -> dict:
        ns, nseg = C.c_size_t(), C.c_size_t()
        self._check(self._lib.kp_get_trajectory(self._h, leaf, None, 0, C.byref(ns), None, 0, C.byref(nseg)))
        smp = np.zeros((ns.value, self.n))
        sc = np.zeros(nseg.value)
        self._check(self._lib.kp_get_trajectory(self._h, leaf, ptr(smp), ns.value, C.byref(ns), ptr(sc),
                                                nseg.value, C.byref(nseg)))
        return {"samples": smp, "segment_costs": sc}

    def debug_propagate(self, parent_states, parent_acc, node_ids, branches, iteration: int) -> dict:
        ps = np.ascontiguousarray(parent_states, np.float32).reshape(-1, self.n)
        k = ps.shape[0]
        pa = np.ascontiguousarray(parent_acc, np.float32)
        ids = np.ascontiguousarray(node_ids, np.uint32)
        brs = np.ascontiguousarray(branches, np.uint32)
        out = {
            "valid": np.zeros(k, np.uint8), "state": np.zeros((k, self.n), np.float32),
            "control": np.zeros((k, self.m), np.float32), "dt": np.zeros(k, np.float32),
            "acc": np.zeros(k, np.float32), "region": np.zeros(k, np.uint32), "steps": np.zeros(k, np.uint32),
            "goal": np.zeros(k, np.uint8),
        }
        self._check(self._lib.kp_debug_propagate(
            self._h, k, ptr(ps), ptr(pa), ptr(ids), ptr(brs), iteration, ptr(out["valid"]), ptr(out["state"]),
            ptr(out["control"]), ptr(out["dt"]), ptr(out["acc"]), ptr(out["region"]), ptr(out["steps"]),
            ptr(out["goal"])))
        return out

    def set_profiling(self, on: bool):
        self._check(self._lib.kp_set_profiling(self._h, 1 if on else 0))

    def profile(self) -> dict:
        pr = _capi.Profile()
        self._check(self._lib.kp_get_profile(self._h, C.byref(pr)))
        return pr.as_dict()

    def trace(self) -> np.ndarray:
        """Per-iteration device trace: structured array (t_ns, iteration, items, live, frontier, nodes, committed)."""
        n = C.c_size_t()
        self._check(self._lib.kp_get_trace(self._h, None, 0, C.byref(n)))
        buf = (_capi.TraceEntry * max(1, n.value))()
        self._check(self._lib.kp_get_trace(self._h, buf, n.value, C.byref(n)))
        dt = np.dtype([("t_ns", np.uint64), ("iteration", np.uint32), ("items", np.uint32), ("live", np.uint32),
                       ("frontier", np.uint32), ("nodes", np.uint32), ("committed", np.uint32),
                       ("t_prop", np.uint32), ("t_sel", np.uint32), ("t_sel_end", np.uint32), ("t_scat", np.uint32)])
        return np.frombuffer(bytes(buf)[: n.value * dt.itemsize], dtype=dt).copy()

    def sweep(self, n_nodes: int, launches: int = 5, seed: int = 1) -> tuple[float, dict]:
        """Propagate-kernel throughput on a synthetic frontier of n_nodes
        (n_nodes * lambda items per launch; BASELINE config 5).  Returns
        (ms per launch, work counters of one launch)."""
        self._check(self._lib.kp_sweep_setup(self._h, n_nodes, seed))
        ms = C.c_double()
        pr = _capi.Profile()
        self._check(self._lib.kp_sweep_run(self._h, launches, C.byref(ms), C.byref(pr)))
        return ms.value, pr.as_dict()

    def stream(self) -> int:
        s = C.c_void_p()
        self._check(self._lib.kp_get_stream(self._h, C.byref(s)))
        return s.value or 0


class BatchPlanner:
    """Concurrent batch engine (BASELINE config 4): `lanes` planner instances
    on one device, independent seeded queries overlapped on the GPU."""

    def __init__(self, scenario: dict, lanes: int = 16, device: int = 0):
        self._lib = load_library()
        self.desc = Descriptors(scenario)
        h = C.c_void_p()
        rc = self._lib.kp_batch_create(C.byref(self.desc.problem), C.byref(self.desc.config), device, lanes,
                                       C.byref(h))
        if rc:
            _raise(rc, self._lib.kp_last_error(None))
        self._h = h
        self.lanes = lanes

    def solve(self, seeds, budget_s: float = -1.0, max_iterations: int = 0):
        seeds = list(seeds)
        arr = (C.c_uint64 * max(1, len(seeds)))(*seeds)
        res = (Result * max(1, len(seeds)))()
        wall = C.c_double()
        rc = self._lib.kp_batch_solve(self._h, arr, len(seeds), budget_s, max_iterations, res, C.byref(wall))
        if rc:
            _raise(rc, self._lib.kp_batch_last_error(self._h))
        return [r.as_dict() for r in res[: len(seeds)]], wall.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.kp_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def plan(scenario: dict, seed: int | None = None, device: int = 0, budget_s: float = -1.0,
         max_iterations: int = 0) -> dict:
    """plan(problem, config): one fresh run; returns the result
    dict plus the timeline and, when found, the root->leaf path."""
    with Planner(scenario, device=device, seed=seed) as p:
        r = p.solve(budget_s, max_iterations)
        r["timeline"] = p.timeline()
        if r["found"]:
            r["path"] = p.path()
        return r
