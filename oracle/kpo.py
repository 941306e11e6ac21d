"""ctypes wrapper of the CPU oracle (oracle/build/libkpo.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg.  Never by the
product package.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_2602_02846_b200._capi import ConfigDesc, Descriptors, ProblemDesc, Result, TimelineEntry  # noqa: E402

MIRROR32 = 0
FAITHFUL64 = 1
_LIB = None


def lib_path() -> str:
    return os.path.join(_HERE, "build", "libkpo.so")


def load() -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(lib_path()):
        raise RuntimeError(f"{lib_path()} missing: run `make -C oracle`")
    L = C.CDLL(lib_path())
    P, CP, D, I, U64, SZ = C.c_void_p, C.POINTER, C.c_double, C.c_int, C.c_uint64, C.c_size_t
    L.kpo_last_error.restype = C.c_char_p
    L.kpo_create.argtypes = [CP(ProblemDesc), CP(ConfigDesc), I, CP(P)]
    L.kpo_destroy.argtypes = [P]
    L.kpo_destroy.restype = None
    L.kpo_reset.argtypes = [P, U64]
    L.kpo_run.argtypes = [P, D, U64, I, CP(Result)]
    L.kpo_get_nodes.argtypes = [P, P, P, P, P, P, P, P, P, SZ, CP(SZ)]
    L.kpo_get_table.argtypes = [P, P, SZ, CP(SZ)]
    L.kpo_get_timeline.argtypes = [P, CP(TimelineEntry), SZ, CP(SZ)]
    L.kpo_get_grid.argtypes = [P, P, P, CP(U64)]
    L.kpo_propagate_items.argtypes = [P, SZ, P, P, P, P, C.c_uint32, P, P, P, P, P, P, P, P]
    L.kpo_mix64.argtypes = [U64]
    L.kpo_mix64.restype = U64
    L.kpo_derive_stream.argtypes = [U64, U64, U64, U64]
    L.kpo_derive_stream.restype = U64
    L.kpo_splitmix.argtypes = [U64, SZ, P, P]
    L.kpo_splitmix.restype = None
    L.kpo_philox.argtypes = [P, P, P]
    L.kpo_philox.restype = None
    L.kpo_wrap_angle.argtypes = [D]
    L.kpo_wrap_angle.restype = D
    L.kpo_wrap_angle_f32.argtypes = [C.c_float]
    L.kpo_wrap_angle_f32.restype = C.c_float
    L.kpo_sincos_f32.argtypes = [C.c_float, CP(C.c_float), CP(C.c_float)]
    L.kpo_sincos_f32.restype = None
    L.kpo_segment_cost.argtypes = [P, SZ, I, I, I, D, CP(D)]
    L.kpo_in_goal.argtypes = [P, I, P, P, I, D]
    L.kpo_propagate_ode.argtypes = [P, P, P, D, D, P, SZ, CP(SZ)]
    L.kpo_derivative.argtypes = [P, P, P, P]
    L.kpo_is_state_valid.argtypes = [P, P]
    L.kpo_is_segment_valid.argtypes = [P, P, SZ]
    L.kpo_region_index.argtypes = [P, P]
    L.kpo_region_index.restype = C.c_uint32
    L.kpo_atomic_min_stress.argtypes = [SZ, SZ, P, P, I, P, P]
    _LIB = L
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[kpo status {code}] {msg}")
        self.code = code


class Oracle:
    """One CPU planner instance: policy MIRROR32 (bit-exact device mirror) or
    FAITHFUL64 (the reference's fp64 / SplitMix64 CPU planner)."""

    def __init__(self, scenario: dict, policy: int = MIRROR32, seed: int | None = None, workers: int | None = None):
        self.L = load()
        self.desc = Descriptors(scenario)
        if seed is not None:
            self.desc.config.seed = seed
        if workers is not None:
            self.desc.config.workers = workers
        self.n, self.m = self.desc.n, self.desc.m
        h = C.c_void_p()
        rc = self.L.kpo_create(C.byref(self.desc.problem), C.byref(self.desc.config), policy, C.byref(h))
        if rc:
            raise OracleError(rc, self.L.kpo_last_error().decode())
        self.h = h

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.kpo_last_error().decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.kpo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, seed: int):
        self._check(self.L.kpo_reset(self.h, seed))

    def run(self, budget_s: float = -1.0, max_iterations: int = 0, stop_first: int = -1) -> dict:
        r = Result()
        self._check(self.L.kpo_run(self.h, budget_s, max_iterations, stop_first, C.byref(r)))
        return r.as_dict()

    def nodes(self) -> dict:
        n = C.c_size_t()
        self._check(self.L.kpo_get_nodes(self.h, *([None] * 8), 0, C.byref(n)))
        k = n.value
        out = {
            "state": np.zeros((k, self.n)), "control": np.zeros((k, self.m)), "dt": np.zeros(k),
            "acc": np.zeros(k), "parent": np.zeros(k, np.int64), "region": np.zeros(k, np.uint32),
            "status": np.zeros(k, np.uint8), "icount": np.zeros(k, np.uint32),
        }
        self._check(self.L.kpo_get_nodes(self.h, _p(out["state"]), _p(out["control"]), _p(out["dt"]),
                                         _p(out["acc"]), _p(out["parent"]), _p(out["region"]), _p(out["status"]),
                                         _p(out["icount"]), k, C.byref(n)))
        return out

    def table(self) -> np.ndarray:
        n = C.c_size_t()
        self._check(self.L.kpo_get_table(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value)
        self._check(self.L.kpo_get_table(self.h, _p(out), n.value, C.byref(n)))
        return out

    def timeline(self) -> list[dict]:
        n = C.c_size_t()
        self._check(self.L.kpo_get_timeline(self.h, None, 0, C.byref(n)))
        buf = (TimelineEntry * max(1, n.value))()
        self._check(self.L.kpo_get_timeline(self.h, buf, n.value, C.byref(n)))
        return [{"iteration": e.iteration, "elapsed_s": e.elapsed_s, "cost": e.cost, "leaf": e.leaf}
                for e in buf[: n.value]]

    def grid(self):
        cells = np.zeros(8, np.int64)
        side = np.zeros(8)
        nr = C.c_uint64()
        self._check(self.L.kpo_get_grid(self.h, _p(cells), _p(side), C.byref(nr)))
        return cells, side, nr.value

    def propagate_items(self, parent_states, parent_acc, node_ids, branches, iteration: int) -> dict:
        ps = np.ascontiguousarray(parent_states, np.float64).reshape(-1, self.n)
        k = ps.shape[0]
        pa = np.ascontiguousarray(parent_acc, np.float64)
        ids = np.ascontiguousarray(node_ids, np.uint32)
        brs = np.ascontiguousarray(branches, np.uint32)
        out = {
            "valid": np.zeros(k, np.uint8), "state": np.zeros((k, self.n)), "control": np.zeros((k, self.m)),
            "dt": np.zeros(k), "acc": np.zeros(k), "region": np.zeros(k, np.uint32),
            "steps": np.zeros(k, np.uint32), "goal": np.zeros(k, np.uint8),
        }
        self._check(self.L.kpo_propagate_items(
            self.h, k, _p(ps), _p(pa), _p(ids), _p(brs), iteration, _p(out["valid"]), _p(out["state"]),
            _p(out["control"]), _p(out["dt"]), _p(out["acc"]), _p(out["region"]), _p(out["steps"]),
            _p(out["goal"])))
        return out

    def propagate_ode(self, x, u, dt: float, h: float) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        cap = int(np.ceil(dt / h)) + 4
        out = np.zeros((cap, self.n))
        n = C.c_size_t()
        self._check(self.L.kpo_propagate_ode(self.h, _p(x), _p(u), dt, h, _p(out), cap, C.byref(n)))
        return out[: n.value]

    def derivative(self, x, u) -> np.ndarray:
        out = np.zeros(self.n)
        self._check(self.L.kpo_derivative(self.h, _p(np.ascontiguousarray(x, np.float64)),
                                          _p(np.ascontiguousarray(u, np.float64)), _p(out)))
        return out

    def is_state_valid(self, x) -> bool:
        return bool(self.L.kpo_is_state_valid(self.h, _p(np.ascontiguousarray(x, np.float64))))

    def is_segment_valid(self, samples) -> bool:
        s = np.ascontiguousarray(samples, np.float64)
        return bool(self.L.kpo_is_segment_valid(self.h, _p(s), s.shape[0]))

    def region_index(self, x) -> int:
        return int(self.L.kpo_region_index(self.h, _p(np.ascontiguousarray(x, np.float64))))


# ---- standalone ops ---------------------------------------------------------
def mix64(z: int) -> int:
    return load().kpo_mix64(z)


def derive_stream(seed, it, node, br) -> int:
    return load().kpo_derive_stream(seed, it, node, br)


def splitmix(seed: int, count: int):
    raw = np.zeros(count, np.uint64)
    unit = np.zeros(count)
    load().kpo_splitmix(seed, count, _p(raw), _p(unit))
    return raw, unit


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    load().kpo_philox(_p(c), _p(k), _p(out))
    return out


def wrap_angle(a: float) -> float:
    return load().kpo_wrap_angle(a)


def wrap_angle_f32(a: float) -> float:
    return load().kpo_wrap_angle_f32(a)


def sincos_f32(x: float):
    s, c = C.c_float(), C.c_float()
    load().kpo_sincos_f32(x, C.byref(s), C.byref(c))
    return s.value, c.value


def segment_cost(samples, position_dims: int, kind: int, duration: float) -> float:
    s = np.ascontiguousarray(samples, np.float64)
    out = C.c_double()
    rc = load().kpo_segment_cost(_p(s), s.shape[0], s.shape[1] if s.ndim == 2 else 0, position_dims, kind,
                                 duration, C.byref(out))
    if rc:
        raise OracleError(rc, load().kpo_last_error().decode())
    return out.value


def in_goal(x, dims, center, radius) -> bool:
    x = np.ascontiguousarray(x, np.float64)
    d = np.ascontiguousarray(dims, np.int32)
    c = np.ascontiguousarray(center, np.float64)
    return bool(load().kpo_in_goal(_p(x), len(x), _p(d), _p(c), len(d), radius))


def atomic_min_stress(n_regions: int, regions, costs, workers: int):
    r = np.ascontiguousarray(regions, np.uint32)
    c = np.ascontiguousarray(costs, np.float64)
    table = np.zeros(n_regions)
    outcomes = np.zeros(len(r), np.uint8)
    rc = load().kpo_atomic_min_stress(n_regions, len(r), _p(r), _p(c), workers, _p(table), _p(outcomes))
    if rc:
        raise OracleError(rc, load().kpo_last_error().decode())
    return table, outcomes
