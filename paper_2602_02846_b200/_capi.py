"""ctypes mirror of include/kinoplan_b200.h (the C-ABI drop-in boundary).

Shared by the product wrapper (planner.py) and the test harness: the oracle's
C entry points take the same POD descriptors, so both sides are driven from
byte-identical problem/config values.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

KP_OK = 0
KP_ERR_SCHEMA = 1
KP_ERR_INVALID_PROBLEM = 2
KP_ERR_CONFIG = 3
KP_ERR_GRID_TOO_FINE = 4
KP_ERR_INVALID_SEGMENT = 5
KP_ERR_CUDA = 6
KP_ERR_ARGUMENT = 7
KP_ERR_SLOT_OVERFLOW = 8

MODEL_IDS = {
    "double_integrator_4d": 0,
    "double_integrator_6d": 1,
    "dubins_airplane_6d": 2,
    "quadcopter_12d": 3,
}
MODEL_SHAPES = {  # model.hpp:64-68; (state_dim, control_dim, position_dims, angle_dims)
    "double_integrator_4d": (4, 2, (0, 1), ()),
    "double_integrator_6d": (6, 3, (0, 1, 2), ()),
    "dubins_airplane_6d": (6, 3, (0, 1, 2), (3,)),
    "quadcopter_12d": (12, 4, (0, 1, 2), (6, 7, 8)),
}
COST_KINDS = {"path_length": 0, "control_duration": 1}
RNG_KINDS = {"philox": 0, "splitmix": 1}


class Obstacle(C.Structure):
    _fields_ = [("type", C.c_int32), ("reserved", C.c_int32), ("a", C.c_double * 3), ("b", C.c_double * 3)]


class ProblemDesc(C.Structure):
    _fields_ = [
        ("model", C.c_int32),
        ("n_params", C.c_int32),
        ("param_names", C.POINTER(C.c_char_p)),
        ("param_values", C.POINTER(C.c_double)),
        ("state_dim", C.c_int32),
        ("control_dim", C.c_int32),
        ("x_init", C.POINTER(C.c_double)),
        ("state_lo", C.POINTER(C.c_double)),
        ("state_hi", C.POINTER(C.c_double)),
        ("control_lo", C.POINTER(C.c_double)),
        ("control_hi", C.POINTER(C.c_double)),
        ("workspace_dim", C.c_int32),
        ("n_obstacles", C.c_int32),
        ("workspace_lo", C.POINTER(C.c_double)),
        ("workspace_hi", C.POINTER(C.c_double)),
        ("obstacles", C.POINTER(Obstacle)),
        ("goal_n_dims", C.c_int32),
        ("reserved0", C.c_int32),
        ("goal_dims", C.POINTER(C.c_int32)),
        ("goal_center", C.POINTER(C.c_double)),
        ("goal_radius", C.c_double),
        ("cost_kind", C.c_int32),
        ("cost_position_dims", C.c_int32),
        ("grid_n_dims", C.c_int32),
        ("reserved1", C.c_int32),
        ("grid_dims", C.POINTER(C.c_int32)),
        ("grid_cells", C.POINTER(C.c_int32)),
        ("grid_delta", C.c_double),
        ("grid_max_cells", C.c_uint64),
    ]


class ConfigDesc(C.Structure):
    _fields_ = [
        ("lambda_", C.c_int32),
        ("i_max", C.c_int32),
        ("t_max_s", C.c_double),
        ("t_prop", C.c_double),
        ("ode_step", C.c_double),
        ("collision_step", C.c_double),
        ("capacity", C.c_uint64),
        ("seed", C.c_uint64),
        ("max_iterations", C.c_uint64),
        ("workers", C.c_int32),
        ("deactivate_after_expansion", C.c_int32),
        ("rng_kind", C.c_int32),
        ("stop_at_first_solution", C.c_int32),
        ("max_slots", C.c_uint64),
    ]


class Result(C.Structure):
    _fields_ = [
        ("found", C.c_int32),
        ("capacity_exhausted", C.c_int32),
        ("best_cost", C.c_double),
        ("best_leaf", C.c_int64),
        ("best_found_at_s", C.c_double),
        ("best_found_iteration", C.c_uint64),
        ("first_solution_s", C.c_double),
        ("first_solution_cost", C.c_double),
        ("first_solution_iteration", C.c_uint64),
        ("elapsed_s", C.c_double),
        ("iterations", C.c_uint64),
        ("propagations_attempted", C.c_uint64),
        ("propagations_valid", C.c_uint64),
        ("propagations_admitted", C.c_uint64),
        ("nodes_committed", C.c_uint64),
        ("nodes_pruned_terminal", C.c_uint64),
        ("nodes_deactivated", C.c_uint64),
        ("nodes_reactivated", C.c_uint64),
        ("candidates_dropped_capacity", C.c_uint64),
        ("node_count", C.c_uint64),
        ("timeline_len", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class Profile(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("graph_launches", C.c_uint64), ("t_propagate_s", C.c_double),
                ("t_select_s", C.c_double), ("t_scatter_s", C.c_double), ("n_propagate", C.c_uint64),
                ("n_select", C.c_uint64), ("n_scatter", C.c_uint64), ("items", C.c_uint64),
                ("rk4_steps", C.c_uint64), ("samples_checked", C.c_uint64), ("interp_points", C.c_uint64),
                ("box_tests", C.c_uint64), ("sphere_tests", C.c_uint64), ("live_scanned", C.c_uint64),
                ("ancestor_hops", C.c_uint64), ("slots_scanned", C.c_uint64), ("admitted_checked", C.c_uint64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class TraceEntry(C.Structure):
    _fields_ = [("t_ns", C.c_uint64), ("iteration", C.c_uint32), ("items", C.c_uint32), ("live", C.c_uint32),
                ("frontier", C.c_uint32), ("nodes", C.c_uint32), ("committed", C.c_uint32),
                ("t_prop", C.c_uint32), ("t_sel", C.c_uint32), ("t_sel_end", C.c_uint32), ("t_scat", C.c_uint32)]


class TimelineEntry(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("elapsed_s", C.c_double), ("cost", C.c_double), ("leaf", C.c_int64)]


def _arr(values, ctype):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


class Descriptors:
    """Owns the ctypes arrays a ProblemDesc/ConfigDesc point into."""

    def __init__(self, scenario: dict):
        pr = scenario["problem"]
        model = pr["model"]
        if model not in MODEL_IDS:
            raise ValueError(f"unknown dynamics model id: {model!r}")
        n, m, pos, _ = MODEL_SHAPES[model]
        env = pr["environment"]
        self._keep = []
        k = self._keep.append
        params = pr.get("model_params", {}) or {}
        names = [s.encode() for s in params.keys()]
        self.names = (C.c_char_p * max(1, len(names)))(*names)
        self.values = _arr(params.values(), C.c_double)
        sb = pr["state_bounds"]
        cb = pr["control_bounds"]
        wb = env["workspace_bounds"]
        obs = env.get("obstacles", [])
        self.obst = (Obstacle * max(1, len(obs)))()
        for i, o in enumerate(obs):
            if o["type"] == "box":
                self.obst[i].type = 0
                lo, hi = list(o["min"]) + [0.0] * 3, list(o["max"]) + [0.0] * 3
                for j in range(3):
                    self.obst[i].a[j] = lo[j]
                    self.obst[i].b[j] = hi[j]
            elif o["type"] == "sphere":
                self.obst[i].type = 1
                c = list(o["center"]) + [0.0] * 3
                for j in range(3):
                    self.obst[i].a[j] = c[j]
                self.obst[i].b[0] = o["radius"]
            else:
                raise ValueError(f"obstacle {i}: unknown type {o['type']!r}")
        goal = pr["goal"]
        dec = scenario["decomposition"]
        arrays = dict(
            x_init=_arr(pr["x_init"], C.c_double),
            state_lo=_arr([b[0] for b in sb], C.c_double),
            state_hi=_arr([b[1] for b in sb], C.c_double),
            control_lo=_arr([b[0] for b in cb], C.c_double),
            control_hi=_arr([b[1] for b in cb], C.c_double),
            workspace_lo=_arr([b[0] for b in wb], C.c_double),
            workspace_hi=_arr([b[1] for b in wb], C.c_double),
            goal_dims=_arr(goal.get("dims", list(pos)), C.c_int32),
            goal_center=_arr(goal["center"], C.c_double),
            grid_dims=_arr(dec["dims"], C.c_int32),
        )
        for v in arrays.values():
            k(v)
        cells = dec.get("cells")
        self.cells = _arr(cells, C.c_int32) if cells else None
        cost = pr.get("cost", "path_length")
        if isinstance(cost, dict):
            cost_kind, cost_pd = cost.get("kind", "path_length"), cost.get("position_dims", len(pos))
        else:
            cost_kind, cost_pd = cost, len(pos)
        p = ProblemDesc()
        p.model = MODEL_IDS[model]
        p.n_params = len(names)
        p.param_names = C.cast(self.names, C.POINTER(C.c_char_p))
        p.param_values = C.cast(self.values, C.POINTER(C.c_double))
        p.state_dim = len(pr["x_init"])
        p.control_dim = len(cb)
        for name in ("x_init", "state_lo", "state_hi", "control_lo", "control_hi", "workspace_lo", "workspace_hi"):
            setattr(p, name, C.cast(arrays[name], C.POINTER(C.c_double)))
        p.workspace_dim = len(wb)
        p.n_obstacles = len(obs)
        p.obstacles = C.cast(self.obst, C.POINTER(Obstacle))
        p.goal_n_dims = len(goal.get("dims", list(pos)))
        p.goal_dims = C.cast(arrays["goal_dims"], C.POINTER(C.c_int32))
        p.goal_center = C.cast(arrays["goal_center"], C.POINTER(C.c_double))
        p.goal_radius = goal["radius"]
        if cost_kind not in COST_KINDS:
            raise ValueError(f"unknown cost metric kind: {cost_kind!r}")
        p.cost_kind = COST_KINDS[cost_kind]
        p.cost_position_dims = cost_pd
        p.grid_n_dims = len(dec["dims"])
        p.grid_dims = C.cast(arrays["grid_dims"], C.POINTER(C.c_int32))
        p.grid_cells = C.cast(self.cells, C.POINTER(C.c_int32)) if self.cells is not None else None
        p.grid_delta = float(dec.get("delta", 0.0) or 0.0)
        p.grid_max_cells = int(dec.get("max_cells", 0))
        self.problem = p
        pl = scenario["planner"]
        c = ConfigDesc()
        c.lambda_ = int(pl.get("lambda", 32))
        c.i_max = int(pl.get("i_max", 5))
        c.t_max_s = float(pl.get("t_max_ms", 100.0)) / 1000.0
        c.t_prop = float(pl["t_prop"])
        c.ode_step = float(pl.get("ode_step", 0.0) or 0.0)
        c.collision_step = float(pl.get("collision_step", 0.05))
        c.capacity = int(pl.get("capacity", 1 << 20))
        c.seed = int(pl.get("seed", scenario.get("trials", {}).get("base_seed", 0)))
        c.max_iterations = int(pl.get("max_iterations", 0) or 0)
        c.workers = int(scenario.get("trials", {}).get("workers", 1))
        c.deactivate_after_expansion = int(bool(pl.get("deactivate_after_expansion", False)))
        c.rng_kind = RNG_KINDS[pl.get("rng", "philox")]
        c.stop_at_first_solution = int(bool(pl.get("stop_at_first_solution", False)))
        c.max_slots = int(pl.get("max_slots", 0) or 0)
        self.config = c
        self.n, self.m = n, m


_LIB = None


def lib_path() -> str:
    here = os.path.dirname(os.path.abspath(__file__))
    return os.path.join(here, "lib", "libkinoplan_b200.so")


def load_library() -> C.CDLL:
    """Load the sm_100a planner library.  Fails loudly when it is missing:
    there is no CPU fallback on the product path."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make`). The planner has no CPU fallback."
        )
    L = C.CDLL(path)
    P, CP, D, I = C.c_void_p, C.POINTER, C.c_double, C.c_int
    L.kp_create.argtypes = [CP(ProblemDesc), CP(ConfigDesc), I, CP(P)]
    L.kp_create.restype = I
    L.kp_destroy.argtypes = [P]
    L.kp_destroy.restype = None
    L.kp_last_error.argtypes = [P]
    L.kp_last_error.restype = C.c_char_p
    L.kp_reset.argtypes = [P, C.c_uint64]
    L.kp_reset.restype = I
    L.kp_reset_query.argtypes = [P, C.c_uint64, P]
    L.kp_reset_query.restype = I
    L.kp_set_stop_at_first_solution.argtypes = [P, I]
    L.kp_set_stop_at_first_solution.restype = I
    L.kp_solve.argtypes = [P, D, C.c_uint64, CP(Result)]
    L.kp_solve.restype = I
    L.kp_solve_batch.argtypes = [P, CP(C.c_uint64), C.c_size_t, D, C.c_uint64, CP(Result)]
    L.kp_solve_batch.restype = I
    L.kp_get_timeline.argtypes = [P, CP(TimelineEntry), C.c_size_t, CP(C.c_size_t)]
    L.kp_get_timeline.restype = I
    L.kp_get_path.argtypes = [P, C.c_int64, P, P, P, P, C.c_size_t, CP(C.c_size_t)]
    L.kp_get_path.restype = I
    L.kp_get_trajectory.argtypes = [P, C.c_int64, P, C.c_size_t, CP(C.c_size_t), P, C.c_size_t, CP(C.c_size_t)]
    L.kp_get_trajectory.restype = I
    L.kp_get_nodes.argtypes = [P, P, P, P, P, P, P, P, P, C.c_size_t, CP(C.c_size_t)]
    L.kp_get_nodes.restype = I
    L.kp_get_region_table.argtypes = [P, P, C.c_size_t, CP(C.c_size_t)]
    L.kp_get_region_table.restype = I
    L.kp_get_grid.argtypes = [P, P, P, CP(C.c_uint64)]
    L.kp_get_grid.restype = I
    L.kp_debug_propagate.argtypes = [P, C.c_size_t, P, P, P, P, C.c_uint32, P, P, P, P, P, P, P, P]
    L.kp_debug_propagate.restype = I
    L.kp_set_profiling.argtypes = [P, I]
    L.kp_set_profiling.restype = I
    L.kp_get_profile.argtypes = [P, CP(Profile)]
    L.kp_get_profile.restype = I
    L.kp_get_trace.argtypes = [P, CP(TraceEntry), C.c_size_t, CP(C.c_size_t)]
    L.kp_get_trace.restype = I
    L.kp_get_stream.argtypes = [P, CP(C.c_void_p)]
    L.kp_get_stream.restype = I
    L.kp_sweep_setup.argtypes = [P, C.c_uint64, C.c_uint64]
    L.kp_sweep_setup.restype = I
    L.kp_sweep_run.argtypes = [P, C.c_uint32, CP(D), CP(Profile)]
    L.kp_sweep_run.restype = I
    L.kp_batch_create.argtypes = [CP(ProblemDesc), CP(ConfigDesc), I, I, CP(P)]
    L.kp_batch_create.restype = I
    L.kp_batch_destroy.argtypes = [P]
    L.kp_batch_destroy.restype = None
    L.kp_batch_last_error.argtypes = [P]
    L.kp_batch_last_error.restype = C.c_char_p
    L.kp_batch_solve.argtypes = [P, CP(C.c_uint64), C.c_size_t, D, C.c_uint64, CP(Result), CP(D)]
    L.kp_batch_solve.restype = I
    L.kp_abi_version.argtypes = []
    L.kp_abi_version.restype = I
    _LIB = L
    return L


EXPORTED_SYMBOLS = [
    "kp_create", "kp_destroy", "kp_last_error", "kp_reset", "kp_reset_query", "kp_set_stop_at_first_solution",
    "kp_solve", "kp_get_timeline", "kp_get_path",
    "kp_get_trajectory", "kp_get_nodes", "kp_get_region_table", "kp_get_grid", "kp_debug_propagate",
    "kp_set_profiling", "kp_get_profile", "kp_get_trace", "kp_get_stream", "kp_solve_batch", "kp_sweep_setup", "kp_sweep_run", "kp_batch_create", "kp_batch_destroy",
    "kp_batch_last_error", "kp_batch_solve", "kp_abi_version",
]


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None
