"""Scenario files (SPEC.md:518 schema) and the bundled benchmark scenes.

A scenario is a plain dict / JSON document with the reference's top-level keys
`name`, `problem` {model, model_params, environment, x_init, goal, cost,
state_bounds, control_bounds}, `decomposition` {dims, delta | cells},
`planner` {lambda, i_max, t_prop, capacity, ode_step, collision_step,
t_max_ms, max_iterations, deactivate_after_expansion, + rng, max_slots,
stop_at_first_solution}, `trials` {n, base_seed, workers}.

The reference's bundled scenes (`proj/scenarios/`) are absent, so
the geometry of the BASELINE.json configs is pinned here:
  forest_di6       6D double integrator, trees (PAPER.md:687 env a)   27,000 regions
  narrow_dubins6   6D Dubins airplane, wall with one slot (env b)     52,000 regions
  building_quad12  12D quadcopter, rooms + doorways (env c)           100,000 regions
plus the SPEC's bundled set (free2d, zigzag2d, forest6d,
narrow6d, building6d, zigzag6d, dubins_narrow, quad12d_forest, each also as
`<name>_small`, the small-δ variant).
"""
from __future__ import annotations

import copy
import json
import math
import os

SCENARIO_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenarios")

MASK64 = (1 << 64) - 1


class SchemaError(ValueError):
    """Malformed scenario (errors.hpp:11 SchemaError)."""


def _splitmix64(seed: int):
    """rng.hpp:12-31 SplitMix64, used to place the forest's trees reproducibly."""
    state = seed & MASK64
    while True:
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def _unit(gen) -> float:
    return (next(gen) >> 11) * 2.0**-53


def forest_di6(n_trees: int = 50, seed: int = 2602) -> dict:
    """Config 1: 6D double integrator in a forest of full-height 0.5 x 0.5 m trees."""
    start, goal = (0.5, 0.5, 5.0), (9.5, 9.5, 5.0)
    gen = _splitmix64(seed)
    obstacles = []
    while len(obstacles) < n_trees:
        cx, cy = 1.0 + 8.0 * _unit(gen), 1.0 + 8.0 * _unit(gen)
        if math.hypot(cx - start[0], cy - start[1]) < 1.0 or math.hypot(cx - goal[0], cy - goal[1]) < 1.0:
            continue
        obstacles.append({"type": "box", "min": [cx - 0.25, cy - 0.25, 0.0], "max": [cx + 0.25, cy + 0.25, 10.0]})
    return {
        "name": "forest_di6",
        "problem": {
            "model": "double_integrator_6d",
            "model_params": {},
            "environment": {"workspace_bounds": [[0, 10], [0, 10], [0, 10]], "obstacles": obstacles},
            "x_init": [start[0], start[1], start[2], 0.0, 0.0, 0.0],
            "goal": {"dims": [0, 1, 2], "center": list(goal), "radius": 0.5},
            "cost": "path_length",
            "state_bounds": [[0, 10], [0, 10], [0, 10], [-2, 2], [-2, 2], [-2, 2]],
            "control_bounds": [[-2, 2], [-2, 2], [-2, 2]],
        },
        "decomposition": {"dims": [0, 1, 2], "cells": [30, 30, 30]},
        "planner": {
            "lambda": 32, "i_max": 5, "t_prop": 0.5, "capacity": 1 << 20, "ode_step": 0.02,
            "collision_step": 0.05, "t_max_ms": 100, "max_iterations": 0, "deactivate_after_expansion": False,
            "rng": "philox", "max_slots": 1 << 22,
        },
        "trials": {"n": 100, "base_seed": 0, "workers": 1},
    }


def narrow_dubins6() -> dict:
    """Config 2: 6D Dubins airplane, two rooms split by a wall with one slot."""
    # wall x in [4.75, 5.25] over y in [0, 10], z in [0, 5]; slot y in [4, 6], z in [1.5, 3.5]
    wx0, wx1 = 4.75, 5.25
    obstacles = [
        {"type": "box", "min": [wx0, 0.0, 0.0], "max": [wx1, 4.0, 5.0]},
        {"type": "box", "min": [wx0, 6.0, 0.0], "max": [wx1, 10.0, 5.0]},
        {"type": "box", "min": [wx0, 4.0, 0.0], "max": [wx1, 6.0, 1.5]},
        {"type": "box", "min": [wx0, 4.0, 3.5], "max": [wx1, 6.0, 5.0]},
    ]
    pi = math.pi
    return {
        "name": "narrow_dubins6",
        "problem": {
            "model": "dubins_airplane_6d",
            "model_params": {},
            "environment": {"workspace_bounds": [[0, 10], [0, 10], [0, 5]], "obstacles": obstacles},
            "x_init": [1.0, 1.0, 2.5, 0.0, 0.0, 1.0],
            "goal": {"dims": [0, 1, 2], "center": [9.0, 9.0, 2.5], "radius": 0.5},
            "cost": "path_length",
            "state_bounds": [[0, 10], [0, 10], [0, 5], [-pi, pi], [-0.5, 0.5], [0.5, 2.0]],
            "control_bounds": [[-1.0, 1.0], [-0.5, 0.5], [-1.0, 1.0]],
        },
        "decomposition": {"dims": [0, 1, 2, 3], "cells": [20, 20, 10, 13]},
        "planner": {
            "lambda": 32, "i_max": 5, "t_prop": 0.5, "capacity": 1 << 20, "ode_step": 0.02,
            "collision_step": 0.05, "t_max_ms": 100, "max_iterations": 0, "deactivate_after_expansion": False,
            "rng": "philox", "max_slots": 1 << 22,
        },
        "trials": {"n": 100, "base_seed": 0, "workers": 1},
    }


def building_quad12() -> dict:
    """Config 3: 12D quadcopter in a four-room building with doorways."""
    t = 0.2  # wall half-thickness
    h = 4.0
    obstacles = [
        # wall x = 5 (y in [0, 10]) with doorways at y in [2, 3.2] and y in [7, 8.2], height 2.5
        {"type": "box", "min": [5 - t, 0.0, 0.0], "max": [5 + t, 2.0, h]},
        {"type": "box", "min": [5 - t, 3.2, 0.0], "max": [5 + t, 7.0, h]},
        {"type": "box", "min": [5 - t, 8.2, 0.0], "max": [5 + t, 10.0, h]},
        {"type": "box", "min": [5 - t, 2.0, 2.5], "max": [5 + t, 3.2, h]},
        {"type": "box", "min": [5 - t, 7.0, 2.5], "max": [5 + t, 8.2, h]},
        # wall y = 5 (x in [0, 10]) with doorways at x in [2, 3.2] and x in [7, 8.2]
        {"type": "box", "min": [0.0, 5 - t, 0.0], "max": [2.0, 5 + t, h]},
        {"type": "box", "min": [3.2, 5 - t, 0.0], "max": [7.0, 5 + t, h]},
        {"type": "box", "min": [8.2, 5 - t, 0.0], "max": [10.0, 5 + t, h]},
        {"type": "box", "min": [2.0, 5 - t, 2.5], "max": [3.2, 5 + t, h]},
        {"type": "box", "min": [7.0, 5 - t, 2.5], "max": [8.2, 5 + t, h]},
        # furniture
        {"type": "box", "min": [1.0, 3.0, 0.0], "max": [2.5, 4.0, 1.0]},
        {"type": "box", "min": [6.5, 1.0, 0.0], "max": [8.0, 2.0, 1.2]},
        {"type": "sphere", "center": [7.5, 7.5, 1.0], "radius": 0.5},
    ]
    a = 0.6
    return {
        "name": "building_quad12",
        "problem": {
            "model": "quadcopter_12d",
            "model_params": {"mass": 1.0, "gravity": 9.81, "arm_length": 1.0, "Ixx": 1.0, "Iyy": 1.0, "Izz": 2.0},
            "environment": {"workspace_bounds": [[0, 10], [0, 10], [0, 4]], "obstacles": obstacles},
            "x_init": [1.5, 1.5, 1.5, 0, 0, 0, 0, 0, 0, 0, 0, 0],
            "goal": {"dims": [0, 1, 2], "center": [8.5, 8.5, 1.5], "radius": 0.5},
            "cost": "path_length",
            "state_bounds": [[0, 10], [0, 10], [0, 4], [-2, 2], [-2, 2], [-2, 2],
                             [-a, a], [-a, a], [-math.pi, math.pi], [-2, 2], [-2, 2], [-2, 2]],
            "control_bounds": [[7.0, 12.5], [-1.0, 1.0], [-1.0, 1.0], [-1.0, 1.0]],
        },
        "decomposition": {"dims": [0, 1, 2], "cells": [50, 50, 40]},
        "planner": {
            "lambda": 32, "i_max": 5, "t_prop": 0.5, "capacity": 1 << 21, "ode_step": 0.02,
            "collision_step": 0.05, "t_max_ms": 1000, "max_iterations": 0, "deactivate_after_expansion": False,
            "rng": "philox", "max_slots": 1 << 23,
        },
        "trials": {"n": 100, "base_seed": 0, "workers": 1},
    }


def free2d() -> dict:
    """2-D double integrator, empty environment, goal 5 m away."""
    return {
        "name": "free2d",
        "problem": {
            "model": "double_integrator_4d",
            "model_params": {},
            "environment": {"workspace_bounds": [[0, 10], [0, 10]], "obstacles": []},
            "x_init": [1.0, 1.0, 0.0, 0.0],
            "goal": {"dims": [0, 1], "center": [4.0, 5.0], "radius": 0.5},
            "cost": "path_length",
            "state_bounds": [[0, 10], [0, 10], [-1, 1], [-1, 1]],
            "control_bounds": [[-1, 1], [-1, 1]],
        },
        "decomposition": {"dims": [0, 1, 2, 3], "cells": [20, 20, 6, 6]},  # full state
        "planner": {
            "lambda": 8, "i_max": 5, "t_prop": 1.0, "capacity": 1 << 16, "ode_step": 0.05,
            "collision_step": 0.05, "t_max_ms": 100, "max_iterations": 0, "rng": "philox", "max_slots": 1 << 18,
        },
        "trials": {"n": 10, "base_seed": 0, "workers": 1},
    }


def zigzag2d() -> dict:
    """corridor of 6 staggered boxes (2-D double integrator)."""
    obstacles = []
    for i in range(6):
        x0 = 1.2 + 1.4 * i
        if i % 2 == 0:
            obstacles.append({"type": "box", "min": [x0, 0.0], "max": [x0 + 0.3, 7.0]})
        else:
            obstacles.append({"type": "box", "min": [x0, 3.0], "max": [x0 + 0.3, 10.0]})
    return {
        "name": "zigzag2d",
        "problem": {
            "model": "double_integrator_4d",
            "model_params": {},
            "environment": {"workspace_bounds": [[0, 10], [0, 10]], "obstacles": obstacles},
            "x_init": [0.5, 0.5, 0.0, 0.0],
            "goal": {"dims": [0, 1], "center": [9.5, 9.0], "radius": 0.5},
            "cost": "path_length",
            "state_bounds": [[0, 10], [0, 10], [-1.5, 1.5], [-1.5, 1.5]],
            "control_bounds": [[-1.5, 1.5], [-1.5, 1.5]],
        },
        "decomposition": {"dims": [0, 1, 2, 3], "cells": [40, 40, 6, 6]},  # full state
        "planner": {
            "lambda": 16, "i_max": 5, "t_prop": 0.8, "capacity": 1 << 20, "ode_step": 0.02,
            "collision_step": 0.05, "t_max_ms": 100, "max_iterations": 0, "rng": "philox", "max_slots": 1 << 20,
        },
        "trials": {"n": 25, "base_seed": 0, "workers": 1},
    }


# ---- the SPEC's bundled set: free2d, zigzag2d, forest6d,
# narrow6d, building6d, zigzag6d, dubins_narrow, quad12d_forest, each with a
# large-delta (as named) and a small-delta variant (`<name>_small`: every
# decomposed position dimension split FINE times finer
# "large-δ and small-δ variants").  forest6d / dubins_narrow are the BASELINE config 1 / 2
# scenes under the SPEC's names.
FINE = 2


def _renamed(fn, name):
    s = fn()
    s["name"] = name
    return s


def _walls_narrow():
    return copy.deepcopy(narrow_dubins6()["problem"]["environment"])


def _di6(name, env, start, goal, cells, dims=(0, 1, 2), vmax=2.0, amax=2.0, t_max_ms=100, lam=32):
    wb = env["workspace_bounds"]
    return {
        "name": name,
        "problem": {
            "model": "double_integrator_6d",
            "model_params": {},
            "environment": env,
            "x_init": list(start) + [0.0, 0.0, 0.0],
            "goal": {"dims": [0, 1, 2], "center": list(goal), "radius": 0.5},
            "cost": "path_length",
            "state_bounds": [list(b) for b in wb] + [[-vmax, vmax]] * 3,
            "control_bounds": [[-amax, amax]] * 3,
        },
        "decomposition": {"dims": list(dims), "cells": list(cells)},
        "planner": {
            "lambda": lam, "i_max": 5, "t_prop": 0.5, "capacity": 1 << 20, "ode_step": 0.02,
            "collision_step": 0.05, "t_max_ms": t_max_ms, "max_iterations": 0,
            "deactivate_after_expansion": False, "rng": "philox",
        },
        "trials": {"n": 25, "base_seed": 0, "workers": 1},
    }


def narrow6d() -> dict:
    """6D double integrator through the one-slot wall of narrow_dubins6."""
    return _di6("narrow6d", _walls_narrow(), (1.0, 1.0, 2.5), (9.0, 9.0, 2.5), (30, 30, 15))


def building6d() -> dict:
    """6D double integrator in the four-room building of building_quad12."""
    env = copy.deepcopy(building_quad12()["problem"]["environment"])
    return _di6("building6d", env, (1.5, 1.5, 1.5), (8.5, 8.5, 1.5), (50, 50, 20))


def zigzag6d() -> dict:
    """6D double integrator through six staggered full-height walls (the 3-D
    extrusion of zigzag2d); decomposition over position + planar velocity."""
    obstacles = []
    for i in range(6):
        x0 = 1.2 + 1.4 * i
        y0, y1 = (0.0, 7.0) if i % 2 == 0 else (3.0, 10.0)
        obstacles.append({"type": "box", "min": [x0, y0, 0.0], "max": [x0 + 0.3, y1, 3.0]})
    env = {"workspace_bounds": [[0, 10], [0, 10], [0, 3]], "obstacles": obstacles}
    s = _di6("zigzag6d", env, (0.5, 0.5, 1.5), (9.5, 9.0, 1.5), (40, 40, 3, 4, 4), dims=(0, 1, 2, 3, 4),
             vmax=1.5, amax=1.5)
    s["planner"]["t_prop"] = 0.8
    return s


def quad12d_forest() -> dict:
    """12D quadcopter among the forest_di6 trees (cut to the 4 m ceiling)."""
    s = building_quad12()
    trees = forest_di6()["problem"]["environment"]["obstacles"]
    s["name"] = "quad12d_forest"
    s["problem"]["environment"] = {
        "workspace_bounds": [[0, 10], [0, 10], [0, 4]],
        "obstacles": [{"type": "box", "min": t["min"], "max": [t["max"][0], t["max"][1], 4.0]} for t in trees],
    }
    s["problem"]["x_init"] = [0.5, 0.5, 2.0] + [0.0] * 9
    s["problem"]["goal"]["center"] = [9.5, 9.5, 2.0]
    s["decomposition"]["cells"] = [50, 50, 20]
    s["planner"].pop("max_slots", None)
    return s


def small_delta(fn, fine: int = FINE):
    """The small-δ variant of a scene: FINE× the cells on every decomposed
    position dimension (velocity / angle cells unchanged)."""
    def build():
        s = fn()
        s["name"] = s["name"] + "_small"
        wdim = len(s["problem"]["environment"]["workspace_bounds"])
        dec = s["decomposition"]
        dec["cells"] = [c * fine if d < wdim else c for d, c in zip(dec["dims"], dec["cells"])]
        # more regions keep more nodes alive: grow the store, size slots by default
        s["planner"]["capacity"] = min(s["planner"]["capacity"] * 16, 1 << 23)
        s["planner"].pop("max_slots", None)
        return s
    build.__name__ = fn.__name__ + "_small"
    return build


SPEC_SET = {
    "free2d": free2d,
    "zigzag2d": zigzag2d,
    "forest6d": lambda: _renamed(forest_di6, "forest6d"),
    "narrow6d": narrow6d,
    "building6d": building6d,
    "zigzag6d": zigzag6d,
    "dubins_narrow": lambda: _renamed(narrow_dubins6, "dubins_narrow"),
    "quad12d_forest": quad12d_forest,
}

BUILDERS = {
    # BASELINE.json configs 1-3
    "forest_di6": forest_di6,
    "narrow_dubins6": narrow_dubins6,
    "building_quad12": building_quad12,
}
for _n, _f in SPEC_SET.items():
    BUILDERS[_n] = _f
    BUILDERS[_n + "_small"] = small_delta(_f)


_REQUIRED = {
    "problem": ["model", "environment", "x_init", "goal", "state_bounds", "control_bounds"],
    "decomposition": ["dims"],
    "planner": ["t_prop"],
}


def validate(s: dict) -> dict:
    """Schema check with field paths in the messages."""
    if not isinstance(s, dict):
        raise SchemaError("scenario: expected an object")
    for top in ("name", "problem", "decomposition", "planner"):
        if top not in s:
            raise SchemaError(f"scenario.{top}: missing")
    for sec, keys in _REQUIRED.items():
        for k in keys:
            if k not in s[sec]:
                raise SchemaError(f"scenario.{sec}.{k}: missing")
    env = s["problem"]["environment"]
    if "workspace_bounds" not in env:
        raise SchemaError("scenario.problem.environment.workspace_bounds: missing")
    for i, o in enumerate(env.get("obstacles", [])):
        t = o.get("type")
        if t == "box":
            if any(a > b for a, b in zip(o["min"], o["max"])):
                raise SchemaError(f"scenario.problem.environment.obstacles[{i}]: box min > max")
        elif t == "sphere":
            if not o.get("radius", 0) > 0:
                raise SchemaError(f"scenario.problem.environment.obstacles[{i}]: sphere radius <= 0")
        else:
            raise SchemaError(f"scenario.problem.environment.obstacles[{i}].type: unknown {t!r}")
    dec = s["decomposition"]
    if ("delta" in dec) == ("cells" in dec):
        raise SchemaError("scenario.decomposition: exactly one of delta / cells is required")
    return s


def load(name_or_path: str, **planner_overrides) -> dict:
    """Load a bundled scenario by name or a JSON file by path; keyword
    arguments override `planner` keys (CLI-style overrides)."""
    if name_or_path in BUILDERS and not os.path.exists(name_or_path):
        path = os.path.join(SCENARIO_DIR, name_or_path + ".json")
        if os.path.exists(path):
            with open(path) as f:
                s = json.load(f)
        else:
            s = BUILDERS[name_or_path]()
    else:
        with open(name_or_path) as f:
            try:
                s = json.load(f)
            except json.JSONDecodeError as e:
                raise SchemaError(f"{name_or_path}: {e}") from e
    s = copy.deepcopy(validate(s))
    s["planner"].update({k: v for k, v in planner_overrides.items() if v is not None})
    return s


def write_bundled(directory: str = SCENARIO_DIR) -> None:
    os.makedirs(directory, exist_ok=True)
    for name, fn in BUILDERS.items():
        with open(os.path.join(directory, name + ".json"), "w") as f:
            json.dump(fn(), f, indent=1)
            f.write("\n")
