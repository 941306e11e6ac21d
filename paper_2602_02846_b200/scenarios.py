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
plus the small 2-D scenes the SPEC examples use (free2d, zigzag2d).
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
            "lambda": 16, "i_max": 5, "t_prop": 0.8, "capacity": 1 << 18, "ode_step": 0.02,
            "collision_step": 0.05, "t_max_ms": 100, "max_iterations": 0, "rng": "philox", "max_slots": 1 << 20,
        },
        "trials": {"n": 25, "base_seed": 0, "workers": 1},
    }


BUILDERS = {
    "forest_di6": forest_di6,
    "narrow_dubins6": narrow_dubins6,
    "building_quad12": building_quad12,
    "free2d": free2d,
    "zigzag2d": zigzag2d,
}

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
