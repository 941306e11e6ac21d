"""C-ABI boundary checks that need no GPU: the library loads, exports every
function include/kinoplan_b200.h declares, the ctypes mirror matches the C
struct layout byte for byte, and descriptor validation maps onto the
reference's exception classes (errors.hpp:11-33) before any device work."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2602_02846_b200 import _capi, scenarios
from paper_2602_02846_b200.planner import (ConfigError, DeviceError, GridTooFineError, InvalidProblemError, Planner,
                                           SchemaError)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kinoplan_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(kp_[a-z_0-9]+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _capi.load_library()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(_capi.EXPORTED_SYMBOLS) <= set(names)
    assert lib.kp_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.lib_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(?!100a)\d+", out.stdout)


def test_struct_layout_matches_c_header():
    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "kinoplan_b200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu\n", sizeof(kp_problem_desc), sizeof(kp_config_desc), sizeof(kp_result),
             sizeof(kp_timeline_entry), sizeof(kp_obstacle));
      printf("%zu %zu %zu %zu\n", offsetof(kp_problem_desc, goal_radius), offsetof(kp_problem_desc, grid_max_cells),
             offsetof(kp_config_desc, max_slots), offsetof(kp_result, timeline_len));
      return 0;
    }"""
    with tempfile.TemporaryDirectory() as d:
        with open(os.path.join(d, "t.c"), "w") as f:
            f.write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "t"),
                        os.path.join(d, "t.c")], check=True)
        out = subprocess.run([os.path.join(d, "t")], capture_output=True, text=True, check=True).stdout.split()
    want = [C.sizeof(_capi.ProblemDesc), C.sizeof(_capi.ConfigDesc), C.sizeof(_capi.Result),
            C.sizeof(_capi.TimelineEntry), C.sizeof(_capi.Obstacle),
            _capi.ProblemDesc.goal_radius.offset, _capi.ProblemDesc.grid_max_cells.offset,
            _capi.ConfigDesc.max_slots.offset, _capi.Result.timeline_len.offset]
    assert [int(x) for x in out] == want


def _gpu_present():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.parametrize("mutate,exc", [
    (lambda s: s["problem"].__setitem__("model", "double_integrator_6d") or s["problem"].__setitem__("x_init", [0] * 4),
     SchemaError),
    (lambda s: s["planner"].__setitem__("lambda", 0), ConfigError),
    (lambda s: s["planner"].__setitem__("t_prop", -1.0), ConfigError),
    (lambda s: s.__setitem__("decomposition", {"dims": [0, 1], "delta": 1e-6}), GridTooFineError),
    (lambda s: s["problem"].__setitem__("x_init", [4.0, 5.0, 0.0, 0.0]) or s["problem"]["environment"].__setitem__(
        "obstacles", [{"type": "box", "min": [3, 4], "max": [5, 6]}]), InvalidProblemError),
    (lambda s: s["problem"]["environment"].__setitem__("obstacles", [{"type": "sphere", "center": [1, 1],
                                                                      "radius": -1}]), SchemaError),
    (lambda s: s["problem"]["goal"].__setitem__("center", [40.0, 5.0]), InvalidProblemError),
])
def test_descriptor_errors_map_to_reference_exceptions(mutate, exc):
    s = scenarios.load("free2d")
    mutate(s)
    with pytest.raises(exc):
        Planner(s)


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU failure mode")
def test_valid_problem_without_gpu_fails_loudly():
    with pytest.raises(DeviceError):
        Planner(scenarios.load("forest_di6"))


def test_bundled_scenarios_match_builders_and_validate():
    import json

    for name, fn in scenarios.BUILDERS.items():
        path = os.path.join(scenarios.SCENARIO_DIR, name + ".json")
        assert json.load(open(path)) == json.loads(json.dumps(fn())), name
        scenarios.load(name)


def test_scenario_schema_errors_name_the_field():
    s = scenarios.forest_di6()
    del s["problem"]["goal"]
    with pytest.raises(scenarios.SchemaError, match="problem.goal"):
        scenarios.validate(s)
    s = scenarios.forest_di6()
    s["problem"]["environment"]["obstacles"][3]["max"][0] = -5
    with pytest.raises(scenarios.SchemaError, match=r"obstacles\[3\]"):
        scenarios.validate(s)
