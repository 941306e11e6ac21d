"""Pin the oracle to the reference's own code.

tests/golden/reference_kat.json comes from the reference's shipped headers
compiled in place (oracle/_ref/ref_kat, see tests/golden/make_golden.py); the
oracle restatement must reproduce every value bit-for-bit.
"""
import json
import math
import os

import numpy as np
import pytest

import kpo

HERE = os.path.dirname(os.path.abspath(__file__))
KAT = json.load(open(os.path.join(HERE, "golden", "reference_kat.json")))
PHILOX = json.load(open(os.path.join(HERE, "golden", "philox_kat.json")))


@pytest.mark.parametrize("case", KAT["splitmix"], ids=lambda c: c["seed"])
def test_splitmix64_and_uniform_unit(case):  # rng.hpp:12-31, :55-57
    raw, unit = kpo.splitmix(int(case["seed"]), 8)
    assert [int(v) for v in raw] == [int(v) for v in case["raw"]]
    assert list(unit) == case["unit"]


def test_mix64():  # rng.hpp:34-39
    for z, want in KAT["mix64"]:
        assert kpo.mix64(int(z)) == int(want)


def test_derive_stream():  # rng.hpp:44-52
    assert len(KAT["derive_stream"]) == 108
    for seed, it, node, br, want, u0, u1 in KAT["derive_stream"]:
        s = kpo.derive_stream(int(seed), int(it), int(node), int(br))
        assert s == int(want)
        _, unit = kpo.splitmix(s, 2)
        assert list(unit) == [u0, u1]


def test_survey_appendix_a_vectors():
    assert kpo.mix64(0) == 0xE220A8397B1DCDAF
    assert kpo.derive_stream(0, 0, 0, 0) == 0x2130748AAAC80268
    assert kpo.derive_stream(7, 3, 42, 5) == 0xDD819ECECF8475A6
    _, u = kpo.splitmix(kpo.derive_stream(7, 0, 0, 0), 2)
    assert list(u) == [0.045311539271475909, 0.62635179504451322]


def test_wrap_angle():  # types.hpp:49-58
    for a, want in KAT["wrap_angle"]:
        got = kpo.wrap_angle(a)
        assert got == want, (a, got, want)
        assert -math.pi < got <= math.pi or got == want


def test_segment_cost_reference_values():  # cost.hpp:44-67
    by = {c["name"]: c for c in KAT["segment_cost"]}
    assert kpo.segment_cost([[0, 0, 0], [3, 4, 0]], 3, 0, 1.0) == by["pythagorean"]["value"] == 5.0
    assert kpo.segment_cost([[1, 2, 3, 4], [1, 2, 3, 9]], 3, 0, 0.5) == by["zero_displacement_dt0.5"]["value"]
    assert kpo.segment_cost([[0, 0, 0], [3, 4, 0]], 3, 1, 0.25) == by["control_duration_0.25"]["value"] == 0.25
    q = [[math.cos(t), math.sin(t), 0.0] for t in (math.pi / 2 * i / 63.0 for i in range(64))]
    v = kpo.segment_cost(q, 3, 0, 1.0)
    assert v == by["quarter_circle_64"]["value"]
    assert math.pi / 2 - 0.001 <= v <= math.pi / 2
    polys = [c for c in KAT["segment_cost"] if c["name"].startswith("poly")]
    assert len(polys) == 20
    for c in polys:
        assert kpo.segment_cost(c["samples"], c["position_dims"], 0, c["duration"]) == c["value"], c["name"]


def test_segment_cost_errors():  # cost.hpp:47-52 InvalidSegmentError
    assert KAT["one_sample_throws_invalid_segment"] == 1
    with pytest.raises(kpo.OracleError) as e:
        kpo.segment_cost([[0, 0, 0]], 3, 0, 1.0)
    assert e.value.code == 5
    with pytest.raises(kpo.OracleError):
        kpo.segment_cost([[0, 0, 0], [1, 0, 0]], 3, 0, 0.0)


def test_in_goal():  # cost.hpp:77-84
    by = {c["name"]: c["value"] for c in KAT["in_goal"]}
    dims, c, r = [0, 1, 2], [9.5, 9.5, 5.0], 0.5
    assert kpo.in_goal([9.5, 9.5, 5.0, 0, 0, 0], dims, c, r) == bool(by["center"])
    assert kpo.in_goal([10.0, 9.5, 5.0, 0, 0, 0], dims, c, r) == bool(by["at_radius"]) is True
    assert kpo.in_goal([10.0 + 1e-12, 9.5, 5.0, 0, 0, 0], dims, c, r) == bool(by["radius_plus_eps"]) is False
    assert kpo.in_goal([9.8, 9.9, 5.0, 1, 1, 1], dims, c, r) == bool(by["diag_3_4_5"])


@pytest.mark.parametrize("case", PHILOX["cases"], ids=lambda c: str(c["ctr"]))
def test_philox_kat(case):
    assert list(kpo.philox(case["ctr"], case["key"])) == case["out"]


def test_philox_random123_published_vectors():
    assert list(kpo.philox([0, 0, 0, 0], [0, 0])) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert list(kpo.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]


def test_sincos_recipe_accuracy():
    """The pinned fp32 sincos recipe is within 2 ulp-ish of libm over (-pi, pi]."""
    xs = np.linspace(-math.pi, math.pi, 20001, dtype=np.float32)
    worst = 0.0
    for x in xs[::7]:
        s, c = kpo.sincos_f32(float(x))
        worst = max(worst, abs(s - math.sin(float(x))), abs(c - math.cos(float(x))))
    assert worst < 3e-7
