"""The C++ drop-in API (include/kinoplan_b200/kinoplan.hpp): compiles and links
against the library on CPU; runs on the GPU (-m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "dropin")
    lib = os.path.join(ROOT, "paper_2602_02846_b200", "lib")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp"), "-L", lib, "-lkinoplan_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_cpp_dropin_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_dropin_runs(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    found, cost, iters, tcost, nsamp = out.stdout.split()
    assert found == "1" and float(cost) > 12.0 and int(iters) > 10 and float(tcost) == float(cost)


def test_cpp_host_api_spec_examples(tmp_path):
    """Host (fp64) building blocks of the drop-in API against the SPEC examples:
    propagate_ode, sampling, validity, load_environment, grid, atomic region
    minimum (tests/cpp/host_api_test.cpp).  CPU only."""
    exe = str(tmp_path / "host_api")
    lib = os.path.join(ROOT, "paper_2602_02846_b200", "lib")
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_api_test.cpp"), "-L", lib, "-lkinoplan_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, (out.stdout, out.stderr)
    assert out.stdout.startswith("ok ")


@pytest.mark.gpu
def test_gpu_solutions_verified_in_fp64(tmp_path):
    """GPU plans (fp32 recipe) re-checked with the host fp64 API: re-propagated
    segments land on the stored states within 1e-4, the fp64 samples are valid,
    and the fp64 path length equals the planner's cost within 1e-4."""
    exe = str(tmp_path / "verify")
    lib = os.path.join(ROOT, "paper_2602_02846_b200", "lib")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "verify_solution.cpp"), "-L", lib, "-lkinoplan_b200",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    scen = os.path.join(ROOT, "paper_2602_02846_b200", "scenarios")
    names = ["forest_di6", "narrow_dubins6", "building_quad12", "zigzag2d", "free2d", "zigzag6d", "building6d"]
    out = subprocess.run([exe] + [os.path.join(scen, n + ".json") for n in names], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, (out.stdout, out.stderr)
    assert len(out.stdout.strip().splitlines()) == len(names)
