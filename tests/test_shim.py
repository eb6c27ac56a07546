"""Drop-in proof: the reference's own C++ tests and simulator, linked against the GPU shim
(paper_2602_21626_b200/shim over libgimbal_gpu.so) instead of proj/src/{moe,placement}.cpp.

The binaries are built here (where /root/reference exists) by `make -C paper_2602_21626_b200/shim`
into oracle/_ref/ and ship prebuilt to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _bin(name):
    p = os.path.join(REF_DIR, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (needs /root/reference at build time)")
    return p


def _run(args, timeout=600):
    return subprocess.run(args, capture_output=True, text=True, timeout=timeout)


# ---- CPU: the reference over its own expert layer reproduces the committed fixtures ----

def test_reference_sim_tests_pass():
    out = _run([_bin("ref_sim_tests")])
    assert out.returncode == 0 and "| 0 failed" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("scenario", [0, 1, 2])
def test_reference_sim_report_matches_fixture(scenario):
    out = _run([_bin("sim_report_ref"), str(scenario)])
    assert out.returncode == 0, out.stderr
    with open(os.path.join(GOLDEN, f"sim_report_{scenario}.json")) as f:
        assert out.stdout == f.read()


# ---- GPU: the same tests and reports through the shim ----

@pytest.mark.gpu
def test_reference_unit_tests_pass_on_gpu_shim():
    """proj/tests/unit/test_moe.cpp + test_placement.cpp (32 TEST_CASEs) against the GPU path."""
    out = _run([_bin("shim_unit_tests")])
    assert out.returncode == 0 and "| 0 failed" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.gpu
def test_reference_sim_tests_pass_on_gpu_shim():
    """proj/tests/unit/test_sim.cpp: the simulator's MoeSubsystem over the GPU expert layer."""
    out = _run([_bin("shim_sim_tests")])
    assert out.returncode == 0 and "| 0 failed" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("scenario", [0, 1, 2])
def test_sim_report_byte_identical_on_gpu_shim(scenario):
    """Full simulation report (routing, per-iteration load/crossings, calibration, relocations,
    anchors, migrations, latencies) byte-identical to the reference's."""
    out = _run([_bin("sim_report_shim"), str(scenario)])
    assert out.returncode == 0, out.stderr
    with open(os.path.join(GOLDEN, f"sim_report_{scenario}.json")) as f:
        assert out.stdout == f.read()


# ---- GPU: the simulator with its expert-layer hook on the GPU (GpuMoeSubsystem) ----

@pytest.mark.gpu
def test_reference_sim_tests_pass_with_gpu_hook():
    """proj/tests/unit/test_sim.cpp with gimbal::run's hook swapped for GpuMoeSubsystem (the
    per-iteration loop of sim.cpp:113-147 as one CUDA graph per engine iteration)."""
    out = _run([_bin("shim_sim_tests_gpuhook")])
    assert out.returncode == 0 and "| 0 failed" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("scenario", [0, 1, 2])
def test_sim_report_byte_identical_with_gpu_hook(scenario):
    """Byte-identical simulation reports with the GPU hook: latencies (which feed on the
    bottleneck excess and crossings of every iteration), expert loads, relocations, migrations."""
    out = _run([_bin("sim_report_gpuhook"), str(scenario)])
    assert out.returncode == 0, out.stderr
    with open(os.path.join(GOLDEN, f"sim_report_{scenario}.json")) as f:
        assert out.stdout == f.read()
