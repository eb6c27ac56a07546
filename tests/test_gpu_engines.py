"""Alternate kernels behind the experiment knobs, checked against the oracle.

The knobs exist only in the test/tool build ``lib/libgimbal_gpu_ab.so`` (``internal.cuh``
GIMBAL_KNOB); each case runs in a fresh process (``tests/ab_engines.py``) with GIMBAL_LIB pointing
at that build, so the shipped library the rest of the suite loads never reads the environment.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AB_LIB = os.path.join(ROOT, "paper_2602_21626_b200", "lib", "libgimbal_gpu_ab.so")


def run_case(knobs: dict, *args) -> None:
    env = dict(os.environ)
    env.update({k: str(v) for k, v in knobs.items()})
    env["GIMBAL_LIB"] = AB_LIB
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ab_engines.py"), *map(str, args)], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]


def test_shipped_library_has_no_knobs():
    """The library the package loads reads no environment variable (nm: no getenv import)."""
    lib = os.path.join(ROOT, "paper_2602_21626_b200", "lib", "libgimbal_gpu.so")
    out = subprocess.run(["nm", "-D", lib], capture_output=True, text=True).stdout
    assert "getenv" not in out


@pytest.mark.parametrize("path", ["fp4", "fp4x2"])
@pytest.mark.parametrize("L,T,dup", [(58, 70001, 0), (58, 129, 0), (2, 5000, 0), (58, 5000, 1), (4, 300000, 0)])
def test_fp4_count_path(path, L, T, dup):
    """Block-scaled FP4 counters: one SM per M = 128 half (fp4) and CTA pairs (fp4x2)."""
    run_case({"GIMBAL_COUNT_PATH": path}, "fp4", L, T, dup)


@pytest.mark.parametrize("L,ne,k,g,C", [(58, 256, 8, 8, 70), (48, 128, 8, 8, 33), (26, 64, 6, 8, 70),
                                        (9, 64, 4, 16, 17)])
def test_eval_integer_alu_path(L, ne, k, g, C):
    run_case({"GIMBAL_EVAL_ALU": "1"}, "eval", L, ne, k, g, C, 2.0, 0.5)


@pytest.mark.parametrize("L,ne,k,g,C", [(32, 8, 2, 8, 4096), (5, 8, 3, 4, 9), (7, 16, 4, 8, 33)])
def test_eval_generic_for_small_shapes(L, ne, k, g, C):
    run_case({"GIMBAL_EVAL_NO_SMALL": "1"}, "eval", L, ne, k, g, C, 1.5, 0.25)


@pytest.mark.parametrize("L,ne,k,g,C", [(32, 8, 2, 8, 4096), (7, 16, 4, 8, 33)])
def test_unfused_pass_for_small_shapes(L, ne, k, g, C):
    run_case({"GIMBAL_NO_TINY_PASS": "1"}, "pass", L, ne, k, g, C)


@pytest.mark.parametrize("knobs,L,ne,k,T", [
    ({"GIMBAL_TMA_MODE": "u15"}, 58, 256, 8, 70001),
    ({"GIMBAL_U15_ROLLING": "1"}, 58, 256, 8, 300001),
    ({"GIMBAL_U15_ROLLING": "1", "GIMBAL_U15_ROLL_SYNC": "8"}, 58, 256, 8, 300001),
    ({"GIMBAL_U15_DRAIN_BLOCKS": "16"}, 58, 256, 8, 300001),
    ({"GIMBAL_U15_SCALAR_SCAN": "1"}, 58, 256, 8, 300001),
    ({"GIMBAL_NO_TMA": "1"}, 58, 256, 8, 70001),
    ({"GIMBAL_COUNT_PATH": "split"}, 58, 256, 8, 30001),
    ({"GIMBAL_COUNT_PATH": "atomic"}, 48, 128, 8, 30001),
    ({"GIMBAL_NO_DIRECT": "1"}, 26, 64, 6, 30001),
    ({"GIMBAL_NO_SMALL": "1"}, 32, 8, 2, 30001),
    ({"GIMBAL_SMALL_BYTEWISE": "1"}, 32, 8, 2, 30001),
    ({"GIMBAL_SMALL_NO_EVENTS": "1"}, 32, 8, 2, 30001),
])
def test_alternate_counters(knobs, L, ne, k, T):
    run_case(knobs, "count", L, ne, k, T)
