"""The reference's OWN test suites (proj/tests/*.cpp and acceptance.cpp, unmodified), compiled
with tests/cpp/doctest.h and linked so that dssync::apply_step, sync_round
and make_partition run on the B200 through the C-ABI (tests/cpp/b200_shim.cpp;
oracle/Makefile target `reftests`).  Every other reference function, incl.
run_training, is the reference's own code calling into the device path."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests_b200")
PURE = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")


def _run(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference: make -C oracle reftests)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(p.stdout[-3000:])
    return p


def test_reference_unit_suite_pure_reference():
    """The harness itself reproduces the reference suite's verdict on CPU."""
    p = _run(PURE)
    assert p.returncode == 0 and "Status: SUCCESS" in p.stdout


@pytest.mark.gpu
def test_reference_unit_suite_on_b200():
    p = _run(B200)
    assert p.returncode == 0 and "Status: SUCCESS" in p.stdout


ACC_B200 = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
ACC_PURE = os.path.join(ROOT, "oracle", "_ref", "acceptance")


def test_reference_acceptance_pure_reference():
    """proj/tests/acceptance.cpp (12 criteria) on the unmodified reference."""
    p = _run(ACC_PURE)
    assert p.returncode == 0 and "all 12 criteria passed" in p.stdout


@pytest.mark.gpu
def test_reference_acceptance_on_b200():
    """The same 12 criteria (schedule, Eq. 2 reconstruction, BSP equivalence,
    divergence/theorem bounds, DS-vs-BSP parity, sync rules under Adam,
    byte-identical metrics lockstep vs parallel) with every apply_step,
    sync_round and make_partition served by the B200 library."""
    p = _run(ACC_B200)
    assert p.returncode == 0 and "all 12 criteria passed" in p.stdout
