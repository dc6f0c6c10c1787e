"""The reference's OWN test suites (proj/tests/*.cpp and acceptance.cpp, unmodified), compiled
with tests/cpp/doctest.h and linked so that dssync::apply_step, sync_round,
make_partition and the ring/tree/ps collectives run on the B200 through the
C-ABI (tests/cpp/b200_shim.cpp; oracle/Makefile targets `reftests`,
`acceptance`, `shimbench`).  Every other reference function, incl.
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


SHIM_PURE = os.path.join(ROOT, "oracle", "_ref", "shim_bench")
SHIM_B200 = os.path.join(ROOT, "oracle", "_ref", "shim_bench_b200")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["lockstep", "parallel"])
def test_run_training_through_the_shim_is_bit_identical(tmp_path, mode):
    """run_training (DS, W=16 / N=4, momentum, isotropic quadratic, 12
    iterations) linked with the B200 shim ends with the same params, bit for
    bit, as the pure reference build."""
    import json

    import numpy as np
    for p in (SHIM_PURE, SHIM_B200):
        if not os.path.exists(p):
            pytest.skip(f"{p} not built (make -C oracle shimbench)")
    out = {}
    for tag, exe in (("ref", SHIM_PURE), ("b200", SHIM_B200)):
        f = str(tmp_path / f"{tag}.bin")
        r = subprocess.run([exe, "20001", "12", "16", "4", mode, f], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = (json.loads(r.stdout.strip().splitlines()[-1]), np.fromfile(f))
    assert out["ref"][1].size == 16 * 20001
    assert np.array_equal(out["ref"][1], out["b200"][1])
    assert out["ref"][0]["final_suboptimality"] == out["b200"][0]["final_suboptimality"]
