import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        meta = json.load(f)
    arrs = np.load(os.path.join(GOLDEN, "golden.npz"))
    return meta, arrs


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library, when it was built here (oracle/_ref)."""
    from oracle import oracle as o
    if not os.path.exists(o.REF_SO):
        if os.path.isdir(o.REF_SRC):
            o.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return o.Reference()


@pytest.fixture(scope="session")
def dss():
    import paper_2007_03298_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test requires a CUDA device (run on the B200 box)")
    return 0
