"""The C-ABI library loads without a GPU and exports every symbol that
include/dssync_b200.h declares; device entry points fail loudly (no CPU
fallback) when no GPU is present."""
import ctypes as C
import os
import re

import pytest

from paper_2007_03298_b200 import _lib as L

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "dssync_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dss_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("dss_partition", "dss_step", "dss_sync_round", "dss_apply_step", "dss_create", "dss_ipc_attach"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = L.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(L.SIGNATURES), "ctypes binding out of sync with the header"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2007_03298_b200 import DsSyncEngine, StrategyKind, SyncStrategy, Topology, WorldConfig
    with pytest.raises(RuntimeError):
        DsSyncEngine(SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(4, 2)), 0, 16)


def test_invalid_config_is_einval_before_device():
    from paper_2007_03298_b200 import DsSyncEngine, StrategyKind, SyncStrategy, Topology, WorldConfig
    with pytest.raises(ValueError):
        DsSyncEngine(SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(8, 2)), 0, 16)
    with pytest.raises(ValueError):
        DsSyncEngine(SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(4, 2)), 0, 0)


def test_null_handles_are_rejected():
    lib = L.load()
    assert lib.dss_step(None, 0, 0.1, 0, None) == L.DSS_EINVAL
    assert lib.dss_check(None) == L.DSS_EINVAL
    assert lib.dss_destroy(None) == L.DSS_OK


def _fake_engine(dtype, P, d):
    """A DsSyncEngine shell (no device context) to exercise the host-side
    argument checks that run before any C call."""
    import numpy as np

    from paper_2007_03298_b200 import DsSyncEngine
    e = DsSyncEngine.__new__(DsSyncEngine)
    e.dtype, e.local_workers, e.dim, e.stats_dim = dtype, P, d, 0
    e.h = None

    class _NoCalls:  # any C call reached means a check was skipped
        def __getattr__(self, name):
            def call(*a):
                raise AssertionError(f"{name} called with an unchecked buffer")
            return call
    e.lib = _NoCalls()
    return e


def test_host_buffer_checks_reject_mismatched_buffers():
    """step_host / upload_all / download_all hand raw pointers to C calls
    that copy local_workers * dim elements: wrong shape, dtype or layout
    must raise ValueError before any copy (not an assert)."""
    import numpy as np
    import torch
    e = _fake_engine(np.float64, 2, 5)
    good = np.zeros((2, 5))
    assert e._host_ptr(good, (2, 5), "x") == good.ctypes.data
    for bad in (np.zeros((2, 5), np.float32), np.zeros((2, 4)), np.zeros((5, 2)).T, np.zeros(10)):
        with pytest.raises(ValueError):
            e._host_ptr(bad, (2, 5), "x")
    t = torch.zeros((2, 5), dtype=torch.float64)
    assert e._host_ptr(t, (2, 5), "x") == t.data_ptr()
    for bad in (torch.zeros((2, 5)), torch.zeros((5, 2), dtype=torch.float64).t(), torch.zeros((2, 6), dtype=torch.float64)):
        with pytest.raises(ValueError):
            e._host_ptr(bad, (2, 5), "x")
    with pytest.raises(TypeError):
        e._host_ptr([[0.0] * 5] * 2, (2, 5), "x")
    with pytest.raises(ValueError):
        e.step_host(0, 0.1, np.zeros((2, 5), np.float32), good)
    with pytest.raises(ValueError):
        e.download_all(0, np.zeros((3, 5)))
    with pytest.raises(ValueError):
        e.broadcast_row(0, np.zeros(4))


def test_iteration_trace_payload_counts_running_stats():
    """simulated_comm_time uses payload_bytes = 8 * (dim + stats_dim)
    (sync.cpp:314-318)."""
    import numpy as np

    from paper_2007_03298_b200 import SyncRoundOutcome, SyncStrategy, StrategyKind, Topology, WorldConfig
    from paper_2007_03298_b200.api import iteration_trace

    class Fake:
        dim, stats_dim = 10, 3
        strategy = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(4, 2))

        def global_mean(self):
            return np.zeros(10)

        def quadratic_losses(self, mu, exact=False):
            return np.ones(4), 0.0

    tr = iteration_trace(Fake(), 0, SyncRoundOutcome(3, 6), 1.0, bandwidth=2.0)
    assert tr.simulated_comm_time == 3 * 8.0 * 13 / 2.0
