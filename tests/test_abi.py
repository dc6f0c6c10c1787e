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
