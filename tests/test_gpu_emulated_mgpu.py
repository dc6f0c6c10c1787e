"""The multi-GPU kernels on ONE device (driver-visible multi-GPU parity).

G contexts are created on device 0 as ranks 0..G-1 of a G-GPU world and
wired to each other's buffers (dss_emulate_attach).  dss_emulate_step runs
each DS-Sync iteration in two passes in rank order, so every cross-rank
flag a kernel waits on was released by an earlier launch on the one shared
stream -- no concurrently spinning kernels on one GPU (what the profiling
guide forbids).  The kernels, tables and flag protocol are the multi-GPU
ones: the fused push two-shot, the one-shot with its flow control, the
ordered chain (partial and mean passes, in-place mean delivery), the pull
two-shot, on contiguous and tiled placements.  Every case is bit-exact
against the fp32 oracle."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import hparams
from paper_2007_03298_b200 import (BUF_GRADS, BUF_MOMENT1, BUF_PARAMS, DsSyncEngine, OptimizerHyperparams,
                                   OptimizerKind, StrategyKind, SyncStrategy, Topology, WorldConfig)
from paper_2007_03298_b200 import _lib as L

pytestmark = pytest.mark.gpu

CASES = [
    # W, N, rect, opt, d
    (8, 2, True, 0, 100_003),   # C2 shape: pairs / quads across the ranks
    (8, 2, True, 1, 4097),
    (16, 4, False, 3, 5000),
    (32, 4, True, 1, 3001),     # C3 shape
    (4, 2, False, 2, 999),
    (64, 8, False, 0, 2000),    # C4 shape
    (8, 2, True, 1, 200_001),   # rows past the one-shot size: push / chain
]


def run(W, N, rect, opt, d, G, orc, path=0, placement=0, iters=4):
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, rect)
    wd = 0.01 if opt in (1, 3) else 0.0
    rng = np.random.default_rng(2000 + W + opt + d)
    w = rng.standard_normal((W, d)).astype(np.float32)
    engines = [DsSyncEngine(s, OptimizerKind(opt), d, OptimizerHyperparams(weight_decay=wd), "f32", 0, r, G,
                            path=path, placement=placement) for r in range(G)]
    try:
        hs = (C.c_void_p * G)(*[e.h.value for e in engines])
        rc = L.load().dss_emulate_attach(hs, G)
        assert rc == 0, L.global_error()
        for e in engines:
            e.upload_all(BUF_PARAMS, w[e.local_ranks])
            e.enable_timing(True)
        m1, m2 = np.zeros_like(w), np.zeros_like(w)
        steps = np.zeros(W, np.int64)
        alpha = 0.05 if opt < 2 else 0.01
        for t in range(iters):
            g = rng.standard_normal((W, d)).astype(np.float32)
            for e in engines:
                e.upload_all(BUF_GRADS, g[e.local_ranks])
            rc = L.load().dss_emulate_step(hs, G, t, alpha, 1)
            assert rc == 0, (t, L.global_error())
            assert orc.ds_step(W, N, t, opt, hparams(weight_decay=wd), alpha, steps, w, g, m1, m2, rect)[0] == 0
            steps += 1
        got = np.empty_like(w)
        got_m1 = np.empty_like(w)
        for e in engines:
            got[e.local_ranks] = e.download_all(BUF_PARAMS)
            if opt >= 1:
                got_m1[e.local_ranks] = e.download_all(BUF_MOMENT1)
        kinds = engines[0].kernel_times_by_kind()
        cross = kinds["fold"][1] + kinds["chain"][1] + kinds["chain_mean"][1]
        assert cross > 0, ("no cross-GPU kernel ran", kinds)  # the multi-GPU kernels, not a local shortcut
        assert np.array_equal(got, w), (W, N, opt, d, G, path, placement)
        if opt >= 1:
            assert np.array_equal(got_m1, m1)
    finally:
        for e in engines:
            e.close()


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("path", [0, 2, 3, 4])
def test_emulated_multi_gpu_paths_bit_exact(cuda_device, oracle, G, path):
    for (W, N, rect, opt, d) in CASES:
        if W % G:
            continue
        run(W, N, rect, opt, d, G, oracle, path)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_emulated_tiled_placement_bit_exact(cuda_device, oracle, G):
    for (W, N, rect, opt, d) in CASES:
        if W % G:
            continue
        run(W, N, rect, opt, d, G, oracle, 0, placement=1)


def test_emulated_eight_gpu_plans(cuda_device, oracle):
    """The 8-GPU plans (this pool offers at most 4 GPUs): C2 pairs one-shot /
    quads push, C3 and C4 combs, on one device."""
    for (W, N, rect, opt, d) in CASES:
        if W % 8:
            continue
        for path in (0, 2):
            run(W, N, rect, opt, d, 8, oracle, path)
