"""BASELINE configs C3 and the C4 per-GPU slice at their full sizes on one
B200, checked against the fp32 oracle on sampled columns.

The fold is elementwise (sync.cpp:347-374: every element's step and
ascending member fold is independent of every other element's), so the
oracle only needs the sampled columns of every worker: 64k random columns
plus the row ends and chunk edges.  Each case runs one block and one comb
iteration (C3: groups of 4 then 8, momentum; C4 slice: one group of 8,
AdamW, DS and BSP) from the device-generated synthetic state, and also
checks the size-independent properties on whole rows: every group's
members bit-identical after the sync.
"""
import numpy as np
import pytest

from oracle.oracle import hparams
from paper_2007_03298_b200 import (BUF_GRADS, BUF_MOMENT1, BUF_MOMENT2, BUF_PARAMS, DsSyncEngine,
                                   OptimizerHyperparams, OptimizerKind, StrategyKind, SyncStrategy, Topology,
                                   WorldConfig, make_partition)

pytestmark = pytest.mark.gpu

CASES = {
    # name: (kind, W, N, rect, d, opt, alpha, weight_decay)
    "c3": ("ds", 32, 4, True, 36_500_000, 1, 0.1, 1e-4),
    "c4slice": ("ds", 8, 8, False, 340_000_000, 3, 3e-5, 0.01),
    "c4slice_bsp": ("bsp", 8, 8, False, 340_000_000, 3, 3e-5, 0.01),
}


def _view(e, buffer, rank, n):
    import torch

    class _A:
        def __init__(self, ptr):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_A(e.device_ptr(buffer, rank)), device="cuda")


def _gather(e, buffer, W, d, idx_t):
    import torch
    return torch.stack([_view(e, buffer, k, d).index_select(0, idx_t) for k in range(W)]).cpu().numpy()


@pytest.mark.parametrize("name", sorted(CASES))
def test_full_size_sampled_columns_vs_oracle(cuda_device, oracle, name):
    import torch
    kind, W, N, rect, d, opt, alpha, wd = CASES[name]
    ds = kind == "ds"
    s = SyncStrategy(StrategyKind.DS_SYNC if ds else StrategyKind.BSP, Topology.RING, WorldConfig(W, N), 1, rect)
    rng = np.random.default_rng(17)
    edges = [0, 1, 63, 64, 8191, 8192, 8193, d // 2, d - 64, d - 2, d - 1]
    idx = np.unique(np.concatenate([rng.choice(d, 65536, replace=False), edges])).astype(np.int64)
    idx_t = torch.as_tensor(idx, device="cuda")
    with DsSyncEngine(s, OptimizerKind(opt), d, OptimizerHyperparams(weight_decay=wd), "f32", 0) as e:
        e.quadratic_init(7, 4.0)
        e.quadratic_gradients(0, 1, 1.0, 0.5)
        torch.cuda.synchronize()
        w = _gather(e, BUF_PARAMS, W, d, idx_t)
        g = _gather(e, BUF_GRADS, W, d, idx_t)
        m1 = np.zeros_like(w) if opt else None
        m2 = np.zeros_like(w) if opt >= 2 else None
        steps = np.zeros(W, np.int64)
        hp = hparams(weight_decay=wd)
        for t in range(2):
            e.step(t, alpha, check=True)
            if ds:
                rc, _, _ = oracle.ds_step(W, N, t, opt, hp, alpha, steps, w, g, m1, m2, rect=rect)
            else:
                rc, _, _ = oracle.bsp_step(t, opt, hp, alpha, steps, w, g, m1, m2)
            assert rc == 0
            steps += 1
            torch.cuda.synchronize()
            assert np.array_equal(_gather(e, BUF_PARAMS, W, d, idx_t), w), (name, t)
            if m1 is not None:
                assert np.array_equal(_gather(e, BUF_MOMENT1, W, d, idx_t), m1), (name, t, "m1")
            if m2 is not None:
                assert np.array_equal(_gather(e, BUF_MOMENT2, W, d, idx_t), m2), (name, t, "m2")
            if ds:
                # whole rows: every group's members carry identical bits after the sync
                for grp in make_partition(s, t).groups:
                    v0 = _view(e, BUF_PARAMS, grp[0], d)
                    for r in grp[1:]:
                        assert torch.equal(v0, _view(e, BUF_PARAMS, r, d)), (name, t, grp)
            else:
                # BSP: every replica stepped with the same mean gradient from the
                # same start stays identical
                v0 = _view(e, BUF_PARAMS, 0, d)
                for r in range(1, W):
                    assert torch.equal(v0, _view(e, BUF_PARAMS, r, d)), (name, t, r)
