"""Host-side multi-GPU logic over a real gloo process group on CPU
(world_size 2, 4 and 8): IPC handle exchange/attach plumbing, and every rank's
two-shot plan agreeing with every other's (each element of each spanning
group owned exactly once, ownership identical from every rank's view)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeEngine:
    """Stands in for DsSyncEngine: records the handles it is attached with."""

    def __init__(self, rank, n_gpus):
        self.rank, self.n_gpus = rank, n_gpus
        self.attached = None

    def ipc_export(self):
        return bytes([self.rank]) * 576

    def ipc_attach(self, handles):
        self.attached = handles


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C
        from paper_2007_03298_b200 import _lib as L
        from paper_2007_03298_b200 import SyncStrategy, StrategyKind, Topology, WorldConfig
        from paper_2007_03298_b200.api import _c_strategy
        from paper_2007_03298_b200.dist import attach, local_slice

        e = FakeEngine(rank, world)
        attach(e)
        assert e.attached == [bytes([r]) * 576 for r in range(world)]
        assert list(local_slice(8 * world, world, rank)) == list(range(8 * rank, 8 * rank + 8))

        results = {}
        for (W, N, rect) in [(8, 2, True), (16, 4, False), (32, 4, True), (64, 8, False), (4, 2, False)]:
            if W % world:
                continue
            s = _c_strategy(SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, rect))
            for t in (0, 1):
                out = L.dss_plan_summary()
                lo, hi, grp = (np.zeros(128, np.int64), np.zeros(128, np.int64), np.zeros(128, np.int32))
                st = L.load().dss_plan(C.byref(s), t, 12345, world, rank, C.byref(out), lo.ctypes.data,
                                       hi.ctypes.data, grp.ctypes.data, 128)
                assert st == 0
                n = out.owned_slices
                mine = list(zip(grp[:n].tolist(), lo[:n].tolist(), hi[:n].tolist()))
                allv = [None] * world
                dist.all_gather_object(allv, mine)
                chains = [None] * world
                dist.all_gather_object(chains, out.chain_groups)
                # every spanning group's slices tile [0, d_pad) exactly once
                d_pad = (12345 + 63) // 64 * 64
                by_group = {}
                for r, sl in enumerate(allv):
                    for g, a, b in sl:
                        by_group.setdefault(g, []).append((a, b, r))
                for g, ivs in by_group.items():
                    ivs.sort()
                    assert ivs[0][0] == 0 and ivs[-1][1] == d_pad, (W, N, t, g)
                    for x, y in zip(ivs, ivs[1:]):
                        assert x[1] == y[0]
                results[(W, N, t)] = (len(by_group), tuple(chains))
        # every rank derives the same worker placement (dss_placement is
        # host-side and deterministic), for every mode and DS shape
        from paper_2007_03298_b200 import placement
        for (W, N, rect) in [(8, 2, True), (32, 4, True), (64, 8, False), (16, 4, False)]:
            if W % world:
                continue
            st = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, rect)
            for mode in (0, 1, 2):
                mine = placement(st, world, mode)
                allp = [None] * world
                dist.all_gather_object(allp, mine)
                assert all(p == allp[0] for p in allp), (W, N, mode)
                gpu, row, _ = mine
                assert sorted(zip(gpu, row)) == [(g, r) for g in range(world) for r in range(W // world)]
        q.put((rank, "ok", results))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_plan_and_handle_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, _ in res:
        assert status == "ok", (rank, status)
    views = [r[2] for r in res]
    assert all(v == views[0] for v in views)
