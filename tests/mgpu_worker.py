"""Worker for the multi-GPU parity test (one process per GPU, launched by
tests/test_multi_gpu.py through torch.distributed.run).

Every rank builds the same seeded full [W][d] inputs, uploads its own rows,
maps its peers' rows over NVLink (CUDA IPC), runs DS-Sync / BSP iterations
whose spanning groups are folded by the in-kernel two-shot P2P path, and
rank 0 checks the gathered result bit for bit against the fp32 oracle.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, hparams  # noqa: E402
from paper_2007_03298_b200 import (BUF_GRADS, BUF_MOMENT1, BUF_PARAMS, BUF_STATS, BUF_STATS_OBS,  # noqa: E402
                                   DsSyncEngine,
                                   OptimizerHyperparams, OptimizerKind, StrategyKind, SyncStrategy, Topology,
                                   WorldConfig)
from paper_2007_03298_b200.dist import attach, local_slice  # noqa: E402

CASES = [
    # kind, W, N, rect, opt, d
    ("ds", 8, 2, True, 0, 100_003),   # C2 shape: pairs / quads spanning GPUs
    ("ds", 8, 2, True, 1, 4097),
    ("ds", 16, 4, False, 3, 5000),    # blocks local or spanning by G, combs spanning
    ("ds", 32, 4, True, 1, 3001),     # C3 shape
    ("ds", 4, 2, False, 2, 999),
    ("bsp", 8, 8, False, 0, 70_001),
    ("bsp", 4, 4, False, 3, 2049),
    ("bsp", 16, 16, False, 1, 300_007),  # packed BSP: chain over gradient rows
    ("ds", 64, 8, False, 0, 20_000),     # C4 shape
    ("bsp", 64, 64, False, 1, 3001),     # W=64 small rows: one-shot gather of all 64 gradient rows
    ("bsp", 64, 64, False, 3, 20_001),   # W=64 chain with short (small-row) chunks
    ("bsp", 4, 4, False, 2, 250_001),    # 1 MB rows, W=4: one-shot gather past the small-row limit
    ("bsp", 16, 16, False, 1, 1_000_003),  # 4 MB rows: pull two-shot at <= 4 replicas per GPU, else chain
]


def device_of(rank):
    """Process rank -> CUDA device (several ranks per device when oversubscribed)."""
    return rank % torch.cuda.device_count()


def run_case(kind, W, N, rect, opt, d, rank, G, orc, path=0, sd=0, placement=0, iters=5):
    s = SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING,
                     WorldConfig(W, N), 1, rect)
    wd = 0.01 if opt in (1, 3) else 0.0
    hp = OptimizerHyperparams(weight_decay=wd)
    rng = np.random.default_rng(1000 + W + opt)
    w = rng.standard_normal((W, d)).astype(np.float32)
    e = DsSyncEngine(s, OptimizerKind(opt), d, hp, "f32", device_of(rank), rank, G, path=path, stats_dim=sd,
                     placement=placement)
    mine = e.local_ranks  # this GPU's workers in local-row order (contiguous unless placed)
    if not placement:
        assert mine == list(local_slice(W, G, rank))
    attach(e)
    e.upload_all(BUF_PARAMS, w[mine])
    rs = rng.standard_normal((W, sd)).astype(np.float32) if sd else None
    if sd:
        e.upload_all(BUF_STATS, rs[mine])
    m1, m2 = np.zeros_like(w), np.zeros_like(w)
    steps = np.zeros(W, np.int64)
    alpha = 0.05 if opt < 2 else 0.01
    for t in range(iters):
        g = rng.standard_normal((W, d)).astype(np.float32)
        e.upload_all(BUF_GRADS, g[mine])
        if sd:  # fold_running_stats EMA, then the stats ride the step's fold
            obs = rng.standard_normal((W, sd)).astype(np.float32)
            e.upload_all(BUF_STATS_OBS, obs[mine])
            e.running_stats_update()
            rs = (np.float32(0.9) * rs + np.float32(0.1) * obs).astype(np.float32)
            if kind == "ds":
                orc.sync_round(W, N, t, rs, rect=rect)
            else:
                orc.sync_round(W, W, t, rs, kind=0)
        e.step(t, alpha)
        if kind == "ds":
            rc = orc.ds_step(W, N, t, opt, hparams(weight_decay=wd), alpha, steps, w, g, m1, m2, rect)
        else:
            rc = orc.bsp_step(t, opt, hparams(weight_decay=wd), alpha, steps, w, g, m1, m2)
        assert rc[0] == 0
        steps += 1
    # sync-only round too (sync_round semantics over peers)
    e.sync_round(iters, check=False)
    if kind == "ds":
        orc.sync_round(W, N, iters, w, rect=rect)
        if sd:
            orc.sync_round(W, N, iters, rs, rect=rect)
    else:
        orc.sync_round(W, W, iters, w, kind=0)
        if sd:
            orc.sync_round(W, W, iters, rs, kind=0)
    e.check()
    got = e.download_all(BUF_PARAMS)
    got_m1 = e.download_all(BUF_MOMENT1) if opt >= 1 else None
    got_rs = e.download_all(BUF_STATS) if sd else None
    e.check_guards()  # DSS_GUARD_BYTES runs: no kernel wrote outside its buffers (raises otherwise)
    parts = [None] * G
    dist.all_gather_object(parts, (mine, got, got_m1, got_rs))
    e.close()
    if rank == 0:
        order = np.argsort(np.concatenate([p[0] for p in parts]))  # rows back into rank order
        full = np.concatenate([p[1] for p in parts])[order]
        ok = np.array_equal(full, w)
        if opt >= 1:
            ok = ok and np.array_equal(np.concatenate([p[2] for p in parts])[order], m1)
        if sd:
            ok = ok and np.array_equal(np.concatenate([p[3] for p in parts])[order], rs)
        diff = float(np.abs(full - w).max())
        print(f"case {kind} W={W} N={N} rect={rect} opt={opt} d={d} path={path} stats={sd} placement={placement}: "
              f"{'OK' if ok else 'MISMATCH'} maxdiff={diff}",
              flush=True)
        return ok
    return True


def logistic_case(rank, G, sampling, kind):
    """C1 end to end on G GPUs (device batch sampling + logistic gradient +
    the step, f64) equals the same run with all workers on one GPU, bit for
    bit: the schedule, the sampling streams and every fold are independent
    of the packing."""
    from paper_2007_03298_b200 import SamplingMode, logistic_dataset
    W, N, T = 4, (2 if kind == "ds" else 4), 40
    if W % G:
        return True
    x, y = logistic_dataset(11, 20, 2000)
    alphas = 1.0 * 0.5 ** (np.arange(T) // 15)
    s = SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING, WorldConfig(W, N))
    e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 20, OptimizerHyperparams(), "f64", device_of(rank), rank, G)
    attach(e)
    e.logistic_setup(x, y, 0.05, 8, sampling, 1)
    e.logistic_steps(0, alphas, check=True)
    parts = [None] * G
    dist.all_gather_object(parts, e.download_all(BUF_PARAMS))
    e.close()
    if rank != 0:
        return True
    with DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 20, OptimizerHyperparams(), "f64", 0) as one:
        one.logistic_setup(x, y, 0.05, 8, sampling, 1)
        for t in range(T):  # per-iteration launches (the one-CTA path has its own test)
            one.logistic_gradients(t)
            one.step(t, float(alphas[t]))
        ref = one.download_all(BUF_PARAMS)
    ok = np.array_equal(np.concatenate(parts), ref)
    print(f"case logistic {kind} sampling={int(sampling)} G={G}: {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def placed_logistic_case(rank, G):
    """C1-style logistic run (device sampling from the workers' shards, f64)
    over a placed 16-worker world equals the same run on one GPU: shards,
    batch streams and gradient noise follow the global rank, not the row."""
    from paper_2007_03298_b200 import SamplingMode, logistic_dataset
    W, N, T = 16, 4, 12
    if W % G:
        return True
    x, y = logistic_dataset(11, 20, 2000)
    alphas = np.full(T, 0.5)
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N))
    e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 20, OptimizerHyperparams(), "f64", device_of(rank), rank, G,
                     placement=1)
    attach(e)
    e.logistic_setup(x, y, 0.05, 8, SamplingMode.EPOCH, 1)
    for t in range(T):
        e.logistic_gradients(t)
        e.step(t, float(alphas[t]))
    e.check()
    parts = [None] * G
    dist.all_gather_object(parts, (e.local_ranks, e.download_all(BUF_PARAMS)))
    e.close()
    if rank != 0:
        return True
    order = np.argsort(np.concatenate([p[0] for p in parts]))
    got = np.concatenate([p[1] for p in parts])[order]
    with DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 20, OptimizerHyperparams(), "f64", 0) as one:
        one.logistic_setup(x, y, 0.05, 8, SamplingMode.EPOCH, 1)
        for t in range(T):
            one.logistic_gradients(t)
            one.step(t, float(alphas[t]))
        ref = one.download_all(BUF_PARAMS)
    ok = np.array_equal(got, ref)
    print(f"case placed logistic W=16 G={G}: {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def busy_case(rank, G):
    """Cross-GPU push steps issued while another stream keeps every SM busy
    with matmuls complete (no flag-wait timeout: the cooperative launch
    keeps the push kernel's CTAs co-resident) and give the same bits as the
    same steps on an idle GPU."""
    if torch.cuda.device_count() < G:
        return True  # oversubscribed ranks share a device: not this case
    ok = True
    for kind, W, N, rect, opt, d in (("ds", 8, 2, True, 1, 4097), ("ds", 16, 4, False, 3, 100_003),
                                     ("bsp", 8, 8, False, 1, 3001)):
        s = SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING,
                         WorldConfig(W, N), 1, rect)
        outs = []
        for busy in (False, True):
            e = DsSyncEngine(s, OptimizerKind(opt), d, OptimizerHyperparams(weight_decay=0.01), "f32",
                             device_of(rank), rank, G)
            attach(e)
            e.quadratic_init(7, 4.0)
            e.quadratic_gradients(0, 1, 1.0, 0.5)
            torch.cuda.synchronize()
            dist.barrier()
            side = torch.cuda.Stream()
            if busy:
                with torch.cuda.stream(side):
                    a = torch.full((8192, 8192), 1e-4, device="cuda")
                    c = torch.empty_like(a)
                    for _ in range(12):  # ~0.2 s of full-device matmuls
                        torch.mm(a, a, out=c)
            e.steps(0, np.full(24, 0.01))
            e.check()  # raises on a latched flag-wait timeout
            torch.cuda.synchronize()
            outs.append(e.download_all(BUF_PARAMS))
            e.close()
        same = bool(np.array_equal(outs[0], outs[1]))
        flags = [None] * G
        dist.all_gather_object(flags, same)
        ok = ok and all(flags)
        if rank == 0:
            print(f"case busy-GPU {kind} W={W} N={N} d={d} G={G}: {'OK' if all(flags) else 'MISMATCH'}", flush=True)
    return ok


def bsp_stream_case(rank, G, orc):
    """Hundreds of back-to-back BSP steps in one dss_steps call (chain-only
    plans skip the per-step barrier, pull / one-shot plans keep their own
    protocol) equal the oracle's loop bit for bit."""
    ok = True
    for W, d, opt, iters in ((64, 20_001, 1, 200), (16, 300_007, 1, 100), (8, 250_001, 0, 100)):
        if W % G:
            continue
        s = SyncStrategy(StrategyKind.BSP, Topology.RING, WorldConfig(W, W))
        hp = OptimizerHyperparams(weight_decay=0.01)
        rng = np.random.default_rng(77 + W)
        w = rng.standard_normal((W, d)).astype(np.float32)
        g = rng.standard_normal((W, d)).astype(np.float32)
        e = DsSyncEngine(s, OptimizerKind(opt), d, hp, "f32", device_of(rank), rank, G)
        attach(e)
        mine = e.local_ranks
        e.upload_all(BUF_PARAMS, w[mine])
        e.upload_all(BUF_GRADS, g[mine])
        e.steps(0, np.full(iters, 0.01))
        e.check()
        got = e.download_all(BUF_PARAMS)
        parts = [None] * G
        dist.all_gather_object(parts, (mine, got))
        e.close()
        if rank == 0:
            m1, m2 = np.zeros_like(w), np.zeros_like(w)
            steps = np.zeros(W, np.int64)
            for t in range(iters):
                assert orc.bsp_step(t, opt, hparams(weight_decay=0.01), 0.01, steps, w, g, m1, m2)[0] == 0
                steps += 1
            order = np.argsort(np.concatenate([p[0] for p in parts]))
            same = bool(np.array_equal(np.concatenate([p[1] for p in parts])[order], w))
            print(f"case bsp stream W={W} d={d} steps={iters} G={G}: {'OK' if same else 'MISMATCH'}", flush=True)
            ok = ok and same
    return ok


def ds_stream_case(rank, G, orc):
    """Tens to hundreds of back-to-back DS steps in one dss_steps call equal
    the oracle's loop bit for bit, and a sync_round afterwards (barrier
    restored) too.  Chain-only plans skip the per-step barrier (per-parity
    chain rows and flags); two-shot push plans replace it with the split
    barrier (the push kernel arrives, the next step's first kernel waits):
    push -> local group kernel (C2 shape and W=16 on 4 GPUs, contiguous) and
    push -> push (W=4 with pairs forced off one-shot, path 4).  On 2 GPUs
    the C2 shape's comb chains leave their mean pass to the next block step
    (deferred, fused with the local groups: LazyPlan), SGD / momentum /
    AdamW."""
    ok = True
    for W, N, rect, opt, d, iters, placement, path in ((8, 2, True, 1, 250_001, 100, 0, 0),
                                                       (16, 4, False, 3, 200_003, 60, 1, 0),
                                                       (32, 4, True, 1, 150_001, 60, 1, 0),
                                                       (8, 2, True, 0, 250_001, 100, 0, 0),
                                                       (16, 4, False, 3, 200_003, 60, 0, 0),
                                                       (4, 2, False, 1, 250_001, 100, 0, 4),
                                                       (4, 2, False, 3, 4097, 200, 0, 4),
                                                       (8, 2, True, 3, 250_001, 60, 0, 0)):
        if W % G:
            continue
        s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, rect)
        hp = OptimizerHyperparams(weight_decay=0.01)
        rng = np.random.default_rng(91 + W)
        w = rng.standard_normal((W, d)).astype(np.float32)
        g = rng.standard_normal((W, d)).astype(np.float32)
        e = DsSyncEngine(s, OptimizerKind(opt), d, hp, "f32", device_of(rank), rank, G, path=path,
                         placement=placement)
        attach(e)
        mine = e.local_ranks
        e.upload_all(BUF_PARAMS, w[mine])
        e.upload_all(BUF_GRADS, g[mine])
        alpha = 0.01 if opt >= 2 else 0.05
        e.enable_timing(True)
        e.steps(0, np.full(iters, alpha))
        barriers = e.kernel_times_by_kind()["barrier"][1]
        e.enable_timing(False)
        # two-shot push plans: no barrier launch between the steps (split barrier)
        push_plan = placement == 0 and ((W, G) in ((8, 4), (16, 4)) or path == 4)
        e.sync_round(iters, check=False)
        e.check()
        got = e.download_all(BUF_PARAMS)
        parts = [None] * G
        dist.all_gather_object(parts, (mine, got))
        e.close()
        if rank == 0:
            m1, m2 = np.zeros_like(w), np.zeros_like(w)
            steps = np.zeros(W, np.int64)
            for t in range(iters):
                assert orc.ds_step(W, N, t, opt, hparams(weight_decay=0.01), alpha, steps, w, g, m1, m2, rect)[0] == 0
                steps += 1
            orc.sync_round(W, N, iters, w, rect=rect)
            order = np.argsort(np.concatenate([p[0] for p in parts]))
            same = bool(np.array_equal(np.concatenate([p[1] for p in parts])[order], w))
            same = same and not (push_plan and barriers)
            print(f"case ds stream W={W} N={N} opt={opt} d={d} steps={iters} placement={placement} path={path} G={G}: "
                  f"barriers={barriers} {'OK' if same else 'MISMATCH'}", flush=True)
            ok = ok and same
    return ok


def fingerprint_case(rank, G):
    """Ranks created with different geometry (here: a different d per rank)
    must refuse to map each other's buffers (dss_ipc_attach fingerprint)."""
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(8, 2), 1, True)
    e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 1000 + rank, OptimizerHyperparams(), "f32", device_of(rank), rank, G)
    try:
        attach(e)
        ok = False
    except ValueError as ex:
        ok = "different configuration" in str(ex)
    e.close()
    if rank == 0:
        print(f"case fingerprint mismatch G={G}: {'OK' if ok else 'MISSED'}", flush=True)
    return ok


def main():
    rank = int(os.environ["RANK"])
    G = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(device_of(rank))
    dist.init_process_group("gloo")
    orc = Oracle()
    ok = fingerprint_case(rank, G)
    ok = busy_case(rank, G) and ok
    ok = bsp_stream_case(rank, G, orc) and ok
    ok = ds_stream_case(rank, G, orc) and ok
    for case in CASES:
        if case[1] % G:
            continue
        # auto (one-shot / fused push two-shot / chain by shape), chain forced,
        # unfused pull two-shot, auto without one-shot
        for path in (0, 2, 3, 4):
            ok = run_case(*case, rank, G, orc, path) and ok
    for case in (("ds", 8, 2, True, 2, 1001), ("bsp", 8, 8, False, 1, 777)):  # running-stats tail
        ok = run_case(*case, rank, G, orc, 0, sd=6) and ok
    # tiled placement (blocks over gc GPUs, combs over gr): every DS shape whose
    # grid tiles differently from contiguous packing at this G, every path
    for case in CASES:
        if case[0] != "ds" or case[1] % G:
            continue
        for path in (0, 2, 3, 4):
            ok = run_case(*case, rank, G, orc, path, placement=1) and ok
    ok = run_case("ds", 32, 4, True, 2, 1001, rank, G, orc, 0, sd=6, placement=1) and ok
    # rows past the 80 MiB long-chunk threshold (16384-element chain chunks,
    # C2-sized rows): a block and a comb iteration plus a sync round
    ok = run_case("ds", 8, 2, True, 1, 21_000_003, rank, G, orc, 0, iters=2) and ok
    # the same row size on a tiled placement (two-GPU-deep chains in both parities)
    if G == 4:
        ok = run_case("ds", 16, 4, False, 3, 21_000_003, rank, G, orc, 0, placement=1, iters=2) and ok
    for kind in ("ds",):
        ok = placed_logistic_case(rank, G) and ok
    from paper_2007_03298_b200 import SamplingMode
    for kind in ("ds", "bsp"):
        for sampling in (SamplingMode.REPLACEMENT, SamplingMode.EPOCH):
            ok = logistic_case(rank, G, sampling, kind) and ok
    dist.barrier()
    if rank == 0:
        print("MGPU " + ("PASS" if ok else "FAIL"), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
