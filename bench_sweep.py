"""Sync microbench (BASELINE config 5): per-worker buffer 1 KB .. 1 GB x group
size N in {2, 4, 8} (W = N^2 workers, DS-Sync square schedule) on G GPUs:
DS-Sync vs our bit-exact BSP vs an NCCL BSP all-reduce baseline.

    python bench_sweep.py [--opt sgd|sync] [--max-mb 1024] > sweep.jsonl
    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 bench_sweep.py --gpus G

One JSON line per (N, bytes, G) on rank 0.  `ds_iters_s` / `bsp_iters_s`
run through the C-ABI (dss_steps, device-resident rows);
`nccl_bsp_iters_s` (G > 1) = local pre-sum (one strided reduction) +
torch.distributed NCCL world all-reduce + x1/W + our apply_step.  DS engines
use the auto worker placement (--placement).  Effective GB/s = W * d * 4 / t.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--min-kb", type=int, default=1)
    ap.add_argument("--max-mb", type=int, default=1024)
    ap.add_argument("--groups", default="2,4,8")
    ap.add_argument("--opt", default="sgd", choices=["sgd", "sync"])
    ap.add_argument("--mem-gb", type=float, default=150.0, help="per-GPU cap for the worker arrays")
    ap.add_argument("--path", type=int, default=0, help="fold path (0 auto; 4 auto without one-shot)")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--placement", type=int, default=2, help="DS placement: 0 contiguous, 1 tiled, 2 auto")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2007_03298_b200 import (BUF_GRADS, BUF_PARAMS, DsSyncEngine, OptimizerKind, StrategyKind,
                                       SyncStrategy, Topology, WorldConfig)

    G = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if G > 1:
        from paper_2007_03298_b200.dist import pin_host_cores
        pin_host_cores(local, int(os.environ.get("LOCAL_WORLD_SIZE", G)))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    # ~1 s of device work first: the first shapes are microsecond steps whose
    # timed region (a few ms) is too short to bring an idle GPU's clocks up
    a = torch.full((4096, 4096), 1e-3, device="cuda")
    t_end = time.time() + 1.0
    while time.time() < t_end:
        for _ in range(20):
            a = torch.mm(a, a).clamp_(-1.0, 1.0)
        torch.cuda.synchronize()
    del a

    def sync_max(x):
        if G == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def timed(fn, K):
        if G > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn(K)
        b.record(stream)
        torch.cuda.synchronize()
        return sync_max(a.elapsed_time(b)) / K

    sizes = []
    b = args.min_kb * 1024
    while b <= args.max_mb * 1024 * 1024:
        sizes.append(b)
        b *= 4
    shapes = []
    for N in [int(x) for x in args.groups.split(",")]:
        W = N * N
        if W % G:
            continue
        P = W // G
        for nbytes in sizes:
            d = nbytes // 4
            if P * d * 4 * 2 > args.mem_gb * 1e9:
                continue
            shapes.append((N, W, P, nbytes, d, int(max(5, min(2000, 4e9 / (P * nbytes * 3 + 1))))))

    def engine(kind, W, N, d):
        s = SyncStrategy(kind, Topology.RING, WorldConfig(W, N if kind == StrategyKind.DS_SYNC else W))
        e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, d, None, "f32", local, rank, G, path=args.path,
                         placement=args.placement if kind == StrategyKind.DS_SYNC else 0)
        e.set_stream(stream.cuda_stream)
        if G > 1:
            from paper_2007_03298_b200.dist import attach
            attach(e)
        e.quadratic_init(7, 4.0)
        e.quadratic_gradients(0, 1, 1.0, 0.5)
        return e

    rows = []
    for N, W, P, nbytes, d, K in shapes:
        row = {"N": N, "W": W, "bytes_per_worker": nbytes, "d": d, "n_gpus": G, "steps": K, "opt": args.opt,
               "path": args.path, "placement": args.placement}
        for kind, key in ((StrategyKind.DS_SYNC, "ds"), (StrategyKind.BSP, "bsp")):
            e = engine(kind, W, N, d)
            if args.opt == "sync" and kind == StrategyKind.DS_SYNC:
                run = lambda K: [e.sync_round(t, check=False) for t in range(K)]  # noqa: E731
            else:
                run = lambda K: e.steps(0, np.full(K, 0.01))  # noqa: E731
            run(min(50, K))  # warm-up: plans built, caches and the cross-GPU flag protocol in steady state
            ms = timed(run, K)
            e.check()
            row[key + "_ms"] = ms
            row[key + "_iters_s"] = 1000.0 / ms
            row[key + "_eff_gbs"] = W * d * 4 / (ms / 1e3) / 1e9
            e.close()
            del e
            torch.cuda.synchronize()
        rows.append(row)
        if G == 1 or args.no_nccl:
            if rank == 0:
                print(json.dumps(row), flush=True)
    if G > 1 and not args.no_nccl:
        # The NCCL baseline in a second pass after all of ours: our kernels
        # run right after NCCL all-reduces in the same process are
        # intermittently up to 2x slower (profiles/r02/sweeps/nccl_order_g2.md)
        for (N, W, P, nbytes, d, K), row in zip(shapes, rows):
            e = engine(StrategyKind.BSP, W, N, d)
            # the local gradient rows as one strided view of the engine's
            # contiguous [P][row_stride] buffer: no gather copies
            ptr, stride = e.device_ptr(BUF_GRADS, e.local_ranks[0]), e.row_stride

            class _A:
                __cuda_array_interface__ = {"shape": (P, stride), "typestr": "<f4", "data": (ptr, False),
                                            "version": 3}
            grads = torch.as_tensor(_A(), device="cuda")[:, :d]
            acc = torch.empty(d, dtype=torch.float32, device="cuda")

            def nccl(K):
                for _ in range(K):
                    torch.sum(grads, dim=0, out=acc)
                    dist.all_reduce(acc)
                    acc.mul_(1.0 / W)
                    grads.copy_(acc.expand_as(grads))
                    e.apply_step(0.01, check=False)
            nccl(3)
            ms = timed(nccl, K)
            row["nccl_bsp_ms"] = ms
            row["nccl_bsp_iters_s"] = 1000.0 / ms
            del grads, acc
            e.close()
            del e
            torch.cuda.synchronize()
            if rank == 0:
                print(json.dumps(row), flush=True)
    if G > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
