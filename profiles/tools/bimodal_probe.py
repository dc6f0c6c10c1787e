"""Run-to-run spread of one small-row multi-GPU shape: R fresh engines,
each timed over K iterations (dss_steps), per-rank device time.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        profiles/tools/bimodal_probe.py --gpus G --W 16 --N 4 --bytes 262144 [--kind ds|bsp]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--W", type=int, default=16)
    ap.add_argument("--N", type=int, default=4)
    ap.add_argument("--bytes", type=int, default=262144)
    ap.add_argument("--kind", default="ds")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--steps", type=int, default=2000)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2007_03298_b200 import (DsSyncEngine, OptimizerHyperparams, OptimizerKind, StrategyKind, SyncStrategy,
                                       Topology, WorldConfig)
    from paper_2007_03298_b200.dist import attach
    G = args.gpus
    rank, local = int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    K, W, N, d = args.steps, args.W, args.N, args.bytes // 4
    ds = args.kind == "ds"
    out = []
    for rep in range(args.reps):
        s = SyncStrategy(StrategyKind.DS_SYNC if ds else StrategyKind.BSP, Topology.RING, WorldConfig(W, N if ds else W))
        e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, d, OptimizerHyperparams(), "f32", local, rank, G)
        e.set_stream(stream.cuda_stream)
        attach(e)
        e.quadratic_init(7, 4.0)
        e.quadratic_gradients(0, 1, 1.0, 0.5)
        al = np.full(K, 1e-3)
        e.steps(0, al[:50])
        torch.cuda.synchronize()
        dist.barrier()
        ms = []
        for blk in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e.steps(50 + blk * K, al)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(round(a.elapsed_time(b) * 1e3 / K, 2))
        e.check()
        e.close()
        del e
        torch.cuda.synchronize()
        rows = [None] * G
        dist.all_gather_object(rows, ms)
        if rank == 0:
            print(json.dumps({"rep": rep, "W": W, "N": N, "bytes": args.bytes, "kind": args.kind,
                              "us_per_iter_by_rank_and_block": rows,
                              "variant": os.environ.get("DSS_LIB_VARIANT", "base").split("/")[-1]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
