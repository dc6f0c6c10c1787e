"""Is the small-row multi-GPU step bound by host launches or by the GPU?

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        profiles/tools/launch_gap_probe.py --gpus G

For DS (W=N^2, square) and BSP at 1 KB and 64 KB rows: the device time of K
iterations in one dss_steps call, the host time the call takes to enqueue
them (wall clock of the call, no sync), and the summed device time of the
library's kernels (per-kernel events).  Enqueue time ~ device time means
the host launch loop is the bound; kernel time well below the device time
means gaps between kernels.  One JSON line per case on rank 0."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
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
    K = args.steps
    for kind in ("ds", "bsp"):
        for N in (2, 4, 8):
            W = N * N
            if W % G:
                continue
            for nbytes in (1024, 65536):
                d = nbytes // 4
                s = SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING,
                                 WorldConfig(W, N if kind == "ds" else W))
                e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, d, OptimizerHyperparams(), "f32", local, rank, G)
                e.set_stream(stream.cuda_stream)
                attach(e)
                e.quadratic_init(7, 4.0)
                e.quadratic_gradients(0, 1, 1.0, 0.5)
                al = np.full(K, 1e-3)
                e.steps(0, al[:50])
                torch.cuda.synchronize()
                dist.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                h0 = time.perf_counter()
                e.steps(50, al)
                h1 = time.perf_counter()
                b.record(stream)
                torch.cuda.synchronize()
                dev_us = a.elapsed_time(b) * 1e3 / K
                host_us = (h1 - h0) * 1e6 / K
                dist.barrier()
                e.enable_timing(True)
                e.steps(50 + K, al)
                torch.cuda.synchronize()
                kinds = e.kernel_times_by_kind()
                e.enable_timing(False)
                e.check()
                kern = {k: round(v[0] * 1e3 / K, 2) for k, v in kinds.items() if v[1]}
                launches = sum(v[1] for v in kinds.values()) / K
                row = dict(kind=kind, W=W, N=N, G=G, bytes=nbytes, device_us_per_iter=round(dev_us, 2),
                           host_enqueue_us_per_iter=round(host_us, 2), kernel_us_per_iter=kern,
                           kernel_sum_us=round(sum(kern.values()), 2), launches_per_iter=launches)
                rows = [None] * G
                dist.all_gather_object(rows, row)
                if rank == 0:
                    print(json.dumps(dict(rank0=row, max_device_us=max(r["device_us_per_iter"] for r in rows),
                                          max_host_us=max(r["host_enqueue_us_per_iter"] for r in rows))), flush=True)
                e.close()
                del e
                torch.cuda.synchronize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
