"""Per-iteration wall time vs kernel time for tiny rows on G GPUs (is the
small-row multi-GPU regime launch-bound?).  torchrun ... small_rows_probe.py W N d"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2007_03298_b200 import (DsSyncEngine, OptimizerKind, StrategyKind, SyncStrategy,  # noqa: E402
                                   Topology, WorldConfig)
from paper_2007_03298_b200.dist import attach  # noqa: E402

W, N, d = (int(x) for x in sys.argv[1:4])
rank, G = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N))
e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, d, None, "f32", rank, rank, G, placement=2)
attach(e)
e.quadratic_init(7, 4.0)
e.quadratic_gradients(0, 1, 1.0, 0.5)
K = 4000
e.steps(0, np.full(200, 0.01))
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
e.steps(200, np.full(K, 0.01))
t_enq = (time.perf_counter() - t0) / K  # host time to enqueue (dss_steps returns before the GPU is done)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K
e.enable_timing(True)
e.steps(200 + K, np.full(K, 0.01))
torch.cuda.synchronize()
kinds = {k: (v[0] * 1e3 / K, v[1] / K) for k, v in e.kernel_times_by_kind().items() if v[1]}
e.enable_timing(False)
t1 = time.perf_counter()
for t in range(K):
    e.lib.dss_launch_count(e.h)  # host-side floor of a trivial C call
host_call = (time.perf_counter() - t1) / K
if rank == 0:
    print(json.dumps({"W": W, "N": N, "d": d, "G": G, "wall_us_per_iter": wall * 1e6,
                      "host_enqueue_us_per_iter": t_enq * 1e6,
                      "kernel_us_per_iter_by_kind": {k: round(v[0], 3) for k, v in kinds.items()},
                      "launches_per_iter": {k: v[1] for k, v in kinds.items()}}))
dist.destroy_process_group()
