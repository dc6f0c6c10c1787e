"""The one-CTA small-world batch kernel (512-thread variant) on its own,
for profiling: W=8 workers, C2's rectangular groups of 2/4, d=1000 fp32
(32 KB per array, the one-CTA limit), SGD, n iterations in one launch.
python profiles/small_world_run.py [iterations]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_03298_b200 import (BUF_GRADS, BUF_PARAMS, DsSyncEngine, OptimizerHyperparams,  # noqa: E402
                                   OptimizerKind, StrategyKind, SyncStrategy, Topology, WorldConfig)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
W, N, d = 8, 2, 1000
rng = np.random.default_rng(0)
s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, True)
with DsSyncEngine(s, OptimizerKind.VANILLA_SGD, d, OptimizerHyperparams(), "f32", 0) as e:
    e.upload_all(BUF_PARAMS, rng.standard_normal((W, d)).astype(np.float32))
    e.upload_all(BUF_GRADS, rng.standard_normal((W, d)).astype(np.float32))
    alphas = np.full(n, 1e-3)
    e.steps(0, alphas, check=True)  # warm-up
    t0 = time.perf_counter()
    for k in range(5):
        e.steps((k + 1) * n, alphas, check=True)
    dt = (time.perf_counter() - t0) / (5 * n)
    print(f"ok {1e6 * dt:.3f} us per iteration (host clock, {n} iterations per launch)")
