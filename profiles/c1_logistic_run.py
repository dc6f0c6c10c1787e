"""C1 end to end on the device (dss_logistic_steps -> the one-CTA
small-world kernel: sampling, logistic gradient, step, group fold), for
profiling: python profiles/c1_logistic_run.py [iterations]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_03298_b200 import (DsSyncEngine, OptimizerHyperparams, OptimizerKind, SamplingMode,  # noqa: E402
                                   StrategyKind, SyncStrategy, Topology, WorldConfig, logistic_dataset)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
x, y = logistic_dataset(11, 20, 2000)
s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(4, 2))
with DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 20, OptimizerHyperparams(), "f32", 0) as e:
    e.logistic_setup(x, y, 0.05, 8, SamplingMode.REPLACEMENT, 1)
    alphas = 1.0 * 0.5 ** (np.arange(n) // 75)
    e.logistic_steps(0, alphas, check=True)
    print("ok", e.download_all(0)[0, :3])
