"""e2e (dss_step_host, pinned host buffers) A/B of library variants:
    python profiles/tools/e2e_ab.py <variant.so|base> [config ...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import json, os, sys, numpy as np, torch
sys.path.insert(0, ROOT)
import bench
from paper_2007_03298_b200 import (BUF_GRADS, DsSyncEngine, OptimizerHyperparams, OptimizerKind, StrategyKind,
                                   SyncStrategy, Topology, WorldConfig)
name = sys.argv[1]
cfg = bench.CONFIGS[name]
W, N, d = cfg["W"], cfg["N"], cfg["d"]
s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, cfg["rect"])
e = DsSyncEngine(s, OptimizerKind(cfg["opt"]), d, OptimizerHyperparams(weight_decay=cfg["wd"]), "f32", 0)
e.quadratic_init(7, 4.0); e.quadratic_gradients(0, 1, 1.0, 0.5)
hg = torch.empty((W, d), dtype=torch.float32, pin_memory=True)
hw = torch.empty((W, d), dtype=torch.float32, pin_memory=True)
e.download_all(BUF_GRADS, hg)
for t in range(5): e.step_host(t, cfg["alpha"], hg, hw)
e.host_sync(); torch.cuda.synchronize()
import time
K = 20
t0 = time.perf_counter()
for t in range(5, 5 + K): e.step_host(t, cfg["alpha"], hg, hw)
e.host_sync()
dt = (time.perf_counter() - t0) / K
print(json.dumps({"variant": os.environ.get("DSS_LIB_VARIANT", "base").split("/")[-1], "config": name,
                  "e2e_iters_s": 1.0 / dt, "ms": dt * 1e3}))
'''.replace("ROOT", repr(ROOT))

if __name__ == "__main__":
    var = sys.argv[1]
    env = dict(os.environ)
    if var != "base":
        env["DSS_LIB_VARIANT"] = os.path.abspath(var)
    for c in sys.argv[2:] or ["c2"]:
        r = subprocess.run([sys.executable, "-c", CHILD, c], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or json.dumps({"variant": var, "config": c, "error": r.stderr[-600:]}), flush=True)
