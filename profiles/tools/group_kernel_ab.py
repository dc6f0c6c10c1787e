"""A/B of library variants on the single-GPU group / BSP kernels.

    python profiles/tools/group_kernel_ab.py <variant.so|base> [config ...]

Runs in a subprocess per variant (DSS_LIB_VARIANT), DS and BSP for each
config at its full size, 3 warm-up + K timed iterations, CUDA-event time of
the whole step and of the dominant kernel; one JSON line per config."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import json, os, sys, numpy as np, torch
sys.path.insert(0, ROOT)
import bench
from paper_2007_03298_b200 import (DsSyncEngine, OptimizerHyperparams, OptimizerKind, StrategyKind, SyncStrategy,
                                   Topology, WorldConfig)
name, K = sys.argv[1], int(sys.argv[2])
cfg = bench.CONFIGS[name]
W, N, d = cfg["W"], cfg["N"], cfg["d"]
out = {"variant": os.environ.get("DSS_LIB_VARIANT", "base"), "config": name}
for kind, key in ((StrategyKind.DS_SYNC, "ds"), (StrategyKind.BSP, "bsp")):
    s = SyncStrategy(kind, Topology.RING, WorldConfig(W, N if kind == StrategyKind.DS_SYNC else W), 1,
                     cfg["rect"] and kind == StrategyKind.DS_SYNC)
    e = DsSyncEngine(s, OptimizerKind(cfg["opt"]), d, OptimizerHyperparams(weight_decay=cfg["wd"]), "f32", 0)
    e.quadratic_init(7, 4.0); e.quadratic_gradients(0, 1, 1.0, 0.5)
    for t in range(3): e.step(t, cfg["alpha"])
    torch.cuda.synchronize()
    e.enable_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for t in range(3, 3 + K): e.step(t, cfg["alpha"])
    b.record(); torch.cuda.synchronize()
    kinds = e.kernel_times_by_kind(); e.check()
    ms = a.elapsed_time(b) / K
    kms = max(v[0] for v in kinds.values()) / K
    byts = W * d * bench.BYTES_PER_ELEM[cfg["opt"]]
    out[key] = {"ms": round(ms, 4), "kernel_ms": round(kms, 4), "kernel_gbs": round(byts / kms / 1e6, 1)}
    e.close(); del e; torch.cuda.synchronize()
print(json.dumps(out), flush=True)
'''.replace("ROOT", repr(ROOT))

if __name__ == "__main__":
    var = sys.argv[1]
    cfgs = sys.argv[2:] or ["c4slice"]
    env = dict(os.environ)
    if var != "base":
        env["DSS_LIB_VARIANT"] = os.path.abspath(var)
    for c in cfgs:
        r = subprocess.run([sys.executable, "-c", CHILD, c, "10"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or json.dumps({"variant": var, "config": c, "error": r.stderr[-800:]}), flush=True)
