"""Small, fast workload touching every single-GPU kernel of the library.
compute-sanitizer is closed on this pool, so out-of-bounds writes are
checked with the library's own guard bands instead:

    DSS_GUARD_BYTES=1048576 python profiles/tools/sanitize_run.py

(every device allocation framed by 1 MB of 0xA5 on both sides; every
engine's bands are verified with dss_check_guards before it is closed).

ds_group_kernel (group sizes 1/2/3/4/8 and the any-size path, SGD / momentum /
Adam / AdamW, f32 / f64), bsp_kernel (W = 2/4/8 and any W), the one-CTA and
cooperative-grid small_steps_kernel, the pull two-shot fold_kernel on one
device (path=1), sync_round, the running-stats tail, quadratic gradients and
init, the global mean and losses, and the logistic batch kernels.
Prints SANITIZE-RUN OK at the end."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2007_03298_b200 import (BUF_GRADS, BUF_PARAMS, BUF_STATS, BUF_STATS_OBS, DsSyncEngine,  # noqa: E402
                                   OptimizerHyperparams, OptimizerKind, StrategyKind, SyncStrategy, Topology,
                                   WorldConfig, logistic_dataset)


GUARDED = []


def strat(kind, W, N, rect=False):
    return SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING,
                        WorldConfig(W, N), 1, rect)


def run(kind, W, N, opt, d, dtype, rect=False, path=0, sd=0, steps=3):
    rng = np.random.default_rng(W * 131 + d)
    ft = np.float64 if dtype == "f64" else np.float32
    with DsSyncEngine(strat(kind, W, N, rect), OptimizerKind(opt), d, OptimizerHyperparams(weight_decay=0.01),
                      dtype, 0, path=path, stats_dim=sd) as e:
        e.upload_all(BUF_PARAMS, rng.standard_normal((W, d)).astype(ft))
        e.upload_all(BUF_GRADS, rng.standard_normal((W, d)).astype(ft))
        if sd:
            e.upload_all(BUF_STATS, rng.standard_normal((W, sd)).astype(ft))
            e.upload_all(BUF_STATS_OBS, rng.standard_normal((W, sd)).astype(ft))
            e.running_stats_update()
        for t in range(steps):
            e.step(t, 0.01)
        e.steps(steps, np.full(4, 0.01))  # batched path (one launch when the world is small)
        e.sync_round(steps + 4)
        e.quadratic_gradients(1, 3, 1.0, 0.5)
        e.global_mean()
        e.check()
        GUARDED.append(e.check_guards())


def main():
    for opt in range(4):
        for dtype in ("f32", "f64"):
            run("ds", 8, 2, opt, 30_011, dtype, rect=True)   # groups of 2 / 4
            run("ds", 9, 3, opt, 4_099, dtype)               # groups of 3
            run("ds", 64, 8, opt, 2_053, dtype)              # groups of 8
            run("bsp", 8, 8, opt, 20_011, dtype)             # bsp W=8
            run("bsp", 6, 6, opt, 5_003, dtype)              # bsp any W
    run("ds", 16, 4, 3, 10, "f32")                           # one-CTA small world
    run("ds", 16, 4, 1, 20_000, "f32")                       # cooperative resident grid
    run("ds", 12, 4, 1, 40_009, "f32", rect=True)            # any-size group path (groups of 3 / 4)
    run("ds", 8, 2, 2, 50_021, "f32", rect=True, path=1)     # pull two-shot fold on one device
    run("bsp", 4, 4, 0, 9_001, "f64", path=1)
    run("ds", 8, 2, 2, 1_001, "f32", rect=True, sd=6)        # running-stats tail
    with DsSyncEngine(strat("ds", 8, 2, True), OptimizerKind.SGD_MOMENTUM, 100_003, None, "f32", 0) as e:
        e.quadratic_init(7, 4.0)
        e.quadratic_gradients(0, 1, 1.0, 0.5)
        e.step(0, 0.05)
        e.quadratic_losses(1.0)
        e.check()
        GUARDED.append(e.check_guards())
    x, y = logistic_dataset(11, 20, 2000)
    for kind in ("ds", "bsp"):
        with DsSyncEngine(strat(kind, 4, 2 if kind == "ds" else 4), OptimizerKind.VANILLA_SGD, 20, None, "f64", 0) as e:
            e.logistic_setup(x, y, 0.05, 8, 0, 1)
            e.logistic_gradients(0)
            e.step(0, 0.5)
            e.logistic_steps(1, np.full(20, 0.5))
            e.logistic_losses()
            e.check()
            GUARDED.append(e.check_guards())
    print(f"SANITIZE-RUN OK ({len(GUARDED)} engines, guard bands "
          f"{'on' if os.environ.get('DSS_GUARD_BYTES') else 'off'}, {sum(GUARDED)} bytes overwritten)", flush=True)


if __name__ == "__main__":
    main()
