"""The tiny MLP with running statistics on the device (§8(f)3: the
gradient producer behind acceptance.cpp:328-402's sync rules), against the
reference's own recorded runs (tests/golden: mlp_ds_*, mlp_bsp_*; DS W=4
groups of 2 and BSP W=4, Adam, batch 2, replacement sampling).

  batch indices               bit-exact
  gradient / observation      |err| <= 1e-13 * (1 + |ref|) per call (device tanh)
  8 iterations with the EMA   params and running stats within 1e-11 * (1 + |ref|)
"""
import numpy as np
import pytest

from paper_2007_03298_b200 import (BUF_GRADS, BUF_PARAMS, BUF_STATS, BUF_STATS_OBS, DsSyncEngine,
                                   OptimizerHyperparams, OptimizerKind, SamplingMode, StrategyKind, SyncStrategy,
                                   Topology, WorldConfig, mlp_dataset)

pytestmark = pytest.mark.gpu


def engine(m, dtype="f64"):
    s = SyncStrategy(StrategyKind.DS_SYNC if m["kind"] == "ds" else StrategyKind.BSP, Topology.RING,
                     WorldConfig(m["W"], m["N"]))
    return DsSyncEngine(s, OptimizerKind.ADAM, m["dim"], OptimizerHyperparams(), dtype, 0,
                        stats_dim=m["stats_dim"])


def close(got, ref, tol):
    return np.all(np.abs(got - ref) <= tol * (1.0 + np.abs(ref)))


def test_mlp_gradient_per_call(cuda_device, golden):
    meta, a = golden
    for m in meta["mlp"]:
        k = m["kind"]
        p = m["problem"]
        x, y = mlp_dataset(p["seed"], p["d"], p["M"])
        grads, obs, params, batches = (a[f"mlp_{k}_grads"], a[f"mlp_{k}_obs"], a[f"mlp_{k}_params"],
                                       a[f"mlp_{k}_batches"])
        T, W, _ = grads.shape
        with engine(m) as e:
            e.mlp_setup(x, y, p["hidden"], m["batch"], SamplingMode.REPLACEMENT, m["run_seed"])
            for t in range(T):
                e.upload_all(BUF_PARAMS, np.tile(a[f"mlp_{k}_w0"], (W, 1)) if t == 0 else params[t - 1])
                e.mlp_gradients(t)
                assert np.array_equal(e.logistic_batch(), batches[t]), (k, t)
                assert close(e.download_all(BUF_GRADS), grads[t], 1e-13), (k, t)
                assert close(e.download_all(BUF_STATS_OBS), obs[t], 1e-13), (k, t)
            e.check()


def test_mlp_run_with_running_stats(cuda_device, golden):
    """gradient (+ observation) -> fold_running_stats EMA -> the DS / BSP
    step, whose fold carries the stats with the params (sync.cpp:193-213)."""
    meta, a = golden
    for m in meta["mlp"]:
        k = m["kind"]
        p = m["problem"]
        x, y = mlp_dataset(p["seed"], p["d"], p["M"])
        params, stats = a[f"mlp_{k}_params"], a[f"mlp_{k}_stats"]
        T = params.shape[0]
        with engine(m) as e:
            e.broadcast_row(BUF_PARAMS, a[f"mlp_{k}_w0"])
            e.mlp_setup(x, y, p["hidden"], m["batch"], SamplingMode.REPLACEMENT, m["run_seed"])
            for t in range(T):
                e.mlp_gradients(t)
                e.running_stats_update()
                e.step(t, m["alpha"])
            e.check()
            assert close(e.download_all(BUF_PARAMS), params[-1], 1e-11), k
            assert close(e.download_all(BUF_STATS), stats[-1], 1e-11), k


def test_mlp_setup_checks(cuda_device, golden):
    meta, _ = golden
    m = meta["mlp"][0]
    x, y = mlp_dataset(71, 4, 24)
    with engine(m) as e:
        with pytest.raises(ValueError, match="setup has not been called"):
            e.mlp_gradients(0)
        with pytest.raises(ValueError, match="hidden"):
            e.mlp_setup(x, y, 40, 2)
        with pytest.raises(ValueError, match="context dim"):
            e.mlp_setup(x, y, 5, 2)
        e.mlp_setup(x, y, 6, 2)
        with pytest.raises(ValueError, match="dss_logistic_setup has not been called"):
            e.logistic_gradients(0)
