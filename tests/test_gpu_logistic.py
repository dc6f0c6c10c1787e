"""Config C1 end to end on the device: logistic regression with the batch
sampled on the GPU (sample_batch, sync.cpp:153-179), the gradient computed
on the GPU (LogisticProblem::stochastic_gradient, problems.cpp:265-290) and
the DS-Sync / BSP step, against the reference's own recorded run
(tests/golden: c1_* replacement sampling, c1e_* epoch sampling).

  batch indices        bit-exact (integer SplitMix64 streams)
  gradient, one call   |err| <= 1e-14 * (1 + |g|): the sigmoid's exp is
                       libdevice's, not glibc's (<= 1 ulp apart)
  300-iteration run    params within 1e-12 * (1 + |w|) of the reference
"""
import numpy as np
import pytest

from paper_2007_03298_b200 import (BUF_GRADS, BUF_PARAMS, DivergenceError, DsSyncEngine, OptimizerHyperparams,
                                   OptimizerKind, SamplingMode, StrategyKind, SyncStrategy, Topology, WorldConfig,
                                   logistic_dataset)

pytestmark = pytest.mark.gpu

L2, B, RUN_SEED = 0.05, 8, 1


def engine(kind, W, N, dtype="f64", opt=0):
    s = SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING, WorldConfig(W, N))
    return DsSyncEngine(s, OptimizerKind(opt), 20, OptimizerHyperparams(), dtype, 0)


@pytest.fixture(scope="module")
def c1_data():
    return logistic_dataset(11, 20, 2000)


def sampling_of(m):
    return SamplingMode.EPOCH if m["sampling"] == "epoch" else SamplingMode.REPLACEMENT


def test_c1_device_gradient_per_call(cuda_device, golden, c1_data):
    """Each iteration's gradient from the reference's own params: batches
    bit-exact, gradient within a few ulp."""
    meta, a = golden
    x, y = c1_data
    for m in meta["c1"]:
        tag = m["tag"]
        grads, params, batches = a[f"{tag}_grads"], a[f"{tag}_params"], a[f"{tag}_batches"]
        T, W, d = grads.shape
        exact = 0
        with engine(m["kind"], W, m["N"]) as e:
            e.logistic_setup(x, y, L2, B, sampling_of(m), RUN_SEED)
            for t in range(T):
                e.upload_all(BUF_PARAMS, np.zeros((W, d)) if t == 0 else params[t - 1])
                e.logistic_gradients(t)
                assert np.array_equal(e.logistic_batch(), batches[t]), (tag, t)
                g = e.download_all(BUF_GRADS)
                err = np.abs(g - grads[t])
                assert np.all(err <= 1e-14 * (1.0 + np.abs(grads[t]))), (tag, t, err.max())
                exact += int(np.array_equal(g, grads[t]))
            e.check()
        assert exact >= T // 10, (tag, exact)  # many iterations are bit-identical (110/300 on B200)


@pytest.mark.parametrize("batched", [False, True])
def test_c1_end_to_end_on_device(cuda_device, golden, c1_data, batched):
    """300 iterations with nothing from the host but the learning rates."""
    meta, a = golden
    x, y = c1_data
    for m in meta["c1"]:
        tag = m["tag"]
        params, alphas = a[f"{tag}_params"], a[f"{tag}_alphas"]
        T, W, d = params.shape
        with engine(m["kind"], W, m["N"]) as e:
            e.logistic_setup(x, y, L2, B, sampling_of(m), RUN_SEED)
            if batched:
                e.logistic_steps(0, alphas, check=True)
            else:
                for t in range(T):
                    e.logistic_gradients(t)
                    e.step(t, float(alphas[t]))
                    if t % 50 == 49:
                        w = e.download_all(BUF_PARAMS)
                        assert np.all(np.abs(w - params[t]) <= 1e-12 * (1.0 + np.abs(params[t]))), (tag, t)
                e.check()
            w = e.download_all(BUF_PARAMS)
            assert np.all(np.abs(w - params[-1]) <= 1e-12 * (1.0 + np.abs(params[-1]))), tag
            # full_loss (problems.cpp:292-305) in fp64 on the host
            z = x @ w.T
            ref = np.mean(np.logaddexp(0.0, -y[:, None] * z), axis=0) + 0.5 * L2 * np.sum(w * w, axis=1)
            for exact in (True, False):
                assert np.allclose(e.logistic_losses(exact=exact), ref, rtol=1e-12, atol=0), (tag, exact)


def test_c1_f32_context_tolerance(cuda_device, golden, c1_data):
    """f32 params: the gradient is computed in fp64 from them and stored as
    f32; the run stays within 1e-4 relative of the f64 reference."""
    meta, a = golden
    x, y = c1_data
    m = meta["c1"][0]
    params, alphas = a[f"{m['tag']}_params"], a[f"{m['tag']}_alphas"]
    W = params.shape[1]
    with engine(m["kind"], W, m["N"], "f32") as e:
        e.logistic_setup(x, y, L2, B, sampling_of(m), RUN_SEED)
        e.logistic_steps(0, alphas, check=True)
        w = e.download_all(BUF_PARAMS).astype(np.float64)
    assert np.allclose(w, params[-1], rtol=1e-4, atol=1e-5), np.abs(w - params[-1]).max()


def test_gradient_divergence_precedence(cuda_device, c1_data):
    """checked_gradient (sync.cpp:181-191): a non-finite batch loss is a
    DivergenceError at the gradient, reported before a later worker's step
    failure; an earlier worker's step failure is reported first (DS runs
    gradient + step per worker in rank order, sync.cpp:348-361)."""
    x, y = c1_data
    W, d = 4, 20
    w = np.zeros((W, d))
    w[2] = 1e200  # |w|^2 overflows in the batch loss; the gradient itself is finite
    with engine("ds", W, 2) as e:
        e.logistic_setup(x, y, L2, B, SamplingMode.REPLACEMENT, RUN_SEED)
        e.upload_all(BUF_PARAMS, w)
        e.logistic_gradients(0)
        e.step(0, 0.1)
        with pytest.raises(DivergenceError) as ex:
            e.check()
        assert ex.value.rank == 2 and ex.value.iteration == 0
        assert "worker 2 diverged at iteration 0: non-finite stochastic gradient" in str(ex.value)
    # rank 0's step overflows (runaway lr: l2 * w = 5 per element, times
    # 1e308) before rank 2's gradient is computed
    w2 = np.full((W, d), 100.0)
    w2[2] = 1e200
    with engine("ds", W, 2) as e:
        e.logistic_setup(x, y, L2, B, SamplingMode.REPLACEMENT, RUN_SEED)
        e.upload_all(BUF_PARAMS, w2)
        e.logistic_gradients(0)
        e.step(0, 1e308)
        with pytest.raises(DivergenceError) as ex:
            e.check()
        assert ex.value.rank == 0 and "apply_step" in str(ex.value)
    # BSP computes every gradient before the collective and the step
    with engine("bsp", W, W) as e:
        e.logistic_setup(x, y, L2, B, SamplingMode.REPLACEMENT, RUN_SEED)
        e.upload_all(BUF_PARAMS, w2)
        e.logistic_gradients(0)
        e.step(0, 1e308)
        with pytest.raises(DivergenceError) as ex:
            e.check()
        assert ex.value.rank == 2 and "non-finite stochastic gradient" in str(ex.value)


def test_logistic_setup_errors(cuda_device, c1_data):
    x, y = c1_data
    with engine("ds", 4, 2) as e:
        with pytest.raises(ValueError, match="setup has not been called"):
            e.logistic_gradients(0)
        with pytest.raises(ValueError, match="batch_size"):
            e.logistic_setup(x, y, L2, 0)
        with pytest.raises(ValueError, match="dataset smaller than worker count"):
            e.logistic_setup(x[:3], y[:3], L2, 2)
        e.logistic_setup(x, y, L2, B, SamplingMode.EPOCH, RUN_SEED)
        with pytest.raises(ValueError, match="iteration must be >= 0"):
            e.logistic_gradients(-1)


@pytest.mark.parametrize("kind,N,alpha,rank,what", [("ds", 2, 0.1, 2, "non-finite stochastic gradient"),
                                                     ("ds", 2, 1e308, 0, "apply_step"),
                                                     ("bsp", 4, 1e308, 2, "non-finite stochastic gradient")])
def test_fused_small_world_divergence(cuda_device, c1_data, kind, N, alpha, rank, what):
    """The one-CTA small-world path (dss_logistic_steps with n >= 2: sampling,
    gradient, step and fold in one kernel) latches the same errors."""
    x, y = c1_data
    w = np.full((4, 20), 100.0)
    w[2] = 1e200
    if alpha < 1:
        w[[0, 1, 3]] = 0.0
    with engine(kind, 4, N) as e:
        e.logistic_setup(x, y, L2, B, SamplingMode.REPLACEMENT, RUN_SEED)
        e.upload_all(BUF_PARAMS, w)
        with pytest.raises(DivergenceError) as ex:
            e.logistic_steps(0, [alpha, alpha], check=True)
        assert ex.value.rank == rank and ex.value.iteration == 0 and what in str(ex.value)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_one_cta_path_equals_per_launch_path(cuda_device, golden, c1_data, dtype):
    """The one-CTA small-world kernel (dss_logistic_steps, n >= 2) and one
    gradient launch + one step launch per iteration do the same additions
    in the same order: identical bits."""
    meta, a = golden
    x, y = c1_data
    for m in meta["c1"]:
        alphas = a[f"{m['tag']}_alphas"][:120]
        with engine(m["kind"], 4, m["N"], dtype) as e1, engine(m["kind"], 4, m["N"], dtype) as e2:
            for e in (e1, e2):
                e.logistic_setup(x, y, L2, B, sampling_of(m), RUN_SEED)
            e1.logistic_steps(0, alphas, check=True)
            for t, al in enumerate(alphas):
                e2.logistic_gradients(t)
                e2.step(t, float(al))
            e2.check()
            assert np.array_equal(e1.download_all(BUF_PARAMS), e2.download_all(BUF_PARAMS)), (m["tag"], dtype)
