"""Parity of the CUDA path (through the C-ABI) with the reference.

  f64 instantiation  vs the reference's own outputs (golden)   bit-exact
  f32 instantiation  vs the f32 restatement (oracle)           bit-exact
  f32                vs the f64 reference                      tolerance stated in-test
  full-size C2 rows  vs the oracle + size-independent properties
"""
import numpy as np
import pytest

from oracle.oracle import hparams
from paper_2007_03298_b200 import (BUF_GRADS, BUF_MOMENT1, BUF_MOMENT2, BUF_PARAMS, DivergenceError, DsSyncEngine,
                                   OptimizerHyperparams, OptimizerKind, OptimizerState, StrategyKind, SyncStrategy,
                                   Topology, WorkerState, WorldConfig, apply_step, sync_round)

pytestmark = pytest.mark.gpu

OPTS = {"vanilla-sgd": 0, "sgd-momentum": 1, "adam": 2, "adamw": 3}


def strategy(kind, W, N, rect=False, topo=Topology.RING):
    return SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, topo, WorldConfig(W, N), 1, rect)


def engine_for(kind, W, N, opt, d, wd=0.0, dtype="f64", path=0, rect=False):
    return DsSyncEngine(strategy(kind, W, N, rect), OptimizerKind(opt), d,
                        OptimizerHyperparams(weight_decay=wd), dtype, 0, path=path)


@pytest.mark.parametrize("path", [0, 1])
def test_golden_trajectories_bit_exact(cuda_device, golden, path):
    """run_training (quadratic, DS and BSP, 4 optimizers) replayed on the
    device from the reference's per-iteration gradients: every worker's f64
    params equal the reference's bit for bit after every iteration.  path=1
    routes every group through the cross-GPU two-shot kernels."""
    meta, a = golden
    for m in meta["trajectories"]:
        grads, params = a[m["key"] + "_grads"], a[m["key"] + "_params"]
        T, W, d = grads.shape
        with engine_for(m["kind"], W, m["N"], OPTS[m["opt"]], d, m["weight_decay"], "f64", path) as e:
            e.broadcast_row(BUF_PARAMS, a["quad_w0"])
            for t in range(T):
                e.upload_all(BUF_GRADS, grads[t])
                e.step(t, m["alpha"], check=True)
                got = e.download_all(BUF_PARAMS)
                assert np.array_equal(got, params[t]), (m["key"], t, np.abs(got - params[t]).max())


def test_trace_parity(cuda_device, golden):
    """run_training's IterationTrace (sync.cpp:430-458) on the device:
    global_mean_params bit-exact (ordered fold over all W workers), critical
    path / messages / simulated comm time exact, post-sync losses, their mean
    and the suboptimality within 1e-12 relative (fp64 device reduction in a
    parallel order, vs the reference's sequential dot)."""
    from paper_2007_03298_b200 import iteration_trace
    meta, a = golden
    mu = meta["quadratic"]["mu"]
    for m in meta["trajectories"]:
        key = m["key"]
        grads = a[key + "_grads"]
        tg, tl, ts = a[key + "_trace_gmean"], a[key + "_trace_loss"], a[key + "_trace_scalars"]
        T, W, d = grads.shape
        with engine_for(m["kind"], W, m["N"], OPTS[m["opt"]], d, m["weight_decay"], "f64") as e:
            e.set_optimum(a["quad_wstar"])
            e.broadcast_row(BUF_PARAMS, a["quad_w0"])
            for t in range(T):
                e.upload_all(BUF_GRADS, grads[t])
                out = e.step(t, m["alpha"], check=True)
                tr = iteration_trace(e, t, out, mu)
                assert np.array_equal(tr.global_mean_params, tg[t]), (key, t)
                np.testing.assert_allclose(tr.post_sync_loss, tl[t], rtol=1e-12, atol=0)
                assert tr.mean_post_sync_loss == pytest.approx(ts[t][0], rel=1e-12)
                assert tr.suboptimality == pytest.approx(ts[t][1], rel=1e-12)
                assert (tr.critical_path_steps, tr.total_messages) == (int(ts[t][2]), int(ts[t][3]))
                assert tr.simulated_comm_time == ts[t][4]


def test_metrics_csv_byte_identical(cuda_device, golden):
    """Device run -> IterationTrace (exact-order losses) -> metrics_csv is
    byte-identical to the reference's own metrics file for the same run
    (metrics.cpp:37-56, determinism contract acceptance.cpp:404-440)."""
    from paper_2007_03298_b200 import iteration_trace
    from paper_2007_03298_b200.metrics import metrics_csv
    meta, a = golden
    mu = meta["quadratic"]["mu"]
    for m in meta["trajectories"]:
        grads = a[m["key"] + "_grads"]
        T, W, d = grads.shape
        traces = []
        with engine_for(m["kind"], W, m["N"], OPTS[m["opt"]], d, m["weight_decay"], "f64") as e:
            e.set_optimum(a["quad_wstar"])
            e.broadcast_row(BUF_PARAMS, a["quad_w0"])
            for t in range(T):
                e.upload_all(BUF_GRADS, grads[t])
                out = e.step(t, m["alpha"], check=True)
                traces.append(iteration_trace(e, t, out, mu, exact=True))
        assert metrics_csv(traces) == m["metrics_csv"], m["key"]


def test_running_stats_tail_bit_exact(cuda_device, golden):
    """Running statistics (sync.cpp:193-213, 386-411): tiny-MLP (stats_dim =
    hidden) under Adam, DS W=4 groups of 2 and BSP W=4, replayed on the device
    from the reference's gradients and batch observations: the EMA update,
    then params ++ stats through the group (DS) / world (BSP) fold.  Params
    and running stats bit-exact after every iteration."""
    from paper_2007_03298_b200 import BUF_STATS, BUF_STATS_OBS
    meta, a = golden
    for m in meta["mlp"]:
        kind = m["kind"]
        g, obs, p, st = (a[f"mlp_{kind}_{n}"] for n in ("grads", "obs", "params", "stats"))
        T, W, dim = g.shape
        s = SyncStrategy(StrategyKind.DS_SYNC if kind == "ds" else StrategyKind.BSP, Topology.RING,
                         WorldConfig(W, m["N"]))
        with DsSyncEngine(s, OptimizerKind.ADAM, dim, OptimizerHyperparams(), "f64", 0,
                          stats_dim=m["stats_dim"]) as e:
            e.broadcast_row(BUF_PARAMS, a[f"mlp_{kind}_w0"])
            for t in range(T):
                e.upload_all(BUF_GRADS, g[t])
                e.upload_all(BUF_STATS_OBS, obs[t])
                e.running_stats_update()
                e.step(t, m["alpha"], check=True)
                assert np.array_equal(e.download_all(BUF_PARAMS), p[t]), (kind, t)
                assert np.array_equal(e.download_all(BUF_STATS), st[t]), (kind, t)


def test_sync_round_with_running_stats(cuda_device, oracle):
    """sync_round averages params ++ running_stats as one payload
    (sync.cpp:203-213): equal to the fold of the concatenated rows."""
    rng = np.random.default_rng(4)
    for W, N in ((4, 2), (9, 3), (16, 16)):
        d, sd = 33, 5
        workers = [WorkerState(k, rng.standard_normal(d), running_stats=rng.standard_normal(sd)) for k in range(W)]
        cat = np.stack([np.concatenate([w.params, w.running_stats]) for w in workers])
        kind = 0 if N == W else 1
        oracle.sync_round(W, N, 1, cat, kind=kind)
        sync_round(workers, strategy("ds" if kind else "bsp", W, N), 1)
        got = np.stack([np.concatenate([w.params, w.running_stats]) for w in workers])
        assert np.array_equal(got, cat)


def test_c1_logistic_bit_exact(cuda_device, golden):
    """Config C1 (4 workers, 2 groups of 2, logistic d=20, SGD, step-decay lr,
    300 iterations) on the device: bit-exact every iteration."""
    meta, a = golden
    for m in meta["c1"]:
        kind, tag = m["kind"], m["tag"]
        grads, params, alphas = a[f"{tag}_grads"], a[f"{tag}_params"], a[f"{tag}_alphas"]
        T, W, d = grads.shape
        with engine_for(kind, W, m["N"], 0, d) as e:
            for t in range(T):
                e.upload_all(BUF_GRADS, grads[t])
                e.step(t, float(alphas[t]))
                if t % 25 == 24 or t == T - 1:
                    assert np.array_equal(e.download_all(BUF_PARAMS), params[t]), (kind, t)
            e.check()


def test_apply_step_golden(cuda_device, golden):
    """apply_step (optim.cpp:46-98) on the device vs the reference, bit-exact,
    including the hand values of test_optim.cpp."""
    meta, a = golden
    for c in meta["apply_step"]["cases"]:
        j = c["id"]
        kind = OptimizerKind(OPTS[c["opt"]])
        st = OptimizerState(kind, OptimizerHyperparams(alpha=c["alpha"], weight_decay=c["weight_decay"]),
                            a[f"c{j}_m1"], a[f"c{j}_m2"], c["step_count"])
        r = apply_step(st, a[f"c{j}_w"], a[f"c{j}_g"])
        assert np.array_equal(r.params, a[f"c{j}_w_out"]), c
        assert r.state.step_count == c["step_count_out"]
        if kind != OptimizerKind.VANILLA_SGD:
            assert np.array_equal(r.state.first_moment, a[f"c{j}_m1_out"])
        if kind in (OptimizerKind.ADAM, OptimizerKind.ADAMW):
            assert np.array_equal(r.state.second_moment, a[f"c{j}_m2_out"])
    with pytest.raises(ValueError):
        apply_step(OptimizerState(hp=OptimizerHyperparams(alpha=-0.1)), [1.0], [1.0])
    with pytest.raises(RuntimeError):  # optim.cpp:96, test_optim.cpp:109-112
        apply_step(OptimizerState(hp=OptimizerHyperparams(alpha=1e308)), [1e308], [-1.0])


def test_sync_round_golden(cuda_device, golden):
    """sync_round (sync.cpp:268-282) on the device: bit-exact means, same
    outcome counts, optimizer state untouched (it is never passed)."""
    meta, a = golden
    for m in meta["sync_rounds"]:
        w = a[f"s{m['id']}_in"]
        workers = [WorkerState(k, w[k].copy()) for k in range(m["W"])]
        s = SyncStrategy(StrategyKind(m["kind"]), Topology(m["topology"]), WorldConfig(m["W"], m["N"]),
                         m["num_servers"])
        out = sync_round(workers, s, m["t"])
        assert np.array_equal(np.stack([x.params for x in workers]), a[f"s{m['id']}_out"]), m
        assert (out.critical_path_steps, out.total_messages) == (m["critical_path_steps"], m["total_messages"])
    with pytest.raises(ValueError):  # test_sync.cpp:210
        sync_round([WorkerState(k, np.zeros(3)) for k in range(4)], strategy("ds", 9, 3), 0)


CASES = [("ds", 4, 2, False), ("ds", 9, 3, False), ("ds", 16, 4, False), ("ds", 8, 2, True), ("ds", 32, 4, True),
         ("ds", 64, 8, False), ("ds", 6, 6, False), ("ds", 25, 5, False), ("ds", 35, 5, True), ("ds", 12, 12, False),
         ("bsp", 8, 8, False), ("bsp", 3, 3, False), ("bsp", 32, 32, False), ("bsp", 13, 13, False)]


@pytest.mark.parametrize("kind,W,N,rect", CASES)
@pytest.mark.parametrize("opt", [0, 1, 2, 3])
def test_f32_bit_exact_vs_restatement(cuda_device, oracle, kind, W, N, rect, opt):
    """fp32 kernels == the fp32 restatement of the reference (same op order,
    constants rounded once from double), bit for bit, ragged d."""
    rng = np.random.default_rng(W * 10 + opt)
    d = 1000 + 13
    wd = 0.01 if opt in (1, 3) else 0.0
    for path in (0, 1):
        w = rng.standard_normal((W, d)).astype(np.float32)
        m1, m2 = np.zeros_like(w), np.zeros_like(w)
        steps = np.zeros(W, np.int64)
        with engine_for(kind, W, N, opt, d, wd, "f32", path, rect) as e:
            e.upload_all(BUF_PARAMS, w)
            for t in range(4):
                g = rng.standard_normal((W, d)).astype(np.float32)
                alpha = 0.05 if opt < 2 else 0.01
                e.upload_all(BUF_GRADS, g)
                e.step(t, alpha, check=True)
                if kind == "ds":
                    rc = oracle.ds_step(W, N, t, opt, hparams(weight_decay=wd), alpha, steps, w, g, m1, m2, rect)
                else:
                    rc = oracle.bsp_step(t, opt, hparams(weight_decay=wd), alpha, steps, w, g, m1, m2)
                assert rc[0] == 0
                steps += 1
                assert np.array_equal(e.download_all(BUF_PARAMS), w), (t, path)
            if opt >= 1:
                assert np.array_equal(e.download_all(BUF_MOMENT1), m1)
            if opt >= 2:
                assert np.array_equal(e.download_all(BUF_MOMENT2), m2)


@pytest.mark.parametrize("kind,W,N", [("ds", 1, 1), ("bsp", 1, 1), ("ds", 4, 2), ("ds", 4, 4), ("bsp", 2, 2)])
@pytest.mark.parametrize("d", [1, 3, 63, 64, 65, 257])
def test_edge_shapes_vs_restatement(cuda_device, oracle, kind, W, N, d):
    """Edge shapes: a single worker, a single full group, rows shorter than
    one 16-B vector and around the 64-element padding; f32 AdamW with decay
    (the most state) and SGD, batched and single steps, bit for bit."""
    for opt in (0, 3):
        rng = np.random.default_rng(d * 7 + W + opt)
        wd = 0.01 if opt == 3 else 0.0
        w = rng.standard_normal((W, d)).astype(np.float32)
        m1, m2 = np.zeros_like(w), np.zeros_like(w)
        steps = np.zeros(W, np.int64)
        g = rng.standard_normal((W, d)).astype(np.float32)
        alphas = [0.05, 0.02, 0.01]
        with engine_for(kind, W, N, opt, d, wd, "f32") as e:
            e.upload_all(BUF_PARAMS, w)
            e.upload_all(BUF_GRADS, g)
            e.steps(0, alphas, check=True)  # the one-launch batch
            e.step(3, 0.01, check=True)     # and a single step
            for t, alpha in enumerate(alphas + [0.01]):
                if kind == "ds":
                    rc = oracle.ds_step(W, N, t, opt, hparams(weight_decay=wd), alpha, steps, w, g.copy(), m1, m2)
                else:
                    rc = oracle.bsp_step(t, opt, hparams(weight_decay=wd), alpha, steps, w, g.copy(), m1, m2)
                assert rc[0] == 0
                steps += 1
            assert np.array_equal(e.download_all(BUF_PARAMS), w), (kind, W, N, d, opt)
            if opt:
                assert np.array_equal(e.download_all(BUF_MOMENT2), m2)


def test_f32_vs_f64_reference_tolerance(cuda_device, golden):
    """fp32 device params vs the fp64 reference on identical synthetic inputs.
    Tolerance (north star): max relative error <= 1e-6 with a magnitude floor
    of 1 (|x - ref| / max(|ref|, 1)) for SGD / momentum; Adam(W) divides by
    sqrt(v) and amplifies fp32 rounding, so it is held to 1e-5 (SURVEY 8(c)
    measured 2e-6 at T=100)."""
    meta, a = golden
    for m in meta["trajectories"]:
        grads, params = a[m["key"] + "_grads"], a[m["key"] + "_params"]
        T, W, d = grads.shape
        with engine_for(m["kind"], W, m["N"], OPTS[m["opt"]], d, m["weight_decay"], "f32") as e:
            e.broadcast_row(BUF_PARAMS, a["quad_w0"].astype(np.float32))
            for t in range(T):
                e.upload_all(BUF_GRADS, grads[t].astype(np.float32))
                e.step(t, m["alpha"])
            got = e.download_all(BUF_PARAMS).astype(np.float64)
        ref = params[T - 1]
        err = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0))
        tol = 1e-6 if m["opt"] in ("vanilla-sgd", "sgd-momentum") else 1e-5
        assert err <= tol, (m["key"], err)


def test_quadratic_gradient_kernel(cuda_device, oracle):
    """Synthetic gradients (problems.cpp:173-193, A = mu*I) vs the oracle.
    SplitMix64 integers are exact; the device's fp64 log/cos may differ from
    glibc by an ulp, so f64 is held to 4e-16 relative of the noise scale and
    f32 (rounded once from the f64 noise) to 1 ulp."""
    W, N, d, seed, mu, sigma = 4, 2, 4099, 1, 1.0, 0.5
    rng = np.random.default_rng(3)
    for dtype, np_t in (("f64", np.float64), ("f32", np.float32)):
        wstar = rng.standard_normal(d).astype(np_t)
        w = rng.standard_normal((W, d)).astype(np_t)
        with engine_for("ds", W, N, 0, d, dtype=dtype) as e:
            e.set_optimum(wstar)
            e.upload_all(BUF_PARAMS, w)
            for t in (0, 5):
                e.quadratic_gradients(t, seed, mu, sigma)
                got = e.download_all(BUF_GRADS)
                want = oracle.quadratic_grad(0, t, seed, mu, sigma, w, wstar)
                if dtype == "f64":
                    assert np.max(np.abs(got - want)) <= 4e-16 * 8 * sigma
                    assert np.mean(got == want) > 0.99
                else:
                    ulp = np.spacing(np.abs(want).astype(np.float32))
                    assert np.all(np.abs(got - want) <= ulp)
                    assert np.mean(got == want) > 0.999


def test_quadratic_init(cuda_device, golden):
    """w* and w0 (problems.cpp:157-165) on the device vs the reference."""
    meta, a = golden
    q = meta["quadratic"]
    with engine_for("ds", 4, 2, 0, q["d"]) as e:
        e.quadratic_init(q["problem_seed"], q["delta0"])
        w = e.download_all(BUF_PARAMS)
    for k in range(4):
        np.testing.assert_allclose(w[k], a["quad_w0"], rtol=0, atol=1e-14)


def test_divergence_reports_rank_and_iteration(cuda_device, oracle):
    """DivergenceError(rank, iteration) with the reference's precedence:
    earliest iteration, local step before group sync, lowest rank."""
    W, N, d = 4, 2, 77
    with engine_for("ds", W, N, 0, d) as e:
        e.upload_all(BUF_PARAMS, np.ones((W, d)))
        g = np.ones((W, d))
        e.upload_all(BUF_GRADS, g)
        for t in range(3):
            e.step(t, 0.1)
        g[3, 5] = np.inf
        g[2, 70] = np.nan
        e.upload_all(BUF_GRADS, g)
        e.step(3, 0.1)
        e.step(4, 0.1)
        with pytest.raises(DivergenceError) as ex:
            e.check()
        assert ex.value.rank == 2 and ex.value.iteration == 3
        assert "worker 2 diverged at iteration 3: apply_step" in str(ex.value)
    # collective overflow -> members[0] of the group (sync.cpp:233-235)
    w = np.full((W, d), 1.7e308)
    w[:2] = 1.0
    with engine_for("ds", W, N, 0, d) as e:
        e.upload_all(BUF_PARAMS, w)
        e.upload_all(BUF_GRADS, np.zeros((W, d)))
        with pytest.raises(DivergenceError) as ex:
            e.step(0, 0.1, check=True)
        assert ex.value.rank == 2 and "ring_allreduce_avg: non-finite" in str(ex.value)
    # runaway learning rate (test_sync.cpp:298-317)
    with engine_for("ds", W, N, 0, d) as e:
        e.upload_all(BUF_PARAMS, np.ones((W, d)))
        with pytest.raises(DivergenceError) as ex:
            for t in range(400):
                e.set_optimum(np.zeros(d))
                e.quadratic_gradients(t, 3, 1.0, 0.0)
                e.step(t, 10.0)
            e.check()
        assert 0 <= ex.value.rank < 4 and 0 <= ex.value.iteration < 400


def _torch_view(e, buffer, rank, n):
    import torch

    class _Arr:
        def __init__(self, ptr, n, typestr):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}

    typestr = "<f4" if e.dtype == np.float32 else "<f8"
    return torch.as_tensor(_Arr(e.device_ptr(buffer, rank), n, typestr), device="cuda")


def test_c2_full_size_rows_vs_oracle(cuda_device, oracle):
    """Config C2 at full size on one GPU (W=8, groups of 2 then 4,
    d=25,000,000 fp32, SGD): two iterations (block + comb) bit-exact vs the
    oracle, every group bit-identical inside, global mean of a sync-only
    round preserved (size-independent properties)."""
    import torch
    W, N, d = 8, 2, 25_000_000
    s = strategy("ds", W, N, rect=True)
    rng = np.random.default_rng(5)
    w = rng.standard_normal((W, d), dtype=np.float32)
    g = (0.01 * rng.standard_normal((W, d), dtype=np.float32)).astype(np.float32)
    with DsSyncEngine(s, OptimizerKind.VANILLA_SGD, d, None, "f32", 0) as e:
        e.upload_all(BUF_PARAMS, w)
        e.upload_all(BUF_GRADS, g)
        steps = np.zeros(W, np.int64)
        for t in range(2):
            e.step(t, 0.05, check=True)
            oracle.ds_step(W, N, t, 0, hparams(), 0.05, steps, w, g, rect=True)
            steps += 1
            for grp in ([[0, 1], [2, 3], [4, 5], [6, 7]] if t == 0 else [[0, 2, 4, 6], [1, 3, 5, 7]]):
                v0 = _torch_view(e, BUF_PARAMS, grp[0], d)
                for r in grp[1:]:
                    assert torch.equal(v0, _torch_view(e, BUF_PARAMS, r, d))
        assert np.array_equal(e.download_all(BUF_PARAMS), w)
        before = torch.stack([_torch_view(e, BUF_PARAMS, k, d).double() for k in range(W)]).mean(0)
        e.sync_round(2)
        after = torch.stack([_torch_view(e, BUF_PARAMS, k, d).double() for k in range(W)]).mean(0)
        assert torch.max(torch.abs(after - before)).item() < 1e-6


@pytest.mark.parametrize("kind,W,N,d,opt,dtype", [
    ("ds", 16, 4, 3001, 3, "f32"),      # 192 KB per array: resident-grid multi-iteration kernel
    ("ds", 4, 2, 50001, 1, "f32"),      # 800 KB: resident grid, momentum
    ("ds", 16, 4, 40001, 1, "f64"),     # 5 MB: one launch per iteration
    ("ds", 8, 2, 30001, 0, "f32"),      # rectangular C2 shape, 960 KB
    ("bsp", 8, 8, 20001, 2, "f32"),     # BSP fold + step, 640 KB
    ("bsp", 4, 4, 9001, 3, "f64"),
])
def test_batched_steps_equal_single_steps(cuda_device, kind, W, N, d, opt, dtype):
    """dss_steps(t0, alphas) == the same iterations one dss_step at a time
    (the batched path runs them in one launch up to 4 MB per array)."""
    rng = np.random.default_rng(9)
    ft = np.float64 if dtype == "f64" else np.float32
    w = rng.standard_normal((W, d)).astype(ft)
    g = rng.standard_normal((W, d)).astype(ft)
    alphas = np.linspace(0.01, 0.05, 7)
    outs = []
    for batched in (False, True):
        with engine_for(kind, W, N, opt, d, 0.01, dtype, rect=(kind == "ds" and W != N * N)) as e:
            e.upload_all(BUF_PARAMS, w)
            e.upload_all(BUF_GRADS, g)
            if batched:
                e.steps(0, alphas, check=True)
            else:
                for t, a_t in enumerate(alphas):
                    e.step(t, float(a_t))
            outs.append((e.download_all(BUF_PARAMS), e.step_count(W - 1)))
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1] == len(alphas)


@pytest.mark.parametrize("kind,W,N", [("ds", 4, 2), ("ds", 9, 3), ("bsp", 4, 4)])
@pytest.mark.parametrize("opt", [0, 1, 2, 3])
def test_small_world_multi_iteration_kernel(cuda_device, oracle, kind, W, N, opt):
    """Tiny worlds (C1-sized): dss_steps runs all n iterations in one CTA
    (one launch).  Bit-exact vs the f32 and f64 restatement iteration by
    iteration semantics, incl. per-iteration learning rates and Adam bias
    corrections."""
    rng = np.random.default_rng(W * 7 + opt)
    d = 20
    wd = 0.01 if opt in (1, 3) else 0.0
    for dtype, npt in (("f32", np.float32), ("f64", np.float64)):
        w = rng.standard_normal((W, d)).astype(npt)
        g = rng.standard_normal((W, d)).astype(npt)
        alphas = np.array([0.05, 0.05, 0.025, 0.025, 0.0125, 0.01, 0.01], dtype=np.float64)
        with engine_for(kind, W, N, opt, d, wd, dtype) as e:
            e.upload_all(BUF_PARAMS, w)
            e.upload_all(BUF_GRADS, g)
            e.steps(3, alphas, check=True)
            got = e.download_all(BUF_PARAMS)
            assert e.step_count(0) == len(alphas)
        ref = w.copy()
        m1, m2 = np.zeros_like(ref), np.zeros_like(ref)
        steps = np.zeros(W, np.int64)
        for i, a_i in enumerate(alphas):
            if kind == "ds":
                rc = oracle.ds_step(W, N, 3 + i, opt, hparams(weight_decay=wd), float(a_i), steps, ref, g, m1, m2)
            else:
                rc = oracle.bsp_step(3 + i, opt, hparams(weight_decay=wd), float(a_i), steps, ref, g, m1, m2)
            assert rc[0] == 0
            steps += 1
        assert np.array_equal(got, ref), (dtype, kind, opt)


@pytest.mark.parametrize("W,N,rect,opt,dtype,d", [(8, 2, True, 1, "f32", 50_021), (4, 2, False, 3, "f64", 9_000),
                                                   (16, 4, False, 0, "f32", 70_001), (8, 8, False, 2, "f32", 777)])
def test_step_host_pipeline(cuda_device, oracle, W, N, rect, opt, dtype, d):
    """dss_step_host: grads fed from host, params returned to host every
    iteration with the copies pipelined across calls (element-chunked on one
    GPU: each chunk's copy-in, step and copy-out overlap).  Iteration t's
    params are complete once call t+1 (or host_sync) returns; every one is
    bit-exact vs the oracle, and a plain dss_step right after the pipeline
    sees the same state."""
    import torch
    rng = np.random.default_rng(12)
    T = 6
    ft = np.float64 if dtype == "f64" else np.float32
    tt = torch.float64 if dtype == "f64" else torch.float32
    w = rng.standard_normal((W, d)).astype(ft)
    grads = [rng.standard_normal((W, d)).astype(ft) for _ in range(T + 1)]
    hg = [torch.from_numpy(g).pin_memory() for g in grads]
    hp = [torch.empty((W, d), dtype=tt).pin_memory() for _ in range(T)]
    with engine_for("ds", W, N, opt, d, 1e-4, dtype, rect=rect) as e:
        e.upload_all(BUF_PARAMS, w)
        for t in range(T):
            e.step_host(t, 0.05, hg[t], hp[t])
        e.upload_all(BUF_GRADS, grads[T])  # ordered after the pipeline's last copies
        e.step(T, 0.05)
        last = e.download_all(BUF_PARAMS)
        e.host_sync()
    ref = w.copy()
    m1 = np.zeros_like(ref) if opt else None
    m2 = np.zeros_like(ref) if opt >= 2 else None
    steps = np.zeros(W, np.int64)
    for t in range(T + 1):
        oracle.ds_step(W, N, t, opt, hparams(weight_decay=1e-4), 0.05, steps, ref, grads[t], m1, m2, rect)
        steps += 1
        if t < T:
            assert np.array_equal(hp[t].numpy(), ref), t
    assert np.array_equal(last, ref)


def test_timing_and_launch_accounting(cuda_device):
    with engine_for("ds", 8, 2, 0, 1 << 20, dtype="f32", rect=True) as e:
        e.enable_timing(True)
        n0 = e.launch_count
        for t in range(4):
            e.step(t, 0.01)
        tot, n, mx = e.kernel_times()
        assert n == 4 and e.launch_count - n0 == 4 and 0 < mx <= tot


@pytest.mark.parametrize("kind,W,N,d,rect", [("ds", 8, 2, 300, True), ("ds", 9, 3, 700, False),
                                             ("bsp", 4, 4, 1500, False)])
@pytest.mark.parametrize("opt", [0, 3])
def test_small_world_wide_cta(cuda_device, oracle, kind, W, N, d, rect, opt):
    """The one-CTA batch kernel's 512-thread variant (more than 256 element
    vectors per parity, still <= 32 KB per array): bit-exact vs the
    restatement, f32 and f64."""
    rng = np.random.default_rng(d + opt)
    wd = 0.01 if opt == 3 else 0.0
    for dtype, npt in (("f32", np.float32), ("f64", np.float64)):
        w = rng.standard_normal((W, d)).astype(npt)
        g = rng.standard_normal((W, d)).astype(npt)
        alphas = np.array([0.05, 0.04, 0.03, 0.02, 0.01], dtype=np.float64)
        with engine_for(kind, W, N, opt, d, wd, dtype, rect=rect) as e:
            e.upload_all(BUF_PARAMS, w)
            e.upload_all(BUF_GRADS, g)
            e.steps(0, alphas, check=True)
            got = e.download_all(BUF_PARAMS)
        ref = w.copy()
        m1, m2 = np.zeros_like(ref), np.zeros_like(ref)
        steps = np.zeros(W, np.int64)
        for i, a_i in enumerate(alphas):
            if kind == "ds":
                rc = oracle.ds_step(W, N, i, opt, hparams(weight_decay=wd), float(a_i), steps, ref, g, m1, m2,
                                    rect=rect)
            else:
                rc = oracle.bsp_step(i, opt, hparams(weight_decay=wd), float(a_i), steps, ref, g, m1, m2)
            assert rc[0] == 0
            steps += 1
        assert np.array_equal(got, ref), (dtype, kind, opt)


def test_guard_bands_see_no_out_of_bounds_writes(cuda_device):
    """compute-sanitizer is closed on this pool: the library's guard bands
    (DSS_GUARD_BYTES) frame every device allocation, and a workload touching
    every single-GPU kernel must leave all of them intact."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DSS_GUARD_BYTES=str(1 << 20))
    p = subprocess.run([sys.executable, os.path.join(root, "profiles", "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "SANITIZE-RUN OK" in p.stdout and "guard bands on, 0 bytes overwritten" in p.stdout, p.stdout


def test_guard_bands_catch_a_stray_write(cuda_device):
    """The detector itself: a write just past a row buffer is reported."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2007_03298_b200 import *
s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(4, 2))
e = DsSyncEngine(s, OptimizerKind.VANILLA_SGD, 1000, None, "f32", 0)
assert e.check_guards() == 0
class A:
    def __init__(self, p):
        self.__cuda_array_interface__ = {"shape": (4,), "typestr": "<f4", "data": (p, False), "version": 3}
end = e.device_ptr(BUF_PARAMS, 3) + 4 * e.row_stride  # one past the last row of the params buffer
torch.as_tensor(A(end), device="cuda").fill_(1.0)
torch.cuda.synchronize()
try:
    e.check_guards()
    print("MISSED")
except RuntimeError as ex:
    print("CAUGHT", ex)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DSS_GUARD_BYTES="4096")
    p = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "CAUGHT guard bands overwritten: 16 bytes" in p.stdout, p.stdout
