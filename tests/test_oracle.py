"""Pin the oracle (oracle/dssync_oracle.c) before trusting it.

CPU only.  The f64 restatement must reproduce the reference's own outputs
bit for bit: the committed golden fixtures (made by the unmodified
reference, tests/golden/make_golden.py) and, when oracle/_ref was built
here, the live reference library on fresh random cases.
"""
import numpy as np
import pytest

from oracle.oracle import hparams

OPTS = {"vanilla-sgd": 0, "sgd-momentum": 1, "adam": 2, "adamw": 3}
K_DATA_GEN = 0x9e3779b97f4a7c15
K_INIT_PARAMS = 0xbf58476d1ce4e5b9
K_GRADIENT_NOISE = 0xa0761d6478bd642f


def test_splitmix_known_answer(oracle, golden):
    """test_rng.cpp:14-37: SplitMix64 seed 0 first output."""
    import ctypes as C
    s = C.c_uint64(0)
    assert oracle.lib.orc_next_u64(C.byref(s)) == 0xE220A8397B1DCDAF
    assert golden[0]["splitmix_seed0_first"] == "0xe220a8397b1dcdaf"


def test_gaussian_streams_match_reference(oracle, golden):
    meta, a = golden
    for rank in range(4):
        for t in range(3):
            got = oracle.gaussians(1, K_GRADIENT_NOISE, rank, t, 512)
            assert np.array_equal(got, a[f"noise_r{rank}_t{t}"])
    assert np.array_equal(oracle.gaussians(7, K_DATA_GEN, 1, 0, 512), a["wstar_stream"])
    assert np.array_equal(oracle.gaussians(7, K_INIT_PARAMS, 0, 0, 512), a["init_stream"])


def test_partition_matches_reference(oracle, golden):
    meta, _ = golden
    for c in meta["partitions"]["cases"]:
        assert oracle.partition(c["W"], c["N"], c["t"]) == c["groups"], c


def test_quadratic_init_matches_reference(oracle, golden):
    meta, a = golden
    q = meta["quadratic"]
    wstar, w0 = oracle.quadratic_init(q["problem_seed"], q["d"], q["delta0"])
    assert np.array_equal(wstar, a["quad_wstar"])
    assert np.array_equal(w0, a["quad_w0"])


def test_apply_step_matches_reference(oracle, golden):
    meta, a = golden
    for c in meta["apply_step"]["cases"]:
        j = c["id"]
        w = a[f"c{j}_w"][None].copy()
        m1 = a[f"c{j}_m1"][None].copy()
        m2 = a[f"c{j}_m2"][None].copy()
        rc, _ = oracle.apply_step(OPTS[c["opt"]], hparams(weight_decay=c["weight_decay"]), c["alpha"],
                                  [c["step_count"]], w, a[f"c{j}_g"][None].copy(), m1, m2)
        assert rc == 0
        assert np.array_equal(w[0], a[f"c{j}_w_out"]), c
        if c["opt"] != "vanilla-sgd":
            assert np.array_equal(m1[0], a[f"c{j}_m1_out"]), c
        if c["opt"] in ("adam", "adamw"):
            assert np.array_equal(m2[0], a[f"c{j}_m2_out"]), c


def test_hand_values(oracle):
    """test_optim.cpp:23-61 hand-checked numbers."""
    w = np.array([[1.0, 2.0]])
    oracle.apply_step(0, hparams(), 0.1, [0], w, np.array([[0.5, -1.0]]))
    assert w[0, 0] == pytest.approx(0.95, rel=1e-15) and w[0, 1] == pytest.approx(2.1, rel=1e-15)
    w, m1, m2 = np.array([[1.0]]), np.zeros((1, 1)), np.zeros((1, 1))
    oracle.apply_step(2, hparams(), 0.1, [0], w, np.array([[2.0]]), m1, m2)
    assert w[0, 0] == pytest.approx(0.9000000005, rel=1e-12)
    assert m1[0, 0] == pytest.approx(0.2, rel=1e-15) and m2[0, 0] == pytest.approx(0.004, rel=1e-15)


def _replay(oracle, meta_t, a, dtype=np.float64):
    key = meta_t["key"]
    grads, params = a[key + "_grads"], a[key + "_params"]
    T, W, d = grads.shape
    w = np.tile(a["quad_w0"], (W, 1)).astype(dtype)
    m1, m2 = np.zeros_like(w), np.zeros_like(w)
    steps = np.zeros(W, np.int64)
    hp = hparams(weight_decay=meta_t["weight_decay"])
    out = []
    for t in range(T):
        g = grads[t].astype(dtype)
        if meta_t["kind"] == "ds":
            rc = oracle.ds_step(W, meta_t["N"], t, OPTS[meta_t["opt"]], hp, meta_t["alpha"], steps, w, g, m1, m2)
        else:
            rc = oracle.bsp_step(t, OPTS[meta_t["opt"]], hp, meta_t["alpha"], steps, w, g, m1, m2)
        assert rc[0] == 0
        steps += 1
        out.append(w.copy())
    return out, params


def test_trajectories_match_reference(oracle, golden):
    """DS and BSP run_training trajectories (quadratic, 4 optimizers): bit-exact."""
    meta, a = golden
    for m in meta["trajectories"]:
        out, params = _replay(oracle, m, a)
        for t, w in enumerate(out):
            assert np.array_equal(w, params[t]), (m["key"], t)


def test_c1_logistic_matches_reference(oracle, golden):
    """Config C1 (acceptance.cpp:239-258) replayed from the reference's gradients."""
    meta, a = golden
    for m in meta["c1"]:
        kind, tag = m["kind"], m["tag"]
        grads, params, alphas = a[f"{tag}_grads"], a[f"{tag}_params"], a[f"{tag}_alphas"]
        T, W, d = grads.shape
        w = np.zeros((W, d))
        steps = np.zeros(W, np.int64)
        for t in range(T):
            if kind == "ds":
                rc = oracle.ds_step(W, m["N"], t, 0, hparams(), float(alphas[t]), steps, w, grads[t].copy())
            else:
                rc = oracle.bsp_step(t, 0, hparams(), float(alphas[t]), steps, w, grads[t].copy())
            assert rc[0] == 0
            assert np.array_equal(w, params[t]), (kind, t)


def test_sync_round_matches_reference(oracle, golden):
    meta, a = golden
    for m in meta["sync_rounds"]:
        w = a[f"s{m['id']}_in"].copy()
        rc, _ = oracle.sync_round(m["W"], m["N"], m["t"], w, kind=m["kind"])
        assert rc == 0
        assert np.array_equal(w, a[f"s{m['id']}_out"]), m


@pytest.mark.parametrize("opt", [0, 1, 2, 3])
def test_oracle_vs_live_reference(oracle, reference, opt):
    """Fresh random cases against the unmodified reference (built here)."""
    rng = np.random.default_rng(100 + opt)
    for W, N in [(4, 2), (9, 3), (16, 4), (4, 4)]:
        d = int(rng.integers(1, 90))
        wd = [0.0, 0.05][opt % 2]
        w = rng.standard_normal((W, d))
        m1, m2 = np.zeros((W, d)), np.zeros((W, d))
        wo, m1o, m2o = w.copy(), m1.copy(), m2.copy()
        steps = np.zeros(W, np.int64)
        for t in range(4):
            g = rng.standard_normal((W, d))
            alpha = float(rng.uniform(0.0, 0.2))
            rc_o = oracle.ds_step(W, N, t, opt, hparams(weight_decay=wd), alpha, steps, wo, g, m1o, m2o)
            rc_r = reference.ds_iteration(0, W, N, t, opt, reference.hp_array(weight_decay=wd), alpha, steps, w, g,
                                          m1, m2)
            assert rc_o[0] == 0 and rc_r[0] == 0
            assert np.array_equal(w, wo) and np.array_equal(m1, m1o) and np.array_equal(m2, m2o)


def test_oracle_divergence_matches_reference(oracle, reference):
    """A runaway step reports the same (rank, iteration) as DivergenceError."""
    W, N, d = 4, 2, 5
    w = np.ones((W, d))
    g = np.ones((W, d))
    g[2, 3] = np.inf
    wo = w.copy()
    rc_o, r_o, ph = oracle.ds_step(W, N, 3, 0, hparams(), 0.1, np.zeros(W, np.int64), wo, g.copy())
    rc_r, r_r, it_r = reference.ds_iteration(0, W, N, 3, 0, reference.hp_array(), 0.1, np.zeros(W, np.int64), w,
                                             g.copy())
    assert rc_o == 2 and rc_r == 2
    assert r_o == r_r == 2 and it_r == 3 and ph == 0
    # collective overflow: finite steps, infinite sum -> members[0] of that group
    w = np.full((W, d), 1.7e308)
    w[:2] = 1.0
    g = np.zeros((W, d))
    wo = w.copy()
    rc_o, r_o, ph = oracle.ds_step(W, N, 0, 0, hparams(), 0.1, np.zeros(W, np.int64), wo, g.copy())
    rc_r, r_r, it_r = reference.ds_iteration(0, W, N, 0, 0, reference.hp_array(), 0.1, np.zeros(W, np.int64), w,
                                             g.copy())
    assert rc_o == rc_r == 2 and r_o == r_r == 2 and ph == 1


def test_rect_extension_reduces_to_square(oracle):
    for n in (2, 3, 4):
        for t in range(4):
            assert oracle.partition(n * n, n, t, rect=True) == oracle.partition(n * n, n, t)
