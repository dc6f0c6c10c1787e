"""Generate the golden fixtures from the UNMODIFIED reference.

Runs only in the build container (needs /root/reference and oracle/_ref).
Every array here is produced by the reference library itself
(oracle/_ref/libdssync_ref.so = /root/reference/proj/src compiled as-is,
driven through its public API by oracle/ref_shim.cpp); the fixtures are
committed so the GPU box, which has no /root/reference, can check the CUDA
path bit for bit.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402

K_DATA_GEN = 0x9e3779b97f4a7c15
K_INIT_PARAMS = 0xbf58476d1ce4e5b9
K_GRADIENT_NOISE = 0xa0761d6478bd642f

OPTS = {"vanilla-sgd": 0, "sgd-momentum": 1, "adam": 2, "adamw": 3}


def partitions(R: Reference) -> dict:
    out = {"cases": [], "invalid": [], "mixing": []}
    for W, N in [(1, 1), (4, 2), (4, 4), (9, 3), (9, 9), (16, 4), (25, 5), (36, 6), (64, 8)]:
        for t in range(0, 11):
            out["cases"].append({"W": W, "N": N, "t": t, "groups": R.make_partition(W, N, t)})
            out["mixing"].append({"W": W, "N": N, "t": t, "mixing": R.check_mixing(W, N, t)})
    # test_schedule.cpp:103-113 plus the C2/C3 shapes
    for W, N in [(6, 2), (4, 3), (0, 0), (4, -2), (8, 2), (8, 4), (32, 4), (32, 8)]:
        try:
            R.make_partition(W, N, 0)
            msg = None
        except ValueError as e:
            msg = str(e)
        out["invalid"].append({"W": W, "N": N, "error": msg})
    try:
        R.make_partition(4, 2, -1)
        out["negative_t"] = None
    except ValueError as e:
        out["negative_t"] = str(e)
    return out


def apply_steps(R: Reference) -> dict:
    rng = np.random.default_rng(11)
    arrs = {}
    cases = []
    # hand values of test_optim.cpp:23-109 and random rows
    hand = [
        ("vanilla-sgd", 0.1, 0.0, 0, [1.0, 2.0], [0.5, -1.0]),
        ("vanilla-sgd", 0.1, 0.5, 0, [2.0], [1.0]),
        ("sgd-momentum", 0.1, 0.0, 0, [1.0], [1.0]),
        ("adam", 0.1, 0.0, 0, [1.0], [2.0]),
        ("adamw", 0.1, 0.1, 0, [1.0], [0.0]),
        ("adam", 0.1, 0.1, 0, [1.0], [0.0]),
        ("sgd-momentum", 0.0, 0.0, 0, [0.25, -0.5], [1.0, 1.0]),
    ]
    for i in range(12):
        opt = list(OPTS)[i % 4]
        d = int(rng.integers(1, 70))
        hand.append((opt, float(rng.uniform(0.001, 0.2)), [0.0, 0.01][i % 2], int(rng.integers(0, 20)),
                     rng.standard_normal(d).tolist(), rng.standard_normal(d).tolist()))
    for j, (opt, alpha, wd, sc, w, g) in enumerate(hand):
        w = np.array(w, np.float64)
        g = np.array(g, np.float64)
        d = w.size
        m1 = np.zeros(d) if sc == 0 else rng.standard_normal(d) * 0.1
        m2 = np.zeros(d) if sc == 0 else np.abs(rng.standard_normal(d)) * 0.01
        hp = R.hp_array(weight_decay=wd)
        arrs[f"c{j}_w"], arrs[f"c{j}_g"], arrs[f"c{j}_m1"], arrs[f"c{j}_m2"] = w.copy(), g.copy(), m1.copy(), m2.copy()
        rc, sc_out = R.apply_step(OPTS[opt], hp, alpha, sc, w, g, m1, m2)
        assert rc == 0, R.error()
        arrs[f"c{j}_w_out"], arrs[f"c{j}_m1_out"], arrs[f"c{j}_m2_out"] = w, m1, m2
        cases.append({"id": j, "opt": opt, "alpha": alpha, "weight_decay": wd, "step_count": sc,
                      "step_count_out": sc_out})
    return {"cases": cases}, arrs


def trajectories(R: Reference) -> tuple[dict, dict]:
    """run_training on the isotropic quadratic (A = mu*I), DS and BSP, with
    every per-iteration gradient recorded (the replay is verified against
    run_training itself)."""
    meta, arrs = [], {}
    d, mu, sigma, delta0, pseed, rseed, T = 37, 1.0, 0.5, 4.0, 7, 1, 6
    hp_by_opt = {"vanilla-sgd": (0.05, 0.0), "sgd-momentum": (0.05, 1e-4), "adam": (0.01, 0.0),
                 "adamw": (0.01, 0.01)}
    shapes = [("ds", 4, 2), ("ds", 9, 3), ("ds", 16, 4), ("bsp", 4, 4), ("bsp", 8, 8), ("ds", 4, 4)]
    for kind, W, N in shapes:
        for opt, (alpha, wd) in hp_by_opt.items():
            hp = R.hp_array(weight_decay=wd)
            grads, params, match, (tg, tl, ts, csv) = R.quadratic_run(1 if kind == "ds" else 0, 0, W, N, d, mu, sigma,
                                                                 delta0, pseed, rseed, T, OPTS[opt], hp, alpha,
                                                                 trace=True)
            assert match, f"replay != run_training for {kind} {W}x{N} {opt}"
            key = f"{kind}_{W}x{N}_{opt}"
            arrs[key + "_grads"] = grads
            arrs[key + "_params"] = params
            # run_training's IterationTrace per t (sync.cpp:430-458)
            arrs[key + "_trace_gmean"] = tg
            arrs[key + "_trace_loss"] = tl
            arrs[key + "_trace_scalars"] = ts
            meta.append({"key": key, "kind": kind, "W": W, "N": N, "opt": opt, "alpha": alpha,
                         "weight_decay": wd, "d": d, "T": T, "metrics_csv": csv})
    wstar, w0 = R.quadratic_init(pseed, d, mu, delta0)
    arrs["quad_wstar"], arrs["quad_w0"] = wstar, w0
    return {"trajectories": meta, "quadratic": {"d": d, "mu": mu, "sigma": sigma, "delta0": delta0,
                                                 "problem_seed": pseed, "run_seed": rseed}}, arrs


def logistic_c1(R: Reference) -> tuple[dict, dict]:
    """Config C1 (acceptance.cpp:239-258): W=4 groups of 2, logistic d=20
    M=2000 l2=0.05 seed 11, batch 8, vanilla SGD, step_decay_lr(1, 0.5, 75);
    replacement sampling (the default) and epoch sampling, with every
    sampled batch recorded."""
    T = 300
    hp = R.hp_array()
    arrs, meta = {}, []
    for kind, N, sampling in (("ds", 2, 0), ("bsp", 4, 0), ("ds", 2, 1), ("bsp", 4, 1)):
        tag = f"c1_{kind}" if sampling == 0 else f"c1e_{kind}"
        grads, params, alphas, batches, match = R.logistic_run(1 if kind == "ds" else 0, 4, N, 20, 2000, 0.05, 11,
                                                               1, 8, T, 0, hp, 1.0, 0.5, 75, sampling=sampling,
                                                               with_batches=True)
        assert match, "logistic replay != run_training"
        arrs[f"{tag}_grads"] = grads
        arrs[f"{tag}_params"] = params
        arrs[f"{tag}_alphas"] = alphas
        arrs[f"{tag}_batches"] = batches
        meta.append({"tag": tag, "kind": kind, "W": 4, "N": N, "d": 20, "T": T, "batch": 8,
                     "sampling": ["replacement", "epoch"][sampling]})
    return {"c1": meta}, arrs


def logistic_data(R: Reference) -> tuple[dict, dict]:
    """Pins for the host-side problem setup: y*x of the synthetic logistic
    data (the model sees the data only through these products), make_shards
    and epoch_order, all from the reference."""
    import hashlib
    arrs = {}
    arrs["logi_yx_small"] = R.logistic_yx(5, 6, 40)
    c1 = R.logistic_yx(11, 20, 2000)
    meta = {"c1_yx_sha256": hashlib.sha256(np.ascontiguousarray(c1).tobytes()).hexdigest(), "shards": [],
            "epoch_orders": []}
    for M, W, seed in ((2000, 4, 1), (10, 3, 7), (7, 7, 2), (1001, 16, 3)):
        idx, off = R.make_shards(M, W, seed)
        key = f"shards_{M}_{W}_{seed}"
        arrs[key + "_idx"], arrs[key + "_off"] = idx, off
        meta["shards"].append({"M": M, "W": W, "seed": seed, "key": key})
    idx, off = R.make_shards(2000, 4, 1)
    for rank, epoch in ((0, 0), (1, 3), (3, 7)):
        key = f"epoch_{rank}_{epoch}"
        arrs[key] = R.epoch_order(idx[off[rank]:off[rank + 1]], 1, rank, epoch)
        meta["epoch_orders"].append({"rank": rank, "epoch": epoch, "key": key, "shards": "shards_2000_4_1"})
    return {"logistic_data": meta}, arrs


def mlp_stats(R: Reference) -> tuple[dict, dict]:
    """Running-statistics tail (sync.cpp:193-213): tiny-MLP (stats_dim =
    hidden), DS W=4 N=2 and BSP W=4, Adam, as in acceptance.cpp:328-402."""
    arrs, meta = {}, []
    hp = R.hp_array()
    for kind, N in (("ds", 2), ("bsp", 4)):
        g, obs, p, st, w0, bt, match = R.mlp_run(1 if kind == "ds" else 0, 4, N, 4, 24, 6, 71, 5, 2, 8, 2, hp, 0.01,
                                                 with_batches=True)
        assert match, "mlp replay != run_training"
        for name, arr in (("grads", g), ("obs", obs), ("params", p), ("stats", st), ("batches", bt)):
            arrs[f"mlp_{kind}_{name}"] = arr
        meta.append({"kind": kind, "W": 4, "N": N, "dim": g.shape[2], "stats_dim": obs.shape[2], "T": g.shape[0],
                     "opt": "adam", "alpha": 0.01, "init": "tiny-mlp initial_params (seed 71)",
                     "problem": {"d": 4, "M": 24, "hidden": 6, "seed": 71}, "run_seed": 5, "batch": 2})
        arrs[f"mlp_{kind}_w0"] = w0
    return {"mlp": meta}, arrs


def sync_rounds(R: Reference) -> tuple[dict, dict]:
    rng = np.random.default_rng(19)
    arrs, meta = {}, []
    for kind, topo, W, N in [(1, 0, 4, 2), (1, 1, 4, 2), (1, 0, 9, 3), (1, 0, 16, 4), (0, 0, 4, 4), (0, 2, 5, 5),
                             (1, 1, 64, 8)]:
        d = int(rng.integers(1, 40))
        w = rng.standard_normal((W, d))
        for t in range(3):
            arrs[f"s{len(meta)}_in"] = w.copy()
            rc, counts, _ = R.sync_round(kind, topo, W, N, t, w, servers=3)
            assert rc == 0, R.error()
            arrs[f"s{len(meta)}_out"] = w.copy()
            meta.append({"id": len(meta), "kind": kind, "topology": topo, "W": W, "N": N, "t": t, "d": d,
                         "num_servers": 3, "critical_path_steps": counts[0], "total_messages": counts[1]})
    return {"sync_rounds": meta}, arrs


def rng_vectors(R: Reference) -> tuple[dict, dict]:
    arrs = {}
    st = np.array([0], np.uint64)
    import ctypes as C
    s = C.c_uint64(0)
    first = R.lib.ref_next_u64(C.byref(s))
    for rank in range(4):
        for t in range(3):
            arrs[f"noise_r{rank}_t{t}"] = R.gaussians(1, K_GRADIENT_NOISE, rank, t, 512)
    arrs["wstar_stream"] = R.gaussians(7, K_DATA_GEN, 1, 0, 512)
    arrs["init_stream"] = R.gaussians(7, K_INIT_PARAMS, 0, 0, 512)
    del st
    return {"splitmix_seed0_first": f"{first:#x}"}, arrs


CLI_CONFIGS = [
    # (name, config, expected parity)
    ("quad_ds_momentum", {"strategy": "ds-sync", "world_size": 4, "group_size": 2, "iterations": 40, "seeds": [1, 2],
                          "problem": {"kind": "quadratic", "d": 16, "mu": 0.5, "L": 0.5, "sigma": 0.0, "delta0": 4.0,
                                      "seed": 3},
                          "optimizer": {"kind": "sgd-momentum", "momentum": 0.8, "weight_decay": 0.001},
                          "lr": {"kind": "step-decay", "alpha": 0.2, "factor": 0.5, "every": 15}}, "bytes"),
    ("quad_bsp_adam", {"strategy": "bsp", "world_size": 4, "iterations": 30, "seeds": [3],
                       "problem": {"kind": "quadratic", "d": 33, "mu": 1.0, "L": 1.0, "delta0": 2.0, "seed": 5},
                       "optimizer": {"kind": "adam"}, "lr": {"kind": "constant", "alpha": 0.05}}, "bytes"),
    ("quad_bsp_ps_theorem", {"strategy": "bsp", "topology": "ps", "servers": 2, "world_size": 9, "iterations": 25,
                            "seeds": [4, 5, 6], "cost_model": {"data_size": 1000.0, "bandwidth": 10.0},
                            "problem": {"kind": "quadratic", "d": 7, "mu": 2.0, "L": 2.0, "delta0": 1.0, "seed": 9},
                            "optimizer": {"kind": "adamw", "weight_decay": 0.01}, "lr": {"kind": "theorem"}}, "bytes"),
    ("quad_ds_tree_noise", {"strategy": "ds-sync", "topology": "tree", "world_size": 16, "iterations": 30,
                            "seeds": [7], "problem": {"kind": "quadratic", "d": 24, "mu": 1.0, "L": 1.0, "sigma": 0.5,
                                                      "delta0": 4.0, "seed": 7},
                            "lr": {"kind": "constant", "alpha": 0.1}}, "tolerance"),
    ("logistic_ds_epoch", {"strategy": "ds-sync", "world_size": 4, "group_size": 2, "iterations": 60, "seeds": [1],
                           "batch_size": 4, "sampling": "epoch",
                           "problem": {"kind": "logistic", "d": 8, "M": 400, "mu": 0.05, "seed": 11},
                           "lr": {"kind": "theorem"}}, "tolerance"),
    ("logistic_bsp", {"strategy": "bsp", "world_size": 4, "iterations": 40, "seeds": [2, 3], "batch_size": 8,
                      "problem": {"kind": "logistic", "d": 20, "M": 2000, "mu": 0.05, "seed": 11},
                      "lr": {"kind": "step-decay", "alpha": 1.0, "factor": 0.5, "every": 10}}, "tolerance"),
    ("mlp_ds_adam", {"strategy": "ds-sync", "world_size": 4, "group_size": 2, "iterations": 30, "seeds": [2],
                     "batch_size": 4, "problem": {"kind": "tiny-mlp", "d": 5, "M": 64, "hidden": 8, "seed": 3},
                     "optimizer": {"kind": "adam"}, "lr": {"kind": "constant", "alpha": 0.01}}, "tolerance"),
    ("mlp_bsp_epoch", {"strategy": "bsp", "world_size": 4, "iterations": 25, "seeds": [1, 4], "batch_size": 3,
                       "sampling": "epoch",
                       "problem": {"kind": "tiny-mlp", "d": 3, "M": 40, "hidden": 4, "seed": 9},
                       "optimizer": {"kind": "sgd-momentum"}, "lr": {"kind": "step-decay", "alpha": 0.05,
                                                                       "every": 10}}, "tolerance"),
    ("quad_diverges", {"strategy": "ds-sync", "world_size": 4, "iterations": 10,
                       "problem": {"kind": "quadratic", "d": 5, "mu": 1.0, "L": 1.0, "seed": 1},
                       "lr": {"kind": "constant", "alpha": 1e300}}, "error"),
]

BAD_CONFIGS = [
    "{", "[]", '{"world_size": 4}', '{"strategy": "x", "world_size": 4, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 5, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "bogus": 1}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic", "dd": 3}}',
    '{"strategy": "ds-sync", "world_size": 4.0, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "topology": "mesh", "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "iterations": 0, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "seeds": [], "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "seeds": [1, -2], "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "sampling": "stratified", "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "svm"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic", "csv": "a.csv"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "optimizer": {"kind": "lion"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "optimizer": {"momentum": 1.0}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "optimizer": {"epsilon": 0}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "lr": {"kind": "cosine"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "lr": {"kind": "step-decay", '
    '"factor": 1.5}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "lr": {"alpha": -1}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "cost_model": {"bandwidth": 0}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"}, "check": {"samples": 1}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "logistic", "M": 3}}',
    '{"strategy": "bsp", "world_size": 4, "group_size": 2, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 6, "group_size": 2, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "servers": 0, "topology": "ps", "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "execution": "async", "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "threads": -1, "problem": {"kind": "quadratic"}}',
    '{"strategy": 3, "world_size": 4, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic", "seed": -1}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic", "mu": "x"}}',
    '{"strategy": "ds-sync", "world_size": 4, "problem": "quadratic"}',
    '{"strategy": "ds-sync", "world_size": 4, "batch_size": 0, "problem": {"kind": "quadratic"}}',
    '{"strategy": "ds-sync", "world_size": 1, "group_size": 1, "problem": {"kind": "quadratic"}}',
]


CSV_CASES = [
    "1.5, -2,1\n\n0.25,4e-1,0\r\n-1,0x10,-1\n",
    "1,1\n3\n", "1,2,1\n1,2,3,1\n", "1,2,2\n", "1,x,1\n", "1,2z,1\n", "", "\n\n", "1,,1\n", "1,2,1,\n",
    " 7 ,\t8\t,1\n", "1e999,1\n", "inf,-1\n", "nan,1\n", "1,-0\n", ",\n", "1,2,1", "1,2,+1\n", ".5,-.5,1\n",
    "1,2,1\n\r\n",
]


def csv_cases(R: Reference) -> dict:
    """load_logistic_csv (problems.cpp:584-640) on edge-case files: the
    reference's error text, or y*x of the parsed rows."""
    import tempfile
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        for i, text in enumerate(CSV_CASES):
            path = os.path.join(tmp, f"c{i}.csv")
            with open(path, "w", newline="") as f:
                f.write(text)
            err, yx = R.load_csv(path, 0.1)
            out.append({"text": text, "error": err.replace(path, "<path>") if err else None,
                        "yx": None if yx is None else [[float(v) for v in row] for row in yx]})
    return {"csv_cases": out}


def cli_runs(R: Reference) -> dict:
    """The reference's own `dssync run` (tools/main.cpp:34-55 through
    oracle/ref_shim.cpp ref_cmd_run): metrics_seed*.csv and summary.json
    texts per config, plus parse_run_config's verdict on malformed configs."""
    import tempfile
    runs = []
    for name, cfg, parity in CLI_CONFIGS:
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "cfg.json")
            with open(path, "w") as f:
                json.dump(cfg, f)
            out = os.path.join(tmp, "out")
            rc, msg, rank, it = R.cmd_run(path, out)
            files = {}
            if rc == 0:
                for fn in sorted(os.listdir(out)):
                    with open(os.path.join(out, fn)) as f:
                        files[fn] = f.read()
        runs.append({"name": name, "config": cfg, "parity": parity, "status": rc, "error": msg, "rank": rank,
                     "iteration": it, "files": files})
    bad = [{"text": t, "error": R.parse_config(t)} for t in BAD_CONFIGS]
    return {"cli_runs": runs, "bad_configs": bad}


def main():
    R = Reference()
    meta = {"generated_by": "tests/golden/make_golden.py from oracle/_ref (unmodified /root/reference/proj/src)"}
    meta["partitions"] = partitions(R)
    m, a1 = apply_steps(R)
    meta["apply_step"] = m
    m, a2 = trajectories(R)
    meta.update(m)
    m, a3 = logistic_c1(R)
    meta.update(m)
    m, a7 = logistic_data(R)
    meta.update(m)
    a3.update(a7)
    m, a4 = sync_rounds(R)
    meta.update(m)
    m, a6 = mlp_stats(R)
    meta.update(m)
    a4.update(a6)
    m, a5 = rng_vectors(R)
    meta.update(m)
    meta.update(cli_runs(R))
    meta.update(csv_cases(R))
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **a1, **a2, **a3, **a4, **a5)
    print("wrote", os.path.join(HERE, "golden.json"), os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
