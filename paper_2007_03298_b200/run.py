"""`run` driver: the reference's `dssync run --config cfg.json --out dir`
(/root/reference/proj/tools/main.cpp:34-55) on the device.

    python -m paper_2007_03298_b200.run --config cfg.json --out out [--device 0] [--dtype f64]

Per seed it builds the problem on the host (bit-exact setup: the quadratic's
w* and w0, the logistic data, shards, smoothness and optimum), then runs
run_training's loop (sync.cpp:286-459).  Every iteration runs on the GPU:
- the stochastic gradient (quadratic: SplitMix64/Box-Muller noise;
  logistic: batch sampling and gradient);
- the DS-Sync or BSP step;
- the trace: the ordered global mean and the per-worker losses.

It writes metrics_seed<seed>.csv (metrics.cpp:37-56) and summary.json
(metrics.cpp:73-115) in the reference's formats.  Exit codes follow
main.cpp:23-26 and 170-191.

Parity:
- Isotropic quadratic with sigma = 0: the metrics files are byte-identical
  to the reference's.
- sigma > 0: the gradient noise uses libdevice log/cos. It matches glibc
  to <= 1 ulp, so the files agree to within that rounding.
- Logistic: the same holds for exp/log1p.

Device path only: the anisotropic quadratic (problem.L != problem.mu, a
dense d x d matvec) is rejected with a clear message.  The tiny MLP runs
with its running statistics; its tanh is libdevice's (tolerance).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import re
import sys
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import _lib as L
from ._lib import BUF_PARAMS
from .api import (DivergenceError, DsSyncEngine, IterationTrace, StrategyKind, Topology,
                  logistic_constants, logistic_dataset, mlp_dataset, mlp_initial_params, quadratic_problem)
from .config import ConfigError, RunConfig, load_run_config
from .metrics import atomic_write_file, format_double, metrics_csv, summary_json

EXIT_OK, EXIT_USAGE, EXIT_DIVERGED = 0, 1, 2  # main.cpp:23-26



class DeviceProblem:
    """A problem whose gradient and losses are produced on the device."""

    kind = ""
    dim = 0
    stats_dim = 0
    mu = 0.0          # strong convexity (problem.strong_convexity())
    smoothness = 0.0  # problem.smoothness()
    has_optimum = True

    def setup(self, engine: DsSyncEngine, run_seed: int, cfg: RunConfig) -> None:
        raise NotImplementedError

    def gradients(self, engine: DsSyncEngine, t: int, run_seed: int) -> None:
        raise NotImplementedError

    def losses(self, engine: DsSyncEngine, with_mean: bool = True) -> Tuple[np.ndarray, float]:
        """(full_loss of every worker, suboptimality of the global mean or None
        when the caller evaluates it)."""
        raise NotImplementedError


def _check_common(p) -> None:  # problems.cpp:115-118
    if p.d < 1:
        raise ConfigError(f"problem.d must be >= 1 (got {p.d})")
    if not (p.mu >= 0.0):
        raise ConfigError("problem.mu must be >= 0")


class Quadratic(DeviceProblem):
    """QuadraticProblem with A = mu*I (problems.cpp:120-224)."""

    kind = "quadratic"

    def __init__(self, spec):
        _check_common(spec)
        if spec.mu <= 0.0:
            raise ConfigError("quadratic requires problem.mu > 0")
        if not (spec.L >= spec.mu):
            raise ConfigError("problem.L must be >= problem.mu")
        if spec.sigma < 0.0:
            raise ConfigError("problem.sigma must be >= 0")
        if spec.delta0 <= 0.0:
            raise ConfigError("problem.delta0 must be > 0")
        if spec.d == 1 and spec.L != spec.mu:
            raise ConfigError("quadratic with d=1 requires problem.L == problem.mu")
        if spec.L != spec.mu:
            raise ConfigError("the device path runs the isotropic quadratic only (problem.L == problem.mu); "
                              "an anisotropic A needs a dense d x d matvec per worker")
        self.spec = spec
        self.dim = spec.d
        self.mu = spec.mu
        self.smoothness = spec.L
        self.wstar, self.w0 = quadratic_problem(spec.seed, spec.d, spec.delta0)

    def setup(self, engine, run_seed, cfg):
        engine.set_optimum(self.wstar)
        engine.broadcast_row(BUF_PARAMS, self.w0)

    def gradients(self, engine, t, run_seed):
        engine.quadratic_gradients(t, run_seed, self.spec.mu, self.spec.sigma)

    def losses(self, engine, with_mean=True):
        return engine.quadratic_losses(self.spec.mu, with_suboptimality=with_mean, exact=True)


_STOD = re.compile(r"[ \t\n\v\f\r]*([+-]?(?:0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?"
                   r"|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|[iI][nN][fF](?:[iI][nN][iI][tT][yY])?"
                   r"|[nN][aA][nN](?:\([0-9A-Za-z_]*\))?))")


def _stod(cell: str) -> Tuple[float, int]:
    """std::stod: (value, characters used); ValueError when nothing parses or
    the value is out of range."""
    m = _STOD.match(cell)
    if not m:
        raise ValueError(cell)
    tok = m.group(1)
    low = tok.lower().lstrip("+-")
    if low.startswith("0x"):
        v = float.fromhex(tok)
    elif low.startswith("nan"):
        v = float("nan")
    else:
        v = float(tok)
    if math.isinf(v) and not low.startswith("inf"):
        raise ValueError(cell)  # ERANGE -> std::out_of_range
    return v, m.end()


def load_logistic_csv(path: str, l2: float):
    """load_logistic_csv (problems.cpp:584-640): features then a label in {-1, 0, 1} (0 -> -1)."""
    try:
        with open(path, "rb") as fh:
            text = fh.read().decode("latin-1")
    except OSError:
        raise ConfigError("cannot open csv file: " + path) from None
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    xs: List[float] = []
    ys: List[float] = []
    d = -1
    for row, line in enumerate(lines, start=1):
        if not line:
            continue
        cells = line.split(",")
        if cells[-1] == "":
            cells.pop()  # getline(',') yields no trailing empty cell
        fields = []
        for cell in cells:
            try:
                v, used = _stod(cell)
            except ValueError:
                raise ConfigError(f"csv row {row}: not a number: '{cell}'") from None
            if used != len(cell) and cell[used:].strip(" \t\r"):
                raise ConfigError(f"csv row {row}: not a number: '{cell}'")
            fields.append(v)
        if len(fields) < 2:
            raise ConfigError(f"csv row {row}: need features plus a label")
        row_d = len(fields) - 1
        if d == -1:
            d = row_d
        elif row_d != d:
            raise ConfigError(f"csv row {row}: expected {d + 1} columns, got {len(fields)}")
        label = fields[-1]
        if label not in (1.0, -1.0, 0.0):
            raise ConfigError(f"csv row {row}: label must be -1, 0 or 1")
        ys.append(-1.0 if label == 0.0 else label)
        xs.extend(fields[:-1])
    if d == -1:
        raise ConfigError("csv file has no data rows: " + path)
    if l2 < 0.0:
        raise ConfigError("logistic l2 must be >= 0")
    return np.array(xs, dtype=np.float64).reshape(len(ys), d), np.array(ys, dtype=np.float64)


class Logistic(DeviceProblem):
    """LogisticProblem (problems.cpp:226-430), synthetic or from CSV."""

    kind = "logistic"

    def __init__(self, spec):
        if spec.csv:
            self.x, self.y = load_logistic_csv(spec.csv, spec.mu)
        else:
            _check_common(spec)
            if spec.M < 1:
                raise ConfigError("logistic requires problem.M >= 1")
            self.x, self.y = logistic_dataset(spec.seed, spec.d, spec.M)
        self.l2 = spec.mu
        self.M, self.dim = self.x.shape
        self.mu = self.l2
        self.smoothness, self.f_star, _ = logistic_constants(self.x, self.y, self.l2)
        self.has_optimum = self.l2 > 0.0

    def setup(self, engine, run_seed, cfg):
        engine.broadcast_row(BUF_PARAMS, np.zeros(self.dim))  # initial_params: zeros
        engine.logistic_setup(self.x, self.y, self.l2, cfg.batch_size, cfg.sampling, run_seed)

    def gradients(self, engine, t, run_seed):
        engine.logistic_gradients(t)

    def losses(self, engine, with_mean=True):
        losses = engine.logistic_losses(exact=True)
        # true_suboptimality(global mean) = full_loss(mean) - f*: the caller
        # evaluates the mean row (None); NaN without an optimum
        return losses, (None if self.has_optimum else float("nan"))


class TinyMlp(DeviceProblem):
    """TinyMlpProblem (problems.cpp:436-570): running statistics = the EMA
    of the hidden pre-activations, folded with the params."""

    kind = "tiny-mlp"
    has_optimum = False
    smoothness = float("nan")

    def __init__(self, spec):
        _check_common(spec)
        if spec.M < 1:
            raise ConfigError("tiny-mlp requires problem.M >= 1")
        if spec.hidden < 1 or spec.hidden > 32:
            raise ConfigError(f"problem.hidden must be in [1, 32] (got {spec.hidden})")
        self.spec = spec
        self.x, self.y = mlp_dataset(spec.seed, spec.d, spec.M)
        self.dim = spec.hidden * spec.d + 2 * spec.hidden + 1
        self.stats_dim = spec.hidden
        self.mu = 0.0
        self.w0 = mlp_initial_params(spec.seed, spec.d, spec.hidden)

    def setup(self, engine, run_seed, cfg):
        engine.broadcast_row(BUF_PARAMS, self.w0)
        engine.mlp_setup(self.x, self.y, self.spec.hidden, cfg.batch_size, cfg.sampling, run_seed)

    def gradients(self, engine, t, run_seed):
        engine.mlp_gradients(t)
        engine.running_stats_update()  # fold_running_stats (sync.cpp:193-201)

    def losses(self, engine, with_mean=True):
        return engine.mlp_losses(exact=True), float("nan")


def make_device_problem(spec) -> DeviceProblem:  # problems.cpp:572-582
    if spec.kind == "quadratic":
        return Quadratic(spec)
    if spec.kind == "logistic":
        return Logistic(spec)
    if spec.kind == "tiny-mlp":
        return TinyMlp(spec)
    raise ConfigError("unknown problem.kind: " + spec.kind)


def build_lr(cfg: RunConfig, problem: DeviceProblem) -> Callable[[int], float]:  # config.cpp:304-314
    spec = cfg.lr
    if spec.kind == "constant":
        if not (spec.alpha >= 0.0) or not math.isfinite(spec.alpha):  # sync.cpp:68-73
            raise ValueError("constant_lr: alpha must be finite and >= 0")
        a = spec.alpha
        return lambda t: a
    if spec.kind == "step-decay":  # sync.cpp:75-88
        if not (spec.alpha >= 0.0) or not math.isfinite(spec.alpha):
            raise ValueError("step_decay_lr: alpha0 must be finite and >= 0")
        a0, f, every = spec.alpha, spec.factor, spec.every
        return lambda t: a0 * math.pow(f, float(t // every))
    mu, Lc = problem.mu, problem.smoothness
    if not (mu > 0.0) or not math.isfinite(Lc):
        raise ConfigError("lr.kind 'theorem' needs a strongly convex problem with known mu and L")
    gamma = max(8.0 * Lc / mu, 2.0)
    return lambda t: 2.0 / (mu * (gamma + float(t)))  # theorem_lr (sync.cpp:90-95)


def run_training(problem: DeviceProblem, cfg: RunConfig, seed: int, device: int = 0,
                 dtype: str = "f64") -> List[IterationTrace]:
    """run_training (sync.cpp:286-459) with every iteration on the device."""
    s = cfg.strategy
    W = s.world.world_size
    lr = build_lr(cfg, problem)
    payload = cfg.cost.data_size if cfg.cost.data_size > 0.0 else 8.0 * (problem.dim + problem.stats_dim)
    bw = cfg.cost.bandwidth
    if s.topology == Topology.PS:  # effective_bandwidth (sync.cpp:215-221)
        bw = cfg.cost.bandwidth * s.num_servers / W
    traces = []
    with DsSyncEngine(s, cfg.optimizer, problem.dim, cfg.hp, dtype, device, stats_dim=problem.stats_dim) as e:
        problem.setup(e, seed, cfg)
        mean_engine = None
        if isinstance(problem, Logistic) and problem.has_optimum:
            # full_loss of the global mean: a one-worker context holding the
            # mean row, same data, same loss kernel
            from .api import SyncStrategy, WorldConfig
            mean_engine = DsSyncEngine(SyncStrategy(StrategyKind.BSP, Topology.RING, WorldConfig(1, 1)),
                                       cfg.optimizer, problem.dim, cfg.hp, dtype, device)
            mean_engine.logistic_setup(problem.x, problem.y, problem.l2, 1, 0, seed)
        try:
            for t in range(cfg.iterations):
                alpha = lr(t)
                if not math.isfinite(alpha) or alpha < 0.0:
                    raise ValueError(f"learning rate at t={t} must be finite and >= 0")
                problem.gradients(e, t, seed)
                if s.kind == StrategyKind.DS_SYNC:
                    # local_iteration + the pre-sync loss check, per worker in
                    # rank order (sync.cpp:348-361), then the group rounds.
                    # The split apply_step / sync_round path gives the same
                    # bits as the fused dss_step.
                    err = None
                    try:
                        e.apply_step(alpha, check=True)
                    except DivergenceError as ex:
                        err = ex
                    pre, _ = problem.losses(e, with_mean=False)
                    for k in range(W):
                        if err is not None and err.rank == k:
                            raise err
                        if not math.isfinite(pre[k]):
                            raise DivergenceError(k, t, f"worker {k} diverged at iteration {t}: "
                                                        "non-finite loss after local step")
                    if err is not None:
                        raise err
                    out = e.sync_round(t, check=True)
                else:
                    out = e.step(t, alpha, check=True)
                gmean = e.global_mean()
                params = e.download_all(BUF_PARAMS)
                losses, sub = problem.losses(e)
                for k in range(W):  # sync.cpp:431-440, ascending rank
                    if not np.all(np.isfinite(params[k])):
                        raise DivergenceError(k, t, f"worker {k} diverged at iteration {t}: "
                                                    "non-finite parameters after sync")
                    if not math.isfinite(losses[k]):
                        raise DivergenceError(k, t, f"worker {k} diverged at iteration {t}: non-finite loss after sync")
                if sub is None:
                    mean_engine.upload(BUF_PARAMS, 0, gmean)
                    sub = float(mean_engine.logistic_losses(exact=True)[0]) - problem.f_star
                acc = 0.0
                for v in losses:
                    acc += float(v)
                traces.append(IterationTrace(t, losses, acc / W, sub, out.critical_path_steps, out.total_messages,
                                             out.critical_path_steps * payload / bw, gmean))
        finally:
            if mean_engine is not None:
                mean_engine.close()
    return traces


def cmd_run(config_path: str, out_dir: str = "out", device: int = 0, dtype: str = "f64") -> int:
    """main.cpp:34-55."""
    cfg = load_run_config(config_path)
    problem = make_device_problem(cfg.problem)
    outcomes = []
    for seed in cfg.seeds:
        traces = run_training(problem, cfg, seed, device, dtype)
        last = traces[-1]
        outcomes.append((seed, last.mean_post_sync_loss, last.suboptimality))
        atomic_write_file(os.path.join(out_dir, f"metrics_seed{seed}.csv"), metrics_csv(traces))
    atomic_write_file(os.path.join(out_dir, "summary.json"), summary_json(cfg, outcomes))
    print(f"wrote {len(cfg.seeds)} metrics file(s) and summary.json to {out_dir}")
    return EXIT_OK


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2007_03298_b200.run",
                                 description="DS-Sync / BSP training run on a B200 (the reference's `dssync run`)")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default="out")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    args = ap.parse_args(argv)
    try:
        return cmd_run(args.config, args.out, args.device, args.dtype)
    except DivergenceError as e:  # main.cpp:182-184
        print(f"error: {e}", file=sys.stderr)
        return EXIT_DIVERGED
    except (ConfigError, ValueError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())


__all__ = ["cmd_run", "run_training", "summary_json", "build_lr", "load_logistic_csv", "make_device_problem",
           "format_double", "L"]
