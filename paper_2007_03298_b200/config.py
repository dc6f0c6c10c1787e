"""Run configuration: the reference's JSON schema and strict validation
(/root/reference/proj/src/config.cpp:17-302, include/dssync/config.hpp:15-42).

Every rejection names the violated rule and the offending field with the
reference's wording; unknown fields are rejected.  The parsed config drives
the device run in run.py.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List

from .api import OptimizerHyperparams, OptimizerKind, SamplingMode, StrategyKind, SyncStrategy, Topology, WorldConfig
from .api import validate as validate_strategy


class ConfigError(ValueError):
    """errors.hpp ConfigError: a rejected configuration (exit code 1)."""


_STRATEGIES = {"bsp": StrategyKind.BSP, "ds-sync": StrategyKind.DS_SYNC}  # sync.cpp:15-19
_TOPOLOGIES = {"ring": Topology.RING, "tree": Topology.TREE, "ps": Topology.PS}  # sync.cpp:21-26
_OPTIMIZERS = {"vanilla-sgd": OptimizerKind.VANILLA_SGD, "sgd-momentum": OptimizerKind.SGD_MOMENTUM,
               "adam": OptimizerKind.ADAM, "adamw": OptimizerKind.ADAMW}  # optim.cpp:9-15


@dataclass
class DatasetSpec:  # problems.hpp:16-27
    kind: str = ""
    d: int = 2
    M: int = 0
    mu: float = 1.0
    L: float = 1.0
    sigma: float = 0.0
    delta0: float = 1.0
    hidden: int = 16
    seed: int = 1
    csv: str = ""


@dataclass
class LrSpec:  # config.hpp:17-22
    kind: str = "constant"
    alpha: float = 0.1
    factor: float = 0.5
    every: int = 100


@dataclass
class CostModel:
    data_size: float = 0.0
    bandwidth: float = 1.0
    servers: int = 1


@dataclass
class RunConfig:  # config.hpp:30-42
    strategy: SyncStrategy = None
    problem: DatasetSpec = field(default_factory=DatasetSpec)
    optimizer: OptimizerKind = OptimizerKind.VANILLA_SGD
    hp: OptimizerHyperparams = field(default_factory=OptimizerHyperparams)
    lr: LrSpec = field(default_factory=LrSpec)
    iterations: int = 100
    batch_size: int = 1
    seeds: List[int] = field(default_factory=lambda: [1])
    execution: str = "lockstep"
    threads: int = 0
    sampling: SamplingMode = SamplingMode.REPLACEMENT
    cost: CostModel = field(default_factory=CostModel)
    check_samples: int = 10000
    check_t_max: int = 11


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _is_num(v) -> bool:
    return (isinstance(v, (int, float))) and not isinstance(v, bool)


class _Fields:
    """Strict object view (config.cpp:17-90): each access marks its key."""

    def __init__(self, j, path: str):
        if not isinstance(j, dict):
            raise ConfigError(path + " must be a JSON object")
        self.j, self.path, self.seen = j, path, set()

    def finish(self):
        for k in self.j:
            if k not in self.seen:
                raise ConfigError("unknown field: " + self.key_path(k))

    def has(self, key):
        return key in self.j

    def raw(self, key):
        self.seen.add(key)
        return self.j[key]

    def key_path(self, key):
        return key if not self.path else self.path + "." + key

    def _string(self, key):
        v = self.raw(key)
        if not isinstance(v, str):
            raise ConfigError(self.key_path(key) + " must be a string")
        return v

    def str(self, key, default):
        return self._string(key) if self.has(key) else default

    def require_str(self, key):
        if not self.has(key):
            raise ConfigError("missing required field: " + self.key_path(key))
        return self._string(key)

    def num(self, key, default):
        if not self.has(key):
            return default
        v = self.raw(key)
        if not _is_num(v):
            raise ConfigError(self.key_path(key) + " must be a number")
        return float(v)

    def integer(self, key, default):
        if not self.has(key):
            return default
        v = self.raw(key)
        if not _is_int(v):
            raise ConfigError(self.key_path(key) + " must be an integer")
        return int(v)

    def uinteger(self, key, default):
        if not self.has(key):
            return default
        v = self.raw(key)
        if not _is_int(v) or v < 0:
            raise ConfigError(self.key_path(key) + " must be a non-negative integer")
        return int(v)


def _parse_problem(j) -> DatasetSpec:  # config.cpp:92-112
    f = _Fields(j, "problem")
    s = DatasetSpec()
    s.kind = f.require_str("kind")
    if s.kind not in ("quadratic", "logistic", "tiny-mlp"):
        raise ConfigError(f"problem.kind must be quadratic, logistic or tiny-mlp (got '{s.kind}')")
    s.csv = f.str("csv", "")
    if s.csv and s.kind != "logistic":
        raise ConfigError("problem.csv is only supported for logistic")
    s.d = f.integer("d", s.d)
    s.M = f.integer("M", s.M)
    s.mu = f.num("mu", s.mu)
    s.L = f.num("L", s.L)
    s.sigma = f.num("sigma", s.sigma)
    s.delta0 = f.num("delta0", s.delta0)
    s.hidden = f.integer("hidden", s.hidden)
    s.seed = f.uinteger("seed", s.seed)
    f.finish()
    return s


def _parse_optimizer(j, cfg: RunConfig) -> None:  # config.cpp:116-143
    f = _Fields(j, "optimizer")
    kind = f.str("kind", "vanilla-sgd")
    if kind not in _OPTIMIZERS:
        raise ConfigError("optimizer.kind: unknown optimizer kind: " + kind)
    cfg.optimizer = _OPTIMIZERS[kind]
    hp = OptimizerHyperparams()
    hp.momentum = f.num("momentum", hp.momentum)
    hp.beta1 = f.num("beta1", hp.beta1)
    hp.beta2 = f.num("beta2", hp.beta2)
    hp.epsilon = f.num("epsilon", hp.epsilon)
    hp.weight_decay = f.num("weight_decay", hp.weight_decay)
    f.finish()
    if not (0.0 <= hp.momentum < 1.0):
        raise ConfigError("optimizer.momentum must be in [0, 1)")
    if not (0.0 <= hp.beta1 < 1.0):
        raise ConfigError("optimizer.beta1 must be in [0, 1)")
    if not (0.0 <= hp.beta2 < 1.0):
        raise ConfigError("optimizer.beta2 must be in [0, 1)")
    if not (hp.epsilon > 0.0):
        raise ConfigError("optimizer.epsilon must be > 0")
    if not (hp.weight_decay >= 0.0):
        raise ConfigError("optimizer.weight_decay must be >= 0")
    cfg.hp = hp


def _parse_lr(j) -> LrSpec:  # config.cpp:145-164
    f = _Fields(j, "lr")
    lr = LrSpec()
    lr.kind = f.str("kind", lr.kind)
    if lr.kind not in ("constant", "step-decay", "theorem"):
        raise ConfigError(f"lr.kind must be constant, step-decay or theorem (got '{lr.kind}')")
    lr.alpha = f.num("alpha", lr.alpha)
    lr.factor = f.num("factor", lr.factor)
    lr.every = f.integer("every", lr.every)
    f.finish()
    if lr.kind != "theorem" and not (lr.alpha >= 0.0):
        raise ConfigError("lr.alpha must be >= 0")
    if lr.kind == "step-decay":
        if not (0.0 < lr.factor <= 1.0):
            raise ConfigError("lr.factor must be in (0, 1]")
        if lr.every < 1:
            raise ConfigError("lr.every must be >= 1")
    return lr


def _integer_sqrt(n: int) -> int:  # config.cpp:166-171
    r = int(round(math.sqrt(float(n))))
    while r * r > n:
        r -= 1
    while (r + 1) * (r + 1) <= n:
        r += 1
    return r


def parse_run_config(text: str) -> RunConfig:  # config.cpp:175-294
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError("config is not valid JSON: " + str(e)) from None
    f = _Fields(j, "")
    cfg = RunConfig()
    name = f.require_str("strategy")
    if name not in _STRATEGIES:
        raise ConfigError("strategy: unknown strategy: " + name)
    kind = _STRATEGIES[name]
    topo_name = f.str("topology", "ring")
    if topo_name not in _TOPOLOGIES:
        raise ConfigError("topology: unknown topology: " + topo_name)
    topo = _TOPOLOGIES[topo_name]
    world = f.integer("world_size", 0)
    if world < 1:
        raise ConfigError("world_size must be a positive integer")
    if f.has("group_size"):
        group = f.integer("group_size", 0)
    elif kind == StrategyKind.BSP:
        group = world
    else:
        n = _integer_sqrt(world)
        if n * n != world:
            raise ConfigError(f"ds-sync requires world_size to be a perfect square (got world_size={world}); "
                              "set group_size explicitly for a single full group")
        group = n
    servers = f.integer("servers", 1)
    cfg.strategy = SyncStrategy(kind, topo, WorldConfig(world, group), servers)

    cfg.iterations = f.integer("iterations", cfg.iterations)
    if cfg.iterations < 1:
        raise ConfigError("iterations must be >= 1")
    cfg.batch_size = f.integer("batch_size", cfg.batch_size)
    if cfg.batch_size < 1:
        raise ConfigError("batch_size must be >= 1")
    if f.has("seeds"):
        seeds = f.raw("seeds")
        if not isinstance(seeds, list) or not seeds:
            raise ConfigError("seeds must be a non-empty array of non-negative integers")
        if not all(_is_int(s) and s >= 0 for s in seeds):
            raise ConfigError("seeds must be a non-empty array of non-negative integers")
        cfg.seeds = [int(s) for s in seeds]
    cfg.execution = f.str("execution", "lockstep")
    if cfg.execution not in ("lockstep", "parallel"):
        raise ConfigError(f"execution must be lockstep or parallel (got '{cfg.execution}')")
    cfg.threads = f.integer("threads", 0)
    if cfg.threads < 0:
        raise ConfigError("threads must be >= 0")
    sampling = f.str("sampling", "replacement")
    if sampling not in ("replacement", "epoch"):
        raise ConfigError(f"sampling must be replacement or epoch (got '{sampling}')")
    cfg.sampling = SamplingMode.EPOCH if sampling == "epoch" else SamplingMode.REPLACEMENT

    if not f.has("problem"):
        raise ConfigError("missing required field: problem")
    cfg.problem = _parse_problem(f.raw("problem"))
    if f.has("optimizer"):
        _parse_optimizer(f.raw("optimizer"), cfg)
    if f.has("lr"):
        cfg.lr = _parse_lr(f.raw("lr"))
    if f.has("cost_model"):
        c = _Fields(f.raw("cost_model"), "cost_model")
        cfg.cost.data_size = c.num("data_size", 0.0)
        cfg.cost.bandwidth = c.num("bandwidth", 1.0)
        c.finish()
        if cfg.cost.data_size < 0.0:
            raise ConfigError("cost_model.data_size must be >= 0")
        if not (cfg.cost.bandwidth > 0.0):
            raise ConfigError("cost_model.bandwidth must be > 0")
    cfg.cost.servers = servers
    if f.has("check"):
        c = _Fields(f.raw("check"), "check")
        cfg.check_samples = c.integer("samples", cfg.check_samples)
        cfg.check_t_max = c.integer("t_max", cfg.check_t_max)
        c.finish()
        if cfg.check_samples < 2:
            raise ConfigError("check.samples must be >= 2")
        if cfg.check_t_max < 1:
            raise ConfigError("check.t_max must be >= 1")
    f.finish()
    try:
        validate_strategy(cfg.strategy)
    except ValueError as e:
        raise ConfigError(str(e)) from None
    if cfg.problem.kind != "quadratic" and not cfg.problem.csv and cfg.problem.M < world:
        raise ConfigError("problem.M must be >= world_size so every worker gets a shard")
    return cfg


def load_run_config(path: str) -> RunConfig:  # config.cpp:296-302
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise ConfigError("cannot open config file: " + path) from None
    return parse_run_config(text)
