"""Reference-shaped interface over the C-ABI.

Mirrors the reference's operator API for the DS-Sync path — same names,
argument meaning and error behaviour — so callers and parity tests read like
the reference's own (proj/include/dssync/*.hpp):

  WorldConfig, validate, is_square_mode, make_partition, group_of,
  check_mixing                                   schedule.hpp:17-45
  OptimizerKind/Hyperparams/State, StepResult,
  apply_step                                     optim.hpp:11-52
  StrategyKind, Topology, SyncStrategy, validate,
  WorkerState, SyncRoundOutcome, sync_round      sync.hpp:14-129
  DivergenceError                                errors.hpp:16-25

``apply_step`` and ``sync_round`` take host-resident workers like the
reference (upload -> CUDA kernel -> download).  ``DsSyncEngine`` keeps the
workers resident in HBM across iterations — the performance path.

Errors: std::invalid_argument -> ValueError, DivergenceError ->
DivergenceError(rank, iteration), CUDA failures -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


class OptimizerKind(enum.IntEnum):  # optim.hpp:11
    VANILLA_SGD = 0
    SGD_MOMENTUM = 1
    ADAM = 2
    ADAMW = 3

    @staticmethod
    def from_string(name: str) -> "OptimizerKind":  # optim.cpp:9-15
        table = {"vanilla-sgd": 0, "sgd-momentum": 1, "adam": 2, "adamw": 3}
        if name not in table:
            raise ValueError("unknown optimizer kind: " + name)
        return OptimizerKind(table[name])

    def __str__(self) -> str:
        return ["vanilla-sgd", "sgd-momentum", "adam", "adamw"][int(self)]


class StrategyKind(enum.IntEnum):  # sync.hpp:14
    BSP = 0
    DS_SYNC = 1

    @staticmethod
    def from_string(name: str) -> "StrategyKind":  # sync.cpp:15-19
        if name == "bsp":
            return StrategyKind.BSP
        if name == "ds-sync":
            return StrategyKind.DS_SYNC
        raise ValueError("unknown strategy: " + name)

    def __str__(self) -> str:
        return "bsp" if self == StrategyKind.BSP else "ds-sync"


class Topology(enum.IntEnum):  # sync.hpp:15
    RING = 0
    TREE = 1
    PS = 2

    @staticmethod
    def from_string(name: str) -> "Topology":  # sync.cpp:21-26
        table = {"ring": 0, "tree": 1, "ps": 2}
        if name not in table:
            raise ValueError("unknown topology: " + name)
        return Topology(table[name])

    def __str__(self) -> str:
        return ["ring", "tree", "ps"][int(self)]


class DivergenceError(RuntimeError):
    """errors.hpp:16-25: a worker produced a non-finite value at iteration t."""

    def __init__(self, rank: int, iteration: int, what: str):
        super().__init__(what)
        self.rank = rank
        self.iteration = iteration


@dataclass
class WorldConfig:  # schedule.hpp:17-20
    world_size: int = 1
    group_size: int = 1


@dataclass
class GroupPartition:  # schedule.hpp:28-31
    iteration: int
    groups: List[List[int]]


@dataclass
class OptimizerHyperparams:  # optim.hpp:16-23
    alpha: float = 0.1
    momentum: float = 0.9
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    weight_decay: float = 0.0


@dataclass
class OptimizerState:  # optim.hpp:25-34
    kind: OptimizerKind = OptimizerKind.VANILLA_SGD
    hp: OptimizerHyperparams = field(default_factory=OptimizerHyperparams)
    first_moment: Optional[np.ndarray] = None
    second_moment: Optional[np.ndarray] = None
    step_count: int = 0


@dataclass
class StepResult:  # optim.hpp:36-39
    params: np.ndarray
    state: OptimizerState


@dataclass
class SyncStrategy:  # sync.hpp:34-39
    kind: StrategyKind = StrategyKind.BSP
    topology: Topology = Topology.RING
    world: WorldConfig = field(default_factory=WorldConfig)
    num_servers: int = 1
    rectangular: bool = False  # builder extension W = N*K (not in the reference)


@dataclass
class WorkerState:  # sync.hpp:55-61
    rank: int = 0
    params: np.ndarray = field(default_factory=lambda: np.zeros(0))
    opt: OptimizerState = field(default_factory=OptimizerState)
    running_stats: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class SyncRoundOutcome:  # sync.hpp:119-122
    critical_path_steps: int = 0
    total_messages: int = 0


@dataclass
class IterationTrace:  # sync.hpp:63-74
    t: int = 0
    post_sync_loss: Optional[np.ndarray] = None
    mean_post_sync_loss: float = 0.0
    suboptimality: float = 0.0
    critical_path_steps: int = 0
    total_messages: int = 0
    simulated_comm_time: float = 0.0
    global_mean_params: Optional[np.ndarray] = None


def iteration_trace(engine: "DsSyncEngine", t: int, outcome: SyncRoundOutcome, mu: float,
                    data_size: float = 0.0, bandwidth: float = 1.0, losses_all=None,
                    exact: bool = False) -> IterationTrace:
    """run_training's post-round bookkeeping (sync.cpp:430-458) on the device
    state: global mean (bit-exact ordered fold), per-worker quadratic losses
    (fp64 device reduction), closed-form comm counts.  On several GPUs pass
    losses_all = every worker's loss gathered in rank order."""
    gmean = engine.global_mean()
    losses, sub = engine.quadratic_losses(mu, exact=exact)
    if losses_all is not None:
        losses = np.asarray(losses_all, dtype=np.float64)
    acc = 0.0
    for x in losses:  # sync.cpp:582-584: ascending sum, then a division
        acc += float(x)
    W = engine.strategy.world.world_size
    # sync.cpp:314-318: the default payload is params ++ running stats, 8 B each
    payload = data_size if data_size > 0.0 else 8.0 * (engine.dim + engine.stats_dim)
    bw = bandwidth
    if engine.strategy.topology == Topology.PS:  # effective_bandwidth (sync.cpp:215-221)
        bw = bandwidth * engine.strategy.num_servers / W
    return IterationTrace(t, losses, acc / W, sub, outcome.critical_path_steps, outcome.total_messages,
                          outcome.critical_path_steps * payload / bw, gmean)


# ---------------------------------------------------------------------------
def _raise(status: int, msg: str, rank: int = -1, iteration: int = -1):
    if status == L.DSS_OK:
        return
    if status == L.DSS_EINVAL:
        raise ValueError(msg)
    if status == L.DSS_EDIVERGED:
        raise DivergenceError(rank, iteration, msg)
    raise RuntimeError(msg)


def _check_global(status: int):
    if status != L.DSS_OK:
        _raise(status, L.global_error())


def _c_strategy(s: SyncStrategy) -> L.dss_strategy:
    return L.dss_strategy(int(s.kind), int(s.topology), int(s.world.world_size),
                          int(s.world.group_size), int(s.num_servers), 1 if s.rectangular else 0)


def _as_strategy(x) -> SyncStrategy:
    if isinstance(x, SyncStrategy):
        return x
    if isinstance(x, WorldConfig):  # make_partition(WorldConfig, t): the DS schedule
        return SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, x)
    raise TypeError("expected WorldConfig or SyncStrategy")


def validate(x) -> None:
    """validate(WorldConfig) (schedule.cpp:8-24) or validate(SyncStrategy) (sync.cpp:47-66)."""
    lib = L.load()
    if isinstance(x, WorldConfig):
        _check_global(lib.dss_validate_world(x.world_size, x.group_size, 0))
    else:
        s = _c_strategy(x)
        _check_global(lib.dss_validate_strategy(C.byref(s)))


def is_square_mode(cfg: WorldConfig) -> bool:  # schedule.cpp:26-29
    return L.load().dss_is_square_mode(cfg.world_size, cfg.group_size) == 1


def make_partition(cfg, t: int) -> GroupPartition:
    """make_partition (schedule.cpp:31-54); a SyncStrategy gives partition_for (sync.cpp:131-141)."""
    s = _c_strategy(_as_strategy(cfg))
    W = max(s.world_size, 1)
    members = np.zeros(W, dtype=np.int32)
    offsets = np.zeros(W + 1, dtype=np.int32)
    n = C.c_int(0)
    _check_global(L.load().dss_partition(C.byref(s), t, members.ctypes.data, offsets.ctypes.data, C.byref(n)))
    groups = [members[offsets[g]:offsets[g + 1]].tolist() for g in range(n.value)]
    return GroupPartition(t, groups)


def group_of(cfg, t: int, rank: int) -> List[int]:  # schedule.cpp:56-65
    s = _c_strategy(_as_strategy(cfg))
    members = np.zeros(max(s.world_size, 1), dtype=np.int32)
    n = C.c_int(0)
    _check_global(L.load().dss_group_of(C.byref(s), t, rank, members.ctypes.data, C.byref(n)))
    return members[:n.value].tolist()


def check_mixing(cfg, t: int) -> bool:  # schedule.cpp:67-90
    s = _c_strategy(_as_strategy(cfg))
    r = L.load().dss_check_mixing(C.byref(s), t)
    if r < 0:
        _raise(-r, L.global_error())
    return r == 1


def placement(strategy: SyncStrategy, n_gpus: int, mode: int = 1, dim: int = 0, dtype: str = "f32"):
    """Worker placement of a context (dss_placement): (gpu_of, row_of, (gr, gc))
    for every global rank; (0, 0) is contiguous packing.  dim / dtype: the
    row size the auto mode considers (0: ignore)."""
    s = _c_strategy(strategy)
    W = strategy.world.world_size
    gpu = np.zeros(W, dtype=np.int32)
    row = np.zeros(W, dtype=np.int32)
    gr, gc = C.c_int(), C.c_int()
    dt = L.DSS_F64 if dtype in ("f64", np.float64) else L.DSS_F32
    _check_global(L.load().dss_placement(C.byref(s), n_gpus, mode, dim, dt, gpu.ctypes.data, row.ctypes.data,
                                         C.byref(gr), C.byref(gc)))
    return gpu.tolist(), row.tolist(), (gr.value, gc.value)


def round_outcome(strategy: SyncStrategy, t: int, payload_dim: int) -> SyncRoundOutcome:
    s = _c_strategy(strategy)
    o = L.dss_outcome()
    _check_global(L.load().dss_round_outcome(C.byref(s), t, payload_dim, C.byref(o)))
    return SyncRoundOutcome(o.critical_path_steps, o.total_messages)


# ---------------------------------------------------------------------------
class SamplingMode(enum.IntEnum):  # sync.hpp SamplingMode
    REPLACEMENT = 0
    EPOCH = 1


@dataclass
class Shard:  # problems.hpp Shard
    owner: int
    indices: List[int]


def logistic_dataset(seed: int, d: int, M: int):
    """LogisticProblem's synthetic data (problems.cpp:230-250), bit-exact:
    (x [M, d] float64, y [M] in {-1, +1})."""
    x = np.empty((M, d), dtype=np.float64)
    y = np.empty(M, dtype=np.float64)
    _check_global(L.load().dss_logistic_dataset(C.c_uint64(seed), d, M, x.ctypes.data, y.ctypes.data))
    return x, y


def quadratic_problem(seed: int, d: int, delta0: float):
    """QuadraticProblem (A = mu*I) optimum w* and start w0 (problems.cpp:157-165), bit-exact."""
    ws = np.empty(d, dtype=np.float64)
    w0 = np.empty(d, dtype=np.float64)
    _check_global(L.load().dss_quadratic_problem(C.c_uint64(seed), d, delta0, ws.ctypes.data, w0.ctypes.data))
    return ws, w0


def logistic_constants(x, y, l2: float):
    """LogisticProblem's smoothness, optimum and f* (problems.cpp:346-416), bit-exact:
    (smoothness, f_star or nan, w_opt or None)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    M, d = x.shape
    sm, fs = C.c_double(), C.c_double()
    w = np.empty(d, dtype=np.float64)
    _check_global(L.load().dss_logistic_constants(x.ctypes.data, y.ctypes.data, M, d, l2, C.byref(sm), C.byref(fs),
                                                  w.ctypes.data))
    return sm.value, fs.value, (w if l2 > 0.0 else None)


def mlp_dataset(seed: int, d: int, M: int):
    """TinyMlpProblem's data (problems.cpp:436-460), bit-exact: (x [M, d], y [M])."""
    x = np.empty((M, d), dtype=np.float64)
    y = np.empty(M, dtype=np.float64)
    _check_global(L.load().dss_mlp_dataset(C.c_uint64(seed), d, M, x.ctypes.data, y.ctypes.data))
    return x, y


def mlp_initial_params(seed: int, d: int, hidden: int) -> np.ndarray:
    """TinyMlpProblem::initial_params (problems.cpp:466-476), bit-exact."""
    w = np.empty(hidden * d + 2 * hidden + 1, dtype=np.float64)
    _check_global(L.load().dss_mlp_initial_params(C.c_uint64(seed), d, hidden, w.ctypes.data))
    return w


def make_shards(dataset_size: int, workers: int, seed: int) -> List[Shard]:  # problems.cpp:642-662
    idx = np.empty(max(dataset_size, 0), dtype=np.int32)
    off = np.empty(max(workers, 0) + 1, dtype=np.int32)
    _check_global(L.load().dss_make_shards(dataset_size, workers, C.c_uint64(seed), idx.ctypes.data,
                                           off.ctypes.data))
    return [Shard(w, idx[off[w]:off[w + 1]].tolist()) for w in range(workers)]


def epoch_order(shard: Shard, seed: int, rank: int, epoch: int) -> List[int]:  # problems.cpp:664-674
    a = np.ascontiguousarray(shard.indices, dtype=np.int32)
    out = np.empty_like(a)
    _check_global(L.load().dss_epoch_order(a.ctypes.data, a.size, C.c_uint64(seed), rank, epoch, out.ctypes.data))
    return out.tolist()


class DsSyncEngine:
    """Device-resident DS-Sync / BSP workers on one GPU (one context).

    This GPU's workers live in HBM as worker-major rows, in the order of
    ``local_ranks`` (``first_rank .. first_rank + local_workers - 1`` under
    contiguous packing; any subset of ranks under the tiled ``placement``,
    where ``first_rank`` is -1).  ``step`` runs one fused iteration on the
    device.
    """

    def __init__(self, strategy: SyncStrategy, optimizer: OptimizerKind, dim: int,
                 hp: Optional[OptimizerHyperparams] = None, dtype: str = "f32", device: int = 0,
                 rank: int = 0, n_gpus: int = 1, path: int = 0, stats_dim: int = 0, placement: int = 0):
        hp = hp or OptimizerHyperparams()
        self.lib = L.load()
        self.strategy = strategy
        self.optimizer = OptimizerKind(optimizer)
        self.dim = int(dim)
        self.dtype = np.float64 if dtype in ("f64", np.float64) else np.float32
        cfg = L.dss_config()
        cfg.strategy = _c_strategy(strategy)
        cfg.optimizer = int(optimizer)
        cfg.hp = L.dss_hparams(hp.momentum, hp.beta1, hp.beta2, hp.epsilon, hp.weight_decay)
        cfg.dtype = L.DSS_F64 if self.dtype == np.float64 else L.DSS_F32
        cfg.dim = self.dim
        cfg.device = device
        cfg.rank = rank
        cfg.n_gpus = n_gpus
        cfg.path = path
        cfg.stats_dim = stats_dim
        cfg.placement = placement
        self.stats_dim = int(stats_dim)
        h = C.c_void_p()
        st = self.lib.dss_create(C.byref(cfg), C.byref(h))
        if st != L.DSS_OK:
            _raise(st, L.global_error())
        self.h = h
        first, count = C.c_int(), C.c_int()
        self.lib.dss_local_workers(self.h, C.byref(first), C.byref(count))
        self.first_rank, self.local_workers = first.value, count.value
        ranks = np.zeros(max(count.value, 1), dtype=np.int32)
        self.lib.dss_local_ranks(self.h, ranks.ctypes.data)
        # global ranks of the local rows: the row order of upload_all / download_all
        self.local_ranks = ranks[:count.value].tolist()
        self.n_gpus = n_gpus
        self.rank = rank

    # -- lifecycle --
    def close(self):
        if getattr(self, "h", None):
            self.lib.dss_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, st: int):
        if st != L.DSS_OK:
            buf = C.create_string_buffer(2048)
            r, it = C.c_int(-1), C.c_long(-1)
            self.lib.dss_last_error(self.h, buf, len(buf), C.byref(r), C.byref(it))
            _raise(st, buf.value.decode(), r.value, it.value)

    # -- data movement --
    def _arr(self, x) -> np.ndarray:
        return np.ascontiguousarray(x, dtype=self.dtype)

    def _host_ptr(self, x, shape, what: str) -> int:
        """Address of a host buffer the library reads or writes in full.
        The C side copies prod(shape) elements of the engine's dtype, so the
        buffer must be exactly that: right shape, right dtype, C-contiguous."""
        if isinstance(x, np.ndarray):
            ok = x.shape == tuple(shape) and x.dtype == self.dtype and x.flags["C_CONTIGUOUS"]
            got = f"{x.dtype}{list(x.shape)}"
            ptr = x.ctypes.data
        elif hasattr(x, "data_ptr"):  # torch tensor (pinned host memory makes copies asynchronous)
            import torch
            want = torch.float64 if self.dtype == np.float64 else torch.float32
            ok = (tuple(x.shape) == tuple(shape) and x.dtype == want and x.is_contiguous()
                  and x.device.type == "cpu")
            got = f"{x.dtype}{list(x.shape)} on {x.device}"
            ptr = x.data_ptr()
        else:
            raise TypeError(f"{what}: expected a numpy array or a torch tensor")
        if not ok:
            raise ValueError(f"{what}: need a C-contiguous host {np.dtype(self.dtype).name}{list(shape)} "
                             f"buffer, got {got}")
        return ptr

    def upload(self, buffer: int, rank: int, host) -> None:
        a = self._arr(host)
        self._ck(self.lib.dss_upload(self.h, buffer, rank, a.ctypes.data, a.size))

    def _len(self, buffer: int) -> int:
        return self.stats_dim if buffer in (L.BUF_STATS, L.BUF_STATS_OBS) else self.dim

    def download(self, buffer: int, rank: int) -> np.ndarray:
        n = self._len(buffer)
        out = np.empty(n, dtype=self.dtype)
        self._ck(self.lib.dss_download(self.h, buffer, rank, out.ctypes.data, n))
        return out

    def upload_all(self, buffer: int, host) -> None:
        """host: [local_workers, row length] (pinned memory makes this asynchronous)."""
        shape = (self.local_workers, self._len(buffer))
        if isinstance(host, np.ndarray):
            host = self._arr(host)
            self._keep = host  # the copy may still be in flight when this returns
        self._ck(self.lib.dss_upload_all(self.h, buffer, self._host_ptr(host, shape, "upload_all")))

    def download_all(self, buffer: int, out=None) -> np.ndarray:
        shape = (self.local_workers, self._len(buffer))
        if out is None:
            out = np.empty(shape, dtype=self.dtype)
        self._ck(self.lib.dss_download_all(self.h, buffer, self._host_ptr(out, shape, "download_all")))
        return out

    def broadcast_row(self, buffer: int, row) -> None:
        a = self._arr(row)
        if a.shape != (self._len(buffer),):
            raise ValueError(f"broadcast_row: need a row of {self._len(buffer)} elements, got shape {a.shape}")
        self._ck(self.lib.dss_broadcast_row(self.h, buffer, a.ctypes.data))

    def device_ptr(self, buffer: int, rank: int) -> int:
        p = C.c_void_p()
        self._ck(self.lib.dss_device_ptr(self.h, buffer, rank, C.byref(p)))
        return p.value

    @property
    def row_stride(self) -> int:
        return self.lib.dss_row_stride(self.h)

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Run on exactly this cudaStream_t (0/None = legacy default stream)."""
        self._ck(self.lib.dss_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def set_step_count(self, rank: int, n: int) -> None:
        self._ck(self.lib.dss_set_step_count(self.h, rank, n))

    def step_count(self, rank: int) -> int:
        return self.lib.dss_get_step_count(self.h, rank)

    # -- hot path --
    def step(self, t: int, alpha: float, check: bool = False) -> SyncRoundOutcome:
        o = L.dss_outcome()
        self._ck(self.lib.dss_step(self.h, t, alpha, 1 if check else 0, C.byref(o)))
        return SyncRoundOutcome(o.critical_path_steps, o.total_messages)

    def steps(self, t0: int, alphas, check: bool = False) -> SyncRoundOutcome:
        """len(alphas) consecutive iterations from t0 in one library call."""
        a = np.ascontiguousarray(alphas, dtype=np.float64)
        o = L.dss_outcome()
        self._ck(self.lib.dss_steps(self.h, t0, a.size, a.ctypes.data, 1 if check else 0, C.byref(o)))
        return SyncRoundOutcome(o.critical_path_steps, o.total_messages)

    def step_host(self, t: int, alpha: float, host_grads, host_params) -> None:
        """dss_step_host: one iteration fed from / returned to pinned host
        buffers ([local_workers, dim]), copies pipelined across calls; the
        previous call's host_params are complete when this returns."""
        shape = (self.local_workers, self.dim)
        gp = self._host_ptr(host_grads, shape, "step_host grads")
        pp = self._host_ptr(host_params, shape, "step_host params")
        self._ck(self.lib.dss_step_host(self.h, t, alpha, C.c_void_p(gp), C.c_void_p(pp)))

    def host_sync(self) -> None:
        self._ck(self.lib.dss_host_sync(self.h))

    def sync_round(self, t: int, check: bool = True) -> SyncRoundOutcome:
        o = L.dss_outcome()
        self._ck(self.lib.dss_sync_round(self.h, t, 1 if check else 0, C.byref(o)))
        return SyncRoundOutcome(o.critical_path_steps, o.total_messages)

    def apply_step(self, alpha: float, check: bool = True) -> None:
        self._ck(self.lib.dss_apply_step(self.h, alpha, 1 if check else 0))

    def running_stats_update(self) -> None:
        """fold_running_stats (sync.cpp:193-201) from the BUF_STATS_OBS rows."""
        self._ck(self.lib.dss_running_stats_update(self.h))

    def quadratic_gradients(self, t: int, seed: int, mu: float, sigma: float) -> None:
        self._ck(self.lib.dss_quadratic_gradients(self.h, t, seed, mu, sigma))

    def quadratic_init(self, problem_seed: int, delta0: float) -> None:
        self._ck(self.lib.dss_quadratic_init(self.h, problem_seed, delta0))

    def set_optimum(self, wstar) -> None:
        a = self._arr(wstar)
        self._ck(self.lib.dss_set_optimum(self.h, a.ctypes.data, a.size))

    def global_mean(self) -> np.ndarray:
        """mean_of_ptrs over all W workers (param.cpp:59-70), bit-exact."""
        out = np.empty(self.dim, dtype=self.dtype)
        self._ck(self.lib.dss_global_mean(self.h, out.ctypes.data))
        return out

    def quadratic_losses(self, mu: float, with_suboptimality: bool = True, exact: bool = False):
        """(post_sync_loss of each local worker, full_loss at the last global mean).
        exact=True evaluates in the reference's sequential order (bit-exact)."""
        losses = np.empty(self.local_workers, dtype=np.float64)
        sub = C.c_double()
        self._ck(self.lib.dss_quadratic_losses(self.h, mu, 1 if exact else 0, losses.ctypes.data,
                                               C.byref(sub) if with_suboptimality else None))
        return losses, (sub.value if with_suboptimality else None)

    # -- logistic regression on the device (config C1) --
    def logistic_setup(self, x, y, l2: float, batch_size: int, sampling: int = SamplingMode.REPLACEMENT,
                       run_seed: int = 1) -> None:
        """Upload the dataset and shard it over the world (make_shards(M, W, run_seed))."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if x.ndim != 2 or x.shape[1] != self.dim or y.shape != (x.shape[0],):
            raise ValueError("logistic: x must be [M, dim] and y [M]")
        self._ck(self.lib.dss_logistic_setup(self.h, x.ctypes.data, y.ctypes.data, x.shape[0], l2, batch_size,
                                             int(sampling), C.c_uint64(run_seed)))
        self._logistic_batch = batch_size

    def logistic_gradients(self, t: int) -> None:
        self._ck(self.lib.dss_logistic_gradients(self.h, t))

    def logistic_steps(self, t0: int, alphas, check: bool = False) -> SyncRoundOutcome:
        """len(alphas) iterations of (device logistic gradient, step) from t0."""
        a = np.ascontiguousarray(alphas, dtype=np.float64)
        o = L.dss_outcome()
        self._ck(self.lib.dss_logistic_steps(self.h, t0, a.size, a.ctypes.data, 1 if check else 0, C.byref(o)))
        return SyncRoundOutcome(o.critical_path_steps, o.total_messages)

    # -- tiny MLP on the device (running statistics) --
    def mlp_setup(self, x, y, hidden: int, batch_size: int, sampling: int = SamplingMode.REPLACEMENT,
                  run_seed: int = 1) -> None:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if x.ndim != 2 or y.shape != (x.shape[0],):
            raise ValueError("tiny-mlp: x must be [M, d] and y [M]")
        self._ck(self.lib.dss_mlp_setup(self.h, x.ctypes.data, y.ctypes.data, x.shape[0], x.shape[1], hidden,
                                        batch_size, int(sampling), C.c_uint64(run_seed)))
        self._logistic_batch = batch_size

    def mlp_gradients(self, t: int) -> None:
        """Gradient rows and running-stat observations of every local worker."""
        self._ck(self.lib.dss_mlp_gradients(self.h, t))

    def mlp_losses(self, exact: bool = False) -> np.ndarray:
        out = np.empty(self.local_workers, dtype=np.float64)
        self._ck(self.lib.dss_mlp_losses(self.h, 1 if exact else 0, out.ctypes.data))
        return out

    def logistic_batch(self) -> np.ndarray:
        out = np.empty((self.local_workers, self._logistic_batch), dtype=np.int32)
        self._ck(self.lib.dss_logistic_batch(self.h, out.ctypes.data))
        return out

    def logistic_losses(self, exact: bool = False) -> np.ndarray:
        """full_loss (problems.cpp:292-305) of every local worker."""
        out = np.empty(self.local_workers, dtype=np.float64)
        self._ck(self.lib.dss_logistic_losses(self.h, 1 if exact else 0, out.ctypes.data))
        return out

    def check(self) -> None:
        self._ck(self.lib.dss_check(self.h))

    def check_guards(self) -> int:
        """Overwritten guard-band bytes (DSS_GUARD_BYTES debug mode); raises if any."""
        n = C.c_long()
        self._ck(self.lib.dss_check_guards(self.h, C.byref(n)))
        return n.value

    def clear_error(self) -> None:
        self._ck(self.lib.dss_clear_error(self.h))

    # -- timing / accounting --
    def enable_timing(self, on: bool = True) -> None:
        self.lib.dss_enable_timing(self.h, 1 if on else 0)

    def kernel_times(self):
        tot, n, mx = C.c_double(), C.c_long(), C.c_double()
        self._ck(self.lib.dss_kernel_times(self.h, C.byref(tot), C.byref(n), C.byref(mx)))
        return tot.value, n.value, mx.value

    def kernel_times_by_kind(self) -> dict:
        """{kind: (total_ms, launches)} since the last timing query."""
        ms = np.zeros(len(L.KIND_NAMES), np.float64)
        n = np.zeros(len(L.KIND_NAMES), np.int64)
        self._ck(self.lib.dss_kernel_times_by_kind(self.h, ms.ctypes.data, n.ctypes.data))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(L.KIND_NAMES)}

    @property
    def launch_count(self) -> int:
        return self.lib.dss_launch_count(self.h)

    # -- multi-GPU --
    def ipc_export(self) -> bytes:
        buf = C.create_string_buffer(L.IPC_BYTES)
        self._ck(self.lib.dss_ipc_export(self.h, buf))
        return buf.raw

    def ipc_attach(self, all_handles: Sequence[bytes]) -> None:
        blob = b"".join(all_handles)
        assert len(blob) == L.IPC_BYTES * self.n_gpus
        buf = C.create_string_buffer(blob, len(blob))
        self._ck(self.lib.dss_ipc_attach(self.h, buf))

    def barrier(self) -> None:
        self._ck(self.lib.dss_barrier(self.h))


# ---------------------------------------------------------------------------
# Host-resident drop-ins for the reference's free functions.  Same semantics
# as the reference (fp64); the arithmetic runs in the CUDA kernels.

def apply_step(state: OptimizerState, params, grad, device: int = 0) -> StepResult:
    """apply_step (optim.cpp:46-98) on the GPU: returns fresh params and state."""
    w = np.asarray(params, dtype=np.float64)
    g = np.asarray(grad, dtype=np.float64)
    if w.shape != g.shape:
        raise ValueError("apply_step: params and grad length mismatch")  # optim.cpp:30-32
    a = state.hp.alpha
    if not (a >= 0.0) or not np.isfinite(a):
        raise ValueError("apply_step: alpha must be finite and >= 0")  # optim.cpp:33-35
    for mom in (state.first_moment, state.second_moment):
        if mom is not None and len(mom) and len(mom) != len(w):
            raise ValueError("apply_step: moment buffer length mismatch")  # optim.cpp:36-41
    if w.size == 0:
        st = OptimizerState(state.kind, state.hp, state.first_moment, state.second_moment, state.step_count + 1)
        return StepResult(w.copy(), st)
    strat = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(1, 1))
    with DsSyncEngine(strat, state.kind, w.size, state.hp, "f64", device) as e:
        e.upload(L.BUF_PARAMS, 0, w)
        e.upload(L.BUF_GRADS, 0, g)
        kind = OptimizerKind(state.kind)
        if kind != OptimizerKind.VANILLA_SGD and state.first_moment is not None and len(state.first_moment):
            e.upload(L.BUF_MOMENT1, 0, state.first_moment)
        if kind in (OptimizerKind.ADAM, OptimizerKind.ADAMW) and state.second_moment is not None \
                and len(state.second_moment):
            e.upload(L.BUF_MOMENT2, 0, state.second_moment)
        e.set_step_count(0, state.step_count)
        try:
            e.apply_step(a, check=True)
        except DivergenceError as err:
            # the reference's apply_step throws std::runtime_error (optim.cpp:96)
            raise RuntimeError("apply_step: non-finite value in result") from err
        new = OptimizerState(kind, state.hp, None, None, state.step_count + 1)
        if kind != OptimizerKind.VANILLA_SGD:
            new.first_moment = e.download(L.BUF_MOMENT1, 0)
        if kind in (OptimizerKind.ADAM, OptimizerKind.ADAMW):
            new.second_moment = e.download(L.BUF_MOMENT2, 0)
        return StepResult(e.download(L.BUF_PARAMS, 0), new)


def sync_round(workers: List[WorkerState], strategy: SyncStrategy, t: int, device: int = 0) -> SyncRoundOutcome:
    """sync_round (sync.cpp:268-282) on the GPU: params and running_stats
    averaged inside the scheduled groups in place; optimizer state is never
    read or written."""
    validate(strategy)
    W = strategy.world.world_size
    if len(workers) != W:
        raise ValueError("sync_round: worker count does not match world_size")  # sync.cpp:271-273
    d = len(workers[0].params)
    sd = len(workers[0].running_stats)
    for ws in workers:  # check_collective_args on the concatenated payload (comm.cpp:56-72)
        if len(ws.params) + len(ws.running_stats) != d + sd:
            raise ValueError("collective vectors must all have the same length")
    if d + sd == 0:
        raise ValueError("collective vectors must be non-empty")
    if d == 0:  # a stats-only payload: fold it as the row
        d, sd = sd, 0
        rows = [np.asarray(ws.running_stats, dtype=np.float64) for ws in workers]
        stats_only = True
    else:
        rows = [np.asarray(ws.params, dtype=np.float64) for ws in workers]
        stats_only = False
    with DsSyncEngine(strategy, OptimizerKind.VANILLA_SGD, d, None, "f64", device, stats_dim=sd) as e:
        e.upload_all(L.BUF_PARAMS, np.stack(rows))
        if sd:
            e.upload_all(L.BUF_STATS, np.stack([np.asarray(ws.running_stats, dtype=np.float64) for ws in workers]))
        out = e.sync_round(t, check=True)
        res = e.download_all(L.BUF_PARAMS)
        st = e.download_all(L.BUF_STATS) if sd else None
    for k, ws in enumerate(workers):
        if stats_only:
            ws.running_stats = res[k].copy()
        else:
            ws.params = res[k].copy()
            if sd:
                ws.running_stats = st[k].copy()
    return out
