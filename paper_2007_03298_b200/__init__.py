"""B200-native DS-Sync (divide-and-shuffle synchronization, arXiv 2007.03298).

The hot path — fused apply_step + ordered group average (+ cross-GPU
two-shot over NVLink) — lives in the CUDA C-ABI library
``libdssync_b200.so`` (include/dssync_b200.h).  This package is its ctypes
binding plus a reference-shaped API (see api.py).
"""
from .api import (  # noqa: F401
    DivergenceError,
    DsSyncEngine,
    GroupPartition,
    IterationTrace,
    OptimizerHyperparams,
    OptimizerKind,
    OptimizerState,
    SamplingMode,
    Shard,
    StepResult,
    StrategyKind,
    SyncRoundOutcome,
    SyncStrategy,
    Topology,
    WorkerState,
    WorldConfig,
    apply_step,
    check_mixing,
    epoch_order,
    group_of,
    iteration_trace,
    logistic_constants,
    logistic_dataset,
    is_square_mode,
    make_partition,
    make_shards,
    mlp_dataset,
    mlp_initial_params,
    placement,
    quadratic_problem,
    round_outcome,
    sync_round,
    validate,
)
from ._lib import BUF_GRADS, BUF_MOMENT1, BUF_MOMENT2, BUF_PARAMS, BUF_STATS, BUF_STATS_OBS  # noqa: F401
