"""DS-Sync sync-iteration benchmark (BASELINE.json metric) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c4slice|c2sq|c1]
                    [--impl ours|reference] [--extras c3,c4slice,c2f64 | none]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step is one DS-Sync iteration of the hot path over the config's worker
buffers: every worker's fused optimizer step + ordered group average
(block groups on even t, comb groups on odd t), device-resident in HBM.
Default workload = BASELINE config C2 (W=8 workers, groups of 2 and 4,
25M-float buffers, vanilla SGD), all W workers packed over the N GPUs
(W/N per GPU, so N=1 holds all 8; scaling is strong: total work fixed).
BSP (ordered gradient fold + step) is measured on the same buffers.

The headline line also carries keyed results for the other BASELINE
configs that fit ("configs": C3, the C4 per-GPU slice, C2 in fp64 and C2's
size on the legal square shape W=16/N=4 at N=1; C3 and, from 4 GPUs, full
C4 at N>1), each with its own roofline and end-to-end number.

Prints ONE JSON line (rank 0).  --impl reference times the reference's own
CPU implementation (oracle/_ref = the unmodified reference sources) on the
box's host cores at the full workload size, without loading the product
library.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DS-Sync sync iters/s & effective GB/s vs BSP at 1/2/4/8 B200 (% of roofline)"

# BASELINE configs.  bytes/elem: algorithmic HBM bytes per
# worker-element per iteration (fp32; x2 for fp64): sgd 12, momentum 20, adam(w) 28.
CONFIGS = {
    "c1": dict(W=4, N=2, rect=False, d=20, opt=0, alpha=0.05, wd=0.0, logistic=True,
               desc="C1: W=4, 2 groups of 2 shuffled every iteration, d=20 (logistic size), vanilla SGD"),
    "c2": dict(W=8, N=2, rect=True, d=25_000_000, opt=0, alpha=0.05, wd=0.0,
               desc="C2: W=8 workers, DS-Sync groups of 2 (even t) / 4 (odd t), d=25,000,000 fp32 "
                    "(ResNet-50 size), vanilla SGD alpha=0.05"),
    "c3": dict(W=32, N=4, rect=True, d=36_500_000, opt=1, alpha=0.1, wd=1e-4,
               desc="C3: W=32 virtual workers, groups of 4 (even) / 8 (odd), d=36,500,000 fp32 "
                    "(WideResNet-28-10 size), SGD-momentum 0.9 wd=1e-4"),
    "c4": dict(W=64, N=8, rect=False, d=340_000_000, opt=3, alpha=3e-5, wd=0.01,
               desc="C4: W=64 virtual workers, groups of 8, d=340,000,000 fp32 (BERT-large size), AdamW"),
    # C2's buffer size on a shape the reference itself accepts (W = N^2):
    # every group index of this line is pinned by the reference's make_partition
    "c2sq": dict(W=16, N=4, rect=False, d=25_000_000, opt=0, alpha=0.05, wd=0.0,
                 desc="C2 size on a legal square shape: W=16 workers, groups of 4 (blocks / combs), d=25,000,000 "
                      "fp32, vanilla SGD alpha=0.05"),
    # one GPU's share of C4's block iteration: 8 workers, one group of 8, AdamW
    "c4slice": dict(W=8, N=8, rect=False, d=340_000_000, opt=3, alpha=3e-5, wd=0.01,
                    desc="C4 per-GPU slice: 8 workers in one group of 8, d=340,000,000 fp32, AdamW"),
}
BYTES_PER_ELEM = {0: 12, 1: 20, 2: 28, 3: 28}
OPT_NAMES = ["vanilla-sgd", "sgd-momentum", "adam", "adamw"]
NVLINK_PEAK = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def config_dict(cfg, G):
    """The `config` object, identical in both arms for the same --config/--gpus."""
    W, N, d = cfg["W"], cfg["N"], cfg["d"]
    P = W // G
    return {"workload": cfg["desc"], "W": W, "N": N, "d": d, "optimizer": OPT_NAMES[cfg["opt"]],
            "rectangular": cfg["rect"], "workers_per_gpu": P, "parallelism": f"dp{G} (W/G workers per GPU)",
            "l2": (f"inputs larger than L2: {P * d * 4 / 1e6:.0f} MB per array per GPU" if P * d * 4 > 126e6
                   else "inputs smaller than L2 (latency-bound config)")}


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem = None
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable"):
                    mem = int(ln.split()[1]) * 1024
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "mem_available_gb": round(mem / 1e9, 1) if mem else None}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(1.0)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        samples = [ln for (ts, ln) in self.lines if t0 - 0.06 <= ts <= t1 + 0.06] or [ln for _, ln in self.lines[-3:]]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in samples:
            parts = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                for n, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# The reference's CPU path (oracle/_ref: the unmodified reference sources
# compiled by oracle/Makefile + oracle/ref_shim.cpp).  Nothing here loads the
# product library.
class RefBench:
    """apply_step for every worker (threaded like run_training's Parallel
    mode, sync.cpp:348-362) + each group's ring_allreduce_avg on the
    concatenated payload, written back (sync.cpp:203-240, 364-370), on
    resident fp64 WorkerStates (the reference is fp64-only)."""

    def __init__(self, cfg, d, threads):
        from oracle.oracle import Reference
        self.R = R = Reference()
        self.cfg, self.d, self.threads = cfg, d, threads
        self.err = C.create_string_buffer(512)
        hp = R.hp_array(weight_decay=cfg["wd"])
        self.h = R.lib.ref_bench_create(cfg["W"], d, cfg["opt"], hp.ctypes.data, 1, threads)
        self.tables = [self._table(p) for p in (0, 1)]

    def _table(self, t):
        W = self.cfg["W"]
        m = np.zeros(W, np.int32)
        o = np.zeros(W + 1, np.int32)
        n = C.c_int()
        rc = self.R.lib.ref_bench_partition(W, self.cfg["N"], int(self.cfg["rect"]), t, m.ctypes.data, o.ctypes.data,
                                            C.byref(n), self.err, 512)
        if rc:
            raise RuntimeError(self.err.value.decode())
        return m, o, n.value

    def ds(self, t):
        m, o, n = self.tables[t & 1]
        rc = self.R.lib.ref_bench_ds_step(self.h, t, self.cfg["alpha"], m.ctypes.data, o.ctypes.data, n,
                                          self.threads, self.err, 512)
        if rc:
            raise RuntimeError(self.err.value.decode())

    def bsp(self, t):
        rc = self.R.lib.ref_bench_bsp_step(self.h, t, self.cfg["alpha"], self.threads, self.err, 512)
        if rc:
            raise RuntimeError(self.err.value.decode())

    def stock(self, t, N):
        rc = self.R.lib.ref_bench_stock_step(self.h, N, t, self.cfg["alpha"], self.threads, self.err, 512)
        if rc:
            raise RuntimeError(self.err.value.decode())

    def close(self):
        if self.h:
            self.R.lib.ref_bench_destroy(self.h)
            self.h = None


def ref_d(cfg):
    """Largest d the host can hold for the reference bench: the full config
    d unless memory forbids (C4 in fp64 needs ~700 GB)."""
    nvec = 2 + {0: 0, 1: 1, 2: 2, 3: 2}[cfg["opt"]]
    threads = os.cpu_count() or 1
    # resident W x (params, grads, moments) + apply_step's copies in flight
    per_elem = 8 * (cfg["W"] * nvec + min(threads, cfg["W"]) * (nvec - 1) + cfg["W"] // max(cfg["N"], 1) * 2)
    avail = (host_info()["mem_available_gb"] or 32.0) * 1e9 * 0.6
    return cfg["d"] if per_elem * cfg["d"] <= avail else int(avail // per_elem) // 64 * 64


def time_ref(rb, fn, k0, K, budget_s=None):
    """Per-iteration wall times of fn(t) for t = k0.. (all K, or until budget_s)."""
    times = []
    for t in range(k0, k0 + K):
        t0 = time.perf_counter()
        fn(t)
        times.append(time.perf_counter() - t0)
        if budget_s is not None and sum(times) > budget_s and len(times) >= 2:
            break
    return times


def reference_arm(args, cfg):
    """--impl reference: the reference's own CPU path at the full workload
    size on every host core; rank 0 only (other ranks exit 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle.oracle import REF_SO
    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdssync_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    d = ref_d(cfg)
    scaled = d != cfg["d"]
    rb = RefBench(cfg, d, threads)
    try:
        for t in range(args.warmup):
            rb.ds(t)
        ts = time_ref(rb, rb.ds, args.warmup, args.steps)
        ms = 1000.0 * sum(ts) / len(ts)
        nb = min(args.steps, 5)
        tb = time_ref(rb, rb.bsp, 0, nb)
        ms_bsp = 1000.0 * sum(tb) / len(tb)
    finally:
        rb.close()
    scale = d / cfg["d"]  # 1.0 unless the host cannot hold the workload
    value = 1000.0 / ms * scale
    sample = (f"the full workload: W={cfg['W']} workers x d={d:,} fp64 (the reference is fp64-only), "
              f"{len(ts)} timed DS iterations after {args.warmup} warm-up, {threads} threads"
              if not scaled else
              f"size-scaled (host memory): W={cfg['W']} x d={d:,} of d={cfg['d']:,} fp64, {len(ts)} timed DS "
              f"iterations, iters/s scaled by {d}/{cfg['d']}")
    out = {
        "metric": METRIC, "value": value, "unit": "iters/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": len(ts), "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter-addressed "
        "reference Rng streams; fixed gradients, as in our arm)",
        "config": config_dict(cfg, args.gpus),
        "effective_gbs": cfg["W"] * cfg["d"] * 4 / (1.0 / value) / 1e9,
        "bsp": {"iters_s": 1000.0 / ms_bsp * scale, "ms_per_step": ms_bsp / scale, "steps": nb},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": host_info(),
        "path": "oracle/_ref (unmodified /root/reference/proj/src): apply_step per worker on a thread pool + "
                "ring_allreduce_avg per group (groups in parallel, run_training's Parallel mode)",
    }
    if args.config == "c2" and not scaled:
        out["stock_sync_round_legal_shape"] = stock_legal_shape(cfg, threads)
    print(json.dumps(out))


def stock_legal_shape(cfg, threads, steps=3):
    """The stock reference iteration on the nearest legal shape (C2's
    rectangular W=8/N=2 is rejected by validate, schedule.cpp:8-24): W=4,
    N=2 at the same d, apply_step on a thread pool + the reference's own
    single-threaded sync_round (sync.cpp:268-282)."""
    c = dict(cfg, W=4, N=2, rect=False)
    rb = RefBench(c, cfg["d"], threads)
    try:
        rb.stock(0, 2)
        ts = time_ref(rb, lambda t: rb.stock(t, 2), 1, steps)
    finally:
        rb.close()
    ms = 1000.0 * sum(ts) / len(ts)
    return {"iters_s": 1000.0 / ms, "ms_per_step": ms, "steps": len(ts),
            "shape": f"W=4 workers, N=2 (legal square shape), d={cfg['d']:,} fp64, {OPT_NAMES[cfg['opt']]}",
            "note": "stock sync_round + apply_step of the unmodified reference; labelled, not the headline shape"}


def cpu_baseline(cfg, seconds=12.0):
    """cpu_baseline leg of our arm: the same reference CPU path at the full
    config d when the host can hold it (size-scaled and labelled otherwise),
    bounded to ~`seconds` of DS iterations after one warm-up iteration."""
    from oracle.oracle import REF_SO
    if not os.path.exists(REF_SO):
        return {"value": None, "unit": "iters/s", "cores": 0, "kind": "reference", "sample": "oracle/_ref missing"}
    threads = os.cpu_count() or 1
    d = ref_d(cfg)
    rb = RefBench(cfg, d, threads)
    try:
        rb.ds(0)
        ts = time_ref(rb, rb.ds, 1, 1000, budget_s=seconds)
    finally:
        rb.close()
    el = sum(ts)
    value = len(ts) / el * d / cfg["d"]
    if d == cfg["d"]:
        sample = (f"{len(ts)} DS iterations of the full workload (W={cfg['W']} x d={d:,} fp64) in {el:.1f} s "
                  f"on {threads} threads (reference apply_step + ring_allreduce_avg)")
    else:
        sample = (f"size-scaled (host memory): {len(ts)} DS iterations of W={cfg['W']} x d={d:,} fp64 in "
                  f"{el:.1f} s on {threads} threads, iters/s scaled by {d}/{cfg['d']}")
    return {"value": value, "unit": "iters/s", "cores": threads, "kind": "reference", "sample": sample}


def cpu_run_training_c1():
    """The reference's own `dssync run` on config C1 (acceptance.cpp:239-258:
    logistic d=20, M=2000, l2=0.05, batch 8, W=4 groups of 2, 300
    iterations, step-decay lr), timed on the host: run_training with its
    per-iteration trace (two full losses per worker)."""
    import tempfile
    from oracle.oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        return None
    cfg = {"strategy": "ds-sync", "world_size": 4, "group_size": 2, "iterations": 300, "batch_size": 8,
           "seeds": [1], "problem": {"kind": "logistic", "d": 20, "M": 2000, "mu": 0.05, "seed": 11},
           "lr": {"kind": "step-decay", "alpha": 1.0, "factor": 0.5, "every": 75}}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c1.json")
        with open(path, "w") as f:
            json.dump(cfg, f)
        t0 = time.perf_counter()
        rc, msg, _, _ = Reference().cmd_run(path, os.path.join(tmp, "out"))
        el = time.perf_counter() - t0
    if rc:
        return None
    return {"iters_s": 300 / el, "cores": 1,
            "note": "the reference's `dssync run` on C1 (run_training lockstep, with its per-iteration trace), "
                    "host, one thread"}


# ---------------------------------------------------------------------------
def gpu_map(cfg, G, placement, esz=4):
    """gpu_of / row_of of every global rank for the DS engines (dss_placement)."""
    from paper_2007_03298_b200 import StrategyKind, SyncStrategy, Topology, WorldConfig
    from paper_2007_03298_b200 import placement as place
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(cfg["W"], cfg["N"]), 1, cfg["rect"])
    gpu, row, tiling = place(s, G, placement, cfg["d"], "f64" if esz == 8 else "f32")
    return gpu, row, tiling


def step_bytes(cfg, G, rank, d_pad, path=0, esz=4, placement=0):
    """Algorithmic bytes one GPU moves per DS / BSP iteration, by kernel kind,
    averaged over the two schedule parities (block / comb iterations).
      group: fused apply_step + fold of local groups, d * bytes_per_elem per
             member (members of spanning groups are stepped inside the push /
             one-shot / chain kernels; only the unfused pull path, path 3,
             steps them in place with the group kernel)
      fold:  two-shot owner slice L over m members: reads m*L*esz, writes
             m*L*esz; the part touching other GPUs' rows crosses NVLink.
      chain: rank-0 outbound rows of its chain roles (partial + mean)."""
    from paper_2007_03298_b200 import StrategyKind, SyncStrategy, Topology, WorldConfig, make_partition
    W, N, d = cfg["W"], cfg["N"], cfg["d"]
    bpe = BYTES_PER_ELEM[cfg["opt"]] * esz // 4
    P = W // G
    gpu_of = gpu_map(cfg, G, placement, esz)[0]
    mine = {k for k in range(W) if gpu_of[k] == rank}
    z = {"group": 0.0, "fold_hbm": 0.0, "fold_nvlink": 0.0, "chain_nvlink": 0.0, "chain_mean_nvlink": 0.0,
         "chain_hbm": 0.0}
    out = {"ds": dict(z), "bsp": dict(z)}
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, cfg["rect"])
    chunks = d_pad // 64

    def chain_out(gpus):
        # rank's outbound rows in the partial-pass kernel (every stage sends
        # one: the partial, or the mean from the last stage) and in the
        # mean-pass kernel (a forwarded mean, stages 0..S-3)
        S, j = len(gpus), gpus.index(rank)
        return d * esz, (d * esz if j < S - 2 else 0)

    for p in (0, 1):
        for g in make_partition(s, p).groups:
            here = [m for m in g if m in mine]
            if not here:
                continue
            gpus = sorted({gpu_of[m] for m in g})
            if len(gpus) == 1 or path == 3:
                out["ds"]["group"] += 0.5 * len(here) * d * bpe
            if len(gpus) == 1:
                continue
            if max(sum(1 for m in g if gpu_of[m] == q) for q in gpus) >= 2:  # ordered chain
                a_bytes, b_bytes = chain_out(gpus)
                out["ds"]["chain_nvlink"] += 0.5 * a_bytes
                out["ds"]["chain_mean_nvlink"] += 0.5 * b_bytes
                # partial-pass HBM bytes: the fused step of the members here
                # (every array but the params write), the received partial
                # (stages > 0), the mean into the members here (last stage)
                S, j = len(gpus), gpus.index(rank)
                hb = len(here) * d * (bpe - esz) + (d * esz if j > 0 else 0) + \
                    (len(here) * d * esz if j == S - 1 else 0)
                out["ds"]["chain_hbm"] += 0.5 * hb
                continue
            S, j = len(gpus), gpus.index(rank)
            L = (chunks // S + (1 if j < chunks % S else 0)) * 64
            out["ds"]["fold_hbm"] += 0.5 * 2 * len(here) * L * esz
            out["ds"]["fold_nvlink"] += 0.5 * 2 * (len(g) - len(here)) * L * esz
    if G == 1:
        out["bsp"]["group"] = W * d * bpe
    elif P >= 2:
        out["bsp"]["chain_nvlink"], out["bsp"]["chain_mean_nvlink"] = chain_out(list(range(G)))
        out["bsp"]["group"] = P * d * bpe
    else:
        L = (chunks // G + (1 if rank < chunks % G else 0)) * 64
        out["bsp"]["fold_hbm"] = (P + 1) * L * esz
        out["bsp"]["fold_nvlink"] = ((W - P) + (G - 1)) * L * esz
        out["bsp"]["group"] = P * d * bpe
    return out


class NcclBaseline:
    """Comparison baselines only (not bit-exact: NCCL's sum order is not the
    ascending fold).  DS: our in-place apply_step, then per group a local
    pre-sum of this GPU's member rows, one ncclAllReduce per distinct GPU set
    (torch.distributed.new_group -> ncclCommSplit), x 1/m, copy back.
    BSP: local pre-sum of the gradients, world ncclAllReduce, x 1/W, copy into
    every local gradient row, our apply_step.

    Copy-free where the layout allows: the local rows are one strided view
    of the engine's contiguous [P][row_stride] allocation, so the pre-sum is
    a single reduction over that view and a group's members are written back
    with one broadcast copy; a GPU holding exactly one member of every group
    all-reduces its own row in place."""

    def __init__(self, e, cfg, G, rank, placement=0):
        import torch
        import torch.distributed as dist
        from paper_2007_03298_b200 import (BUF_GRADS, BUF_PARAMS, StrategyKind, SyncStrategy, Topology,
                                           WorldConfig, make_partition)
        self.e, self.cfg, self.G, self.rank = e, cfg, G, rank
        W, N, d = cfg["W"], cfg["N"], cfg["d"]
        P = W // G
        self.P = P
        gpu_of, row_of, _ = gpu_map(cfg, G, placement)
        first = e.local_ranks[0]  # local row 0
        stride = e.row_stride
        self.params = self._view(e, BUF_PARAMS, first, P, stride)[:, :d]
        self.grads = self._view(e, BUF_GRADS, first, P, stride)[:, :d]
        s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, cfg["rect"])
        self.plans = []
        comms = {}
        for p in (0, 1):
            by_set = {}
            for g in make_partition(s, p).groups:
                gpus = tuple(sorted({gpu_of[m] for m in g}))
                by_set.setdefault(gpus, []).append(g)
            plan = []
            for gpus, groups in sorted(by_set.items()):
                if gpus not in comms:
                    comms[gpus] = dist.new_group(list(gpus)) if len(gpus) > 1 else None
                if rank in gpus:
                    local = [self._rows([row_of[m] for m in g if gpu_of[m] == rank]) for g in groups]
                    plan.append((comms[gpus], groups, local))
            self.plans.append(plan)
        self.acc = torch.empty(d, dtype=torch.float32, device="cuda")
        self.torch, self.dist = torch, dist

    @staticmethod
    def _rows(idx):
        """A group's local member rows as a basic slice (a view, no gather):
        blocks are consecutive rows, combs every N-th row."""
        if len(idx) == 1:
            return idx[0]
        step = idx[1] - idx[0]
        assert all(b - a == step for a, b in zip(idx, idx[1:])), idx
        return slice(idx[0], idx[-1] + 1, step)

    @staticmethod
    def _view(e, buf, first, P, stride):
        import torch

        class _A:
            def __init__(self, ptr):
                self.__cuda_array_interface__ = {"shape": (P, stride), "typestr": "<f4", "data": (ptr, False),
                                                 "version": 3}
        return torch.as_tensor(_A(e.device_ptr(buf, first)), device="cuda")

    def ds_step(self, t, alpha):
        torch, dist = self.torch, self.dist
        self.e.apply_step(alpha, check=False)
        for comm, groups, local in self.plans[t & 1]:
            for g, lg in zip(groups, local):
                if isinstance(lg, int):  # one member here: all-reduce its row in place
                    rows = self.params[lg]
                else:  # several: one strided reduction into the accumulator
                    torch.sum(self.params[lg], dim=0, out=self.acc)
                    rows = self.acc
                if comm is not None:
                    dist.all_reduce(rows, group=comm)
                rows.mul_(1.0 / len(g))
                if not isinstance(lg, int):
                    dst = self.params[lg]
                    dst.copy_(rows.expand_as(dst))  # one broadcast copy into every local member
        return None

    def bsp_step(self, t, alpha):
        torch, dist = self.torch, self.dist
        torch.sum(self.grads, dim=0, out=self.acc)
        dist.all_reduce(self.acc)
        self.acc.mul_(1.0 / self.cfg["W"])
        self.grads.copy_(self.acc.expand_as(self.grads))
        self.e.apply_step(alpha, check=False)


def dominant_roofline(kinds_rows, ms_step, peak, peak_kind, G, chain_hbm=0.0):
    """Roofline of the kernel with the most time in the step.  HBM kernels
    (group / bsp) against the measured copy peak; cross-GPU kernels (fold =
    push / pull two-shot and one-shot, chain = the ordered chain's partial +
    mean passes) against the measured NVLink peer-copy peak per direction."""
    cand = {}
    for k, v in kinds_rows.items():
        if k in ("group", "bsp") and v.get("alg_bytes_per_step"):
            cand[k] = ("hbm", v["ms_per_step"], v["launches_per_step"], v["alg_bytes_per_step"])
        elif k == "fold" and v.get("nvlink_bytes_per_step"):
            cand[k] = ("nvlink", v["ms_per_step"], v["launches_per_step"], v["nvlink_bytes_per_step"])
        elif k == "chain" and v.get("nvlink_bytes_per_step"):
            # the partial-pass kernel carries the rank's outbound row of each
            # chain role and the fused member steps: a fused step + collective
            # kernel, bounded by the slower of its HBM and NVLink bytes
            # (B200_PROFILING.md); the mean pass is its own kernel, reported
            # in its own row
            link_t = v["nvlink_bytes_per_step"] / (NVLINK_PEAK * 1e9)
            hbm_t = chain_hbm / (peak * 1e9)
            if hbm_t > link_t:
                cand[k] = ("hbm", v["ms_per_step"], v["launches_per_step"], chain_hbm)
            else:
                cand[k] = ("nvlink", v["ms_per_step"], v["launches_per_step"], v["nvlink_bytes_per_step"])
    if not cand:
        return None
    k, (bound, ms_, n_, b_) = max(cand.items(), key=lambda kv: kv[1][1])
    per_ms, per_b = ms_ / n_, b_ / n_
    ach = per_b / (per_ms / 1e3) / 1e9 if per_ms else None
    names = {"group": "ds_group_kernel (fused apply_step + ordered fold + broadcast)",
             "bsp": "bsp_kernel (fused ordered gradient fold + step)",
             "fold": "push_twoshot / one-shot / fold_kernel (fused step + ordered fold over NVLink peers)",
             "chain": "chain_partial_kernel + chain_mean_kernel (ordered chain fold with the step fused)"}
    pk = peak if bound == "hbm" else NVLINK_PEAK
    r = {"bound": bound, "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk if ach else None,
         "traffic": None, "peak_kind": peak_kind if bound == "hbm" else
         "measured NVLink peer copy per direction (B200_PROFILING.md); 900 GB/s nominal",
         "kernel": names.get(k, k), "kind": k, "avg_launch_ms": per_ms, "alg_bytes_per_launch": per_b,
         "share_of_step": ms_ / ms_step if ms_step else None}
    if bound == "nvlink" and ach:
        r["frac_of_nominal_900"] = ach / 900.0
    return r


def measure(args, cfg, dtype, G, rank, local, stream, full=True, nccl_only=False):
    """DS + BSP iterations of one config on this rank's engine(s) (or, with
    nccl_only, the NCCL baselines of the same rows).  Returns the per-rank
    measurements (times already max-over-ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2007_03298_b200 import (BUF_GRADS, DsSyncEngine, OptimizerHyperparams, OptimizerKind,
                                       StrategyKind, SyncStrategy, Topology, WorldConfig)
    W, N, d = cfg["W"], cfg["N"], cfg["d"]
    P = W // G
    esz = 8 if dtype == "f64" else 4
    hp = OptimizerHyperparams(weight_decay=cfg["wd"])

    def make(kind):
        s = SyncStrategy(kind, Topology.RING, WorldConfig(W, N if kind == StrategyKind.DS_SYNC else W), 1,
                         cfg["rect"] and kind == StrategyKind.DS_SYNC)
        e = DsSyncEngine(s, OptimizerKind(cfg["opt"]), d, hp, dtype, local, rank, G, path=args.path,
                         placement=args.placement if kind == StrategyKind.DS_SYNC else 0)
        e.set_stream(stream.cuda_stream)
        if G > 1:
            from paper_2007_03298_b200.dist import attach
            attach(e)
        e.quadratic_init(7, 4.0)
        e.quadratic_gradients(0, 1, 1.0, 0.5)
        torch.cuda.synchronize()
        return e

    def max_over_ranks(x):
        if G == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def timed(fn, k0, K, batched=None):
        if G > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if batched is not None:
            batched(k0, K)  # K iterations in one library call (dss_steps)
        else:
            for t in range(k0, k0 + K):
                fn(t)
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b)) / K

    res = {}
    if nccl_only:
        # The NCCL baselines run in their own pass after all of our
        # measurements, over fresh engines: a run of our kernels right after
        # NCCL all-reduces in the same process is intermittently up to 2x
        # slower (small rows across GPUs: profiles/r02/sweeps/nccl_order_g2.md)
        for kind, name in ((StrategyKind.DS_SYNC, "ds"), (StrategyKind.BSP, "bsp")):
            e = make(kind)
            nb = NcclBaseline(e, cfg, G, rank, args.placement if name == "ds" else 0)
            fn = (lambda t: nb.ds_step(t, cfg["alpha"])) if name == "ds" else (lambda t: nb.bsp_step(t, cfg["alpha"]))
            for t in range(3):
                fn(t)
            res["nccl_" + name] = timed(fn, 3, max(3, args.steps // 2))
            del nb
            e.close()
            del e
            torch.cuda.synchronize()
        return res
    clocks = ClockSampler(local)  # every config: its timed region's clocks and throttle reasons
    for kind, name in ((StrategyKind.DS_SYNC, "ds"), (StrategyKind.BSP, "bsp")):
        e = make(kind)
        l0 = e.launch_count
        step = lambda t: e.step(t, cfg["alpha"])  # noqa: E731
        steps = lambda k0, K: e.steps(k0, np.full(K, cfg["alpha"]))  # noqa: E731
        for t in range(args.warmup):
            step(t)
        e.check()
        if clocks and name == "ds":
            clocks.start()
            tc0 = time.time()
        ms = timed(step, args.warmup, args.steps, batched=steps)
        if clocks and name == "ds":
            res["clocks"] = clocks.stop(tc0, time.time())
        launches = (e.launch_count - l0) / (args.warmup + args.steps)
        # second pass: every hot kernel bracketed by events on its stream
        e.enable_timing(True)
        timed(step, args.warmup + args.steps, args.steps, batched=steps)
        kinds = e.kernel_times_by_kind()
        e.enable_timing(False)
        e.check()
        res[name] = dict(ms=ms, kinds={k: (v[0] / args.steps, v[1] / args.steps) for k, v in kinds.items()},
                         launches_per_step=launches)
        host_gb = (host_info()["mem_available_gb"] or 64.0) * 1e9
        pinned = 2 * P * d * esz * G
        cap = 0.5 * host_gb if full else min(0.5 * host_gb, 64e9)  # keyed extras: bounded host pinning
        if name == "ds" and not args.no_e2e and pinned > cap:
            res["e2e_skipped"] = (f"pinned host buffers of {pinned / 1e9:.0f} GB across the ranks exceed the "
                                  f"{cap / 1e9:.0f} GB cap (half the host's {host_gb / 1e9:.0f} GB; 64 GB for keyed "
                                  f"configs)")
        elif name == "ds" and not args.no_e2e:
            # e2e through the C-ABI with host buffers: pinned H2D of every
            # local worker's gradient, the step, D2H of every worker's params
            # (dss_step_host: copies on two copy streams, the D2H of step t
            # overlapping the H2D of step t+1)
            big = P * d * esz > (1 << 30)
            K2 = max(3, min(args.steps, args.e2e_steps if big else args.steps))
            if big:
                # the copy pipeline fills and drains once per timed run (the
                # first H2D and the last D2H overlap nothing): K steps reach
                # at most K / (K + 1) of the bidirectional ceiling (5 steps:
                # 0.84), so large rows get 16 steps (C4 slice: ~4 s)
                K2 = min(K2, 16)
            tdt = torch.float64 if dtype == "f64" else torch.float32
            hg = torch.empty((P, d), dtype=tdt, pin_memory=True)
            hw = torch.empty((P, d), dtype=tdt, pin_memory=True)
            e.download_all(BUF_GRADS, hg)

            def e2e_run(k0, K):
                for t in range(k0, k0 + K):
                    e.step_host(t, cfg["alpha"], hg, hw)
                e.host_sync()  # the last iteration's params are on the host
            t_e2e = args.warmup + 2 * args.steps
            e2e_run(t_e2e, 1 if big else args.warmup)  # sets up the copy streams and the snapshot rows
            res["e2e_ms"] = timed(None, t_e2e + args.warmup, K2, batched=e2e_run)
            res["e2e_steps"] = K2
            e.check()
            try:
                res["pcie"] = pcie_ceiling(hg, hw)
            except RuntimeError as ex:  # out of device memory on a packed config: no ceiling, no failure
                res["pcie_error"] = str(ex).splitlines()[0]
            del hg, hw
        e.close()
        del e
        torch.cuda.synchronize()
    d_pad = (d + 63) // 64 * 64
    res["bytes"] = step_bytes(cfg, G, rank, d_pad, args.path, esz, args.placement)
    return res


def pcie_ceiling(hg, hw, reps=5):
    """The e2e leg's own ceiling: pinned-host copies of this rank's gradient
    and param buffers (up to 1 GiB each) by the copy engines, H2D alone, D2H
    alone and both at once on two streams (what dss_step_host overlaps),
    GB/s per direction, after the timed region."""
    import torch
    n = min(hg.numel(), (1 << 30) // hg.element_size())
    src, dst = hg.view(-1)[:n], hw.view(-1)[:n]
    da = torch.empty(n, dtype=hg.dtype, device="cuda")
    db = torch.empty(n, dtype=hg.dtype, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    da.copy_(src, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    dst.copy_(db, non_blocking=True)
        torch.cuda.synchronize()
        return reps * n * hg.element_size() / (time.perf_counter() - t0) / 1e9

    run(True, True)  # warm-up
    out = {"h2d_gbs": run(True, False), "d2h_gbs": run(False, True), "bidir_gbs_per_direction": run(True, True),
           "bytes_per_copy": n * hg.element_size()}
    del da, db
    return out


def summarize(args, cfg, dtype, G, res, peak, peak_kind):
    """The result object of one config (rank 0)."""
    W, N, d = cfg["W"], cfg["N"], cfg["d"]
    P = W // G
    esz = 8 if dtype == "f64" else 4
    ds, bsp = res["ds"], res["bsp"]
    nb_bytes = res["bytes"]
    bpe = BYTES_PER_ELEM[cfg["opt"]] * esz // 4

    def kernel_rows(r, key):
        rows = {}
        for k, (ms_, n_) in r["kinds"].items():
            if n_ == 0:
                continue
            row = {"ms_per_step": ms_, "launches_per_step": n_}
            if k == "group" or k == "bsp":
                b = nb_bytes[key]["group"]
                row.update(alg_bytes_per_step=b, hbm_gbs=b / (ms_ / 1e3) / 1e9 if ms_ else None)
            elif k == "fold":
                row.update(alg_bytes_per_step=nb_bytes[key]["fold_hbm"] + nb_bytes[key]["fold_nvlink"],
                           nvlink_bytes_per_step=nb_bytes[key]["fold_nvlink"],
                           nvlink_gbs=nb_bytes[key]["fold_nvlink"] / (ms_ / 1e3) / 1e9 if ms_ else None)
            elif k == "chain_mean":
                b = nb_bytes[key]["chain_mean_nvlink"]
                row.update(nvlink_bytes_per_step=b, nvlink_gbs=b / (ms_ / 1e3) / 1e9 if ms_ and b else None,
                           note="mean pass of the chain (rank 0): copies the received mean to the other local "
                                "members; forwards it on middle stages")
            elif k == "chain":
                b = nb_bytes[key]["chain_nvlink"]
                hb = nb_bytes[key]["chain_hbm"]
                row.update(nvlink_bytes_per_step=b, nvlink_gbs=b / (ms_ / 1e3) / 1e9 if ms_ else None,
                           hbm_bytes_per_step=hb or None, hbm_gbs=hb / (ms_ / 1e3) / 1e9 if ms_ and hb else None,
                           note="partial pass (rank 0): fused member step + ordered fold + one outbound row per "
                                "chain role (the partial, or the mean from the last stage)")
            rows[k] = row
        return rows

    ds_k = kernel_rows(ds, "ds")
    roof = dominant_roofline(ds_k, ds["ms"], peak, peak_kind, G, nb_bytes["ds"]["chain_hbm"])
    # the HBM kernel is always reported too (at N > 1 it may not dominate)
    hbm = dominant_roofline({k: v for k, v in ds_k.items() if k in ("group", "bsp")}, ds["ms"], peak, peak_kind, G)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof) and roof:
        try:
            tr = json.load(open(prof)).get(f"{cfg.get('key', args.config)}{'_f64' if esz == 8 else ''}_g{G}")
            if tr and tr.get("kind", "group") == roof.get("kind"):
                traffic = tr["bytes_per_launch"]
        except Exception:
            traffic = None
    if roof:
        roof["traffic"] = traffic
        if roof["bound"] == "hbm" and roof["achieved"] and roof["achieved"] > peak:
            roof["note"] = (f"above the copy peak: the group kernel reads 2+ bytes per byte written (the peak "
                            f"is a 1:1 copy); {P * d * esz / 1e6:.0f} MB per array per GPU against 126 MB of L2")
    out = {
        "value": 1000.0 / ds["ms"], "unit": "iters/s", "ms_per_step": ds["ms"], "dtype": dtype,
        "config": config_dict(cfg, G),
        "effective_gbs": W * d * esz / (ds["ms"] / 1e3) / 1e9,
        "hbm_gbs_algorithmic": W * d * bpe / G / (ds["ms"] / 1e3) / 1e9,
        "bsp": {"iters_s": 1000.0 / bsp["ms"], "ms_per_step": bsp["ms"],
                "effective_gbs": W * d * esz / (bsp["ms"] / 1e3) / 1e9, "ds_speedup_over_bsp": bsp["ms"] / ds["ms"],
                "kernels": kernel_rows(bsp, "bsp")},
        "kernels": ds_k,
        "roofline": roof,
        "gpu_launches": int(round(ds["launches_per_step"] * args.steps)),
    }
    if hbm and roof and hbm.get("kind") != roof.get("kind"):
        out["roofline_hbm_kernel"] = hbm
    if "e2e_ms" in res:
        out["e2e"] = {"value": 1000.0 / res["e2e_ms"], "unit": "iters/s", "h2d_bytes_per_step": P * d * esz * G,
                      "d2h_bytes_per_step": P * d * esz * G, "steps": res["e2e_steps"],
                      "path": "C-ABI dss_step_host: pinned grads H2D + step + params D2H every step (copies on two "
                              "copy streams, D2H of step t overlapping H2D of step t+1)"}
        if "pcie" in res:
            # the e2e roofline: bytes each way per step / step time against
            # the copy engines' own pinned bidirectional rate on this box
            pc = dict(res["pcie"])
            pc["achieved_gbs_per_direction"] = P * d * esz / (res["e2e_ms"] / 1e3) / 1e9
            pc["frac"] = pc["achieved_gbs_per_direction"] / pc["bidir_gbs_per_direction"]
            out["e2e"]["pcie"] = pc
    elif "e2e_skipped" in res:
        out["e2e"] = {"value": None, "unit": "iters/s", "skipped": res["e2e_skipped"]}
    if "nccl_ds" in res:
        out["nccl_baselines"] = {
            "ds_split_allreduce": {"iters_s": 1000.0 / res["nccl_ds"], "ms_per_step": res["nccl_ds"]},
            "bsp_world_allreduce": {"iters_s": 1000.0 / res["nccl_bsp"], "ms_per_step": res["nccl_bsp"]},
            "note": "torch.distributed NCCL (ncclCommSplit sub-communicators); tolerance-parity only"}
    return out


def extras_for(args, G):
    if args.extras == "none":
        return []
    if args.extras != "auto":
        return [x for x in args.extras.split(",") if x]
    if args.config != "c2":
        return []
    return ["c3", "c4slice", "c2f64", "c2sq"] if G == 1 else (["c3", "c4"] if G >= 4 else ["c3"])


def our_arm(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    G = args.gpus
    if world != G:
        raise SystemExit(f"--gpus {G} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if G > 1:
        from paper_2007_03298_b200.dist import pin_host_cores
        pin_host_cores(local, int(os.environ.get("LOCAL_WORLD_SIZE", G)))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if cfg["W"] % G:
        raise SystemExit(f"W={cfg['W']} not divisible by {G} GPUs")
    peak, peak_kind = load_peaks()
    # one dedicated stream for the engine, torch's events and NCCL plumbing
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    res = measure(args, cfg, "f32", G, rank, local, stream, full=True)
    logistic_ms = None
    if cfg.get("logistic") and G == 1:
        logistic_ms = logistic_run(args, cfg, local, stream)
    extra_res = {}
    for name in extras_for(args, G):
        key, dtype = (name[:-3], "f64") if name.endswith("f64") else (name, "f32")
        c = dict(CONFIGS[key], key=key)
        if c["W"] % G:
            continue
        extra_res[name] = (c, dtype, measure(args, c, dtype, G, rank, local, stream, full=False))
    if G > 1 and not args.no_nccl:
        res.update(measure(args, cfg, "f32", G, rank, local, stream, nccl_only=True))
    if G > 1:
        dist.barrier()
    if rank != 0:
        if G > 1:
            dist.destroy_process_group()
        return

    head = summarize(args, dict(cfg, key=args.config), "f32", G, res, peak, peak_kind)
    out = {"metric": METRIC, "value": head["value"], "unit": "iters/s", "n_gpus": G, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic: isotropic-quadratic gradients (SplitMix64/Box-Muller, seeds 7/1), device-resident",
           "config": head["config"]}
    if G > 1:
        out["placement"] = {"mode": ["contiguous", "tiled", "auto"][args.placement],
                            "tiling_gr_gc": list(gpu_map(cfg, G, args.placement)[2])}
    if args.path:
        out["fold_path"] = {2: "chain forced for every spanning group", 3: "unfused pull two-shot"}.get(
            args.path, args.path)
    for k in ("effective_gbs", "hbm_gbs_algorithmic", "bsp", "kernels", "roofline", "roofline_hbm_kernel",
              "gpu_launches", "e2e", "nccl_baselines"):
        if k in head:
            out[k] = head[k]
    out["clocks"] = res.get("clocks")
    if logistic_ms is not None:
        out["device_gradient_run"] = {
            "iters_s": 1000.0 / logistic_ms, "ms_per_step": logistic_ms,
            "note": "DS iterations with the logistic batch sampled and the gradient computed on the device "
                    "(dss_logistic_steps: one launch for the whole batch of iterations; no trace)"}
        if not args.no_cpu_baseline:
            out["device_gradient_run"]["cpu_reference_run_training"] = cpu_run_training_c1()
    if extra_res:
        out["configs"] = {}
        for name, (c, dtype, r) in extra_res.items():
            s = summarize(args, c, dtype, G, r, peak, peak_kind)
            s["clocks"] = r.get("clocks")
            if G == 1 and not args.no_cpu_baseline and dtype == "f32":
                s["cpu_baseline"] = cpu_baseline(c, seconds=8.0)
            out["configs"][name] = s
            out["gpu_launches"] += s["gpu_launches"]
    if G == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg)
        if "configs" in out and "c2f64" in out["configs"]:
            out["configs"]["c2f64"]["cpu_baseline"] = dict(out["cpu_baseline"], note="same reference run as the "
                                                           "headline: the reference is fp64")
        out["host"] = host_info()
    print(json.dumps(out))
    if G > 1:
        dist.destroy_process_group()


def logistic_run(args, cfg, local, stream):
    """C1 end to end on the device: batch sampling + logistic gradient (fp64
    inside, f32 rows) + the DS step, nothing from the host but the learning
    rates (acceptance.cpp:239-258 data: d=20, M=2000)."""
    import torch
    from paper_2007_03298_b200 import (DsSyncEngine, OptimizerHyperparams, OptimizerKind, StrategyKind,
                                       SyncStrategy, Topology, WorldConfig, logistic_dataset)
    W, N, d = cfg["W"], cfg["N"], cfg["d"]
    x, y = logistic_dataset(11, d, 2000)
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N))
    e = DsSyncEngine(s, OptimizerKind(cfg["opt"]), d, OptimizerHyperparams(), "f32", local)
    e.set_stream(stream.cuda_stream)
    e.logistic_setup(x, y, 0.05, 8, 0, 1)
    alphas = np.full(args.steps, cfg["alpha"])
    e.logistic_steps(0, alphas[:args.warmup])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    e.logistic_steps(args.warmup, alphas)
    b.record(stream)
    torch.cuda.synchronize()
    e.check()
    e.close()
    return a.elapsed_time(b) / args.steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--extras", default="auto",
                    help="comma list of extra configs (c3, c4, c4slice, c2f64, ...), 'auto' or 'none'")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--d", type=int, default=None, help="override the config's d (profiling runs)")
    ap.add_argument("--path", type=int, default=0, help="fold path: 0 auto, 2 chain for every spanning group")
    ap.add_argument("--placement", type=int, default=2,
                    help="DS worker placement over the GPUs: 0 contiguous, 1 tiled, 2 auto (dss_config.placement)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = dict(CONFIGS[args.config])
    if args.d:
        cfg["d"] = args.d
        cfg["desc"] += f" [d overridden to {args.d:,} for profiling]"
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        our_arm(args, cfg)


if __name__ == "__main__":
    main()
