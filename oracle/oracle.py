"""ctypes wrappers of the test-only checkers.

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm, never by the product package.

  Oracle    liboracle.so: C restatement (dssync_oracle.c), f64 + f32.
  Reference _ref/libdssync_ref.so: the unmodified reference sources
            (/root/reference/proj/src) + ref_shim.cpp.  Built here; travels
            to the GPU box as a prebuilt .so.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdssync_ref.so")
REF_SRC = "/root/reference/proj"

_P = C.c_void_p
_D = np.float64


def build(ref: bool = True) -> None:
    """Build the oracle (and, when the reference sources are present, _ref)."""
    targets = [ORACLE_SO]
    if ref and os.path.isdir(REF_SRC):
        targets += ["ref", "reftests", "acceptance", "shimbench"]
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data


class HParams(C.Structure):  # orc_hparams
    _fields_ = [("momentum", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("epsilon", C.c_double), ("weight_decay", C.c_double)]


def hparams(momentum=0.9, beta1=0.9, beta2=0.999, epsilon=1e-8, weight_decay=0.0) -> HParams:
    return HParams(momentum, beta1, beta2, epsilon, weight_decay)


class Oracle:
    """C restatement of the reference hot path (f64 and f32)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        self.lib = L = C.CDLL(ORACLE_SO)
        L.orc_for_stream.restype = C.c_uint64
        L.orc_for_stream.argtypes = [C.c_uint64] * 4
        L.orc_next_u64.restype = C.c_uint64
        L.orc_next_u64.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_gaussian_stream.argtypes = [C.c_uint64] * 4 + [C.c_long, _P]
        L.orc_partition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, _P, _P, C.POINTER(C.c_int)]
        L.orc_validate_world.argtypes = [C.c_int, C.c_int, C.c_int]
        for suf in ("f64", "f32"):
            getattr(L, f"orc_ds_step_{suf}").argtypes = [
                C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, C.c_int, C.POINTER(HParams), C.c_double,
                _P, _P, _P, _P, _P, C.POINTER(C.c_int), C.POINTER(C.c_int)]
            getattr(L, f"orc_sync_round_{suf}").argtypes = [
                C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, _P, C.POINTER(C.c_int)]
            getattr(L, f"orc_bsp_step_{suf}").argtypes = [
                C.c_int, C.c_long, C.c_long, C.c_int, C.POINTER(HParams), C.c_double, _P, _P, _P, _P, _P,
                C.POINTER(C.c_int), C.POINTER(C.c_int)]
            getattr(L, f"orc_apply_step_{suf}").argtypes = [
                C.c_int, C.c_long, C.c_int, C.POINTER(HParams), C.c_double, _P, _P, _P, _P, _P,
                C.POINTER(C.c_int)]
            getattr(L, f"orc_quadratic_grad_{suf}").argtypes = [
                C.c_int, C.c_int, C.c_long, C.c_long, C.c_uint64, C.c_double, C.c_double, _P, _P, _P]
        L.orc_quadratic_init_f64.argtypes = [C.c_uint64, C.c_long, C.c_double, _P, _P]

    @staticmethod
    def _suf(a):
        return "f64" if a.dtype == np.float64 else "f32"

    def partition(self, W, N, t, rect=False, kind=1):
        members = np.zeros(W, np.int32)
        offsets = np.zeros(W + 1, np.int32)
        n = C.c_int()
        rc = self.lib.orc_partition(W, N, int(rect), kind, t, _ptr(members), _ptr(offsets), C.byref(n))
        if rc:
            raise ValueError("invalid world")
        return [members[offsets[g]:offsets[g + 1]].tolist() for g in range(n.value)]

    def gaussians(self, seed, purpose, rank, it, n):
        out = np.zeros(n, _D)
        self.lib.orc_gaussian_stream(seed, purpose, rank, it, n, _ptr(out))
        return out

    def ds_step(self, W, N, t, opt, hp, alpha, steps, w, g, m1=None, m2=None, rect=False):
        """In place on [W][d] arrays; returns (rc, err_rank, err_phase)."""
        d = w.shape[1]
        r, ph = C.c_int(), C.c_int()
        steps = np.ascontiguousarray(steps, np.int64)
        rc = getattr(self.lib, f"orc_ds_step_{self._suf(w)}")(
            W, N, int(rect), d, t, opt, C.byref(hp), alpha, _ptr(steps), _ptr(w), _ptr(g), _ptr(m1), _ptr(m2),
            C.byref(r), C.byref(ph))
        return rc, r.value, ph.value

    def sync_round(self, W, N, t, w, rect=False, kind=1):
        r = C.c_int()
        rc = getattr(self.lib, f"orc_sync_round_{self._suf(w)}")(W, N, int(rect), kind, w.shape[1], t, _ptr(w), C.byref(r))
        return rc, r.value

    def bsp_step(self, t, opt, hp, alpha, steps, w, g, m1=None, m2=None):
        W, d = w.shape
        r, ph = C.c_int(), C.c_int()
        steps = np.ascontiguousarray(steps, np.int64)
        rc = getattr(self.lib, f"orc_bsp_step_{self._suf(w)}")(
            W, d, t, opt, C.byref(hp), alpha, _ptr(steps), _ptr(w), _ptr(g), _ptr(m1), _ptr(m2),
            C.byref(r), C.byref(ph))
        return rc, r.value, ph.value

    def apply_step(self, opt, hp, alpha, steps, w, g, m1=None, m2=None):
        W, d = w.shape
        r = C.c_int()
        steps = np.ascontiguousarray(steps, np.int64)
        rc = getattr(self.lib, f"orc_apply_step_{self._suf(w)}")(
            W, d, opt, C.byref(hp), alpha, _ptr(steps), _ptr(w), _ptr(g), _ptr(m1), _ptr(m2), C.byref(r))
        return rc, r.value

    def quadratic_grad(self, first_rank, t, seed, mu, sigma, w, wstar):
        nrows, d = w.shape
        g = np.zeros_like(w)
        getattr(self.lib, f"orc_quadratic_grad_{self._suf(w)}")(
            nrows, first_rank, d, t, seed, mu, sigma, _ptr(w), _ptr(np.ascontiguousarray(wstar, w.dtype)), _ptr(g))
        return g

    def quadratic_init(self, seed, d, delta0):
        wstar = np.zeros(d, _D)
        w0 = np.zeros(d, _D)
        self.lib.orc_quadratic_init_f64(seed, d, delta0, _ptr(wstar), _ptr(w0))
        return wstar, w0


class Reference:
    """The unmodified reference library (oracle/_ref), through ref_shim.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = L = C.CDLL(REF_SO)
        E = [C.c_char_p, C.c_int]
        L.ref_validate_world.argtypes = [C.c_int, C.c_int] + E
        L.ref_validate_strategy.argtypes = [C.c_int] * 5 + E
        L.ref_is_square_mode.argtypes = [C.c_int, C.c_int]
        L.ref_make_partition.argtypes = [C.c_int, C.c_int, C.c_long, _P, _P, C.POINTER(C.c_int)] + E
        L.ref_group_of.argtypes = [C.c_int, C.c_int, C.c_long, C.c_int, _P, C.POINTER(C.c_int)] + E
        L.ref_check_mixing.argtypes = [C.c_int, C.c_int, C.c_long]
        L.ref_allreduce.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, _P, _P, C.POINTER(C.c_long),
                                    C.POINTER(C.c_long)] + E
        L.ref_mean_of.argtypes = [C.c_int, C.c_long, _P, _P] + E
        L.ref_apply_step.argtypes = [C.c_int, _P, C.c_double, C.POINTER(C.c_long), C.c_long, _P, _P, _P, _P] + E
        L.ref_sync_round.argtypes = [C.c_int] * 5 + [C.c_long, C.c_long, _P, C.POINTER(C.c_long),
                                                     C.POINTER(C.c_long), C.POINTER(C.c_int), C.POINTER(C.c_long)] + E
        L.ref_ds_iteration.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, C.c_int, _P, C.c_double,
                                       _P, _P, _P, _P, _P, C.POINTER(C.c_int), C.POINTER(C.c_long)] + E
        L.ref_bsp_iteration.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, C.c_int, _P, C.c_double,
                                        _P, _P, _P, _P, _P, C.POINTER(C.c_int), C.POINTER(C.c_long)] + E
        L.ref_gaussians.argtypes = [C.c_uint64] * 4 + [C.c_long, _P]
        L.ref_next_u64.restype = C.c_uint64
        L.ref_next_u64.argtypes = [C.POINTER(C.c_uint64)]
        L.ref_quadratic_init.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, _P, _P] + E
        L.ref_quadratic_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _P, C.c_double,
                                        _P, _P, C.POINTER(C.c_int)] + E + [_P, _P, _P, C.c_char_p, C.c_long]
        L.ref_format_doubles.argtypes = [_P, C.c_long, C.c_char_p, C.c_long]
        L.ref_logistic_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                       C.c_uint64, C.c_int, C.c_int, C.c_int, _P, C.c_double, C.c_double,
                                       C.c_long, C.c_int, _P, _P, _P, _P, C.POINTER(C.c_int)] + E
        L.ref_cmd_run.argtypes = [C.c_char_p, C.c_char_p] + E + [C.POINTER(C.c_int), C.POINTER(C.c_long)]
        L.ref_parse_config.argtypes = [C.c_char_p] + E
        L.ref_logistic_yx.argtypes = [C.c_uint64, C.c_int, C.c_int, _P] + E
        L.ref_load_csv.argtypes = [C.c_char_p, C.c_double, _P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)] + E
        L.ref_make_shards.argtypes = [C.c_int, C.c_int, C.c_uint64, _P, _P] + E
        L.ref_epoch_order.argtypes = [_P, C.c_int, C.c_uint64, C.c_int, C.c_long, _P]
        L.ref_mlp_run.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, _P, C.c_double,
                                                  _P, _P, _P, _P, _P, _P, C.POINTER(C.c_int)] + E
        L.ref_bench_create.restype = _P
        L.ref_bench_create.argtypes = [C.c_int, C.c_long, C.c_int, _P, C.c_uint64, C.c_int]
        L.ref_bench_partition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, _P, _P, C.POINTER(C.c_int)] + E
        L.ref_bench_stock_step.argtypes = [_P, C.c_int, C.c_long, C.c_double, C.c_int] + E
        L.ref_bench_bytes.restype = C.c_long
        L.ref_bench_bytes.argtypes = [_P]
        L.ref_bench_destroy.argtypes = [_P]
        L.ref_bench_ds_step.argtypes = [_P, C.c_long, C.c_double, _P, _P, C.c_int, C.c_int] + E
        L.ref_bench_bsp_step.argtypes = [_P, C.c_long, C.c_double, C.c_int] + E
        self.err = C.create_string_buffer(1024)

    @staticmethod
    def hp_array(momentum=0.9, beta1=0.9, beta2=0.999, epsilon=1e-8, weight_decay=0.0):
        return np.array([momentum, beta1, beta2, epsilon, weight_decay], _D)

    def _e(self):
        return self.err, len(self.err)

    def error(self) -> str:
        return self.err.value.decode()

    def make_partition(self, W, N, t):
        members = np.zeros(max(W, 1), np.int32)
        offsets = np.zeros(max(W, 1) + 1, np.int32)
        n = C.c_int()
        rc = self.lib.ref_make_partition(W, N, t, _ptr(members), _ptr(offsets), C.byref(n), *self._e())
        if rc:
            raise ValueError(self.error())
        return [members[offsets[g]:offsets[g + 1]].tolist() for g in range(n.value)]

    def check_mixing(self, W, N, t):
        return self.lib.ref_check_mixing(W, N, t)

    def apply_step(self, opt, hp, alpha, step_count, w, g, m1=None, m2=None):
        sc = C.c_long(step_count)
        rc = self.lib.ref_apply_step(opt, _ptr(hp), alpha, C.byref(sc), w.size, _ptr(w), _ptr(g), _ptr(m1), _ptr(m2),
                                     *self._e())
        return rc, sc.value

    def ds_iteration(self, topo, W, N, t, opt, hp, alpha, steps, w, g, m1=None, m2=None):
        r, it = C.c_int(-1), C.c_long(-1)
        rc = self.lib.ref_ds_iteration(topo, W, N, w.shape[1], t, opt, _ptr(hp), alpha, _ptr(steps), _ptr(w), _ptr(g),
                                       _ptr(m1), _ptr(m2), C.byref(r), C.byref(it), *self._e())
        return rc, r.value, it.value

    def bsp_iteration(self, topo, W, t, opt, hp, alpha, steps, w, g, m1=None, m2=None, servers=1):
        r, it = C.c_int(-1), C.c_long(-1)
        rc = self.lib.ref_bsp_iteration(topo, servers, W, w.shape[1], t, opt, _ptr(hp), alpha, _ptr(steps), _ptr(w),
                                        _ptr(g), _ptr(m1), _ptr(m2), C.byref(r), C.byref(it), *self._e())
        return rc, r.value, it.value

    def sync_round(self, kind, topo, W, N, t, w, servers=1):
        st, ms = C.c_long(), C.c_long()
        r, it = C.c_int(-1), C.c_long(-1)
        rc = self.lib.ref_sync_round(kind, topo, W, N, servers, t, w.shape[1], _ptr(w), C.byref(st), C.byref(ms),
                                     C.byref(r), C.byref(it), *self._e())
        return rc, (st.value, ms.value), (r.value, it.value)

    def gaussians(self, seed, purpose, rank, it, n):
        out = np.zeros(n, _D)
        self.lib.ref_gaussians(seed, purpose, rank, it, n, _ptr(out))
        return out

    def format_doubles(self, values):
        v = np.ascontiguousarray(values, _D)
        buf = C.create_string_buffer(64 * (v.size + 1))
        assert self.lib.ref_format_doubles(_ptr(v), v.size, buf, len(buf)) == 0
        return buf.value.decode().split("\n")[:-1]

    def quadratic_init(self, seed, d, mu, delta0):
        wstar, w0 = np.zeros(d, _D), np.zeros(d, _D)
        rc = self.lib.ref_quadratic_init(seed, d, mu, delta0, _ptr(wstar), _ptr(w0), *self._e())
        if rc:
            raise RuntimeError(self.error())
        return wstar, w0

    def quadratic_run(self, kind, topo, W, N, d, mu, sigma, delta0, problem_seed, run_seed, T, opt, hp, alpha,
                      trace=False):
        grads = np.zeros((T, W, d), _D)
        params = np.zeros((T, W, d), _D)
        match = C.c_int()
        tg = np.zeros((T, d), _D) if trace else None
        tl = np.zeros((T, W), _D) if trace else None
        ts = np.zeros((T, 5), _D) if trace else None
        csv = C.create_string_buffer(1 << 16) if trace else None
        rc = self.lib.ref_quadratic_run(kind, topo, W, N, d, mu, sigma, delta0, problem_seed, run_seed, T, opt,
                                        _ptr(hp), alpha, _ptr(grads), _ptr(params), C.byref(match), *self._e(),
                                        _ptr(tg), _ptr(tl), _ptr(ts), csv, len(csv) if trace else 0)
        if rc:
            raise RuntimeError(self.error())
        if trace:
            return grads, params, bool(match.value), (tg, tl, ts, csv.value.decode())
        return grads, params, bool(match.value)

    def mlp_run(self, kind, W, N, d_in, M, hidden, problem_seed, run_seed, batch, T, opt, hp, alpha,
                with_batches=False):
        dim = hidden * d_in + 2 * hidden + 1
        g = np.zeros((T, W, dim), _D)
        obs = np.zeros((T, W, hidden), _D)
        p = np.zeros((T, W, dim), _D)
        st = np.zeros((T, W, hidden), _D)
        w0 = np.zeros(dim, _D)
        batches = np.zeros((T, W, batch), np.int32)
        match = C.c_int()
        rc = self.lib.ref_mlp_run(kind, W, N, d_in, M, hidden, problem_seed, run_seed, batch, T, opt, _ptr(hp), alpha,
                                  _ptr(g), _ptr(obs), _ptr(p), _ptr(st), _ptr(w0), _ptr(batches), C.byref(match),
                                  *self._e())
        if rc:
            raise RuntimeError(self.error())
        if with_batches:
            return g, obs, p, st, w0, batches, bool(match.value)
        return g, obs, p, st, w0, bool(match.value)

    def logistic_run(self, kind, W, N, d, M, l2, problem_seed, run_seed, batch, T, opt, hp, alpha0, factor, every,
                     sampling=0, with_batches=False):
        grads = np.zeros((T, W, d), _D)
        params = np.zeros((T, W, d), _D)
        alphas = np.zeros(T, _D)
        batches = np.zeros((T, W, batch), np.int32)
        match = C.c_int()
        rc = self.lib.ref_logistic_run(kind, W, N, d, M, l2, problem_seed, run_seed, batch, T, opt, _ptr(hp), alpha0,
                                       factor, every, sampling, _ptr(grads), _ptr(params), _ptr(alphas),
                                       _ptr(batches), C.byref(match), *self._e())
        if rc:
            raise RuntimeError(self.error())
        if with_batches:
            return grads, params, alphas, batches, bool(match.value)
        return grads, params, alphas, bool(match.value)

    def cmd_run(self, config_path, out_dir):
        """The reference's `dssync run` (main.cpp:34-55): (status, message, rank, iteration);
        status 0 ok, 2 DivergenceError, 4 ConfigError, else another failure."""
        rank, it = C.c_int(-1), C.c_long(-1)
        rc = self.lib.ref_cmd_run(config_path.encode(), out_dir.encode(), *self._e(), C.byref(rank), C.byref(it))
        return rc, (self.error() if rc else ""), rank.value, it.value

    def parse_config(self, text):
        """None when parse_run_config accepts text, else its ConfigError message."""
        rc = self.lib.ref_parse_config(text.encode(), *self._e())
        return self.error() if rc else None

    def logistic_yx(self, seed, d, M):
        out = np.zeros((M, d), _D)
        if self.lib.ref_logistic_yx(C.c_uint64(seed), d, M, _ptr(out), *self._e()):
            raise RuntimeError(self.error())
        return out

    def load_csv(self, path, l2, cap=1 << 16):
        """(error or None, y*x [M, d] or None)."""
        out = np.zeros(cap, _D)
        M, d = C.c_int(0), C.c_int(0)
        rc = self.lib.ref_load_csv(path.encode(), l2, _ptr(out), cap, C.byref(M), C.byref(d), *self._e())
        if rc:
            return self.error(), None
        return None, out[:M.value * d.value].reshape(M.value, d.value).copy()

    def make_shards(self, M, W, seed):
        idx = np.zeros(M, np.int32)
        off = np.zeros(W + 1, np.int32)
        if self.lib.ref_make_shards(M, W, C.c_uint64(seed), _ptr(idx), _ptr(off), *self._e()):
            raise RuntimeError(self.error())
        return idx, off

    def epoch_order(self, shard, seed, rank, epoch):
        shard = np.ascontiguousarray(shard, np.int32)
        out = np.zeros_like(shard)
        self.lib.ref_epoch_order(_ptr(shard), shard.size, C.c_uint64(seed), rank, C.c_long(epoch), _ptr(out))
        return out
