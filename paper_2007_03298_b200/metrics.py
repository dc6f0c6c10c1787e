"""Metrics writer mirroring the reference's (proj/src/metrics.cpp:13-56):
shortest round-trip doubles formatted exactly like std::to_chars, and the
per-iteration CSV of run_training traces, so a device run's metrics file is
byte-identical to the reference's for the same trajectory."""
from __future__ import annotations

import json
import math
import os
from decimal import Decimal
from typing import Iterable


def format_double(v: float) -> str:
    """std::to_chars(double) shortest form (metrics.cpp:13-17): the shortest
    round-trip digits, written as %f or %e whichever is shorter (ties -> %f)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign, digits, exp = Decimal(repr(v)).as_tuple()
    ds = "".join(map(str, digits)).rstrip("0") or "0"
    # value = 0.ds... scaled: digits ds with decimal exponent so that
    # v = int(ds) * 10**e10
    e10 = exp + (len(digits) - len(ds))
    n = len(ds)
    sci_exp = e10 + n - 1
    mant = ds[0] + ("." + ds[1:] if n > 1 else "")
    sci = f"{mant}e{'-' if sci_exp < 0 else '+'}{abs(sci_exp):02d}"
    if e10 >= 0:
        # integral value: among equal-length round-trip candidates to_chars
        # takes the one closest to the value, i.e. its exact digits
        fixed = str(int(abs(v)))
    elif -e10 < n:
        fixed = ds[:n + e10] + "." + ds[n + e10:]
    else:
        fixed = "0." + "0" * (-e10 - n) + ds
    body = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + body


def metrics_csv(traces: Iterable) -> str:
    """metrics_csv (metrics.cpp:37-56): one row per IterationTrace."""
    out = ["t,mean_post_sync_loss,suboptimality,critical_path_steps,total_messages,simulated_comm_time\n"]
    for tr in traces:
        sub = format_double(tr.suboptimality) if math.isfinite(tr.suboptimality) else ""
        out.append(f"{int(tr.t)},{format_double(tr.mean_post_sync_loss)},{sub},{int(tr.critical_path_steps)},"
                   f"{int(tr.total_messages)},{format_double(tr.simulated_comm_time)}\n")
    return "".join(out)


def atomic_write_file(path: str, content: str) -> None:
    """Write-then-rename (metrics.cpp:58-71)."""
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(content.encode())
    os.replace(tmp, path)


# ---------------------------------------------------------------------------
# nlohmann::json number output (used by the reference's summary_json,
# metrics.cpp:73-115): Grisu2 (Loitsch 2010, "Printing floating-point numbers
# quickly and accurately with integers"), alpha = -60, gamma = -32, cached
# powers of ten every 8 decades from 1e-300 -- not always the shortest
# round-trip digits, so Python's repr cannot stand in for it.

_M64 = (1 << 64) - 1


def _cached_powers():
    out = []
    for k in range(-300, 325, 8):
        # 10^k = f * 2^e with f normalised to [2^63, 2^64), rounded to nearest
        num, den = (10 ** k, 1) if k >= 0 else (1, 10 ** -k)
        e = num.bit_length() - den.bit_length() - 64
        while True:
            n2, d2 = (num, den << e) if e >= 0 else (num << -e, den)
            f = (2 * n2 + d2) // (2 * d2)
            if f >= 1 << 64:
                e += 1
            elif f < 1 << 63:
                e -= 1
            else:
                break
        out.append((f, e, k))
    return out


_POWERS = _cached_powers()


def _mul(xf, xe, yf, ye):
    return (((xf * yf) >> 32) + (1 << 31)) >> 32, xe + ye + 64


def _normalize(f, e):
    s = 64 - f.bit_length()
    return f << s, e - s


def _grisu2(value: float):
    """(digits, decimal_exponent) with value = int(digits) * 10**decimal_exponent."""
    bits = int.from_bytes(math_pack(value), "little")
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    vf, ve = (F, -1074) if E == 0 else (F + (1 << 52), E - 1075)
    closer = F == 0 and E > 1
    pf, pe = _normalize(2 * vf + 1, ve - 1)
    mf, me = (4 * vf - 1, ve - 2) if closer else (2 * vf - 1, ve - 1)
    mf, me = mf << (me - pe), pe
    wf, we = _normalize(vf, ve)
    # cached power with alpha <= e_c + e + 64 <= gamma
    x = -60 - pe - 1
    k = int(x * 78913 / (1 << 18)) + (1 if x > 0 else 0)  # C truncating division
    cf, ce, ck = _POWERS[(300 + k + 7) // 8]
    w = _mul(wf, we, cf, ce)
    lo = _mul(mf, me, cf, ce)
    hi = _mul(pf, pe, cf, ce)
    Mm = lo[0] + 1
    Mp, e = hi[0] - 1, hi[1]
    dec = -ck
    delta = Mp - Mm
    dist = Mp - w[0]
    one = 1 << -e
    p1 = Mp >> -e
    p2 = Mp & (one - 1)
    buf = []

    def round_last(dist_, delta_, rest, ten_k):
        while rest < dist_ and delta_ - rest >= ten_k and (rest + ten_k < dist_ or dist_ - rest > rest + ten_k - dist_):
            buf[-1] -= 1
            rest += ten_k

    n = len(str(p1)) if p1 else 1
    pow10 = 10 ** (n - 1)
    while n > 0:
        d, p1 = divmod(p1, pow10)
        buf.append(d)
        n -= 1
        rest = (p1 << -e) + p2
        if rest <= delta:
            dec += n
            round_last(dist, delta, rest, pow10 << -e)
            return "".join(map(str, buf)), dec
        pow10 //= 10
    m = 0
    while True:
        p2 = (p2 * 10) & _M64
        buf.append(p2 >> -e)
        p2 &= one - 1
        m += 1
        delta = (delta * 10) & _M64
        dist = (dist * 10) & _M64
        if p2 <= delta:
            break
    dec -= m
    round_last(dist, delta, p2, one)
    return "".join(map(str, buf)), dec


def math_pack(v: float) -> bytes:
    import struct
    return struct.pack("<d", v)


def json_double(v: float) -> str:
    """nlohmann::json's text for a double: Grisu2 digits, then
    format_buffer with min_exp -4 and max_exp 15.  That gives fixed notation
    for a decimal point position n in (-4, 15], else d.ddde+XX.  Integral
    values get '.0'; NaN and inf become null."""
    v = float(v)
    if not math.isfinite(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    v = abs(v)
    if v == 0.0:
        return sign + "0.0"
    digits, dec = _grisu2(v)
    k = len(digits)
    n = k + dec
    if k <= n <= 15:
        body = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        body = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        body = "0." + "0" * (-n) + digits
    else:
        x = n - 1
        body = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if x < 0 else "+") + f"{abs(x):02d}"
    return sign + body


def _dump(obj, indent: int = 0) -> str:
    """nlohmann::ordered_json::dump(2) as built for the reference (json.hpp
    3.11 from the image): objects one key per line, arrays of scalars inline."""
    pad = " " * (indent + 2)
    if obj is None:
        return "null"
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return json_double(obj)
    if isinstance(obj, str):
        return json.dumps(obj, ensure_ascii=False)
    if isinstance(obj, list):
        if not obj:
            return "[]"
        if not any(isinstance(x, (list, dict)) for x in obj):
            # arrays of scalars are written on one line, no spaces (the
            # json.hpp build the reference links, metrics.cpp:102-104)
            return "[" + ",".join(_dump(x, indent) for x in obj) + "]"
        return "[\n" + ",\n".join(pad + _dump(x, indent + 2) for x in obj) + "\n" + " " * indent + "]"
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        return ("{\n" + ",\n".join(pad + json.dumps(k) + ": " + _dump(v, indent + 2) for k, v in obj.items())
                + "\n" + " " * indent + "}")
    raise TypeError(type(obj))


def summary_json(cfg, outcomes) -> str:
    """summary_json (metrics.cpp:73-115)."""
    if not outcomes:
        raise ValueError("summary needs at least one seed outcome")

    def mean_of_values(xs):
        acc = 0.0
        for x in xs:
            acc += x
        return acc / len(xs)

    def sample_std(xs, mean):
        if len(xs) < 2:
            return 0.0
        acc = 0.0
        for x in xs:
            acc += (x - mean) * (x - mean)
        return math.sqrt(acc / (len(xs) - 1))

    losses, subs, per_seed = [], [], []
    for seed, loss, sub in outcomes:
        losses.append(loss)
        row = {"seed": seed, "final_loss": loss}
        if math.isfinite(sub):
            row["final_suboptimality"] = sub
            subs.append(sub)
        else:
            row["final_suboptimality"] = None
        per_seed.append(row)
    s = cfg.strategy
    j = {"strategy": ["bsp", "ds-sync"][int(s.kind)], "topology": ["ring", "tree", "ps"][int(s.topology)],
         "world_size": s.world.world_size, "group_size": s.world.group_size, "problem": cfg.problem.kind,
         "optimizer": ["vanilla-sgd", "sgd-momentum", "adam", "adamw"][int(cfg.optimizer)], "iterations": cfg.iterations, "seeds": list(cfg.seeds)}
    lm = mean_of_values(losses)
    j["final_loss"] = {"mean": lm, "std": sample_std(losses, lm)}
    if len(subs) == len(outcomes):
        sm = mean_of_values(subs)
        j["final_suboptimality"] = {"mean": sm, "std": sample_std(subs, sm)}
    else:
        j["final_suboptimality"] = None
    j["per_seed"] = per_seed
    return _dump(j) + "\n"
