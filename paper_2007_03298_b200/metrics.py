"""Metrics writer mirroring the reference's (proj/src/metrics.cpp:13-56):
shortest round-trip doubles formatted exactly like std::to_chars, and the
per-iteration CSV of run_training traces, so a device run's metrics file is
byte-identical to the reference's for the same trajectory."""
from __future__ import annotations

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
