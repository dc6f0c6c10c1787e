"""Metrics writer parity (proj/src/metrics.cpp:13-56): format_double is
std::to_chars' shortest form, metrics_csv the reference's exact layout."""
import struct

import numpy as np

from paper_2007_03298_b200.api import IterationTrace
from paper_2007_03298_b200.metrics import format_double, metrics_csv


def test_format_double_matches_reference(reference):
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**63, size=4000, dtype=np.int64).astype(np.uint64)
    vals = [struct.unpack("<d", struct.pack("<Q", int(b)))[0] for b in bits]
    vals = [v for v in vals if np.isfinite(v)]
    vals += list(rng.standard_normal(2000) * 10.0 ** rng.integers(-12, 12, 2000))
    vals += [0.0, -0.0, 1.0, 2.0, 888.0, 0.1, 1e-4, 1e-5, 1e15, 1e16, 123456789012345680.0, 5e-324,
             1.7976931348623157e308, 0.000123, 1234567.0, -2.5e-7, 3.0e21]
    want = reference.format_doubles(vals)
    got = [format_double(v) for v in vals]
    bad = [(v, g, w) for v, g, w in zip(vals, got, want) if g != w]
    assert not bad, bad[:10]


def test_metrics_csv_layout_from_reference_traces(golden):
    """The reference's own metrics file, rebuilt from its trace scalars."""
    meta, a = golden
    for m in meta["trajectories"]:
        ts = a[m["key"] + "_trace_scalars"]
        traces = [IterationTrace(t, None, ts[t][0], ts[t][1], int(ts[t][2]), int(ts[t][3]), ts[t][4])
                  for t in range(len(ts))]
        assert metrics_csv(traces) == m["metrics_csv"], m["key"]
