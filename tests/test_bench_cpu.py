"""bench.py's host-side pieces: the reference arm runs the unmodified
reference (oracle/_ref) without loading the product library, at the full
workload d, and prints the same `config` object as our arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_built():
    from oracle import oracle as o
    if not os.path.exists(o.REF_SO):
        if os.path.isdir(o.REF_SRC):
            o.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built")


def test_reference_arm_is_product_free_and_same_config():
    _ref_built()
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--d','65536','--steps','3','--warmup','3'];"
            "import bench; bench.main();"
            "print(json.dumps(sorted(m for m in sys.modules if m.startswith('paper_2007_03298_b200'))))")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = p.stdout.strip().splitlines()
    line, mods = json.loads(lines[-2]), json.loads(lines[-1])
    assert mods == [], f"reference arm loaded the product package: {mods}"
    assert line["impl"] == "reference" and line["steps"] == 3 and line["value"] > 0
    assert "scaled" not in line["cpu_baseline"]["sample"]
    import bench
    cfg = dict(bench.CONFIGS["c2"], d=65536)
    cfg["desc"] += " [d overridden to 65,536 for profiling]"
    assert line["config"] == bench.config_dict(cfg, 1)
    assert line["stock_sync_round_legal_shape"]["iters_s"] > 0


def test_reference_partition_rule_matches_the_product_schedule():
    """The reference arm's group tables (the reference's make_partition for
    legal shapes, the documented rectangular rule otherwise) equal the
    product's schedule for every BASELINE shape."""
    _ref_built()
    import numpy as np

    import bench
    from paper_2007_03298_b200 import StrategyKind, SyncStrategy, Topology, WorldConfig, make_partition
    for name in ("c1", "c2", "c3", "c4", "c4slice", "c2sq"):
        c = bench.CONFIGS[name]
        rb = bench.RefBench(dict(c, d=64), 64, 1)
        try:
            for t in (0, 1):
                m, o, n = rb.tables[t]
                got = [m[o[g]:o[g + 1]].tolist() for g in range(n)]
                s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(c["W"], c["N"]), 1, c["rect"])
                assert got == make_partition(s, t).groups, (name, t)
        finally:
            rb.close()
    assert np is not None
