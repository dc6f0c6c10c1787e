"""The run driver's host side (CPU): config validation and summary.json,
against the reference's own parse_run_config / summary_json outputs
(tests/golden: bad_configs, cli_runs)."""
import json
import math

import pytest

from paper_2007_03298_b200.config import ConfigError, parse_run_config
from paper_2007_03298_b200.metrics import json_double, summary_json
from paper_2007_03298_b200.run import build_lr, load_logistic_csv


def test_config_errors_match_reference(golden):
    meta, _ = golden
    for b in meta["bad_configs"]:
        if b["error"] is None:
            parse_run_config(b["text"])
            continue
        with pytest.raises(ConfigError) as ex:
            parse_run_config(b["text"])
        if b["error"].startswith("config is not valid JSON"):
            assert str(ex.value).startswith("config is not valid JSON"), b
        else:
            assert str(ex.value) == b["error"], b


def test_summary_json_byte_identical(golden):
    """summary_json (metrics.cpp:73-115) from the reference's per-seed values
    reproduces the reference's file byte for byte (Grisu2 digits, layout)."""
    meta, _ = golden
    n = 0
    for r in meta["cli_runs"]:
        if r["status"]:
            continue
        cfg = parse_run_config(json.dumps(r["config"]))
        ref = r["files"]["summary.json"]
        per_seed = json.loads(ref)["per_seed"]
        outcomes = [(p["seed"], p["final_loss"],
                     p["final_suboptimality"] if p["final_suboptimality"] is not None else math.nan)
                    for p in per_seed]
        assert summary_json(cfg, outcomes) == ref, r["name"]
        n += 1
    assert n >= 5


def test_json_double_known_answers():
    # Grisu2 is not always the shortest round trip: cases where nlohmann's
    # digits differ from repr() (checked against json.hpp 3.11)
    assert json_double(1422378505248446.2) == "1.4223785052484463e+15"
    assert json_double(3.472778835919032e+17) == "3.4727788359190323e+17"
    assert json_double(-921633924497811.2) == "-921633924497811.3"
    assert json_double(5.0) == "5.0"
    assert json_double(1e-5) == "1e-05"
    assert json_double(0.0001) == "0.0001"
    assert json_double(1e15) == "1e+15"
    assert json_double(123456789012345.0) == "123456789012345.0"
    assert json_double(-0.0) == "-0.0"
    assert json_double(float("nan")) == "null"


def test_lr_schedules():
    cfg = parse_run_config(json.dumps({"strategy": "ds-sync", "world_size": 4, "problem": {"kind": "quadratic"},
                                       "lr": {"kind": "step-decay", "alpha": 1.0, "factor": 0.5, "every": 75}}))

    class P:
        mu, smoothness = 1.0, 1.0
    lr = build_lr(cfg, P)
    assert [lr(t) for t in (0, 74, 75, 150, 299)] == [1.0, 1.0, 0.5, 0.25, 0.125]
    cfg.lr.kind = "theorem"
    lr = build_lr(cfg, P)
    assert lr(0) == 2.0 / (1.0 * (8.0 + 0.0))


def test_csv_loader_matches_reference(golden, tmp_path):
    """load_logistic_csv (problems.cpp:584-640) + the problem setup on the
    reference's edge cases: same error text, or the same y*x rows."""
    from paper_2007_03298_b200 import logistic_constants
    meta, _ = golden
    for i, c in enumerate(meta["csv_cases"]):
        p = tmp_path / f"c{i}.csv"
        p.write_bytes(c["text"].encode())
        try:
            x, y = load_logistic_csv(str(p), 0.1)
            logistic_constants(x, y, 0.1)
            got = None
        except (ConfigError, ValueError, RuntimeError) as e:
            got = str(e).replace(str(p), "<path>")
        assert got == c["error"], (c["text"], got)
        if got is None:
            assert (y[:, None] * x).tolist() == c["yx"], c["text"]
