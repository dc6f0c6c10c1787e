"""The run driver end to end on the device vs the reference's own
`dssync run` outputs (tests/golden cli_runs, made by oracle/ref_shim.cpp
ref_cmd_run = tools/main.cpp:34-55 over the unmodified reference).

  isotropic quadratic, sigma = 0   metrics_seed*.csv and summary.json byte-identical
  sigma > 0 / logistic             same rows; loss and suboptimality within 1e-9
                                   relative (libdevice vs glibc transcendentals)
  diverging run                    exit code 2 and the reference's message
"""
import csv
import io
import json
import os

import pytest

from paper_2007_03298_b200.run import main

pytestmark = pytest.mark.gpu


def _rows(text):
    return list(csv.reader(io.StringIO(text)))


@pytest.mark.parametrize("idx", range(9))
def test_cli_matches_reference(cuda_device, golden, tmp_path, capsys, idx):
    meta, _ = golden
    r = meta["cli_runs"][idx]
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(r["config"]))
    out = tmp_path / "out"
    rc = main(["--config", str(cfg), "--out", str(out)])
    if r["parity"] == "error":
        assert rc == 2
        assert r["error"] in capsys.readouterr().err
        return
    assert rc == 0
    assert sorted(os.listdir(out)) == sorted(r["files"])
    for fn, ref in r["files"].items():
        got = (out / fn).read_text()
        if r["parity"] == "bytes":
            assert got == ref, (r["name"], fn)
        elif fn.endswith(".csv"):
            g, e = _rows(got), _rows(ref)
            assert g[0] == e[0] and len(g) == len(e)
            for a, b in zip(g[1:], e[1:]):
                assert a[0] == b[0] and a[3:5] == b[3:5] and float(a[5]) == float(b[5]), (r["name"], a, b)
                for i in (1, 2):
                    if b[i] == "":
                        assert a[i] == ""
                    else:
                        assert abs(float(a[i]) - float(b[i])) <= 1e-9 * abs(float(b[i])) + 1e-15, (r["name"], i, a, b)
        else:
            gj, ej = json.loads(got), json.loads(ref)
            assert gj.keys() == ej.keys()
            for k in ("strategy", "topology", "world_size", "group_size", "problem", "optimizer", "iterations",
                      "seeds"):
                assert gj[k] == ej[k]
            assert gj["final_loss"]["mean"] == pytest.approx(ej["final_loss"]["mean"], rel=1e-9)
