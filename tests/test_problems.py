"""Host-side problem setup (library, CPU): the synthetic logistic dataset,
make_shards and epoch_order, bit-exact against fixtures produced by the
reference itself (tests/golden/make_golden.py: logistic_data)."""
import hashlib

import numpy as np
import pytest

from paper_2007_03298_b200 import Shard, epoch_order, logistic_dataset, make_shards


def test_logistic_dataset_matches_reference(golden):
    meta, a = golden
    x, y = logistic_dataset(5, 6, 40)
    assert set(np.unique(y)) <= {-1.0, 1.0}
    assert np.array_equal(y[:, None] * x, a["logi_yx_small"])
    # config C1's data (seed 11, d 20, M 2000), pinned by digest
    x, y = logistic_dataset(11, 20, 2000)
    yx = np.ascontiguousarray(y[:, None] * x)
    assert hashlib.sha256(yx.tobytes()).hexdigest() == meta["logistic_data"]["c1_yx_sha256"]


def test_make_shards_matches_reference(golden):
    meta, a = golden
    for s in meta["logistic_data"]["shards"]:
        shards = make_shards(s["M"], s["W"], s["seed"])
        idx, off = a[s["key"] + "_idx"], a[s["key"] + "_off"]
        assert [sh.owner for sh in shards] == list(range(s["W"]))
        for w, sh in enumerate(shards):
            assert sh.indices == idx[off[w]:off[w + 1]].tolist(), (s, w)


def test_epoch_order_matches_reference(golden):
    meta, a = golden
    shards = make_shards(2000, 4, 1)
    for e in meta["logistic_data"]["epoch_orders"]:
        got = epoch_order(shards[e["rank"]], 1, e["rank"], e["epoch"])
        assert got == a[e["key"]].tolist(), e
    assert epoch_order(Shard(0, []), 1, 0, 0) == []


def test_setup_errors_match_reference():
    with pytest.raises(ValueError, match="dataset smaller than worker count"):
        make_shards(3, 4, 1)
    with pytest.raises(ValueError, match="workers must be >= 1"):
        make_shards(3, 0, 1)
    with pytest.raises(ValueError, match="problem.M >= 1"):
        logistic_dataset(1, 3, 0)


def test_mlp_initial_params_match_reference(golden):
    """TinyMlpProblem::initial_params (problems.cpp:466-476), bit for bit."""
    from paper_2007_03298_b200 import mlp_initial_params
    meta, a = golden
    for m in meta["mlp"]:
        p = m["problem"]
        assert np.array_equal(mlp_initial_params(p["seed"], p["d"], p["hidden"]), a[f"mlp_{m['kind']}_w0"])
