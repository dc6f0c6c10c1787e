"""Host-side schedule of the C-ABI library (no GPU): bit-exact group
membership against the reference's own partitions (golden), its error
rules and messages, the rectangular extension, closed-form round outcomes
and the multi-GPU two-shot plan."""
import numpy as np
import pytest

from paper_2007_03298_b200 import (SyncStrategy, StrategyKind, Topology, WorldConfig, check_mixing, group_of,
                                   is_square_mode, make_partition, round_outcome, validate)


def ds(W, N, topo=Topology.RING, rect=False):
    return SyncStrategy(StrategyKind.DS_SYNC, topo, WorldConfig(W, N), 1, rect)


def test_partitions_bit_exact_vs_reference(golden):
    meta, _ = golden
    for c in meta["partitions"]["cases"]:
        assert make_partition(WorldConfig(c["W"], c["N"]), c["t"]).groups == c["groups"], c


def test_mixing_vs_reference(golden):
    meta, _ = golden
    for c in meta["partitions"]["mixing"]:
        assert check_mixing(WorldConfig(c["W"], c["N"]), c["t"]) == bool(c["mixing"]), c


def test_invalid_worlds_same_message(golden):
    meta, _ = golden
    for c in meta["partitions"]["invalid"]:
        if c["error"] is None:
            make_partition(WorldConfig(c["W"], c["N"]), 0)
            continue
        with pytest.raises(ValueError) as e:
            make_partition(WorldConfig(c["W"], c["N"]), 0)
        assert str(e.value) == c["error"]
    with pytest.raises(ValueError) as e:
        make_partition(WorldConfig(4, 2), -1)
    assert str(e.value) == meta["partitions"]["negative_t"]


def test_reference_unit_cases():
    """test_schedule.cpp:11-120."""
    p0, p1 = make_partition(WorldConfig(4, 2), 0), make_partition(WorldConfig(4, 2), 1)
    assert p0.groups == [[0, 1], [2, 3]] and p1.groups == [[0, 2], [1, 3]]
    for t in range(11):
        assert make_partition(WorldConfig(4, 2), t).groups == make_partition(WorldConfig(4, 2), t % 2).groups
    assert make_partition(WorldConfig(9, 3), 1).groups == [[0, 3, 6], [1, 4, 7], [2, 5, 8]]
    assert not is_square_mode(WorldConfig(4, 4)) and is_square_mode(WorldConfig(9, 3))
    assert not is_square_mode(WorldConfig(1, 1))
    assert make_partition(WorldConfig(1, 1), 0).groups == [[0]]
    for t in range(4):
        p = make_partition(WorldConfig(16, 4), t)
        for r in range(16):
            mine = group_of(WorldConfig(16, 4), t, r)
            assert mine in p.groups and r in mine
    for bad in (4, -1):
        with pytest.raises(ValueError):
            group_of(WorldConfig(4, 2), 0, bad)


@pytest.mark.parametrize("W,N", [(8, 2), (8, 4), (32, 4), (32, 8), (12, 3), (64, 8), (6, 2)])
def test_rectangular_extension(W, N):
    """W = N*K: K blocks of N on even t, N combs of K on odd t; disjoint
    ascending cover; consecutive groups share exactly one worker; reduces to
    the reference's square rule when K == N."""
    K = W // N
    s = ds(W, N, rect=True)
    for t in range(6):
        p = make_partition(s, t)
        size = N if t % 2 == 0 else K
        assert len(p.groups) == (K if t % 2 == 0 else N)
        flat = sorted(x for g in p.groups for x in g)
        assert flat == list(range(W))
        for g in p.groups:
            assert len(g) == size and g == sorted(g)
        assert check_mixing(s, t)
    if K == N:
        for t in range(4):
            assert make_partition(s, t).groups == make_partition(WorldConfig(W, N), t).groups
    # the reference itself rejects these shapes
    if W != N * N:
        with pytest.raises(ValueError):
            make_partition(WorldConfig(W, N), 0)


def test_c2_c3_c4_shapes():
    assert make_partition(ds(8, 2, rect=True), 0).groups == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert make_partition(ds(8, 2, rect=True), 1).groups == [[0, 2, 4, 6], [1, 3, 5, 7]]
    p = make_partition(ds(32, 4, rect=True), 1)
    assert len(p.groups) == 4 and all(len(g) == 8 for g in p.groups)
    p = make_partition(ds(64, 8), 1)
    assert p.groups[0] == list(range(0, 64, 8))


def test_strategy_validation():
    """sync.cpp:47-66 / test_sync.cpp:70-90."""
    bad = [
        SyncStrategy(StrategyKind.DS_SYNC, Topology.PS, WorldConfig(4, 2)),
        SyncStrategy(StrategyKind.DS_SYNC, Topology.TREE, WorldConfig(9, 3)),
        SyncStrategy(StrategyKind.BSP, Topology.RING, WorldConfig(4, 2)),
        SyncStrategy(StrategyKind.BSP, Topology.PS, WorldConfig(4, 4), num_servers=0),
    ]
    msgs = [
        "ds-sync has no parameter-server variant; use topology ring or tree",
        "tree topology requires power-of-two groups (group_size=3)",
        "bsp runs one group spanning the world; set group_size equal to world_size",
        "ps topology needs num_servers >= 1 (got 0)",
    ]
    for s, m in zip(bad, msgs):
        with pytest.raises(ValueError) as e:
            validate(s)
        assert str(e.value) == m
    validate(ds(16, 4))
    validate(SyncStrategy(StrategyKind.BSP, Topology.RING, WorldConfig(3, 3)))


def test_round_outcome_vs_reference(golden):
    """Closed-form serial steps / messages equal the reference's executed
    collectives (sync_round outcome, golden)."""
    meta, _ = golden
    for m in meta["sync_rounds"]:
        s = SyncStrategy(StrategyKind(m["kind"]), Topology(m["topology"]), WorldConfig(m["W"], m["N"]),
                         m["num_servers"])
        o = round_outcome(s, m["t"], m["d"])
        assert (o.critical_path_steps, o.total_messages) == (m["critical_path_steps"], m["total_messages"]), m
    # test_sync.cpp:141-152: ring pairs 3/6, bsp world of four 7/7
    o = round_outcome(ds(4, 2), 0, 8)
    assert (o.critical_path_steps, o.total_messages) == (3, 6)
    o = round_outcome(SyncStrategy(StrategyKind.BSP, Topology.RING, WorldConfig(4, 4)), 0, 8)
    assert (o.critical_path_steps, o.total_messages) == (7, 7)


def _plan(s, t, d, G, r):
    import ctypes as C
    from paper_2007_03298_b200 import _lib as L
    from paper_2007_03298_b200.api import _c_strategy
    cs = _c_strategy(s)
    out = L.dss_plan_summary()
    lo, hi, grp = np.zeros(256, np.int64), np.zeros(256, np.int64), np.zeros(256, np.int32)
    st = L.load().dss_plan(C.byref(cs), t, d, G, r, C.byref(out), lo.ctypes.data, hi.ctypes.data, grp.ctypes.data, 256)
    assert st == 0, L.global_error()
    n = out.owned_slices
    return out, list(zip(grp[:n].tolist(), lo[:n].tolist(), hi[:n].tolist()))


@pytest.mark.parametrize("W,N,rect,G", [(8, 2, True, 8), (8, 2, True, 2), (32, 4, True, 8), (64, 8, False, 8),
                                        (16, 4, False, 8), (8, 2, True, 4), (4, 2, False, 2), (32, 4, True, 4)])
def test_multi_gpu_plan_covers_every_element_once(W, N, rect, G):
    """Every spanning group is folded exactly one way: two-shot (its GPUs'
    owned slices tile [0, d_pad) exactly once) when it has one member per
    GPU, the ordered chain (no slices; every member GPU takes part) when
    some GPU holds several of its members.  GPU-local groups own nothing."""
    d = 1000 + 3
    d_pad = (d + 63) // 64 * 64
    s = ds(W, N, rect=rect)
    for t in (0, 1):
        part = make_partition(s, t)
        per = W // G
        cover = {}
        n_local = n_chain = 0
        for r in range(G):
            summ, slices = _plan(s, t, d, G, r)
            n_local += summ.local_groups
            n_chain += summ.chain_groups
            for g, lo, hi in slices:
                cover.setdefault(g, []).append((lo, hi))
        want_chain = 0
        for gi, members in enumerate(part.groups):
            gpus = sorted({m // per for m in members})
            if len(gpus) == 1:
                assert gi not in cover
                continue
            if max(sum(1 for m in members if m // per == g) for g in gpus) >= 2:
                assert gi not in cover
                want_chain += len(gpus)
                continue
            ivs = sorted(cover[gi])
            assert ivs[0][0] == 0 and ivs[-1][1] == d_pad
            for (a0, a1), (b0, b1) in zip(ivs, ivs[1:]):
                assert a1 == b0
            assert len(ivs) <= len(gpus)
        assert n_chain == want_chain
        assert n_local == sum(1 for g in part.groups if len({m // per for m in g}) == 1)


@pytest.mark.parametrize("W,N,rect", [(8, 2, True), (32, 4, True), (64, 8, False), (16, 4, False), (36, 6, False),
                                      (4, 2, False), (128, 8, True)])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_tiled_placement_properties(W, N, rect, G):
    """dss_placement (the tiled worker placement): a bijection onto G GPUs x
    W/G rows, local rows ascending by rank, and every group's members on a
    GPU forming one contiguous run of its ascending (fold) order -- what the
    ordered chain needs.  It never moves more rows across GPUs than
    contiguous packing in the busier parity."""
    from paper_2007_03298_b200 import (SyncStrategy, StrategyKind, Topology, WorldConfig, make_partition,
                                       placement)
    if W % G:
        pytest.skip("W not a multiple of G")
    s = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(W, N), 1, rect)
    P = W // G
    gpu, row, (gr, gc) = placement(s, G, 1)
    assert sorted(zip(gpu, row)) == [(q, r) for q in range(G) for r in range(P)]
    for q in range(G):
        mine = [k for k in range(W) if gpu[k] == q]
        assert [row[k] for k in mine] == list(range(P))
    busy = {}
    for mode, gmap in (("tiled", gpu), ("contiguous", [k // P for k in range(W)])):
        b = 0
        for t in (0, 1):
            cross = 0
            for grp in make_partition(s, t).groups:
                seq = [gmap[m] for m in grp]
                runs = [seq[0]] + [y for x, y in zip(seq, seq[1:]) if y != x]
                assert len(runs) == len(set(runs)), (mode, grp, seq)
                cross += len(set(seq)) - 1
            b = max(b, cross)
        busy[mode] = b
    assert busy["tiled"] <= busy["contiguous"]
    if (gr, gc) == (0, 0):
        assert gpu == [k // P for k in range(W)]


def test_tiled_placement_choices():
    """C3 / C4 at 4 GPUs tile 2 x 2 (blocks and combs each over 2 GPUs);
    at 2 GPUs contiguous packing is already best."""
    from paper_2007_03298_b200 import SyncStrategy, StrategyKind, Topology, WorldConfig, placement
    c3 = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(32, 4), 1, True)
    c4 = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(64, 8))
    assert placement(c3, 4)[2] == (2, 2) and placement(c4, 4)[2] == (2, 2)
    assert placement(c3, 2)[2] == (2, 1) and placement(c4, 8)[2] in ((4, 2), (2, 4))
    bsp = SyncStrategy(StrategyKind.BSP, Topology.RING, WorldConfig(32, 32))
    assert placement(bsp, 4)[2] == (0, 0)


def test_auto_placement_tiles_only_deep_chains():
    """placement=2: C3 / C4 on 4 GPUs (contiguous combs would chain over 4
    GPUs, 2 members each) are tiled; C2 on 4 GPUs (quads one member per GPU:
    push two-shot) and everything on 2 GPUs stay contiguous."""
    from paper_2007_03298_b200 import SyncStrategy, StrategyKind, Topology, WorldConfig, placement
    c2 = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(8, 2), 1, True)
    c3 = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(32, 4), 1, True)
    c4 = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(64, 8))
    assert placement(c3, 4, 2)[2] == (2, 2) and placement(c4, 4, 2)[2] == (2, 2)
    assert placement(c2, 4, 2)[2] == (0, 0) and placement(c3, 2, 2)[2] == (0, 0)
    assert placement(c4, 8, 2)[2] == (0, 0) and placement(c3, 8, 2)[2] == (0, 0)


def test_auto_placement_keeps_one_shot_rows_contiguous():
    """Rows of the one-shot size (<= 512 KiB) stay contiguous in auto mode:
    there contiguous packing keeps one parity GPU-local, while a tiling makes
    both parities exchange."""
    from paper_2007_03298_b200 import SyncStrategy, StrategyKind, Topology, WorldConfig, placement
    w64 = SyncStrategy(StrategyKind.DS_SYNC, Topology.RING, WorldConfig(64, 8))
    assert placement(w64, 4, 2, dim=256)[2] == (0, 0)
    assert placement(w64, 4, 2, dim=131072)[2] == (0, 0)      # exactly 512 KiB of fp32
    assert placement(w64, 4, 2, dim=131072 + 64)[2] == (2, 2)
    assert placement(w64, 4, 2, dim=65536, dtype="f64")[2] == (0, 0)
    assert placement(w64, 4, 1, dim=256)[2] == (2, 2)         # forced tiling ignores the size
