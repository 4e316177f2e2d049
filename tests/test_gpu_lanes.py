"""GPU: batches on the lane-per-query engine (lanes.cuh, TGXD_MODE_LANES —
AUTO's choice for 2..32 earliest-arrival / latest-departure queries from one
source) against
the oracle query by query, and against the slot-major batch engine."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
from tests import _support as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmat():
    gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 21, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    return E, n, Oracle(E, n)


def _queries(rng, E, n, k, kind):
    deg = np.bincount(E[0] if kind == "earliest_arrival" else E[1], minlength=n)
    srcs = [int(x) for x in rng.choice(np.flatnonzero(deg), k)]
    wins = []
    for i in range(k):
        off = int(rng.integers(0, 990_000))
        wins.append([T.QueryWindow(0, 999_999), T.QueryWindow(off, off + 9_999),
                     T.QueryWindow(off, off + 199_999), T.QueryWindow(off, 1 << 40)][i % 4])
    return srcs, wins


@pytest.mark.parametrize("k", [2, 17, 32])
@pytest.mark.parametrize("cutoff", [1, 2, 256])
@pytest.mark.parametrize("kind", ["earliest_arrival", "latest_departure"])
def test_lanes_batch_matches_oracle(rmat, k, cutoff, kind):
    E, n, o = rmat
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=cutoff))
    rng = np.random.default_rng(k * 7 + cutoff)
    srcs, wins = _queries(rng, E, n, k, kind)
    for ordering in (T.Ordering.STRICTLY_SUCCEEDS, T.Ordering.SUCCEEDS):
        out = T.query_batch(g, kind, srcs, wins, ordering=ordering, mode=T.Mode.LANES)
        for q in range(k):
            want = o.query(kind, srcs[q], wins[q].t_a, wins[q].t_b, int(ordering))
            assert np.array_equal(out[q], want), (kind, k, cutoff, ordering, q)
    g.close()


def test_lanes_repeated_sources_and_auto(rmat):
    E, n, o = rmat
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=64))
    deg = np.bincount(E[0], minlength=n)
    hub = int(np.argmax(deg))
    srcs = [hub] * 5 + [int(np.flatnonzero(deg)[0])] * 3
    wins = [T.QueryWindow(0, 999_999), T.QueryWindow(0, 500_000), T.QueryWindow(400_000, 999_999),
            T.QueryWindow(999_999, 999_999), T.QueryWindow(7, 7), T.QueryWindow(0, 999_999),
            T.QueryWindow(0, 999_999), T.QueryWindow(123_456, 654_321)]
    auto = T.query_batch(g, "earliest_arrival", srcs, wins)
    lanes = T.query_batch(g, "earliest_arrival", srcs, wins, mode=T.Mode.LANES)
    slot = T.query_batch(g, "earliest_arrival", srcs, wins, mode=T.Mode.SPARSE)
    assert np.array_equal(auto, lanes) and np.array_equal(lanes, slot)
    for q in range(len(srcs)):
        assert np.array_equal(lanes[q], o.query("earliest_arrival", srcs[q], wins[q].t_a,
                                                wins[q].t_b, 1))
    # E_adm / V_reached bookkeeping reads the batch's labels
    e_l = [T.last_work(g, q) for q in range(len(srcs))]
    T.query_batch(g, "earliest_arrival", srcs, wins, mode=T.Mode.SPARSE)
    assert e_l == [T.last_work(g, q) for q in range(len(srcs))]
    g.close()


def test_lanes_golden_small_instances():
    # the reference's small random fixtures, grouped into batches per instance
    groups = {}
    for E, n, v, ta, tb, kind, ordv, want in S.small_random():
        if kind == "fastest":
            continue
        key = (b"".join(np.ascontiguousarray(x).tobytes() for x in E), n, kind, ordv)
        groups.setdefault(key, (E, n, kind, ordv, []))[4].append((v, ta, tb, want))
    seen = 0
    for E, n, kind, ordv, qs in groups.values():
        if len(qs) < 2:
            qs = qs * 2
        qs = qs[:32]
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=2))
        out = T.query_batch(g, kind, [q[0] for q in qs], [T.QueryWindow(q[1], q[2]) for q in qs],
                            ordering=T.Ordering(ordv), mode=T.Mode.LANES)
        for q, (v, ta, tb, want) in enumerate(qs):
            assert np.array_equal(out[q], want), (kind, ordv, v, ta, tb)
        g.close()
        seen += 1
    assert seen > 50


def test_lanes_mode_rejects_what_it_cannot_run(rmat):
    E, n, _ = rmat
    g = T.TemporalGraph.build(E, n)
    with pytest.raises(T.Unsupported):
        T.query_batch(g, "earliest_arrival", [1], [T.QueryWindow(0, 10)], mode=T.Mode.LANES)
    with pytest.raises(T.Unsupported):
        T.query_batch(g, "fastest", [1, 2], [T.QueryWindow(0, 10)] * 2, mode=T.Mode.LANES)
    with pytest.raises(T.Unsupported):
        T.query_batch(g, "earliest_arrival", list(range(33)), [T.QueryWindow(0, 10)] * 33,
                      mode=T.Mode.LANES)
    g.close()


def test_lanes_auto_window_sweep(rmat):
    # one source, 32 windows: AUTO runs the lane engine; same labels as slot-major
    E, n, o = rmat
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=16))
    src = int(np.argmax(np.bincount(E[0], minlength=n)))
    wins = [T.QueryWindow(15_000 * i, 999_999 - 15_000 * i) for i in range(32)]
    for kind in ("earliest_arrival", "latest_departure"):
        auto = T.query_batch(g, kind, [src] * 32, wins)
        slot = T.query_batch(g, kind, [src] * 32, wins, mode=T.Mode.SPARSE)
        assert np.array_equal(auto, slot), kind
        for q in (0, 13, 31):
            assert np.array_equal(auto[q], o.query(kind, src, wins[q].t_a, wins[q].t_b, 1))
    g.close()


def test_lanes_window_sweep_at_scale():
    # a one-source sweep of 24 windows on a 2^20-vertex graph (AUTO: lane engine,
    # host results through the staged path) equals the queries one by one
    gen = T.GenConfig.rmat(20, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 5, cube_root_starts=True)
    g = T.TemporalGraph.generate(gen, True, T.EngineConfig(index_cutoff=256))
    src = int(np.argmax(g.degrees(T.Direction.OUT)))
    wins = [T.QueryWindow(20_000 * i, 999_999 - 10_000 * i) for i in range(24)]
    for kind in ("earliest_arrival", "latest_departure"):
        v = src if kind == "earliest_arrival" else int(np.argmax(g.degrees(T.Direction.IN)))
        batch = T.query_batch(g, kind, [v] * 24, wins)
        for q in (0, 7, 23):
            fn = T.earliest_arrival if kind == "earliest_arrival" else T.latest_departure
            assert np.array_equal(batch[q], fn(g, v, wins[q]).values), (kind, q)
    g.close()
