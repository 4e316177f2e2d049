"""Fastest path from hub sources: the candidate sweep split into sub-sweeps
(traverse.cuh split_seed_step; r = min over candidates d of A_d - d, so any
partition of the candidates swept separately and reduced by a minimum gives
path_algorithms.cpp:436-528's result). Bit-exact against the C oracle for
forced and automatic splits, every round mode and both orderings, and
against the reference library where it is present."""
import os

import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle, Reference

pytestmark = pytest.mark.gpu

MODES = [T.Mode.AUTO, T.Mode.SPARSE, T.Mode.DENSE, T.Mode.PULL]


@pytest.fixture(scope="module")
def hub_graph():
    # uniform starts over a short timeline: the hubs' out-edges have
    # thousands of distinct departures (config 4's shape at scale 14)
    gen = T.GenConfig.rmat(14, 16, 0.57, 0.19, 0.19, 200_000, 0.005, 44)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=64))
    deg = np.bincount(E[0], minlength=n)
    hubs = [int(v) for v in np.argsort(deg)[::-1][:3]]
    yield E, n, g, Oracle(E, n), hubs
    g.close()


def _fastest(g, v, w, mode=T.Mode.AUTO, ordering=None, split=None):
    old = os.environ.get("TGXD_FASTEST_SPLIT")
    if split is not None:
        os.environ["TGXD_FASTEST_SPLIT"] = str(split)
    try:
        st = T.EdgeMapStats()
        res = T.fastest_path(g, v, w, T.AlgoOptions(ordering=ordering, mode=mode, stats=st))
        return res.values, st
    finally:
        if split is not None:
            if old is None:
                del os.environ["TGXD_FASTEST_SPLIT"]
            else:
                os.environ["TGXD_FASTEST_SPLIT"] = old


@pytest.mark.parametrize("split", [1, 2, 7, 32, None])
def test_forced_splits_match_oracle(hub_graph, split):
    E, n, g, o, hubs = hub_graph
    w = T.QueryWindow(0, 199_999)
    for v in hubs[:2]:
        got, st = _fastest(g, v, w, split=split)
        assert st.candidates > 512  # the automatic split engages on these
        want = o.query("fastest", v, w.t_a, w.t_b)
        assert np.array_equal(got, want), (split, v, int((got != want).sum()))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("ordering", [T.Ordering.STRICTLY_SUCCEEDS, T.Ordering.SUCCEEDS])
def test_modes_and_orderings(hub_graph, mode, ordering):
    E, n, g, o, hubs = hub_graph
    for w in [T.QueryWindow(0, 199_999), T.QueryWindow(50_000, 120_000)]:
        v = hubs[2]
        got, _ = _fastest(g, v, w, mode=mode, ordering=ordering, split=5)
        want = o.query("fastest", v, w.t_a, w.t_b, int(ordering))
        assert np.array_equal(got, want), (mode, ordering, w, int((got != want).sum()))


def test_split_then_other_queries_on_the_same_handle(hub_graph):
    """A split sweep uses split x n slots; the queries after it (lazy EA /
    LD resets, a one-sweep fastest) must see clean state."""
    E, n, g, o, hubs = hub_graph
    w = T.QueryWindow(0, 199_999)
    _fastest(g, hubs[0], w, split=16)
    for kind, fn in (("earliest_arrival", T.earliest_arrival),
                     ("latest_departure", T.latest_departure)):
        got = fn(g, hubs[1], w).values
        assert np.array_equal(got, o.query(kind, hubs[1], w.t_a, w.t_b)), kind
    low = int(np.flatnonzero(np.bincount(E[0], minlength=n) == 3)[0])
    got, st = _fastest(g, low, w)
    assert np.array_equal(got, o.query("fastest", low, w.t_a, w.t_b))


def test_hub_against_reference_library(hub_graph):
    if not Reference.available():
        pytest.skip("oracle/_ref/libtgxref.so not built")
    E, n, g, o, hubs = hub_graph
    ref = Reference(E, n, True, 64)
    w = T.QueryWindow(0, 199_999)
    got, st = _fastest(g, hubs[0], w)
    assert np.array_equal(got, ref.query("fastest", hubs[0], w.t_a, w.t_b))
    ref.close()
