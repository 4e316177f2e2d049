"""GPU: graph views (tgxd_graph_view) — handles sharing one device graph
with their own streams and workspaces — answer queries driven concurrently
from several host threads exactly like the owning handle."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,streams", [(12, 3), (20, 4)])
def test_concurrent_queries_match(scale, streams):
    gen = T.GenConfig.rmat(scale, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 13,
                           cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=128))
    o = Oracle(E, n)
    rng = np.random.default_rng(scale)
    deg = np.bincount(E[0], minlength=n)
    srcs = [int(x) for x in rng.choice(np.flatnonzero(deg), 10)]
    wins = [T.QueryWindow(0, 999_999) if i % 2 else T.QueryWindow(200_000, 900_000)
            for i in range(10)]
    for kind in ("earliest_arrival", "latest_departure", "fastest"):
        out = T.concurrent_queries(g, kind, srcs, wins, streams=streams)
        for i in range(10):
            assert np.array_equal(out[i], o.query(kind, srcs[i], wins[i].t_a, wins[i].t_b)), \
                (kind, i)
    g.close()


def test_view_errors_and_lifetime():
    gen = T.GenConfig.rmat(10, 8, 0.57, 0.19, 0.19, 1_000_000, 0.02, 1)
    g = T.TemporalGraph.generate(gen)
    v = g.view(2)
    with pytest.raises(ValueError):
        v.view(2)  # a view of a view
    with pytest.raises(ValueError):
        g.view(0)
    a = T.earliest_arrival(v, 0, T.QueryWindow(0, 999_999)).values
    b = T.earliest_arrival(g, 0, T.QueryWindow(0, 999_999)).values
    assert np.array_equal(a, b)
    assert v.vertex_count() == g.vertex_count() and v.edge_count() == g.edge_count()
    v.close()
    assert np.array_equal(T.earliest_arrival(g, 0, T.QueryWindow(0, 999_999)).values, b)
    g.close()


def test_views_are_released_when_the_stream_count_changes():
    """concurrent_queries replaces its serve views when `streams` changes;
    closed views leave the parent's list (no growth, no stale handles)."""
    gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 13, cube_root_starts=True)
    g = T.TemporalGraph.generate(gen)
    E = T.generate_edges(gen)
    o = Oracle(E, gen.n_vertices)
    deg = np.bincount(E[0], minlength=gen.n_vertices)
    srcs = [int(x) for x in np.flatnonzero(deg)[:4]]
    wins = [T.QueryWindow(0, 999_999)] * 4
    for streams in (2, 3, 2, 4):
        out = T.concurrent_queries(g, "earliest_arrival", srcs, wins, streams=streams)
        assert len(g._views) == streams
        for i, s in enumerate(srcs):
            assert np.array_equal(out[i], o.query("earliest_arrival", s, 0, 999_999))
    g.close()
    assert g._views == []
