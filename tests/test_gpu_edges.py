"""GPU: shortest duration, temporal BFS and the Overlaps ordering (SURVEY.md
8(f) rows 2-3) through the C-ABI, against the reference-generated fixtures
(all five metrics x all three orderings) and the C oracle."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
from paper_2401_02563_b200.configs import workload
from tests import _support as S

pytestmark = pytest.mark.gpu
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path, "shortest_duration": T.shortest_duration,
      "temporal_bfs": T.temporal_bfs}


def run(g, kind, v, ta, tb, ordv, mode=T.Mode.AUTO):
    return FN[kind](g, v, T.QueryWindow(ta, tb),
                    T.AlgoOptions(ordering=T.Ordering(ordv), mode=mode)).values


def test_hand_ext_cases():
    z = np.load(S.GOLDEN / "hand_ext.npz")
    for name, n, edges, kind, v, ta, tb, ordv in S.HAND_EXT:
        g = T.TemporalGraph.build(S.hand_edges(edges), n)
        got = run(g, kind, v, ta, tb, ordv)
        assert np.array_equal(got, z[name]), name
        for vert, want in S.HAND_EXT_EXPECT[name].items():
            assert got[vert] == want, (name, vert)


@pytest.mark.parametrize("cutoff", [1, 4])
def test_small_random_ext_golden(cutoff):
    """200 reference instances x 5 metrics x 3 orderings (enumerate_paths-checked)."""
    count = 0
    graphs = {}
    for E, n, v, ta, tb, kind, ordv, want in S.small_random_ext():
        key = id(E[0])
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=cutoff))
        got = run(g, kind, v, ta, tb, ordv)
        assert np.array_equal(got, want), (kind, ordv, n, v, ta, tb, got, want)
        g.close()
        count += 1
    assert count == 200 * 5 * 3


def test_rmat12_ext_golden():
    gen, n, m, edig, _, _, _ = S.scaled("rmat12")
    dig, qs, labels = S.rmat12_ext()
    g = T.TemporalGraph.generate(gen, True, T.EngineConfig(index_cutoff=64))
    for (kind, v, ta, tb, ordv), want in zip(qs, labels):
        assert np.array_equal(run(g, kind, v, ta, tb, ordv), want), (kind, v, ta, tb, ordv)


@pytest.mark.parametrize("mode", list(T.Mode))
def test_bfs_is_mode_invariant(mode):
    """Hop counts need round-synchronous admission: every mode request runs
    queue-driven or dense rounds and gives the same levels."""
    gen, n, m, edig, qs, labels, digests = S.scaled("rmat12")
    g = T.TemporalGraph.generate(gen, True, T.EngineConfig(index_cutoff=64))
    o = Oracle(T.generate_edges(gen), n)
    for kind, v, ta, tb in qs[:6]:
        want = o.query("temporal_bfs", v, ta, tb)
        assert np.array_equal(run(g, "temporal_bfs", v, ta, tb, 1, mode), want)


def test_medium_random_against_oracle():
    rng = np.random.default_rng(777)
    for it in range(30):
        E, n = S.rand_instance(rng, max_v=200, max_e=3000, t_range=400, d_max=30)
        g = T.TemporalGraph.build(E, n, bool(it % 3), T.EngineConfig(index_cutoff=1 + it % 16))
        o = Oracle(E, n, bool(it % 3))
        ta, tb = sorted(int(x) for x in rng.integers(0, 450, 2))
        v = int(rng.integers(0, n))
        for kind in FN:
            for ordv in (0, 1, 2):
                assert np.array_equal(run(g, kind, v, ta, tb, ordv),
                                      o.query(kind, v, ta, tb, ordv)), (it, kind, ordv)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_reduced_configs_edge_state_parity(name):
    wl = workload(name, -8)
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
    o = Oracle(T.generate_edges(wl.gen), wl.gen.n_vertices)
    q = qs[0]
    for kind in FN:
        for ordv in (1, 2) if kind != "shortest_duration" else (0, 1, 2):
            want = o.query(kind, q.vertex, q.window.t_a, q.window.t_b, ordv)
            got = run(g, kind, q.vertex, q.window.t_a, q.window.t_b, ordv)
            assert np.array_equal(got, want), (name, kind, ordv)


def test_weighted_shortest_duration_golden():
    """AlgoOptions::weighted (path_algorithms.cpp:196-258) on the device:
    the reference's fixtures, its invalid_argument (a reachable edge with a
    non-integer or negative weight) as InvalidArgument, every ordering."""
    z = np.load(S.GOLDEN / "weighted.npz")
    eoff = z["eoff"]
    errors = 0
    for it, n, v, ta, tb, ordv, code, lo in z["meta"]:
        a, b = eoff[it], eoff[it + 1]
        E = (z["src"][a:b], z["dst"][a:b], z["start"][a:b], z["end"][a:b], z["weight"][a:b])
        g = T.TemporalGraph.build(E, int(n))
        opts = T.AlgoOptions(ordering=T.Ordering(int(ordv)), weighted=True)
        if code:
            errors += 1
            with pytest.raises(T.InvalidArgument):
                T.shortest_duration(g, int(v), T.QueryWindow(int(ta), int(tb)), opts)
        else:
            got = T.shortest_duration(g, int(v), T.QueryWindow(int(ta), int(tb)), opts).values
            assert np.array_equal(got, z["labels"][lo:lo + n]), (it, ordv)
        g.close()
    assert errors > 0


def test_weighted_shortest_duration_rmat12():
    z = np.load(S.GOLDEN / "weighted.npz")
    gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 7, cube_root_starts=True)
    E = T.generate_edges(gen)
    assert S.edge_digest(E) == int(z["rmat_edge_digest"][0])
    W = np.random.default_rng(int(z["rmat_weight_seed"][0])).integers(0, 1000, len(E[0]))
    g = T.TemporalGraph.build(E + (W.astype(np.float64),), gen.n_vertices)
    for (v, ta, tb, ordv), want in zip(z["rmat_meta"], z["rmat_labels"]):
        got = T.shortest_duration(g, int(v), T.QueryWindow(int(ta), int(tb)),
                                  T.AlgoOptions(ordering=T.Ordering(int(ordv)),
                                                weighted=True)).values
        assert np.array_equal(got, want), (v, ordv)
    # unweighted queries on the weighted graph still sum durations
    o = Oracle(E, gen.n_vertices)
    v, ta, tb, _ = (int(x) for x in z["rmat_meta"][0])
    assert np.array_equal(T.shortest_duration(g, v, T.QueryWindow(ta, tb)).values,
                          o.query("shortest_duration", v, ta, tb))


def test_weighted_on_unweighted_graph_counts_edges():
    """Without stored weights every edge weighs 1.0 (TemporalEdge default)."""
    gen = T.GenConfig.rmat(10, 8, 0.57, 0.19, 0.19, 1_000_000, 0.02, 9, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n)
    o = Oracle(E, n, True, np.ones(len(E[0])))
    src = int(np.argmax(np.bincount(E[0], minlength=n)))
    for ordv in (0, 1, 2):
        got = T.shortest_duration(g, src, T.QueryWindow(0, 999_999),
                                  T.AlgoOptions(ordering=T.Ordering(ordv), weighted=True)).values
        assert np.array_equal(got, o.query("shortest_duration_weighted", src, 0, 999_999, ordv))
