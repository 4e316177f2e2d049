"""GPU: the reference-facing API through the C-ABI — golden fixtures from the
reference, hand-computed cases, error semantics, layouts, generators, the
C++ drop-in shim."""
import subprocess
from collections import Counter
from pathlib import Path

import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
from tests import _support as S

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path}


def test_hand_cases():
    z = np.load(S.GOLDEN / "hand_cases.npz")
    for name, n, edges, kind, v, ta, tb, ordv in S.HAND:
        g = T.TemporalGraph.build(S.hand_edges(edges), n)
        got = FN[kind](g, v, T.QueryWindow(ta, tb), T.AlgoOptions(ordering=T.Ordering(ordv)))
        assert np.array_equal(got.values, z[name]), name
        for vert, want in S.HAND_EXPECT[name].items():
            assert got.values[vert] == want, (name, vert)


@pytest.mark.parametrize("mode", [T.Mode.AUTO, T.Mode.SPARSE, T.Mode.DENSE, T.Mode.ASYNC, T.Mode.PULL])
def test_small_random_golden(mode):
    for E, n, v, ta, tb, kind, ordv, want in S.small_random():
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=2))
        got = FN[kind](g, v, T.QueryWindow(ta, tb),
                       T.AlgoOptions(ordering=T.Ordering(ordv), mode=mode)).values
        assert np.array_equal(got, want), (kind, ordv, n, v, ta, tb)


@pytest.mark.parametrize("name", ["rmat12", "uniform14"])
@pytest.mark.parametrize("cutoff", [1, 64, 1 << 30])
def test_scaled_golden_device_generated(name, cutoff):
    """The device-generated graph gives the reference's labels and digests;
    the index cutoff (1 = every vertex indexed) is results-neutral."""
    gen, n, m, edig, qs, labels, digests = S.scaled(name)
    g = T.TemporalGraph.generate(gen, True, T.EngineConfig(index_cutoff=cutoff))
    assert g.edge_count() == m
    for (kind, v, ta, tb), want, dg in zip(qs, labels, digests):
        got = FN[kind](g, v, T.QueryWindow(ta, tb)).values
        assert np.array_equal(got, want), (name, kind, v)
        assert T.digest_of(got) == int(dg)


def test_device_generator_matches_host_generator():
    """Same edge multiset on both sides; each layout segment sorted by key
    (tcsr.hpp:23-27, test_tcsr.cpp:60-76)."""
    gen = T.GenConfig.uniform(1 << 10, 1 << 14, 1_000_000, 0.01, 17)
    host = T.generate_edges(gen)
    g = T.TemporalGraph.generate(gen)
    want = Counter(zip(*(x.tolist() for x in host)))
    for d in (T.Direction.OUT, T.Direction.IN):
        s, t, a, b = g.flatten(d)
        assert Counter(zip(s.tolist(), t.tolist(), a.tolist(), b.tolist())) == want
        own = s if d == T.Direction.OUT else t
        key = a.astype(np.int64) if d == T.Direction.OUT else -b.astype(np.int64)
        assert np.all(np.diff(own.astype(np.int64)) >= 0)
        same = own[1:] == own[:-1]
        assert np.all(np.diff(key)[same] >= 0)


def test_undirected_symmetrization():
    rng = np.random.default_rng(5)
    for _ in range(20):
        E, n = S.rand_instance(rng, 10, 30)
        g = T.TemporalGraph.build(E, n, directed=False)
        o = Oracle(E, n, directed=False)
        assert g.edge_count() == len(E[0]) + int(np.sum(E[0] != E[1]))
        ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2))
        v = int(rng.integers(0, n))
        for kind, fn in FN.items():
            assert np.array_equal(fn(g, v, T.QueryWindow(ta, tb)).values,
                                  o.query(kind, v, ta, tb))


def test_error_semantics():
    g = T.TemporalGraph.build(S.hand_edges([(0, 1, 3, 5)]), 2)
    with pytest.raises(T.OutOfRange):          # path_algorithms.cpp:15-20
        T.earliest_arrival(g, 2)
    with pytest.raises(T.OutOfRange):
        T.latest_departure(g, 7)
    with pytest.raises(T.InvalidArgument):     # path_algorithms.cpp:22-25
        T.fastest_path(g, 0, T.QueryWindow(9, 3))
    with pytest.raises(T.InvalidArgument):     # internal.hpp:19-21
        T.earliest_arrival(g, 0, T.QueryWindow(1 << 63, (1 << 64) - 1))
    # weighted shortest duration: weight 1.0 without stored weights; a
    # reachable non-integer weight is invalid_argument (path_algorithms.cpp:196-203)
    assert T.shortest_duration(g, 0, T.QueryWindow(),
                               T.AlgoOptions(weighted=True)).values[1] == 1
    gw = T.TemporalGraph.build(S.hand_edges([(0, 1, 3, 5), (1, 0, 7, 8)]) + (
        np.array([2.0, 0.5]),), 2)
    with pytest.raises(T.InvalidArgument):
        T.shortest_duration(gw, 0, T.QueryWindow(), T.AlgoOptions(weighted=True))
    assert T.shortest_duration(gw, 0, T.QueryWindow(0, 6),  # the 0.5 edge is outside
                               T.AlgoOptions(weighted=True)).values[1] == 2
    with pytest.raises(T.TimeRangeError):      # beyond the device's int64 weight range
        gb = T.TemporalGraph.build(S.hand_edges([(0, 1, 3, 5)]) + (np.array([2.0 ** 63]),), 2)
        T.shortest_duration(gb, 0, T.QueryWindow(), T.AlgoOptions(weighted=True))
    with pytest.raises(T.OutOfRange):
        T.shortest_duration(g, 2)
    with pytest.raises(T.InvalidArgument):
        T.temporal_bfs(g, 0, T.QueryWindow(9, 3))
    with pytest.raises(T.InvalidArgument):
        T.earliest_arrival(g, 0, T.QueryWindow(9, 3), T.AlgoOptions(ordering=T.Ordering.OVERLAPS))
    with pytest.raises(T.OutOfRange, match="edge 1: endpoint"):   # types.cpp:43-47
        T.TemporalGraph.build(S.hand_edges([(0, 1, 3, 5), (0, 2, 3, 5)]), 2)
    with pytest.raises(T.OutOfRange, match="edge 0: end 4 precedes start 5"):  # :48-51
        T.TemporalGraph.build(S.hand_edges([(0, 1, 5, 4)]), 2)
    with pytest.raises(T.TimeRangeError):
        T.TemporalGraph.build(S.hand_edges([(0, 1, 5, 1 << 40)]), 2)


def test_unbounded_and_out_of_domain_windows():
    """Default window [0, 2^64-1]: LD writes the clamped t_b = 2^63-1 at the
    target; a window starting past every edge reaches nothing."""
    E = S.hand_edges([(0, 1, 3, 5), (1, 2, 7, 9)])
    g = T.TemporalGraph.build(E, 3)
    o = Oracle(E, 3)
    for kind, fn in FN.items():
        for w in [T.QueryWindow(), T.QueryWindow(0, 1 << 62), T.QueryWindow(1 << 40, 1 << 41)]:
            assert np.array_equal(fn(g, 0, w).values, o.query(kind, 0, w.t_a, w.t_b)), (kind, w)
    assert T.latest_departure(g, 2).values[2] == (1 << 63) - 1


def test_stats_and_work_counters():
    gen, n, m, edig, qs, labels, digests = S.scaled("rmat12")
    g = T.TemporalGraph.generate(gen, True, T.EngineConfig(index_cutoff=64))
    st = T.EdgeMapStats()
    kind, v, ta, tb = qs[0]
    # push-only rounds relax every admissible edge at least once
    T.earliest_arrival(g, v, T.QueryWindow(ta, tb), T.AlgoOptions(stats=st, mode=T.Mode.SPARSE))
    e_adm, v_reached = T.last_work(g, 0)
    E = T.generate_edges(gen)
    o = Oracle(E, n)
    lab = o.query("earliest_arrival", v, ta, tb)
    assert (e_adm, v_reached) == o.work("earliest_arrival", v, ta, tb, lab)
    assert st.rounds > 0 and st.edges_relaxed >= e_adm
    assert st.index_decisions > 0  # the source is the hub: it used the index
    # pull rounds may check fewer in-edges than there are admissible edges
    st2 = T.EdgeMapStats()
    r = T.earliest_arrival(g, v, T.QueryWindow(ta, tb), T.AlgoOptions(stats=st2, mode=T.Mode.PULL))
    assert np.array_equal(r.values, lab) and st2.rounds > 0 and st2.edges_relaxed > 0


def test_cpp_shim_runs():
    exe = Path("/tmp/tgx_b200_shim_test_gpu")
    res = subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                          str(ROOT / "tests" / "cpp" / "shim_test.cpp"),
                          "-L", str(ROOT / "paper_2401_02563_b200"), "-ltgxd",
                          f"-Wl,-rpath,{ROOT / 'paper_2401_02563_b200'}", "-o", str(exe)],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-2000:]
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "shim ok" in run.stdout


def test_edge_list_file_to_device_graph(tmp_path):
    """ingest.cpp's on-disk format (edgelist.py) feeding the device build."""
    from paper_2401_02563_b200 import edgelist as EL
    rng = np.random.default_rng(11)
    E, n = S.rand_instance(rng, max_v=50, max_e=400, t_range=300, d_max=20)
    p = str(tmp_path / "g.txt.gz")
    EL.write_edge_list(p, *E)
    L = EL.load_edge_list(p)
    g = T.TemporalGraph.build(L.edges, max(L.n_vertices, n))
    o = Oracle(E, max(L.n_vertices, n))
    for v in range(0, min(n, 10)):
        assert np.array_equal(T.earliest_arrival(g, v, T.QueryWindow(0, 400)).values,
                              o.query("earliest_arrival", v, 0, 400))


def test_lazy_label_reset_across_query_kinds():
    # api.cu launch: round-kernel EA / LD queries reset only the slots the
    # previous such query reached; every other route re-initializes. Mixed
    # sequences on one handle must keep every answer exact.
    gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 31, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=64))
    o = Oracle(E, n)
    deg = np.bincount(E[0], minlength=n)
    srcs = [int(x) for x in np.argsort(-deg)[:6]]
    w_full, w_part = T.QueryWindow(0, 999_999), T.QueryWindow(300_000, 800_000)
    seq = [("earliest_arrival", srcs[:4], [w_full, w_part, w_full, w_part], T.Mode.AUTO),
           ("earliest_arrival", srcs[:1], [w_part], T.Mode.AUTO),
           ("latest_departure", srcs[1:3], [w_full, w_part], T.Mode.SPARSE),
           ("fastest", srcs[2:3], [w_full], T.Mode.AUTO),
           ("earliest_arrival", srcs[:2], [w_full, w_full], T.Mode.AUTO),
           ("earliest_arrival", [srcs[0]] * 3, [w_full, w_part, w_full], T.Mode.AUTO),  # lanes
           ("latest_departure", srcs[3:4], [w_full], T.Mode.ASYNC),
           ("earliest_arrival", srcs, [w_part] * 6, T.Mode.PULL),
           ("temporal_bfs", srcs[4:5], [w_full], T.Mode.AUTO),
           ("earliest_arrival", srcs[5:6], [w_full], T.Mode.DENSE),
           ("earliest_arrival", srcs[:3], [w_part] * 3, T.Mode.AUTO)]
    for kind, vs, ws, mode in seq:
        out = T.query_batch(g, kind, vs, ws, mode=mode)
        for q, (v, w) in enumerate(zip(vs, ws)):
            assert np.array_equal(out[q], o.query(kind, v, w.t_a, w.t_b)), (kind, mode, q)
    g.close()
