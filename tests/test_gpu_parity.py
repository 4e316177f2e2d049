"""GPU parity: the CUDA path through the C-ABI against the C oracle (pinned to
the reference, tests/test_oracle.py), bit-exact int64 labels."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu

KINDS = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
         "fastest": T.fastest_path}
MODES = [T.Mode.AUTO, T.Mode.SPARSE, T.Mode.DENSE, T.Mode.ASYNC, T.Mode.PULL]


def rand_instance(rng, max_v=12, max_e=40, t_range=60, d_max=8, d_min=0):
    n = int(rng.integers(1, max_v + 1))
    m = int(rng.integers(0, max_e + 1))
    s = rng.integers(0, n, m)
    d = rng.integers(0, n, m)
    a = rng.integers(0, t_range + 1, m)
    b = a + rng.integers(d_min, d_max + 1, m)
    return (s, d, a, b), n


@pytest.mark.parametrize("ordering", [T.Ordering.STRICTLY_SUCCEEDS, T.Ordering.SUCCEEDS])
@pytest.mark.parametrize("mode", MODES)
def test_small_random_instances(ordering, mode):
    """Mirrors test_algorithms.cpp:171-194 (random_instance(rng, 9, 28) x windows)."""
    rng = np.random.default_rng(67 + int(ordering) * 3 + int(mode))
    for it in range(150):
        E, n = rand_instance(rng)
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=1 + it % 4))
        o = Oracle(E, n)
        for _ in range(2):
            ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2))
            v = int(rng.integers(0, n))
            for kind, fn in KINDS.items():
                opts = T.AlgoOptions(ordering=ordering, mode=mode)
                got = fn(g, v, T.QueryWindow(ta, tb), opts).values
                want = o.query(kind, v, ta, tb, int(ordering))
                assert np.array_equal(got, want), (it, kind, n, E, v, ta, tb, got, want)
        g.close()


@pytest.mark.parametrize("mode", MODES)
def test_medium_rmat_all_kinds(mode):
    gen = T.GenConfig.rmat(14, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 5, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=64))
    o = Oracle(E, n)
    deg = np.bincount(E[0], minlength=n)
    for src in [int(np.argmax(deg)), int(np.flatnonzero(deg)[7])]:
        for w in [T.QueryWindow(0, 999_999), T.QueryWindow(300_000, 700_000)]:
            for kind, fn in KINDS.items():
                got = fn(g, src, w, T.AlgoOptions(mode=mode)).values
                want = o.query(kind, src, w.t_a, w.t_b)
                assert np.array_equal(got, want), (kind, src, w, int((got != want).sum()))


@pytest.mark.parametrize("mode", MODES)
def test_batched_queries_match_single(mode):
    gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 9, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=256))
    o = Oracle(E, n)
    rng = np.random.default_rng(3)
    deg = np.bincount(E[0], minlength=n)
    srcs = [int(x) for x in rng.choice(np.flatnonzero(deg), 12)]
    wins = []
    for i in range(12):
        off = int(rng.integers(0, 900_000))
        wins.append(T.QueryWindow(0, 999_999) if i % 2 == 0 else T.QueryWindow(off, off + 99_999))
    for kind in ("earliest_arrival", "latest_departure", "fastest"):
        out = T.query_batch(g, kind, srcs, wins, mode=mode)
        for q in range(12):
            want = o.query(kind, srcs[q], wins[q].t_a, wins[q].t_b)
            assert np.array_equal(out[q], want), (kind, q)
