"""GPU parity: the CUDA path through the C-ABI against the C oracle (and the
compiled reference where it travelled), bit-exact int64 labels."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu

KINDS = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
         "fastest": T.fastest_path}


def rand_instance(rng, max_v=12, max_e=40, t_range=60, d_max=8, d_min=0):
    n = int(rng.integers(1, max_v + 1))
    m = int(rng.integers(0, max_e + 1))
    s = rng.integers(0, n, m)
    d = rng.integers(0, n, m)
    a = rng.integers(0, t_range + 1, m)
    b = a + rng.integers(d_min, d_max + 1, m)
    return (s, d, a, b), n


@pytest.mark.parametrize("ordering", [T.Ordering.STRICTLY_SUCCEEDS, T.Ordering.SUCCEEDS])
def test_small_random_instances(ordering):
    rng = np.random.default_rng(67 + int(ordering))
    for it in range(300):
        E, n = rand_instance(rng)
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=1 + it % 4))
        o = Oracle(E, n)
        for _ in range(2):
            ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2))
            v = int(rng.integers(0, n))
            for kind, fn in KINDS.items():
                got = fn(g, v, T.QueryWindow(ta, tb), T.AlgoOptions(ordering=ordering)).values
                want = o.query(kind, v, ta, tb, int(ordering))
                assert np.array_equal(got, want), (it, kind, n, E, v, ta, tb, got, want)
        g.close()


def test_medium_rmat_all_kinds():
    gen = T.GenConfig.rmat(14, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 5, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=64))
    o = Oracle(E, n)
    deg = np.bincount(E[0], minlength=n)
    for src in [int(np.argmax(deg)), int(np.flatnonzero(deg)[7])]:
        for w in [T.QueryWindow(0, 999_999), T.QueryWindow(300_000, 700_000)]:
            for kind, fn in KINDS.items():
                got = fn(g, src, w).values
                want = o.query(kind, src, w.t_a, w.t_b)
                assert np.array_equal(got, want), (kind, src, w, int((got != want).sum()))
