"""GPU: the selective-index cost model on the device (costmodel.cuh) — the
decision, beta_hat and k_hat of choose_access_method and count_in_window,
bit for bit against the reference (golden fixture, and the C restatement on
graphs the fixture does not hold); fit_cost_constants through the C-ABI."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
from tests import _support as S

pytestmark = pytest.mark.gpu


def _dev(g, d, verts, ta, tb, theta):
    ws = [T.QueryWindow(int(a), int(b)) if a <= b else _Raw(int(a), int(b)) for a, b in zip(ta, tb)]
    return T.access_decisions(g, T.Direction(d), verts, ws, theta)


class _Raw:  # an inverted window: the cost model takes any pair (no validation)
    def __init__(self, a, b):
        self.t_a, self.t_b = a, b


def test_cost_model_golden_on_device():
    z, graphs = S.cost_model()
    for name, (E, n, cutoff) in graphs.items():
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=cutoff))
        for d in (0, 1):
            verts, ta, tb, theta, want = S.cost_cases(z, name, d)
            got = _dev(g, d, verts, ta, tb, theta)
            for gv, wv, what in zip(got, want, ("method", "beta", "k_hat", "matches")):
                assert np.array_equal(gv, wv), (name, d, what, int(np.sum(gv != wv)))
        g.close()


@pytest.mark.parametrize("cutoff", [1, 8, 256])
def test_cost_model_matches_restatement(cutoff):
    gen = T.GenConfig.rmat(13, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 5, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=cutoff))
    o = Oracle(E, n)
    rng = np.random.default_rng(cutoff)
    for d in (0, 1):
        deg = g.degrees(T.Direction(d))
        verts = np.concatenate([np.argsort(-deg)[:200], rng.integers(0, n, 200)]).astype(np.uint32)
        ta = rng.integers(0, 1_000_000, len(verts)).astype(np.uint64)
        tb = ta + rng.integers(0, 400_000, len(verts)).astype(np.uint64)
        tb[::4] = (1 << 63) - 1
        got = _dev(g, d, verts, ta, tb, 0.15)
        want = o.access_decisions(d, cutoff, verts, ta, tb, 0.15)
        for gv, wv in zip(got, want):
            assert np.array_equal(gv, wv)
    # single-call mirrors
    v = int(np.argmax(g.degrees(T.Direction.OUT)))
    w = T.QueryWindow(100_000, 300_000)
    dec = T.choose_access_method(v, g, T.Direction.OUT, w, T.CostModelParams(theta_sel=0.5))
    m, b, k, c = o.access_decisions(0, cutoff, [v], [w.t_a], [w.t_b], 0.5)
    assert (int(dec.method), dec.beta_hat, dec.k_hat) == (int(m[0]), b[0], k[0])
    assert T.count_in_window(g, v, T.Direction.OUT, w) == int(c[0])
    with pytest.raises(T.OutOfRange):
        T.count_in_window(g, n, T.Direction.OUT, w)
    g.close()


def test_fit_cost_constants_golden():
    z, _ = S.cost_model()
    for deg, mat, ix, sc, c, cp in S.fit_cases(z):
        pts = [T.CalibrationPoint(int(a), int(b), float(x), float(y))
               for a, b, x, y in zip(deg, mat, ix, sc)]
        p = T.fit_cost_constants(pts, 0.3)
        assert (p.c, p.c_prime, p.theta_sel) == (c, cp, 0.3)
    with pytest.raises(T.InvalidArgument):
        T.fit_cost_constants([])
    with pytest.raises(T.InvalidArgument):
        T.fit_cost_constants([T.CalibrationPoint(0, 5, 1.0, 1.0)])
    assert T.cost_scan(100, 2.0) == 200.0
    assert T.cost_index_lookup(1024, 3.0, 2.0) == 26.0
    with pytest.raises(ValueError):
        T.cost_index_lookup(0, 1.0, 1.0)
