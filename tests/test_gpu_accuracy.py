"""GPU: the estimator-accuracy measurement (tgx.cpp:454-488) through the
device cost model equals the same computation on the reference library."""
import numpy as np
import pytest

import paper_2401_02563_b200 as T
from paper_2401_02563_b200.accuracy import estimator_accuracy
from paper_2401_02563_b200.edgelist import window_for_recent_fraction
from oracle.pyoracle import Reference

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not Reference.available(), reason="reference library not built")
def test_estimator_accuracy_matches_reference():
    gen = T.GenConfig.rmat(13, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 3, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    cutoffs, fractions = [32, 256], [1.0, 10.0, 50.0, 100.0]
    got = estimator_accuracy(E, n, cutoffs, fractions)
    for (cutoff, pct, total, acc) in got:
        r = Reference(E, n, True, cutoff)
        t_a, t_b = window_for_recent_fraction(E[2], E[3], pct / 100.0)
        agree = count = 0
        for d in (0, 1):
            deg = np.bincount(E[d], minlength=n)
            verts = np.flatnonzero(deg >= cutoff).astype(np.uint32)
            k = len(verts)
            m, _, _, matches = r.access_decisions(d, verts, np.full(k, t_a, np.uint64),
                                                  np.full(k, t_b, np.uint64), 0.2)
            should = matches / deg[verts] <= 0.2
            agree += int(np.sum(should == (m == 0)))
            count += k
        assert total == count
        assert acc == (1.0 if count == 0 else agree / count), (cutoff, pct)
    assert any(0.0 < a < 1.0 or a == 1.0 for *_, a in got)
