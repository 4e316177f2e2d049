"""GPU: host results of large EA / LD queries leave the device while the
async tail is still running (api.cu early copy) and the tail's changes are
patched in afterwards — identical to the device-resident result and to the
oracle; the re-copy fallback when the patch list overflows."""
import os

import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2_small():
    # config-2 distributions at scale 20 (2^20 slots: the staged host path)
    gen = T.GenConfig.rmat(20, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 11, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=256))
    yield g, Oracle(E, n), n
    g.close()


def _run(fn, g, v, w, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return fn(g, v, w).values
    finally:
        for k, x in old.items():
            if x is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = x


@pytest.mark.parametrize("kind", ["earliest_arrival", "latest_departure"])
def test_early_copy_matches(c2_small, kind):
    g, o, n = c2_small
    fn = T.earliest_arrival if kind == "earliest_arrival" else T.latest_departure
    deg = g.degrees(T.Direction.OUT if kind == "earliest_arrival" else T.Direction.IN)
    rng = np.random.default_rng(4)
    for v in [int(np.argmax(deg))] + [int(x) for x in rng.choice(np.flatnonzero(deg), 3)]:
        for w in (T.QueryWindow(0, 999_999), T.QueryWindow(250_000, 900_000)):
            got = _run(fn, g, v, w)
            want = o.query(kind, v, w.t_a, w.t_b)
            assert np.array_equal(got, want), (kind, v, w)
            assert np.array_equal(_run(fn, g, v, w, {"TGXD_NO_EARLY_COPY": "1"}), want)
            # a patch list of one entry forces the re-copy after the tail
            assert np.array_equal(_run(fn, g, v, w, {"TGXD_PATCH_CAP": "1"}), want)
            # the copy started from inside the round kernel: as early as
            # possible (every later round lists its changes), never, and with
            # the whole tail left to the round kernel
            for env in ({"TGXD_LOG_F": "1000000000"}, {"TGXD_LOG_F": "0"},
                        {"TGXD_LOG_F": "1000000000", "TGXD_HANDOFF_F": "0",
                         "TGXD_ASYNC_F": "0"},
                        {"TGXD_LOG_F": "1000000000", "TGXD_PATCH_CAP": "64"},
                        {"TGXD_NO_PACK24": "1"}, {"TGXD_NO_PACK24": "1", "TGXD_LOG_F": "0"}):
                assert np.array_equal(_run(fn, g, v, w, env), want), env


def test_early_copy_batch(c2_small):
    g, o, n = c2_small
    deg = g.degrees(T.Direction.OUT)
    srcs = [int(x) for x in np.argsort(deg.astype(np.int64))[::-1][:3]]
    wins = [T.QueryWindow(0, 999_999), T.QueryWindow(100_000, 999_999), T.QueryWindow(0, 500_000)]
    for mode in (T.Mode.SPARSE, T.Mode.AUTO):
        out = T.query_batch(g, "earliest_arrival", srcs, wins, mode=mode)
        for q in range(3):
            assert np.array_equal(out[q], o.query("earliest_arrival", srcs[q], wins[q].t_a,
                                                  wins[q].t_b)), (mode, q)
