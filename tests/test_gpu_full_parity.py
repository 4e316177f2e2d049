"""GPU, full BASELINE sizes: configs 3, 4 and 5 label for label against the
compiled reference library (oracle/_ref/libtgxref.so, the unmodified
reference sources, on all host cores) — north_star's "bit-exact labels on all
five configs". Configs 1 and 2 are pinned at full size in test_gpu_configs.py.

Every query of each config is compared: config 3's 32 EA + 32 LD queries
(one at a time on one handle, kinds interleaved, so every query resets the
previous one's labels and uploads its own parameters, and as two batches),
config 4's fastest (path_algorithms.cpp:436-528) and latest departure
(:310-357), config 5's 32 earliest-arrival queries (:262-308) batched and one
at a time. With TGXD_PARITY_LOG=<path> each comparison appends a JSON line
(query, identical, reference and device digests)."""
import json
import os

import numpy as np
import pytest

import paper_2401_02563_b200 as T
from oracle.pyoracle import Reference, digest
from paper_2401_02563_b200.configs import workload

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(not Reference.available(),
                                 reason="reference library not built (oracle/_ref)")]
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path}


def _log(rec):
    path = os.environ.get("TGXD_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


class Setup:
    def __init__(self, name):
        self.name = name
        self.wl = workload(name)
        self.g = T.TemporalGraph.generate(self.wl.gen, True,
                                          T.EngineConfig(index_cutoff=self.wl.index_cutoff))
        self.n = self.g.vertex_count()
        self.qs = self.wl.queries(self.g.degrees(T.Direction.OUT),
                                  self.g.degrees(T.Direction.IN), self.n)
        Reference.set_workers(os.cpu_count() or 1)
        self.ref = Reference(T.generate_edges(self.wl.gen), self.n, True, self.wl.index_cutoff)
        self._want = {}

    def want(self, i):
        if i not in self._want:
            q = self.qs[i]
            self._want[i] = self.ref.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
        return self._want[i]

    def check(self, i, got, how):
        q = self.qs[i]
        want = self.want(i)
        same = bool(np.array_equal(got, want))
        unreached = T.K_UNREACHED_MAX if q.kind == "latest_departure" else T.K_UNREACHED_MIN
        _log({"config": self.name, "query": i, "kind": q.kind, "vertex": q.vertex,
              "window": [q.window.t_a, q.window.t_b], "how": how, "identical": same,
              "ref_digest": digest(want), "gpu_digest": digest(got),
              "reached": int(np.count_nonzero(want != unreached))})
        assert same, (self.name, i, q.kind, q.vertex, how,
                      int(np.count_nonzero(got != want)))

    def close(self):
        self.ref.close()
        self.g.close()


@pytest.fixture(scope="module")
def c3():
    s = Setup("c3")
    yield s
    s.close()


@pytest.fixture(scope="module")
def c4():
    s = Setup("c4")
    yield s
    s.close()


@pytest.fixture(scope="module")
def c5():
    s = Setup("c5")
    yield s
    s.close()


def test_c3_every_query_one_at_a_time(c3):
    """64 single queries on one handle, EA and LD interleaved (each resets
    the previous query's reached slots and seeds a new root)."""
    for i, q in enumerate(c3.qs):
        c3.check(i, FN[q.kind](c3.g, q.vertex, q.window).values, "single")


def test_c3_batches(c3):
    for kind in ("earliest_arrival", "latest_departure"):
        idx = [i for i, q in enumerate(c3.qs) if q.kind == kind]
        out = T.query_batch(c3.g, kind, [c3.qs[i].vertex for i in idx],
                            [c3.qs[i].window for i in idx])
        for j, i in enumerate(idx):
            c3.check(i, out[j], "batch")


def test_c4_fastest_and_latest_departure(c4):
    for i, q in enumerate(c4.qs):
        c4.check(i, FN[q.kind](c4.g, q.vertex, q.window).values, "single")
    # the other schedules give the same fixpoints
    fq, lq = c4.qs
    c4.check(0, FN["fastest"](c4.g, fq.vertex, fq.window,
                              T.AlgoOptions(mode=T.Mode.SPARSE)).values, "single-sparse")
    c4.check(1, FN["latest_departure"](c4.g, lq.vertex, lq.window,
                                       T.AlgoOptions(mode=T.Mode.PULL)).values, "single-pull")


def test_c5_batch_and_singles(c5):
    """The 16 full-window and 16 10%-window queries as the config's batch
    (AUTO schedule) and one at a time."""
    for half in (range(0, 16), range(16, 32)):
        idx = list(half)
        out = T.query_batch(c5.g, "earliest_arrival", [c5.qs[i].vertex for i in idx],
                            [c5.qs[i].window for i in idx])
        for j, i in enumerate(idx):
            c5.check(i, out[j], "batch16")
        del out
    for i, q in enumerate(c5.qs):
        c5.check(i, T.earliest_arrival(c5.g, q.vertex, q.window).values, "single")
