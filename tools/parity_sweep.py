"""Parity sweep of every metric x ordering against the C oracle on RMAT /
uniform graphs of a few scales (diagnostics; the -m gpu suite has the fixed
cases)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path, "shortest_duration": T.shortest_duration,
      "temporal_bfs": T.temporal_bfs}
rng = np.random.default_rng(2024)
bad = 0
total = 0
for scale, kind_gen in ((14, "rmat"), (16, "rmat"), (15, "uniform"), (17, "rmat")):
    if kind_gen == "rmat":
        gen = T.GenConfig.rmat(scale, 8, 0.57, 0.19, 0.19, 100_000, 0.05, seed=scale,
                               cube_root_starts=True)
    else:
        gen = T.GenConfig.uniform(1 << scale, 8 << scale, 100_000, 0.05, scale)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    t0 = time.time()
    o = Oracle(E, n)
    for cutoff in (64, 4096):
        g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=cutoff))
        deg = g.degrees(T.Direction.OUT)
        srcs = [int(np.argmax(deg))] + [int(x) for x in rng.choice(np.flatnonzero(deg), 2)]
        for s in srcs:
            for w in ((0, 99_999), (20_000, 60_000)):
                for kind, fn in FN.items():
                    for ordv in (0, 1, 2):
                        if kind == "shortest_duration" and ordv != 2 and scale >= 17:
                            continue  # the oracle's edge-state relaxation is slow there
                        got = fn(g, s, T.QueryWindow(*w), T.AlgoOptions(ordering=T.Ordering(ordv))).values
                        want = o.query(kind, s, w[0], w[1], ordv)
                        total += 1
                        if not np.array_equal(got, want):
                            bad += 1
                            print("MISMATCH", kind_gen, scale, cutoff, s, w, kind, ordv,
                                  int(np.sum(got != want)), flush=True)
        g.close()
    print(kind_gen, scale, "done", f"{time.time() - t0:.1f}s", flush=True)
# 2^20 slots and more: the host results take the staged / early-copy path
# (int32 over PCIe while the async tail runs, patched afterwards)
for scale in (20, 21):
    gen = T.GenConfig.rmat(scale, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, seed=scale,
                           cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    t0 = time.time()
    o = Oracle(E, n)
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=256))
    deg = g.degrees(T.Direction.OUT)
    srcs = [int(np.argmax(deg))] + [int(x) for x in rng.choice(np.flatnonzero(deg), 3)]
    for s in srcs:
        for w in ((0, 999_999), (300_000, 900_000)):
            for kind in ("earliest_arrival", "latest_departure"):
                for ordv in (0, 1):
                    got = FN[kind](g, s, T.QueryWindow(*w), T.AlgoOptions(ordering=T.Ordering(ordv))).values
                    want = o.query(kind, s, w[0], w[1], ordv)
                    total += 1
                    if not np.array_equal(got, want):
                        bad += 1
                        print("MISMATCH rmat", scale, s, w, kind, ordv, int(np.sum(got != want)),
                              flush=True)
    g.close()
    print("rmat", scale, "(staged host results) done", f"{time.time() - t0:.1f}s", flush=True)
print("checked", total, "mismatches", bad)
