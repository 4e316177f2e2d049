import sys; sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 13, cube_root_starts=True)
E = T.generate_edges(gen); n = gen.n_vertices
g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=128))
o = Oracle(E, n)
rng = np.random.default_rng(12)
deg = np.bincount(E[0], minlength=n)
srcs = [int(x) for x in rng.choice(np.flatnonzero(deg), 10)]
wins = [T.QueryWindow(0, 999_999) if i % 2 else T.QueryWindow(200_000, 900_000) for i in range(10)]
views = [g.view(3) for _ in range(3)]
fn = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure, "fastest": T.fastest_path}
bad = 0
for kind in fn:
    for i in range(10):
        out = fn[kind](views[i % 3], srcs[i], wins[i]).values   # one at a time: no concurrency
        bad += not np.array_equal(out, o.query(kind, srcs[i], wins[i].t_a, wins[i].t_b))
print("sequential through views, check build: mismatches", bad)
