"""Fastest on the barrier-free engine (ASYNC mode) vs the round engine at
scale 20 (diagnostics: the -m gpu suite checks small instances)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T

rng = np.random.default_rng(1)
for scale in (18, 20):
    gen = T.GenConfig.rmat(scale, 16, 0.57, 0.19, 0.19, 10_000_000, 0.005, scale)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=256))
    deg = g.degrees(T.Direction.OUT)
    srcs = [int(x) for x in rng.choice(np.flatnonzero((deg > 0) & (deg < 200)), 6)]
    for s in srcs:
        w = T.QueryWindow(0, 9_999_999)
        a = T.fastest_path(g, s, w, T.AlgoOptions(mode=T.Mode.ASYNC)).values
        b = T.fastest_path(g, s, w, T.AlgoOptions(mode=T.Mode.SPARSE)).values
        c = T.fastest_path(g, s, w).values
        print(scale, s, "async==sparse", np.array_equal(a, b), int(np.sum(a != b)),
              "auto==sparse", np.array_equal(c, b), flush=True)
    g.close()
