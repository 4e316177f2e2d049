"""Reduced-config parity per mode (diagnostics): python tools/fast_repro.py c4 -8"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
from paper_2401_02563_b200.configs import workload

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
delta = int(sys.argv[2]) if len(sys.argv) > 2 else -8
wl = workload(name, delta)
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
o = Oracle(T.generate_edges(wl.gen), wl.gen.n_vertices)
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path}
for q in qs:
    want = o.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
    for mode in range(5):
        for div in ("8", "1000000"):
            os.environ["TGXD_PULL_DIV"] = div
            st = T.EdgeMapStats()
            got = FN[q.kind](g, q.vertex, q.window, T.AlgoOptions(mode=T.Mode(mode), stats=st)).values
            bad = np.nonzero(got != want)[0]
            print(q.kind, "mode", mode, "div", div, "bad", len(bad), bad[:5].tolist(),
                  got[bad[:5]].tolist(), want[bad[:5]].tolist(), "rounds", st.rounds, flush=True)
