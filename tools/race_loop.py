"""Repeat the reduced config-4 fastest query on fresh graphs (race hunting)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
from paper_2401_02563_b200.configs import workload

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
modes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 4]
wl = workload(name, -8)
o = Oracle(T.generate_edges(wl.gen), wl.gen.n_vertices)
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path}
want = {}
fails = {m: 0 for m in modes}
runs = 0
for rep in range(reps):
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    if os.environ.get("RACE_TRACE"):
        T.set_trace(g, 4096)
    qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
    if len(sys.argv) > 4:  # kind override: the same sources and windows
        import dataclasses
        qs = [dataclasses.replace(q, kind=sys.argv[4]) for q in qs]
    for qi, q in enumerate(qs):
        if qi not in want:
            want[qi] = o.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
        for m in modes:
            for it in range(5):
                got = FN[q.kind](g, q.vertex, q.window, T.AlgoOptions(mode=T.Mode(m))).values
                bad = np.nonzero(got != want[qi])[0]
                runs += 1
                if os.environ.get("RACE_TRACE") and (len(bad) or (rep == 0 and it == 0)):
                    tr = T.get_trace(g, 4096).astype(np.int64)
                    print("TRACE", "bad" if len(bad) else "good", " ".join(
                        f"{'LDPG'[[1, 2, 3, 0].index(r[7])] if r[7] in (0, 1, 2, 3) else '?'}{r[3]}/{r[6]}"
                        for r in tr if r[0]), flush=True)
                if len(bad):
                    fails[m] += 1
                    print("FAIL rep", rep, q.kind, "mode", m, "it", it, "bad", len(bad), bad[:4].tolist(),
                          got[bad[:4]].tolist(), want[qi][bad[:4]].tolist(), flush=True)
    g.close()
print("runs", runs, "fails", fails)
