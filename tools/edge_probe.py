"""Times the edge-state kinds and temporal BFS on a config graph (one query each)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = workload(name, delta)
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())[0]
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path, "shortest_duration": T.shortest_duration,
      "temporal_bfs": T.temporal_bfs}
for kind, ordv in [("temporal_bfs", 1), ("earliest_arrival", 2), ("latest_departure", 2),
                   ("fastest", 2), ("temporal_bfs", 2), ("shortest_duration", 2),
                   ("shortest_duration", 1), ("shortest_duration", 0)]:
    st = T.EdgeMapStats()
    t = time.time()
    r = FN[kind](g, q.vertex, q.window, T.AlgoOptions(ordering=T.Ordering(ordv), stats=st)).values
    dt = time.time() - t
    reached = int((r != (r.min() if kind == "latest_departure" else r.max())).sum())
    print(name, kind, ordv, f"wall {dt*1e3:.2f} ms kernel {st.kernel_ms:.3f} ms rounds {st.rounds} "
          f"checked {st.edges_relaxed} reached {reached}", flush=True)
