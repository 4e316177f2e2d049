"""Times a config's batch split into sub-batches of size s (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
wl = workload(name)
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = [q for q in wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
      if q.kind == "earliest_arrival"]
for s in (1, 2, 4, 8, 16, 32):
    tot = 0.0
    for i in range(0, len(qs), s):
        sub = qs[i:i + s]
        t, k = T.time_queries(g, "earliest_arrival", [q.vertex for q in sub], [q.window for q in sub],
                              warmup=1, steps=3)
        tot += t / 3
    print(name, "sub-batch", s, f"{tot:.3f} ms for {len(qs)} queries", flush=True)
