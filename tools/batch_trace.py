"""Round trace of one batched query group (diagnostics): config [kind]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
kind = sys.argv[2] if len(sys.argv) > 2 else "earliest_arrival"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = workload(name)
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = [q for q in wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
      if q.kind == kind]
if k:
    qs = qs[:k]
T.set_trace(g, 4096)
for rep in range(2):
    st = T.EdgeMapStats()
    T.query_batch(g, kind, [q.vertex for q in qs], [q.window for q in qs], width=4, stats=st)
print(name, kind, len(qs), st)
tr = T.get_trace(g, 4096).astype(np.int64)
out = []
for r, row in enumerate(tr):
    if row[0] == 0:
        break
    t = 'L' if row[7] == 1 else ('D' if row[7] == 2 else ('P' if row[7] == 3 else 'G'))
    out.append(f"{t}{row[3]}:{(row[1]-row[0])/1e3:.0f}+{(row[2]-row[1])/1e3:.0f}")
print(" ".join(out))
