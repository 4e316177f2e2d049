import sys; sys.path.insert(0,'/root/repo')
import numpy as np, paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload
wl = workload("c3")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
ea = [q for q in qs if q.kind == "earliest_arrival"]
T.set_trace(g, 4096)
for rep in range(2):
    st = T.EdgeMapStats()
    T.query_batch(g, "earliest_arrival", [q.vertex for q in ea], [q.window for q in ea], width=4, stats=st)
print(st)
tr = T.get_trace(g, 4096).astype(np.int64)
for r, row in enumerate(tr):
    if row[0] == 0: break
    print(f"  r{r:3d} F={row[3]:8d} A={(row[1]-row[0])/1e3:6.1f} B={(row[2]-row[1])/1e3:6.1f} ch={row[4]:6d} sm={row[5]:6d} push={row[6]:7d} {'L' if row[7]==1 else ('D' if row[7]==2 else ('P' if row[7]==3 else 'G'))}")
