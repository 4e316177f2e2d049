"""One query on a BASELINE workload with device counters (diagnostics)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--delta", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--trace", action="store_true")
args = ap.parse_args()
wl = workload(args.config, args.delta)
t = time.time()
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
print(f"build {time.time()-t:.2f}s n={g.vertex_count()} m={g.edge_count()} indexed={g.indexed_count(0)}", flush=True)
T.set_trace(g, 4096)
qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
for q in qs[:4]:
    for r in range(args.reps):
        st = T.EdgeMapStats()
        T.query_batch(g, q.kind, [q.vertex], [q.window], width=4, stats=st, mode=T.Mode(args.mode))
    e, v = T.last_work(g, 0)
    print(q.kind, q.vertex, q.window, st, "E_adm", e, "V", v, flush=True)
    if args.trace:
        tr = T.get_trace(g, 4096).astype(np.int64)
        for r, row in enumerate(tr):
            if row[0] == 0: break
            print(f"  r{r:3d} F={row[3]:9d} A={(row[1]-row[0])/1e3:8.1f}us B={(row[2]-row[1])/1e3:8.1f}us chunks={row[4]:8d} smalls={row[5]:8d} pushes={row[6]:8d}")
