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
            big = 1 << 62
            a_last = (row[8] - row[0]) / 1e3 if row[8] else 0
            a_first = (big - row[9] - row[0]) / 1e3 if row[9] else 0
            b_last = (row[10] - row[1]) / 1e3 if row[10] else 0
            b_first = (big - row[11] - row[1]) / 1e3 if row[11] else 0
            print(f"  r{r:3d} F={row[3]:9d} A={(row[1]-row[0])/1e3:7.1f}us [warps {a_first:6.1f}..{a_last:6.1f}] B={(row[2]-row[1])/1e3:7.1f}us [warps {b_first:6.1f}..{b_last:6.1f}] ch={row[4]:7d} sm={row[5]:7d} push={row[6]:8d} {'L' if row[7]==1 else ('D' if row[7]==2 else ('P' if row[7]==3 else 'G'))}")
