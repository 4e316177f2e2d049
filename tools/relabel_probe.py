"""Locality experiment: the config-2 edge list built as generated (ids
randomly permuted) and relabelled by in-degree (descending), same EA query
(source mapped); device-timed. Run with TGXD_LIB variants to compare."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--key", default="in", choices=["in", "out", "sum"])
args = ap.parse_args()
wl = workload(args.config)
t = time.time()
s, d, a, b = T.generate_edges(wl.gen)
n = wl.gen.n_vertices
print(f"host gen {time.time()-t:.1f}s m={len(s)}", flush=True)
g = T.TemporalGraph.build((s, d, a, b), n, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), n)[0]
tot, ker = T.time_queries(g, q.kind, [q.vertex], [q.window], warmup=3, steps=args.steps)
ref = T.earliest_arrival(g, q.vertex, q.window).values
print(f"as generated: {tot/args.steps:.4f} ms/query", flush=True)
indeg = np.bincount(d, minlength=n)
outdeg = np.bincount(s, minlength=n)
key = {"in": indeg, "out": outdeg, "sum": indeg + outdeg}[args.key]
order = np.argsort(-key, kind="stable")          # new id -> old id
newid = np.empty(n, np.uint32)
newid[order] = np.arange(n, dtype=np.uint32)      # old id -> new id
g.close()
g2 = T.TemporalGraph.build((newid[s], newid[d], a, b), n, True,
                           T.EngineConfig(index_cutoff=wl.index_cutoff))
src2 = int(newid[q.vertex])
tot2, ker2 = T.time_queries(g2, q.kind, [src2], [q.window], warmup=3, steps=args.steps)
got = T.earliest_arrival(g2, src2, q.window).values
ok = np.array_equal(got[newid], ref)
print(f"relabelled by {args.key}-degree: {tot2/args.steps:.4f} ms/query (labels equal: {ok})",
      flush=True)
