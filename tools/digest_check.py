"""Label digests of the BASELINE workloads' queries (A/B of library builds and
environment knobs: two runs must print identical lines).
usage: [TGXD_LIB=...] python tools/digest_check.py [--configs c2,c1,c4,c5]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import c2_rotation, workload

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c1,c4,c5")
ap.add_argument("--max-queries", type=int, default=8)
args = ap.parse_args()
for name in args.configs.split(","):
    wl = workload(name)
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    deg_o, deg_i = g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN)
    qs = c2_rotation(deg_o) if name == "c2" else wl.queries(deg_o, deg_i, g.vertex_count())
    for q in qs[:args.max_queries]:
        for rep in range(2):  # the second run starts from the first one's lazy reset
            out = T.query_batch(g, q.kind, [q.vertex], [q.window], width=8)[0]
            print(name, q.kind, q.vertex, q.window.t_a, q.window.t_b, rep, hex(T.digest_of(out)), flush=True)
    g.close()
