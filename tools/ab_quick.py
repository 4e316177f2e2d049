"""Quick A/B timing line (device time, ms) for environment experiments:
the config-2 rotation (8 sources), config 2's own source, config 4 fastest
and latest departure, config 1, one config-5 query.
usage: TGXD_...=x python tools/ab_quick.py [--skip c4,c5]"""
import argparse, json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import c2_rotation, workload

ap = argparse.ArgumentParser()
ap.add_argument("--skip", default="")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
skip = set(args.skip.split(","))
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("TGXD_")}}


def graph(name):
    wl = workload(name)
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    return wl, g, wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN),
                             g.vertex_count())


wl, g, qs = graph("c2")
rot = c2_rotation(g.degrees(T.Direction.OUT))
per = []
for q in rot:
    tot, ker = T.time_queries(g, q.kind, [q.vertex], [q.window], warmup=2, steps=args.steps)
    per.append(round(tot / args.steps, 4))
tot, ker = T.time_rotation(g, "earliest_arrival", [q.vertex for q in rot], [q.window for q in rot],
                           warmup=3, steps=8 * args.steps)
out["c2_rotation_ms"] = round(tot / (8 * args.steps), 4)
out["c2_per_source_ms"] = per
g.close()
for name in ("c1", "c4", "c5"):
    if name in skip:
        continue
    wl, g, qs = graph(name)
    for q in qs[:2]:
        tot, ker = T.time_queries(g, q.kind, [q.vertex], [q.window], warmup=2, steps=args.steps)
        out[f"{name}_{q.kind}_ms"] = round(tot / args.steps, 4)
    g.close()
print(json.dumps(out), flush=True)
