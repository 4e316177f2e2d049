"""Config 5's (and 3's) query batch under different AUTO split budgets:
device ms per batch. usage: python tools/batch_groups.py [--config c5]"""
import argparse, json, os, sys, subprocess
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--budgets", default="64,128,256,512,100000")
ap.add_argument("--child", default="")
args = ap.parse_args()
if args.child:
    import paper_2401_02563_b200 as T
    from paper_2401_02563_b200.configs import workload
    wl = workload(args.config)
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
    out = {"config": args.config, "budget_mb": os.environ.get("TGXD_BATCH_BUDGET_MB")}
    for kind in sorted({q.kind for q in qs}):
        sub = [q for q in qs if q.kind == kind]
        tot, ker = T.time_queries(g, kind, [q.vertex for q in sub], [q.window for q in sub],
                                  warmup=1, steps=3)
        out[kind + "_ms"] = round(tot / 3, 3)
    print(json.dumps(out), flush=True)
else:
    for b in args.budgets.split(","):
        env = dict(os.environ, TGXD_BATCH_BUDGET_MB=b)
        subprocess.run([sys.executable, __file__, "--config", args.config, "--child", "1"], env=env)
