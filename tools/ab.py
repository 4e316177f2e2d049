"""A/B timing of library variants on BASELINE workloads: for each config,
the first query of each kind (device-timed, graph resident), repeated
`--rounds` times alternating the variant libraries in subprocesses.

usage: python tools/ab.py --libs base=build/variants/lib_base.so,red=... [--configs c2]"""
import argparse, json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--libs", default="")
ap.add_argument("--configs", default="c2")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--kinds", default="")
ap.add_argument("--child", action="store_true")
ap.add_argument("--env", default="", help="extra env per variant: name:K=V;K=V|name2:...")
args = ap.parse_args()

if args.child:
    import paper_2401_02563_b200 as T
    from paper_2401_02563_b200.configs import workload
    out = {}
    for c in args.configs.split(","):
        wl = workload(c)
        g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
        qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
        seen = set()
        for q in qs:
            if q.kind in seen or (args.kinds and q.kind not in args.kinds.split(",")):
                continue
            seen.add(q.kind)
            tot, ker = T.time_queries(g, q.kind, [q.vertex], [q.window], warmup=3,
                                      steps=args.steps)
            out[f"{c}/{q.kind}"] = round(tot / args.steps, 4)
        g.close()
    print(json.dumps(out))
    sys.exit(0)

libs = [kv.split("=", 1) for kv in args.libs.split(",") if kv]
extra = {}
for part in [p for p in args.env.split("|") if p]:
    name, kvs = part.split(":", 1)
    extra[name] = dict(kv.split("=", 1) for kv in kvs.split(";") if kv)
res = {name: [] for name, _ in libs}
for r in range(args.rounds):
    for name, lib in libs:
        env = dict(os.environ)
        if lib != "-":
            env["TGXD_LIB"] = str(ROOT / lib)
        env.update(extra.get(name, {}))
        p = subprocess.run([sys.executable, __file__, "--child", "--configs", args.configs,
                            "--steps", str(args.steps), "--kinds", args.kinds],
                           env=env, capture_output=True, text=True, timeout=900)
        if p.returncode != 0:
            print(name, "FAILED", p.stderr[-800:], flush=True)
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        res[name].append(d)
        print(name, r, d, flush=True)
print("== min over rounds (ms per query)")
for name, runs in res.items():
    if not runs:
        continue
    keys = runs[0].keys()
    print(name, {k: min(x[k] for x in runs) for k in keys})
