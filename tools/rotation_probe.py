"""Per-source cost of the bench's config-2 rotation: device time, kernel
time, E_adm, rounds and the per-round trace summary (pull / push / local
rounds, tail handoff). usage: python tools/rotation_probe.py [--trace]"""
import argparse, json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import c2_rotation, workload

ap = argparse.ArgumentParser()
ap.add_argument("--trace", action="store_true")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--config", default="c2")
args = ap.parse_args()
wl = workload(args.config)
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = c2_rotation(g.degrees(T.Direction.OUT))
if args.trace:
    T.set_trace(g, 4096)
tot_e = tot_ms = 0.0
for q in qs:
    st = T.EdgeMapStats()
    T.query_batch(g, q.kind, [q.vertex], [q.window], width=4, stats=st)
    e, v = T.last_work(g, 0)
    rows = []
    if args.trace:
        tr = T.get_trace(g, 4096).astype(np.int64)
        for row in tr:
            if row[0] == 0:
                break
            kind = {1: "L", 2: "D", 3: "P", 4: "T"}.get(int(row[7]), "G")
            if kind == "T":  # cluster tail round: phase 1 and chunk phase
                rows.append([kind, int(row[3]), round((row[1] - row[0]) / 1e3, 1),
                             round((row[2] - row[1]) / 1e3, 1) if row[2] else 0, int(row[4])])
            else:
                # expand (or P1) and relax (or P2) separately, chunks, smalls
                rows.append([kind, int(row[3]), round((row[1] - row[0]) / 1e3, 1),
                             round((row[2] - row[1]) / 1e3, 1), int(row[4]), int(row[5])])
    tot, ker = T.time_queries(g, q.kind, [q.vertex], [q.window], warmup=2, steps=args.steps)
    ms = tot / args.steps
    tot_e += e
    tot_ms += ms
    print(json.dumps({"src": q.vertex, "e_adm": e, "v": v, "ms": round(ms, 4),
                      "kernel_ms": round(ker, 4), "gteps": round(e / ms / 1e6, 2),
                      "rounds": st.rounds, "relaxed": st.edges_relaxed, "trace": rows}),
          flush=True)
tr_tot, tr_ker = T.time_rotation(g, "earliest_arrival", [q.vertex for q in qs],
                                 [q.window for q in qs], warmup=3, steps=8 * args.steps)
print(json.dumps({"sum_single_ms": tot_ms, "rotation_ms_per_pass": tr_tot / args.steps,
                  "gteps_single": tot_e / tot_ms / 1e6,
                  "gteps_rotation": tot_e * args.steps / tr_tot / 1e6}))
