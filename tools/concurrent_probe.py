"""Throughput probe for serving: the same set of EA queries run one by one on
one handle (full grid) versus split across S views of the graph
(tgxd_graph_view: one stream and workspace each, grids sized so all fit on
the GPU together) driven from S host threads. Wall time of the whole set.

usage: python tools/concurrent_probe.py --config c5 --streams 2"""
import argparse, os, sys, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--streams", type=int, default=2)
ap.add_argument("--queries", type=int, default=32)
args = ap.parse_args()
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

wl = workload(args.config)
S = args.streams
base = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
# S views of one device graph (tgxd_graph_view: own stream / workspace, grids / S)
gs = [base] if S == 1 else [base.view(S) for _ in range(S)]
qs = [q for q in wl.queries(gs[0].degrees(T.Direction.OUT), gs[0].degrees(T.Direction.IN),
                            gs[0].vertex_count()) if q.kind == "earliest_arrival"]
qs = (qs * (args.queries // max(1, len(qs)) + 1))[:args.queries]
# warm every handle once
for g in gs:
    T.time_queries(g, "earliest_arrival", [qs[0].vertex], [qs[0].window], warmup=1, steps=1)


def run(g, mine):
    for q in mine:
        T.time_queries(g, "earliest_arrival", [q.vertex], [q.window], warmup=0, steps=1)


parts = [qs[i::S] for i in range(S)]
t0 = time.perf_counter()
th = [threading.Thread(target=run, args=(gs[i], parts[i])) for i in range(S)]
for t in th:
    t.start()
for t in th:
    t.join()
wall = time.perf_counter() - t0
print(f"{args.config} streams={S} (views): {len(qs)} EA queries in "
      f"{wall * 1e3:.1f} ms ({wall * 1e3 / len(qs):.3f} ms per query)", flush=True)
