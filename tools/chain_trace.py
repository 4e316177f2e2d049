"""Timestamps along block 0 / warp 0's dependent chain in every grid round
(diagnostics build -DTGXD_CHAIN): where a thin round's time goes.
usage: TGXD_LIB=build/variants/lib_chain.so TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 python tools/chain_trace.py"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

os.environ["TGXD_CHAIN_FILE"] = "/tmp/chain.bin"
wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
T.set_trace(g, 64)
q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())[0]
for _ in range(3):
    T.query_batch(g, q.kind, [q.vertex], [q.window], width=4)
T.get_trace(g, 64)
C = np.fromfile("/tmp/chain.bin", dtype=np.uint64).astype(np.int64).reshape(64, 16)
names = ["A entry", "item", "label/bounds", "search+append", "list drain", "flush_work", "barrier",
         "counters", "B entry", "window load", "first window relaxed", "push drain", "barrier", "counters"]
for r in range(2, 24):
    row = C[r]
    if row[0] == 0:
        continue
    parts = []
    prev = row[0]
    for k in range(1, 14):
        if row[k] == 0:
            continue
        parts.append(f"{names[k]} +{(row[k] - prev) / 1e3:.1f}")
        prev = row[k]
    print(f"r{r:2d} total {(prev - row[0]) / 1e3:6.1f} us: " + ", ".join(parts))
