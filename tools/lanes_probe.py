"""Batch engines on batches whose queries share their source (a window sweep
from one vertex, as `tgx sweep` runs) vs independent sources: lane-per-query
(TGXD_MODE_LANES) against the slot-major batch (SPARSE / AUTO without
lanes), device-timed, config-2 graph."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

wl = workload(os.environ.get("CFG", "c2"))
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())
src = qs[0].vertex
rng = np.random.default_rng(5)
cases = {
    "same source, nested windows": ([src] * 32, [T.QueryWindow(0, 999_999 - 20_000 * i) for i in range(32)]),
    "same source, shifted windows": ([src] * 32, [T.QueryWindow(10_000 * i, 999_999) for i in range(32)]),
    "same source, 1% windows": ([src] * 32, [T.QueryWindow(o, o + 9_999) for o in rng.integers(0, 990_000, 32)]),
}
deg = g.degrees(T.Direction.OUT)
srcs = [int(x) for x in rng.choice(np.flatnonzero(deg), 32)]
cases["independent sources, full window"] = (srcs, [T.QueryWindow(0, 999_999)] * 32)
for name, (vs, ws) in cases.items():
    for mode in (T.Mode.LANES, T.Mode.SPARSE, T.Mode.AUTO):
        env = os.environ
        if mode == T.Mode.AUTO:
            env["TGXD_NO_LANES"] = "1"
        tot, ker = T.time_queries(g, "earliest_arrival", vs, ws, mode=mode, warmup=2, steps=5)
        env.pop("TGXD_NO_LANES", None)
        print(f"{name:36s} {('AUTO-slot' if mode == T.Mode.AUTO else mode.name):10s} "
              f"{tot / 5:8.3f} ms per batch of 32", flush=True)
