"""Async-mode stress: fresh graph per query, one kind per run; reports errors."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
kind = sys.argv[1]
rng = np.random.default_rng(int(sys.argv[2]))
mode = T.Mode(int(sys.argv[3])) if len(sys.argv) > 3 else T.Mode.ASYNC
fn = {"ea": T.earliest_arrival, "ld": T.latest_departure, "fastest": T.fastest_path}[kind]
okind = {"ea": "earliest_arrival", "ld": "latest_departure", "fastest": "fastest"}[kind]
bad = 0
for it in range(300):
    n = int(rng.integers(1, 13)); m = int(rng.integers(0, 41))
    s = rng.integers(0, n, m); d = rng.integers(0, n, m)
    a = rng.integers(0, 61, m); b = a + rng.integers(0, 9, m)
    E = (s, d, a, b)
    ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2)); v = int(rng.integers(0, n))
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=1 + it % 4))
    try:
        got = fn(g, v, T.QueryWindow(ta, tb), T.AlgoOptions(mode=mode)).values
    except Exception as e:
        print(it, "ERR", e, flush=True); bad += 1; continue
    want = Oracle(E, n).query(okind, v, ta, tb)
    if not np.array_equal(got, want):
        bad += 1
        if bad < 4: print(it, "MISMATCH", got, want, n, m, v, (ta, tb), flush=True)
print("bad", bad)
