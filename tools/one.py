import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
rng = np.random.default_rng(67)
for it in range(10):
    n = int(rng.integers(1, 13)); m = int(rng.integers(0, 41))
    s = rng.integers(0, n, m); d = rng.integers(0, n, m)
    a = rng.integers(0, 61, m); b = a + rng.integers(0, 9, m)
    ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2)); v = int(rng.integers(0, n))
E = (s, d, a, b)
print("n", n, "m", m, "v", v, "w", ta, tb); print("edges", list(zip(s, d, a, b)))
g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=2))
T.set_trace(g, 64)
st = T.EdgeMapStats()
try:
    r = T.fastest_path(g, v, T.QueryWindow(ta, tb), T.AlgoOptions(stats=st))
    print("got", r.values, st)
except Exception as e:
    print("ERR", e)
print("want", Oracle(E, n).query("fastest", v, ta, tb))
tr = T.get_trace(g, 64).astype(np.int64)
for i, row in enumerate(tr[:40]):
    print(i, row[3:].tolist(), (row[1]-row[0]), (row[2]-row[1]))
