"""Medium random instances (pull rounds with TGXD_PULL_F small): kind seed count mode"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
kind = sys.argv[1]
seed = int(sys.argv[2])
count = int(sys.argv[3])
mode = T.Mode(int(sys.argv[4]))
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path}
rng = np.random.default_rng(seed)
fails = 0
for it in range(count):
    n = int(rng.integers(2, 60)); m = int(rng.integers(1, 600))
    s = rng.integers(0, n, m); d = rng.integers(0, n, m)
    a = rng.integers(0, 200, m); b = a + rng.integers(0, 20, m)
    E = (s, d, a, b)
    g = T.TemporalGraph.build(E, n, True, T.EngineConfig(index_cutoff=int(rng.integers(1, 64))))
    o = Oracle(E, n)
    ta, tb = sorted(int(x) for x in rng.integers(0, 220, 2))
    v = int(rng.integers(0, n))
    want = o.query(kind, v, ta, tb)
    for rep in range(3):
        got = FN[kind](g, v, T.QueryWindow(ta, tb), T.AlgoOptions(mode=mode)).values
        if not np.array_equal(got, want):
            fails += 1
            if fails <= 3:
                print("MISMATCH it", it, "rep", rep, "n", n, "m", m, "v", v, "w", ta, tb,
                      "bad", np.nonzero(got != want)[0][:8].tolist(), flush=True)
                np.savez(f"gpurun_out/p3/fail_{kind}_{seed}_{it}.npz", s=s, d=d, a=a, b=b, n=n, v=v,
                         ta=ta, tb=tb, got=got, want=want)
            break
    g.close()
print("done", count, "fails", fails)
