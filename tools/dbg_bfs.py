import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from oracle.pyoracle import Oracle
E = [(3, 1, 7, 7), (3, 1, 22, 24), (1, 0, 43, 46), (1, 2, 51, 55), (1, 1, 53, 60), (1, 3, 18, 23), (3, 3, 26, 30), (1, 0, 5, 9), (1, 3, 23, 24), (1, 3, 52, 59), (2, 1, 9, 9), (3, 1, 17, 19), (0, 2, 55, 61), (3, 1, 46, 51), (2, 3, 13, 16), (2, 2, 14, 16), (0, 1, 26, 27), (3, 0, 11, 13), (3, 3, 2, 5), (3, 1, 49, 49), (2, 1, 40, 44), (2, 3, 50, 54), (0, 1, 43, 45), (2, 1, 45, 52)]
e = np.array(E, np.int64)
Ed = (e[:, 0], e[:, 1], e[:, 2], e[:, 3])
o = Oracle(Ed, 4)
for cutoff in (1, 4, 2048):
    g = T.TemporalGraph.build(Ed, 4, True, T.EngineConfig(index_cutoff=cutoff))
    T.set_trace(g, 64)
    for ordv in (0, 1):
        for mode in (T.Mode.SPARSE, T.Mode.DENSE):
            for k, fn in (("temporal_bfs", T.temporal_bfs), ("earliest_arrival", T.earliest_arrival)):
                got = fn(g, 1, T.QueryWindow(3, 46), T.AlgoOptions(ordering=T.Ordering(ordv), mode=mode)).values
                print(cutoff, ordv, mode, k, got, o.query(k, 1, 3, 46, ordv))
        tr = T.get_trace(g, 64).astype(np.int64)
        print([r[3:8].tolist() for r in tr[:6]])
