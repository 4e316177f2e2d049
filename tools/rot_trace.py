"""Round traces of the config-2 rotation's sources (diag.py for each of the 8 queries).
usage: [TGXD_...=x] python tools/rot_trace.py [--sources 1,2,4]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import c2_rotation, workload

ap = argparse.ArgumentParser()
ap.add_argument("--sources", default="0,1,2,3,4,5,6,7")
args = ap.parse_args()
wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
T.set_trace(g, 4096)
rot = c2_rotation(g.degrees(T.Direction.OUT))
for i in [int(x) for x in args.sources.split(",")]:
    q = rot[i]
    for r in range(2):
        st = T.EdgeMapStats()
        T.query_batch(g, q.kind, [q.vertex], [q.window], width=4, stats=st)
    e, v = T.last_work(g, 0)
    print(f"source {i}: {q.vertex} rounds={st.rounds} kernel_ms={st.kernel_ms:.4f} E_adm={e} V={v}", flush=True)
    tr = T.get_trace(g, 4096).astype(np.int64)
    for r, row in enumerate(tr):
        if row[0] == 0:
            break
        kind = {1: "L", 2: "D", 3: "P", 5: "S"}.get(int(row[7]), "G")
        print(f"  r{r:3d} F={row[3]:9d} A={(row[1]-row[0])/1e3:7.1f}us B={(row[2]-row[1])/1e3:7.1f}us "
              f"ch={row[4]:7d} sm={row[5]:7d} push={row[6]:8d} {kind}")
