"""A/B of per-call end-to-end time through tgxd_earliest_arrival over the
config-2 rotation, environment settings interleaved every rotation pass
(the library reads TGXD_LOG_F per call). usage: e2e_ab.py "A=1;B=2" "A=3" ..."""
import ctypes, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import c2_rotation, workload

variants = [dict(kv.split("=", 1) for kv in v.split(";") if kv) for v in sys.argv[1:]] or [{}]
wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
qs = c2_rotation(g.degrees(T.Direction.OUT))
lib = T.load_library()
out = np.empty(g.vertex_count(), np.int64)
optr = out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
walls = {i: [] for i in range(len(variants))}
for rep in range(30):
    for i, env in enumerate(variants):
        os.environ.update(env)
        for q in qs:
            t0 = time.perf_counter()
            T._check(lib.tgxd_earliest_arrival(g.handle, q.vertex, q.window.t_a, q.window.t_b, 1,
                                               optr, None))
            if rep >= 2:
                walls[i].append((time.perf_counter() - t0) * 1e3)
        for k in env:
            del os.environ[k]
for i, env in enumerate(variants):
    w = np.array(walls[i])
    print(f"{env}: mean {w.mean():.4f} ms  median {np.median(w):.4f}  p10 {np.percentile(w, 10):.4f}"
          f"  p90 {np.percentile(w, 90):.4f}  (n={len(w)})", flush=True)
