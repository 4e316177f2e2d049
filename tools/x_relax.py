"""Experiment: one heavy round's relax as a non-persistent kernel
(relax_only_kernel, -DTGXD_EXPERIMENTS build) vs the same phase inside the
persistent round kernel (per-round trace). Config 2's own source, tail on the
grid. usage: TGXD_LIB=build/variants/lib_x8.so python tools/x_relax.py"""
import ctypes, json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

lib = T.load_library()
lib.tgxd_x_relax.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                             ctypes.POINTER(ctypes.c_double)]
wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())[0]
os.environ["TGXD_HANDOFF_F"] = "0"
os.environ["TGXD_ASYNC_F"] = "0"
T.set_trace(g, 64)
inkernel = {}
for _ in range(3):
    T.query_batch(g, q.kind, [q.vertex], [q.window], width=4)
tr = T.get_trace(g, 64).astype(np.int64)
for r, row in enumerate(tr):
    if row[0] == 0:
        break
    inkernel[r] = ((row[2] - row[1]) / 1e3, int(row[7]))
del os.environ["TGXD_HANDOFF_F"], os.environ["TGXD_ASYNC_F"]
out = (ctypes.c_double * 4)()
for r in (2, 4, 5, 6):
    for upw in (1, 2, 4):
        ms = []
        for rep in range(3):
            T._check(lib.tgxd_x_relax(g.handle, q.vertex, r, upw, out))
            ms.append(out[0])
        print(json.dumps({"round": r, "upw": upw, "standalone_us": round(1e3 * min(ms), 1),
                          "in_kernel_phase_b_us": round(inkernel.get(r, (0, 0))[0], 1),
                          "round_kind": inkernel.get(r, (0, 0))[1],
                          "chunks": int(out[1]), "smalls": int(out[2]), "push": int(out[3])}),
              flush=True)
g.close()
