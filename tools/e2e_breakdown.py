"""Where the end-to-end time of one config-2 query through the C-ABI goes:
wall time per call (host int64 result, pageable), the device span from the
first launch to the last result copy (events), and the traversal kernels."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())[0]
lib = T.load_library()
out = np.empty(g.vertex_count(), np.int64)
st = T._Stats()
walls, spans, kers = [], [], []
for i in range(60):
    t0 = time.perf_counter()
    T._check(lib.tgxd_earliest_arrival(g.handle, q.vertex, q.window.t_a, q.window.t_b, 1,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                       ctypes.byref(st)))
    t1 = time.perf_counter()
    if i >= 10:
        walls.append((t1 - t0) * 1e3)
        spans.append(st.total_ms)
        kers.append(st.kernel_ms)
print(f"wall {np.median(walls):.3f} ms  device span (launch..last copy) {np.median(spans):.3f} ms  "
      f"traversal kernels {np.median(kers):.3f} ms  (medians of 50)")
for name in ("TGXD_HOST_THREADS",):
    pass
