"""Per-warp completion of the heavy phases (diagnostics build -DTGXD_WTRACE_ALL,
TGXD_WTRACE=1): how much of the spread is between SMs / blocks and how much
within a block. usage: TGXD_LIB=build/variants/lib_wall.so python tools/warp_spread.py"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

os.environ["TGXD_WTRACE"] = "1"
os.environ["TGXD_WTRACE_ALL_FILE"] = "/tmp/wdone.bin"
wl = workload("c2")
g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
T.set_trace(g, 64)
q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), g.vertex_count())[0]
for _ in range(3):
    T.query_batch(g, q.kind, [q.vertex], [q.window], width=4)
tr = T.get_trace(g, 64).astype(np.int64)
nw = 148 * 4 * 8
W = np.fromfile("/tmp/wdone.bin", dtype=np.uint64).astype(np.int64).reshape(16, 2, nw)
detail = "--detail" in sys.argv
for r in range(2, 12 if detail else 8):
    for ph in range(2):
        t = W[r, ph]
        if not (t > 0).any():
            continue
        start = tr[r][0] if ph == 0 else tr[r][1]
        d = (t - start) / 1e3
        blk = d.reshape(-1, 8)                  # 8 warps per block
        inblock = (blk.max(1) - blk.min(1)).mean()
        bmean = blk.mean(1)
        if detail:
            bmax = blk.max(1)
            order = np.argsort(bmax)
            pct = [np.percentile(bmax, p) for p in (50, 90, 99, 100)]
            slow = ", ".join(f"b{int(b)}(sm~{int(b) % 148}):{bmax[b]:.1f}" for b in order[-6:][::-1])
            print(f"   r{r} {'AB'[ph]} block completion p50 {pct[0]:.1f} p90 {pct[1]:.1f} p99 {pct[2]:.1f} "
                  f"max {pct[3]:.1f} us; slowest: {slow}")
        print(f"r{r} {'AB'[ph]}: warps first {d.min():6.1f} median {np.median(d):6.1f} last {d.max():6.1f} us;"
              f" block means {bmean.min():6.1f}..{bmean.max():6.1f} (sd {bmean.std():5.1f});"
              f" mean in-block spread {inblock:5.1f}; "
              f"block id vs mean corr {np.corrcoef(np.arange(len(bmean)) % 148, bmean)[0, 1]:+.2f}")
