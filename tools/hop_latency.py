"""Per-hop latency of the traversal engines: K parallel chains of L hops
(edge i -> i+1 of a chain leaves at 2i+1, arrives at 2i+2), every vertex
of a chain reached one round after its predecessor. Reports kernel time per
hop for each mode; K=1 is the CTA-local path, K large the grid path."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T

ap = argparse.ArgumentParser()
ap.add_argument("--hops", type=int, default=1000)
ap.add_argument("--chains", default="1,64,4096")
ap.add_argument("--pad", type=int, default=1 << 22, help="total vertices (isolated padding)")
ap.add_argument("--modes", default="0,1,3")
ap.add_argument("--trace", type=int, default=0, help="print this many rounds of the per-round trace")
args = ap.parse_args()
L = args.hops
for K in [int(x) for x in args.chains.split(",")]:
    n = max(args.pad, K * (L + 1) + 1)
    root = n - 1
    # root -> first vertex of every chain at t=0..1, then the chains
    src, dst, st, en = [], [], [], []
    first = np.arange(K, dtype=np.int64) * (L + 1)
    src.append(np.full(K, root)); dst.append(first)
    st.append(np.zeros(K)); en.append(np.ones(K))
    for i in range(L):
        src.append(first + i); dst.append(first + i + 1)
        st.append(np.full(K, 2 * i + 2)); en.append(np.full(K, 2 * i + 3))
    s = np.concatenate(src).astype(np.uint32); d = np.concatenate(dst).astype(np.uint32)
    a = np.concatenate(st).astype(np.uint64); b = np.concatenate(en).astype(np.uint64)
    g = T.TemporalGraph.build((s, d, a, b), n, True, T.EngineConfig(index_cutoff=2048))
    w = T.QueryWindow(0, 10 * L + 10)
    for m in [int(x) for x in args.modes.split(",")]:
        tot, ker = T.time_queries(g, "earliest_arrival", [root], [w], mode=T.Mode(m),
                                  warmup=2, steps=5)
        print(f"K={K:6d} L={L} mode={T.Mode(m).name:6s} kernel {ker*1e3:9.1f} us "
              f"-> {ker*1e3/(L+1):6.2f} us/hop", flush=True)
        if args.trace and m in (1, 2):
            T.set_trace(g, 4096)
            T.query_batch(g, "earliest_arrival", [root], [w], width=4, mode=T.Mode(m))
            tr = T.get_trace(g, 4096).astype(np.int64)
            big = 1 << 62
            for r, row in enumerate(tr[:args.trace]):
                if row[0] == 0: break
                a_last = (row[8] - row[0]) / 1e3 if row[8] else 0
                a_first = (big - row[9] - row[0]) / 1e3 if row[9] else 0
                b_last = (row[10] - row[1]) / 1e3 if row[10] else 0
                b_first = (big - row[11] - row[1]) / 1e3 if row[11] else 0
                print(f"  r{r:3d} F={row[3]:7d} A={(row[1]-row[0])/1e3:6.2f}us [{a_first:5.2f}..{a_last:5.2f}]"
                      f" B={(row[2]-row[1])/1e3:6.2f}us [{b_first:5.2f}..{b_last:5.2f}]", flush=True)
            T.set_trace(g, 0)
    g.close()
