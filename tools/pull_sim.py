# CPU simulation (numpy) of config-2 EA rounds: per round, push work vs pull scan lengths.
"""Round-synchronous EA on config 2 with per-round push cost (edges relaxed,
delta-ranges) vs pull cost (in-edges scanned in te order up to the first
admissible one or te >= current label) computed from the same snapshot."""
import sys, time, numpy as np
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parent.parent))
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload
wl = workload("c2")
s, d, a, b = T.generate_edges(wl.gen)
n = wl.gen.n_vertices
src_deg = np.bincount(s, minlength=n)
q = wl.queries(src_deg, np.bincount(d, minlength=n), n)[0]
root, ta, tb = q.vertex, 0, 999999
a = a.astype(np.int64); b = b.astype(np.int64)
win = (a >= ta) & (b <= tb)
s, d, a, b = s[win], d[win], a[win], b[win]
INF = np.iinfo(np.int64).max
# out-CSR sorted by (src, start)
o = np.lexsort((a, s)); os_, od, oa, ob = s[o], d[o], a[o], b[o]
ooff = np.zeros(n + 1, np.int64); np.add.at(ooff, os_ + 1, 1); ooff = np.cumsum(ooff)
# in-CSR sorted by (dst, end)
i = np.lexsort((b, d)); is_, id_, ia, ib = s[i], d[i], a[i], b[i]
ioff = np.zeros(n + 1, np.int64); np.add.at(ioff, id_ + 1, 1); ioff = np.cumsum(ioff)
ipos = np.arange(len(id_)) - ioff[id_]
L = np.full(n, INF); L[root] = ta
Ex = np.full(n, INF)  # bound at last expansion (work-efficient push)
frontier = np.array([root])
r = 0
tot_push = tot_pull = 0
while len(frontier):
    snap = L.copy()
    # pull cost from this snapshot: for every vertex, in-edges with te < L[d]
    # scanned in te order until the first admissible one
    lim = snap[id_]
    relevant = ib < lim
    adm = relevant & (((snap[is_] != INF) & (ia > snap[is_])) | (is_ == root))
    first = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(first, id_[adm], ipos[adm])
    nrel = np.bincount(id_[relevant], minlength=n)
    big = np.iinfo(np.int64).max
    per = np.where(first == big, nrel, np.minimum(first + 1, nrel))
    pull_cost = int(per.sum())
    if r in (2, 3, 4):
        srt = np.sort(per)[::-1]
        op=nrel>0
        print(f"   r{r} open {op.sum()} reached {(snap!=INF).sum()} sum_min16 {np.minimum(nrel,16).sum()} early {per.sum()} n>16 {(nrel>16).sum()} per>16 {(per>16).sum()} sum_nrel>16 {nrel[nrel>16].sum()} sum_per>16 {per[per>16].sum()} early<=16 {per[per<=16].sum()}")
        print(f"   r{r} scan max {srt[0]} top10 {srt[:10].tolist()} >32: {(per>32).sum()} (sum {per[per>32].sum()}) >256: {(per>256).sum()} (sum {per[per>256].sum()}) unreached-scan {per[snap==INF].sum()}")
    # push (work-efficient delta ranges) from the frontier
    lb = np.where(frontier == root, ta, snap[frontier] + 1)
    cnt = 0
    newL = L.copy()
    segs = []
    for v, lbv in zip(frontier, lb):
        lo, hi = ooff[v], ooff[v + 1]
        p0 = lo + np.searchsorted(oa[lo:hi], lbv, 'left')
        p1 = lo + np.searchsorted(oa[lo:hi], Ex[v], 'left') if Ex[v] != INF else hi
        Ex[v] = lbv
        if p1 > p0:
            segs.append((p0, p1))
    if segs:
        idx = np.concatenate([np.arange(p0, p1) for p0, p1 in segs])
        cnt = len(idx)
        np.minimum.at(newL, od[idx], ob[idx])
    improved = np.flatnonzero(newL < L)
    L = newL
    frontier = improved
    tot_push += cnt; tot_pull += pull_cost
    print(f"round {r:2d} frontier {len(lb):8d} push_edges {cnt:10d} pull_scan {pull_cost:10d}", flush=True)
    r += 1
print("total push", tot_push, "total pull-if-every-round", tot_pull)
