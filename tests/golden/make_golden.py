"""Generate the golden fixtures from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libtgxref.so, compiled
from /root/reference/proj/src by oracle/Makefile) and the reference's own
brute-force oracle (tests/support/oracle.cpp) on seeded inputs, and stores
inputs + outputs as compressed npz files next to this script:

  small_random.npz  300 random small instances (shape of random_instance(rng,
                    9..12, 28..40), test_algorithms.cpp:171-194) x
                    {EA, LD, fastest} x {Succeeds, StrictlySucceeds}, checked
                    against enumerate_paths as well
  hand_cases.npz    the hand-computed cases of test_algorithms.cpp:51-122
  rmat12.npz        RMAT scale 12 (config-2 distributions) with 12 queries,
                    full int64 label vectors + FNV-1a digests
  uniform14.npz     uniform n=2^14, m=2^18 (config-1 distributions), 6 queries
  small_random_ext.npz  200 more random small instances x all five path
                    metrics (+ shortest duration, temporal BFS) x all three
                    orderings (+ Overlaps), checked against enumerate_paths
  hand_ext.npz      shortest-duration / temporal-BFS hand cases
                    (test_algorithms.cpp:124-168) and the Overlaps gate of
                    test_engine.cpp:223-243 as a path query
  rmat12_ext.npz    the rmat12 graph, 4 sources x 2 windows x 5 metrics x 3
                    orderings
  weighted.npz      weighted shortest duration (AlgoOptions::weighted,
                    path_algorithms.cpp:196-258): 240 random small instances
                    with integer weights 0..5 x all three orderings, a third
                    of them with one non-integer or negative weight (the
                    reference's invalid_argument iff a reachable edge carries
                    it: code 2, labels zero), plus the rmat12 graph with
                    seeded integer weights, 4 sources x 3 orderings
  cost_model.npz    the selective-index cost model (choose_access_method:
                    decision, beta_hat, k_hat; count_in_window) on the rmat12
                    graph indexed at 64 (both directions, every indexed vertex
                    and 100 others, seeded windows incl. unbounded / empty /
                    inverted ones) and on a hand graph with degenerate
                    histograms; fit_cost_constants on seeded samples

Only this script touches the reference; tests read the npz files. Re-run
with:  python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.pyoracle import Reference  # noqa: E402

HERE = Path(__file__).resolve().parent
KINDS = ["earliest_arrival", "latest_departure", "fastest"]
KINDS5 = KINDS + ["shortest_duration", "temporal_bfs"]


def small_random():
    rng = np.random.default_rng(20240105)
    rows = {k: [] for k in ["n", "eoff", "src", "dst", "start", "end", "vertex", "ta", "tb",
                            "kind", "ordering", "labels", "loff"]}
    eoff = [0]
    loff = [0]
    src, dst, st, en, labels = [], [], [], [], []
    meta = []
    for it in range(300):
        n = int(rng.integers(1, 13))
        m = int(rng.integers(0, 41))
        s = rng.integers(0, n, m)
        d = rng.integers(0, n, m)
        a = rng.integers(0, 61, m)
        b = a + rng.integers(0, 9, m)
        E = (s, d, a, b)
        ref = Reference(E, n)
        ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2))
        v = int(rng.integers(0, n))
        for ki, kind in enumerate(KINDS):
            for ordv in (0, 1):
                out = ref.query(kind, v, ta, tb, ordv)
                brute = Reference.enumerate(E, n, kind, v, ta, tb, ordv)
                assert np.array_equal(out, brute), (it, kind, ordv)
                meta.append((it, n, v, ta, tb, ki, ordv, loff[-1]))
                labels.append(out)
                loff.append(loff[-1] + n)
        ref.close()
        src.append(s); dst.append(d); st.append(a); en.append(b)
        eoff.append(eoff[-1] + m)
    np.savez_compressed(
        HERE / "small_random.npz",
        eoff=np.array(eoff, np.int64), src=np.concatenate(src).astype(np.uint32),
        dst=np.concatenate(dst).astype(np.uint32), start=np.concatenate(st).astype(np.uint64),
        end=np.concatenate(en).astype(np.uint64), meta=np.array(meta, np.int64),
        labels=np.concatenate(labels).astype(np.int64))


# test_algorithms.cpp:51-122 (inputs, query, expected values of listed vertices)
HAND = [
    # (name, n, edges, kind, vertex, ta, tb, ordering, {vertex: expected})
    ("ea_no_edges", 4, [], "earliest_arrival", 1, 5, 50, 1, None),
    ("ea_single_edge", 2, [(0, 1, 3, 5)], "earliest_arrival", 0, 0, 10, 1, None),
    ("ea_strict_rejects_equal_handoff", 3, [(0, 1, 1, 3), (1, 2, 3, 4)], "earliest_arrival", 0,
     0, (1 << 64) - 1, 1, None),
    ("ea_weak_accepts_equal_handoff", 3, [(0, 1, 1, 3), (1, 2, 3, 4)], "earliest_arrival", 0,
     0, (1 << 64) - 1, 0, None),
    ("ld_no_edges", 3, [], "latest_departure", 1, 2, 9, 1, None),
    ("ld_single_edge", 2, [(0, 1, 3, 5)], "latest_departure", 1, 0, 10, 1, None),
    ("fastest_two_hop", 3, [(0, 1, 2, 6), (0, 2, 3, 4), (2, 1, 4, 5)], "fastest", 0, 0,
     (1 << 64) - 1, 0, None),
    ("fastest_no_edges", 3, [], "fastest", 2, 0, (1 << 64) - 1, 1, None),
]


def hand_cases():
    out = {}
    for name, n, edges, kind, v, ta, tb, ordv, _ in HAND:
        e = np.array(edges, np.int64).reshape(-1, 4)
        E = (e[:, 0], e[:, 1], e[:, 2], e[:, 3])
        ref = Reference(E, n)
        out[name] = ref.query(kind, v, ta, tb, ordv)
        ref.close()
    np.savez_compressed(HERE / "hand_cases.npz", **out)


def scaled(name, gen, queries):
    import paper_2401_02563_b200 as T  # host generator only (no GPU needed)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    ref = Reference(E, n)
    meta, labels, digests = [], [], []
    for (kind, v, ta, tb) in queries:
        out = ref.query(kind, v, ta, tb, 1)
        meta.append((KINDS.index(kind), v, ta, tb))
        labels.append(out)
        digests.append(int(Reference.lib().tgxref_digest(out.ctypes.data_as(
            __import__("ctypes").POINTER(__import__("ctypes").c_int64)), len(out))))
    ref.close()
    # the edge list itself is not stored: tests regenerate it from `gen`
    # (host generator) and check it against edge_digest first
    gen_fields = np.array([gen.kind, gen.scale, gen.n, gen.m, gen.start_dist, gen.t_range,
                           gen.seed], np.uint64)
    gen_probs = np.array([gen.a, gen.b, gen.c, gen.geo_p], np.float64)
    np.savez_compressed(HERE / f"{name}.npz", gen_fields=gen_fields, gen_probs=gen_probs,
                        edge_digest=np.array([edge_digest(E)], np.uint64), n=np.array([n]),
                        m=np.array([len(E[0])]), meta=np.array(meta, np.int64),
                        labels=np.array(labels, np.int64), digests=np.array(digests, np.uint64))


def edge_digest(E):
    """FNV-1a (digest.hpp:12-40) over the src|dst|start|end little-endian bytes:
    pins the generator."""
    import paper_2401_02563_b200 as T
    buf = b"".join(np.ascontiguousarray(x).tobytes() for x in (
        np.asarray(E[0], np.uint32), np.asarray(E[1], np.uint32), np.asarray(E[2], np.uint64),
        np.asarray(E[3], np.uint64)))
    return T.digest_of(np.frombuffer(buf, np.int64))


def small_random_ext():
    rng = np.random.default_rng(20240106)
    eoff, loff = [0], [0]
    src, dst, st, en, labels, meta = [], [], [], [], [], []
    for it in range(200):
        n = int(rng.integers(1, 10))
        m = int(rng.integers(0, 29))
        s = rng.integers(0, n, m)
        d = rng.integers(0, n, m)
        a = rng.integers(0, 61, m)
        b = a + rng.integers(0, 9, m)
        E = (s, d, a, b)
        ref = Reference(E, n)
        ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2))
        v = int(rng.integers(0, n))
        for ki, kind in enumerate(KINDS5):
            for ordv in (0, 1, 2):
                out = ref.query(kind, v, ta, tb, ordv)
                brute = Reference.enumerate(E, n, kind, v, ta, tb, ordv)
                assert np.array_equal(out, brute), (it, kind, ordv)
                meta.append((it, n, v, ta, tb, ki, ordv, loff[-1]))
                labels.append(out)
                loff.append(loff[-1] + n)
        ref.close()
        src.append(s); dst.append(d); st.append(a); en.append(b)
        eoff.append(eoff[-1] + m)
    np.savez_compressed(
        HERE / "small_random_ext.npz",
        eoff=np.array(eoff, np.int64), src=np.concatenate(src).astype(np.uint32),
        dst=np.concatenate(dst).astype(np.uint32), start=np.concatenate(st).astype(np.uint64),
        end=np.concatenate(en).astype(np.uint64), meta=np.array(meta, np.int64),
        labels=np.concatenate(labels).astype(np.int64))


# test_algorithms.cpp:124-168 (unweighted) and test_engine.cpp:223-243 as a
# path query: 0 reaches 1 over [2, 6]; only 1's out-edge [4, 9] overlaps it.
HAND_EXT = [
    ("sd_single_edge", 2, [(0, 1, 3, 5)], "shortest_duration", 0, 0, (1 << 64) - 1, 1),
    ("sd_two_hop_sum_wins", 3, [(0, 1, 0, 4), (0, 2, 0, 1), (2, 1, 5, 7)], "shortest_duration",
     0, 0, (1 << 64) - 1, 1),
    ("bfs_chain", 4, [(0, 1, 1, 2), (1, 2, 3, 4), (2, 3, 5, 6)], "temporal_bfs", 0, 0,
     (1 << 64) - 1, 1),
    ("bfs_more_hops_unlock", 4, [(0, 1, 9, 10), (0, 2, 0, 1), (2, 1, 2, 3), (1, 3, 5, 6)],
     "temporal_bfs", 0, 0, (1 << 64) - 1, 1),
    ("overlaps_gate", 6, [(0, 1, 2, 6), (1, 2, 4, 9), (1, 3, 7, 9), (1, 4, 2, 8), (1, 5, 3, 5)],
     "earliest_arrival", 0, 0, (1 << 64) - 1, 2),
]


def hand_ext():
    out = {}
    for name, n, edges, kind, v, ta, tb, ordv in HAND_EXT:
        e = np.array(edges, np.int64).reshape(-1, 4)
        E = (e[:, 0], e[:, 1], e[:, 2], e[:, 3])
        ref = Reference(E, n)
        out[name] = ref.query(kind, v, ta, tb, ordv)
        ref.close()
    np.savez_compressed(HERE / "hand_ext.npz", **out)


def rmat12_ext(gen):
    import paper_2401_02563_b200 as T
    E = T.generate_edges(gen)
    n = gen.n_vertices
    deg = np.bincount(E[0], minlength=n)
    rng = np.random.default_rng(13)
    srcs = [int(np.argmax(deg))] + [int(x) for x in rng.choice(np.flatnonzero(deg), 3)]
    ref = Reference(E, n)
    meta, labels = [], []
    for s in srcs:
        for w in ((0, 999_999), (200_000, 800_000)):
            for ki, kind in enumerate(KINDS5):
                for ordv in (0, 1, 2):
                    meta.append((ki, s, w[0], w[1], ordv))
                    labels.append(ref.query(kind, s, w[0], w[1], ordv))
    ref.close()
    np.savez_compressed(HERE / "rmat12_ext.npz", edge_digest=np.array([edge_digest(E)], np.uint64),
                        meta=np.array(meta, np.int64), labels=np.array(labels, np.int64))


def extended():
    import paper_2401_02563_b200 as T
    small_random_ext()
    hand_ext()
    rmat12_ext(T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 7,
                                cube_root_starts=True))


def degenerate_graph():
    """Hubs whose histograms collapse: one start (vertex 0), one duration
    (vertex 1), both (vertex 2), and a spread hub (vertex 3)."""
    s, d, a, b = [], [], [], []
    for i in range(40):
        s += [0, 1, 2, 3]
        d += [10 + i % 7, 20 + i % 5, 30 + i % 3, 40 + i % 9]
        a += [500, 100 + 37 * i, 700, 13 * i * i % 997]
        b += [500 + 1 + (i * 31) % 90, 100 + 37 * i + 25, 750, 13 * i * i % 997 + 1 + i % 11]
    return (np.array(s, np.uint32), np.array(d, np.uint32), np.array(a, np.uint64),
            np.array(b, np.uint64)), 64


def cost_model():
    import paper_2401_02563_b200 as T
    gen = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 7, cube_root_starts=True)
    E = T.generate_edges(gen)
    n = gen.n_vertices
    rng = np.random.default_rng(2024)
    out = {"gen_fields": np.array([gen.kind, gen.scale, gen.n, gen.m, gen.start_dist,
                                   gen.t_range, gen.seed], np.uint64),
           "gen_probs": np.array([gen.a, gen.b, gen.c, gen.geo_p], np.float64)}
    ref = Reference(E, n, True, 64)
    DE, dn = degenerate_graph()
    dref = Reference(DE, dn, True, 4)
    for name, r, edges, nn, cutoff in (("rmat", ref, E, n, 64), ("degen", dref, DE, dn, 4)):
        for d in (0, 1):
            deg = np.bincount(edges[d], minlength=nn)
            idx = np.flatnonzero(deg >= cutoff)
            other = rng.integers(0, nn, 100)
            verts = np.concatenate([idx, idx, other]).astype(np.uint32)
            k = len(verts)
            ta = rng.integers(0, 1_000_000, k).astype(np.uint64)
            tb = ta + rng.integers(0, 300_000, k).astype(np.uint64)
            ta[::9] = 0
            tb[::5] = (1 << 63) - 1
            tb[3::17] = ta[3::17]                      # one-instant windows
            tb[5::23] = np.maximum(ta[5::23], 1) - 1   # inverted (t_b < t_a)
            theta = 0.2 if d == 0 else 0.05
            m, beta, khat, matches = r.access_decisions(d, verts, ta, tb, theta)
            key = f"{name}_d{d}_"
            out.update({key + "verts": verts, key + "ta": ta, key + "tb": tb,
                        key + "theta": np.array([theta]), key + "method": m, key + "beta": beta,
                        key + "khat": khat, key + "matches": matches})
    out["degen_edges"] = np.stack([x.astype(np.uint64) for x in DE])
    out["degen_n_cutoff"] = np.array([dn, 4], np.uint64)
    fits = []
    for t in range(5):
        kk = int(rng.integers(1, 40))
        degree = rng.integers(0 if t == 4 else 1, 5000, kk).astype(np.uint64)
        matches = rng.integers(0, 300, kk).astype(np.uint64)
        ix = rng.random(kk) * 1e-5
        sc = rng.random(kk) * 1e-4
        c, cp = Reference.fit_cost_constants(degree, matches, ix, sc)
        fits.append((degree, matches, ix, sc, c, cp))
    out["fit_k"] = np.array([len(f[0]) for f in fits], np.uint64)
    out["fit_degree"] = np.concatenate([f[0] for f in fits])
    out["fit_matches"] = np.concatenate([f[1] for f in fits])
    out["fit_index_s"] = np.concatenate([f[2] for f in fits])
    out["fit_scan_s"] = np.concatenate([f[3] for f in fits])
    out["fit_c"] = np.array([f[4] for f in fits])
    out["fit_c_prime"] = np.array([f[5] for f in fits])
    np.savez_compressed(HERE / "cost_model.npz", **out)


def weighted():
    from oracle.pyoracle import OracleError, generate
    rng = np.random.default_rng(20260105)
    eoff, src, dst, st, en, wt, meta, labels = [0], [], [], [], [], [], [], []
    for it in range(240):
        n = int(rng.integers(1, 13))
        m = int(rng.integers(0, 41))
        s = rng.integers(0, n, m)
        d = rng.integers(0, n, m)
        a = rng.integers(0, 61, m)
        b = a + rng.integers(0, 9, m)
        w = rng.integers(0, 6, m).astype(np.float64)
        if it % 3 == 0 and m:
            w[int(rng.integers(0, m))] = (2.5, -1.0, 0.25)[it // 3 % 3]
        ref = Reference((s, d, a, b), n, True, 0, w)
        ta, tb = sorted(int(x) for x in rng.integers(0, 76, 2))
        v = int(rng.integers(0, n))
        for ordv in (0, 1, 2):
            try:
                out, code = ref.query("shortest_duration_weighted", v, ta, tb, ordv), 0
            except OracleError as e:
                out, code = np.zeros(n, np.int64), e.code
            meta.append((it, n, v, ta, tb, ordv, code, sum(len(x) for x in labels)))
            labels.append(out)
        ref.close()
        src.append(s); dst.append(d); st.append(a); en.append(b); wt.append(w)
        eoff.append(eoff[-1] + m)
    # the rmat12 graph with seeded integer weights
    import paper_2401_02563_b200 as T
    g = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 7, cube_root_starts=True)
    E = generate(g)
    n = g.n_vertices
    W = np.random.default_rng(5).integers(0, 1000, len(E[0])).astype(np.float64)
    ref = Reference(E, n, True, 0, W)
    deg = np.bincount(E[0], minlength=n)
    srcs = [int(np.argmax(deg))] + [int(x) for x in np.random.default_rng(13).choice(
        np.flatnonzero(deg), 3)]
    rq, rl = [], []
    for sidx, v in enumerate(srcs):
        ta, tb = (0, 999_999) if sidx % 2 == 0 else (200_000, 800_000)
        for ordv in (0, 1, 2):
            rq.append((v, ta, tb, ordv))
            rl.append(ref.query("shortest_duration_weighted", v, ta, tb, ordv))
    ref.close()
    np.savez_compressed(
        HERE / "weighted.npz", eoff=np.array(eoff, np.int64),
        src=np.concatenate(src).astype(np.uint32), dst=np.concatenate(dst).astype(np.uint32),
        start=np.concatenate(st).astype(np.uint64), end=np.concatenate(en).astype(np.uint64),
        weight=np.concatenate(wt), meta=np.array(meta, np.int64),
        labels=np.concatenate(labels).astype(np.int64),
        rmat_edge_digest=np.array([edge_digest(E)], np.uint64),
        rmat_weight_seed=np.array([5], np.int64), rmat_meta=np.array(rq, np.int64),
        rmat_labels=np.stack(rl).astype(np.int64))


def main():
    import paper_2401_02563_b200 as T
    small_random()
    hand_cases()
    g = T.GenConfig.rmat(12, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 7, cube_root_starts=True)
    E = T.generate_edges(g)
    deg = np.bincount(E[0], minlength=g.n_vertices)
    rng = np.random.default_rng(12)
    srcs = [int(np.argmax(deg))] + [int(x) for x in rng.choice(np.flatnonzero(deg), 3)]
    qs = []
    for sidx, s in enumerate(srcs):
        w = (0, 999_999) if sidx % 2 == 0 else (200_000, 800_000)
        for kind in KINDS:
            qs.append((kind, s, w[0], w[1]))
    scaled("rmat12", g, qs)
    g2 = T.GenConfig.uniform(1 << 14, 1 << 18, 1_000_000, 0.01, 3)
    qs2 = [(k, 0, 0, 999_999) for k in KINDS] + [(k, 77, 100_000, 600_000) for k in KINDS]
    scaled("uniform14", g2, qs2)
    extended()
    cost_model()
    weighted()
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    if sys.argv[1:] == ["cost_model"]:
        cost_model()
    elif sys.argv[1:] == ["weighted"]:
        weighted()
    else:
        main()
