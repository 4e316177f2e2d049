"""Shared test helpers: golden fixtures (generated from the reference by
tests/golden/make_golden.py) and random-instance generators."""
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
KINDS = ["earliest_arrival", "latest_departure", "fastest"]
# the reference's five path metrics (algorithms.hpp:46-66), fixture order
KINDS5 = KINDS + ["shortest_duration", "temporal_bfs"]
INF = (1 << 63) - 1
NEG = -(1 << 63)


def small_random():
    """Yield (edges, n, vertex, ta, tb, kind, ordering, labels) from the fixture."""
    z = np.load(GOLDEN / "small_random.npz")
    eoff, meta, labels = z["eoff"], z["meta"], z["labels"]
    for it, n, v, ta, tb, ki, ordv, lo in meta:
        a, b = eoff[it], eoff[it + 1]
        E = (z["src"][a:b], z["dst"][a:b], z["start"][a:b], z["end"][a:b])
        yield E, int(n), int(v), int(ta), int(tb), KINDS[ki], int(ordv), labels[lo:lo + n]


def small_random_ext():
    """All five metrics x all three orderings (small_random_ext.npz)."""
    z = np.load(GOLDEN / "small_random_ext.npz")
    eoff, meta, labels = z["eoff"], z["meta"], z["labels"]
    for it, n, v, ta, tb, ki, ordv, lo in meta:
        a, b = eoff[it], eoff[it + 1]
        E = (z["src"][a:b], z["dst"][a:b], z["start"][a:b], z["end"][a:b])
        yield E, int(n), int(v), int(ta), int(tb), KINDS5[ki], int(ordv), labels[lo:lo + n]


def rmat12_ext():
    """(edge_digest, [(kind, v, ta, tb, ordering)], labels) on the rmat12 graph."""
    z = np.load(GOLDEN / "rmat12_ext.npz")
    qs = [(KINDS5[k], int(v), int(ta), int(tb), int(o)) for k, v, ta, tb, o in z["meta"]]
    return int(z["edge_digest"][0]), qs, z["labels"]


def scaled(name):
    """(GenConfig, n, m, edge_digest, [(kind, v, ta, tb)], labels, digests)."""
    import paper_2401_02563_b200 as T
    z = np.load(GOLDEN / f"{name}.npz")
    kind, scale, n, m, sd, tr, seed = (int(x) for x in z["gen_fields"])
    a, b, c, p = (float(x) for x in z["gen_probs"])
    gen = T.GenConfig(kind, scale, n, m, a, b, c, sd, tr, p, seed)
    qs = [(KINDS[k], int(v), int(ta), int(tb)) for k, v, ta, tb in z["meta"]]
    return (gen, int(z["n"][0]), int(z["m"][0]), int(z["edge_digest"][0]), qs, z["labels"],
            z["digests"])


def edge_digest(E):
    import paper_2401_02563_b200 as T
    buf = b"".join(np.ascontiguousarray(x).tobytes() for x in (
        np.asarray(E[0], np.uint32), np.asarray(E[1], np.uint32), np.asarray(E[2], np.uint64),
        np.asarray(E[3], np.uint64)))
    return T.digest_of(np.frombuffer(buf, np.int64))


# hand-computed expectations of test_algorithms.cpp:51-122: name -> {vertex: value}
HAND_EXPECT = {
    "ea_no_edges": {1: 5, 0: INF, 2: INF, 3: INF},
    "ea_single_edge": {1: 5},
    "ea_strict_rejects_equal_handoff": {2: INF},
    "ea_weak_accepts_equal_handoff": {2: 4},
    "ld_no_edges": {1: 9, 0: NEG},
    "ld_single_edge": {0: 3},
    "fastest_two_hop": {1: 2},
    "fastest_no_edges": {2: 0, 0: INF},
}
HAND = [  # name, n, edges, kind, vertex, ta, tb, ordering
    ("ea_no_edges", 4, [], "earliest_arrival", 1, 5, 50, 1),
    ("ea_single_edge", 2, [(0, 1, 3, 5)], "earliest_arrival", 0, 0, 10, 1),
    ("ea_strict_rejects_equal_handoff", 3, [(0, 1, 1, 3), (1, 2, 3, 4)], "earliest_arrival", 0,
     0, (1 << 64) - 1, 1),
    ("ea_weak_accepts_equal_handoff", 3, [(0, 1, 1, 3), (1, 2, 3, 4)], "earliest_arrival", 0,
     0, (1 << 64) - 1, 0),
    ("ld_no_edges", 3, [], "latest_departure", 1, 2, 9, 1),
    ("ld_single_edge", 2, [(0, 1, 3, 5)], "latest_departure", 1, 0, 10, 1),
    ("fastest_two_hop", 3, [(0, 1, 2, 6), (0, 2, 3, 4), (2, 1, 4, 5)], "fastest", 0, 0,
     (1 << 64) - 1, 0),
    ("fastest_no_edges", 3, [], "fastest", 2, 0, (1 << 64) - 1, 1),
]


# test_algorithms.cpp:124-168 and test_engine.cpp:223-243 (as a path query)
HAND_EXT = [  # name, n, edges, kind, vertex, ta, tb, ordering
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
HAND_EXT_EXPECT = {
    "sd_single_edge": {1: 2},
    "sd_two_hop_sum_wins": {1: 3},
    "bfs_chain": {0: 0, 1: 1, 2: 2, 3: 3},
    "bfs_more_hops_unlock": {1: 1, 3: 3},
    "overlaps_gate": {1: 6, 2: 9, 3: INF, 4: INF, 5: INF},
}


def hand_edges(edges):
    e = np.array(edges, np.int64).reshape(-1, 4)
    return (e[:, 0], e[:, 1], e[:, 2], e[:, 3])


def rand_instance(rng, max_v=12, max_e=40, t_range=60, d_max=8, d_min=0):
    """Shape of random_instance (tests/support/random_graphs.hpp:19-39)."""
    n = int(rng.integers(1, max_v + 1))
    m = int(rng.integers(0, max_e + 1))
    s = rng.integers(0, n, m)
    d = rng.integers(0, n, m)
    a = rng.integers(0, t_range + 1, m)
    b = a + rng.integers(d_min, d_max + 1, m)
    return (s, d, a, b), n


def cost_model():
    """The cost-model fixture: (npz, {name: (edges, n, cutoff)}) with the rmat
    graph regenerated from its generator fields and the hand graph stored."""
    import paper_2401_02563_b200 as T
    z = np.load(GOLDEN / "cost_model.npz")
    kind, scale, n, m, sd, tr, seed = (int(x) for x in z["gen_fields"])
    a, b, c, p = (float(x) for x in z["gen_probs"])
    gen = T.GenConfig(kind, scale, n, m, a, b, c, sd, tr, p, seed)
    E = T.generate_edges(gen)
    de = z["degen_edges"]
    DE = (de[0].astype(np.uint32), de[1].astype(np.uint32), de[2], de[3])
    dn, dcut = (int(x) for x in z["degen_n_cutoff"])
    return z, {"rmat": (E, gen.n_vertices, 64), "degen": (DE, dn, dcut)}


def cost_cases(z, name, d):
    """verts, t_a, t_b, theta and the reference's (method, beta, k_hat, matches)."""
    k = f"{name}_d{d}_"
    return (z[k + "verts"], z[k + "ta"], z[k + "tb"], float(z[k + "theta"][0]),
            (z[k + "method"], z[k + "beta"], z[k + "khat"], z[k + "matches"]))


def fit_cases(z):
    o = 0
    for i, k in enumerate(z["fit_k"]):
        k = int(k)
        yield (z["fit_degree"][o:o + k], z["fit_matches"][o:o + k], z["fit_index_s"][o:o + k],
               z["fit_scan_s"][o:o + k], float(z["fit_c"][i]), float(z["fit_c_prime"][i]))
        o += k
