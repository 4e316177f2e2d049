"""CPU: on-disk edge lists (paper_2401_02563_b200/edgelist.py) against the
reference's ingest.cpp (compiled into oracle/_ref) and its own test cases
(test_ingest.cpp)."""
import ctypes
import gzip

import numpy as np
import pytest

from oracle.pyoracle import Reference
from paper_2401_02563_b200 import edgelist as EL

ref_available = pytest.mark.skipif(not Reference.available(),
                                   reason="reference library not built (oracle/_ref)")
u64p = ctypes.POINTER(ctypes.c_uint64)
u32p = ctypes.POINTER(ctypes.c_uint32)


def ref_load(path, map_ids=False, seed=1, dmax=3600):
    lib = Reference.lib()
    m = ctypes.c_uint64()
    n = ctypes.c_uint32()
    cap = 1 << 16
    s = np.empty(cap, np.uint32)
    d = np.empty(cap, np.uint32)
    a = np.empty(cap, np.uint64)
    b = np.empty(cap, np.uint64)
    w = np.empty(cap, np.float64)
    rc = lib.tgxref_load_edge_list(str(path).encode(), int(map_ids), ctypes.c_uint64(seed),
                                   ctypes.c_uint64(dmax), ctypes.c_uint64(cap), ctypes.byref(m),
                                   ctypes.byref(n), s.ctypes.data_as(u32p), d.ctypes.data_as(u32p),
                                   a.ctypes.data_as(u64p), b.ctypes.data_as(u64p),
                                   w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc:
        return rc, lib.tgxref_last_error()
    k = m.value
    return 0, (s[:k], d[:k], a[:k], b[:k], w[:k], n.value)


CASES = {
    "empty.txt": "",
    "g.txt": "# a comment\n0 1 2 5\n0 2 1 3\n2 0 4 6\n",
    "w.txt": "0 1 2 5 0.25\n",
    "s.txt": "0 1 10\n1 0 20\n",
    "sparse.txt": "5 2 1 2\n",
    "crlf.txt": "0 1 2 5\r\n\r\n  # indented comment\n1 2 3 9\r\n",
    "noeol.txt": "3 4 7 8",
}
BAD = {
    "bad.txt": ("0 1 2 5\n0 x 3 4\n", ":2:"),
    "back.txt": ("0 1 5 2\n", "precedes"),
    "cols.txt": ("0 1 2 5\n0 1 2\n", "column count"),
    "six.txt": ("0 1 2 3 4 5\n", "expected 3, 4, or 5 columns"),
    "big.txt": ("4294967296 1 2 3\n", "exceeds 32-bit range"),
}


def test_hand_cases(tmp_path):
    """test_ingest.cpp:46-116."""
    for name, text in CASES.items():
        (tmp_path / name).write_text(text)
    r = EL.load_edge_list(str(tmp_path / "empty.txt"))
    assert r.src.size == 0 and r.n_vertices == 0
    r = EL.load_edge_list(str(tmp_path / "g.txt"))
    assert r.n_vertices == 3 and r.src.size == 3
    assert (int(r.src[0]), int(r.dst[0]), int(r.start[0]), int(r.end[0])) == (0, 1, 2, 5)
    assert EL.load_edge_list(str(tmp_path / "w.txt")).weight[0] == 0.25
    a = EL.load_edge_list(str(tmp_path / "s.txt"), seed=9, end_sample_max=5)
    b = EL.load_edge_list(str(tmp_path / "s.txt"), seed=9, end_sample_max=5)
    assert np.array_equal(a.end, b.end)
    assert np.all(a.end > a.start) and np.all(a.end - a.start <= 5)
    (tmp_path / "ids.txt").write_text("a b 3\nb c 4\n")
    r = EL.load_edge_list(str(tmp_path / "ids.txt"), map_ids=True)
    assert r.n_vertices == 3 and r.src.tolist() == [0, 1] and r.dst.tolist() == [1, 2]
    assert EL.load_edge_list(str(tmp_path / "sparse.txt")).n_vertices == 6
    for name, (text, msg) in BAD.items():
        (tmp_path / name).write_text(text)
        with pytest.raises(EL.EdgeListError, match=msg):
            EL.load_edge_list(str(tmp_path / name))
    with pytest.raises(EL.EdgeListError):
        EL.load_edge_list(str(tmp_path / "nope.txt"))


def test_sample_end_times_degenerate():
    """test_ingest.cpp:151-157: d_max = 1 gives start + 1."""
    assert EL.sample_end_times([5, 9], 3, 1).tolist() == [6, 10]


@ref_available
def test_loads_match_the_reference(tmp_path):
    for name, text in CASES.items():
        p = tmp_path / name
        p.write_text(text)
        for map_ids in (False, True):
            for seed, dmax in ((1, 3600), (9, 5), (77, 1 << 40)):
                rc, want = ref_load(p, map_ids, seed, dmax)
                assert rc == 0, want
                got = EL.load_edge_list(str(p), map_ids, seed, dmax)
                for x, y in zip((got.src, got.dst, got.start, got.end, got.weight), want[:5]):
                    assert np.array_equal(x, y), (name, map_ids, seed)
                assert got.n_vertices == want[5]
    for name, (text, msg) in BAD.items():
        p = tmp_path / name
        p.write_text(text)
        rc, err = ref_load(p)
        assert rc != 0 and msg.encode() in err, (name, err)


@ref_available
def test_sampling_and_window_match_the_reference():
    lib = Reference.lib()
    rng = np.random.default_rng(5)
    for seed in (0, 1, 21, (1 << 63) + 11):
        for dmax in (1, 2, 7, 100, 3600, (1 << 33) + 5, (1 << 64) - 1):
            st = rng.integers(0, 1 << 40, 300).astype(np.uint64)
            out = np.empty_like(st)
            assert lib.tgxref_sample_end_times(ctypes.c_uint64(st.size), st.ctypes.data_as(u64p),
                                               ctypes.c_uint64(seed), ctypes.c_uint64(dmax),
                                               out.ctypes.data_as(u64p)) == 0
            assert np.array_equal(out, EL.sample_end_times(st, seed, dmax)), (seed, dmax)
    for frac in (1.0, 0.5, 0.1, 0.013, 1e-9):
        st = rng.integers(0, 1000, 777).astype(np.uint64)
        en = st + rng.integers(0, 50, 777).astype(np.uint64)
        ta, tb = ctypes.c_uint64(), ctypes.c_uint64()
        assert lib.tgxref_window_for_recent_fraction(
            ctypes.c_uint64(st.size), st.ctypes.data_as(u64p), en.ctypes.data_as(u64p),
            ctypes.c_double(frac), ctypes.byref(ta), ctypes.byref(tb)) == 0
        assert EL.window_for_recent_fraction(st, en, frac) == (ta.value, tb.value)


@ref_available
def test_write_round_trip_and_reference_reads_it(tmp_path):
    """test_ingest.cpp:118-147: plain and gzip, the multiset survives, and the
    reference's loader reads what ours wrote (and vice versa)."""
    rng = np.random.default_rng(7)
    s = rng.integers(0, 41, 500).astype(np.uint32)
    d = rng.integers(0, 41, 500).astype(np.uint32)
    a = rng.integers(0, 1001, 500).astype(np.uint64)
    b = a + rng.integers(0, 10, 500).astype(np.uint64)
    w = rng.integers(1, 9, 500) / 4.0
    for name in ("rt.txt", "rt.gz"):
        p = str(tmp_path / name)
        EL.write_edge_list(p, s, d, a, b, w)
        if name.endswith(".gz"):
            assert open(p, "rb").read(2) == b"\x1f\x8b"
        got = EL.load_edge_list(p)
        for x, y in zip((got.src, got.dst, got.start, got.end, got.weight), (s, d, a, b, w)):
            assert np.array_equal(x, y)
        rc, want = ref_load(p)
        assert rc == 0
        for x, y in zip(want[:5], (s, d, a, b, w)):
            assert np.array_equal(x, y)
        p2 = str(tmp_path / ("ref_" + name))
        lib = Reference.lib()
        assert lib.tgxref_write_edge_list(p2.encode(), ctypes.c_uint64(500), s.ctypes.data_as(u32p),
                                          d.ctypes.data_as(u32p), a.ctypes.data_as(u64p),
                                          b.ctypes.data_as(u64p),
                                          w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) == 0
        got2 = EL.load_edge_list(p2)
        assert np.array_equal(got2.start, a) and np.array_equal(got2.weight, w)
        if not name.endswith(".gz"):
            assert open(p, "rb").read() == open(p2, "rb").read()  # byte-identical text
