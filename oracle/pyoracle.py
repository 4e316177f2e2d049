"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the checkers.

* `Oracle`    : the C restatement (oracle/tgx_oracle.c -> _ref/libtgxoracle.so)
* `Reference` : the compiled, unmodified reference library plus the
                reference's own brute-force oracle (_ref/libtgxref.so, built
                from /root/reference by oracle/Makefile; it travels to the GPU
                box as a built artefact)

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may use this module.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
ORACLE_SO = REF_DIR / "libtgxoracle.so"
REF_SO = REF_DIR / "libtgxref.so"

_P = ctypes.POINTER
_u32p = _P(ctypes.c_uint32)
_u64p = _P(ctypes.c_uint64)
_i64p = _P(ctypes.c_int64)
KIND = {"earliest_arrival": 0, "latest_departure": 1, "fastest": 2, "shortest_duration": 3,
        "temporal_bfs": 4, "shortest_duration_weighted": 5}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ensure(so: Path, target: str) -> Path:
    if not so.exists():
        subprocess.run(["make", "-C", str(HERE), target], check=True, capture_output=True)
    return so


def _arr(edges):
    s, d, a, b = edges
    return (np.ascontiguousarray(s, np.uint32), np.ascontiguousarray(d, np.uint32),
            np.ascontiguousarray(a, np.uint64), np.ascontiguousarray(b, np.uint64))


class Oracle:
    """The plain-C restatement."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            lib = ctypes.CDLL(str(_ensure(ORACLE_SO, "oracle")))
            vp = ctypes.c_void_p
            lib.tgxo_graph_build.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p,
                                             _u64p, _u64p, ctypes.c_int, _P(vp)]
            lib.tgxo_graph_build_weighted.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u32p,
                                                      _u32p, _u64p, _u64p,
                                                      _P(ctypes.c_double), ctypes.c_int, _P(vp)]
            lib.tgxo_graph_free.argtypes = [vp]
            lib.tgxo_graph_free.restype = None
            lib.tgxo_query.argtypes = [vp, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_int, _i64p]
            lib.tgxo_work.argtypes = [vp, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_int, _i64p, _u64p, _u64p]
            lib.tgxo_digest.argtypes = [_i64p, ctypes.c_uint64]
            lib.tgxo_digest.restype = ctypes.c_uint64
            lib.tgxo_last_error.restype = ctypes.c_char_p
            cls._lib = lib
        return cls._lib

    def __init__(self, edges, n: int, directed: bool = True, weights=None):
        lib = self.lib()
        s, d, a, b = _arr(edges)
        self.n = n
        self._h = ctypes.c_void_p()
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self._check(lib.tgxo_graph_build_weighted(
            n, len(s), s.ctypes.data_as(_u32p), d.ctypes.data_as(_u32p),
            a.ctypes.data_as(_u64p), b.ctypes.data_as(_u64p),
            None if w is None else w.ctypes.data_as(_f64p), 1 if directed else 0,
            ctypes.byref(self._h)))

    @classmethod
    def _check(cls, rc):
        if rc:
            lib = cls.lib()
            lib.tgxo_last_error.restype = ctypes.c_char_p
            raise OracleError(rc, lib.tgxo_last_error().decode())

    def query(self, kind: str, vertex: int, t_a: int, t_b: int, ordering: int = 1) -> np.ndarray:
        out = np.empty(self.n, np.int64)
        self._check(self.lib().tgxo_query(self._h, KIND[kind], vertex, t_a, t_b, ordering,
                                          out.ctypes.data_as(_i64p)))
        return out

    def work(self, kind: str, vertex: int, t_a: int, t_b: int, labels: np.ndarray,
             ordering: int = 1) -> tuple[int, int]:
        e = ctypes.c_uint64()
        r = ctypes.c_uint64()
        lab = np.ascontiguousarray(labels, np.int64)
        self._check(self.lib().tgxo_work(self._h, KIND[kind], vertex, t_a, t_b, ordering,
                                         lab.ctypes.data_as(_i64p), ctypes.byref(e),
                                         ctypes.byref(r)))
        return e.value, r.value

    def access_decisions(self, direction: int, cutoff: int, verts, t_a, t_b, theta: float = 0.2):
        """(method, beta_hat, k_hat, matches) per (vertex, window): selective_index.cpp:98-209."""
        return _decisions(self.lib().tgxo_access_decisions, self._check,
                          (self._h, ctypes.c_int(direction), ctypes.c_uint64(cutoff)), verts, t_a, t_b,
                          theta)

    @classmethod
    def fit_cost_constants(cls, degree, matches, index_s, scan_s):
        out = (ctypes.c_double * 2)()
        deg, mat, ix, sc = _fit_arrays(degree, matches, index_s, scan_s)
        cls._check(cls.lib().tgxo_fit_cost_constants(
            ctypes.c_uint64(len(deg)), deg.ctypes.data_as(_u64p), mat.ctypes.data_as(_u64p),
            ix.ctypes.data_as(_f64p), sc.ctypes.data_as(_f64p), ctypes.byref(out, 0),
            ctypes.byref(out, 8)))
        return out[0], out[1]

    def close(self):
        if self._h:
            self.lib().tgxo_graph_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _GenConfig(ctypes.Structure):      # tgxo_gen_config (= tgxd_gen_config's layout)
    _fields_ = [("kind", ctypes.c_int), ("scale", ctypes.c_uint32), ("n", ctypes.c_uint32),
                ("m", ctypes.c_uint64), ("a", ctypes.c_double), ("b", ctypes.c_double),
                ("c", ctypes.c_double), ("start_dist", ctypes.c_int),
                ("t_range", ctypes.c_uint32), ("geo_p", ctypes.c_double),
                ("seed", ctypes.c_uint64)]


def generate(gen):
    """The BASELINE workload edge list from the checker's own generator
    (tgx_gen.c): (src u32, dst u32, start u64, end u64). `gen` is any object
    with the generator fields (e.g. the package's GenConfig)."""
    lib = Oracle.lib()
    c = _GenConfig(*(getattr(gen, f) for f, _ in _GenConfig._fields_))
    fn = lib.tgxo_generate
    fn.argtypes = [_P(_GenConfig), ctypes.c_uint64, _u64p, _u32p, _u32p, _u64p, _u64p]
    fn.restype = ctypes.c_int
    m = ctypes.c_uint64()
    Oracle._check(fn(ctypes.byref(c), 0, ctypes.byref(m), None, None, None, None)
                  if c.kind == 0 else 0)
    cap = int(m.value) if c.kind == 0 else int(c.m)
    s = np.empty(cap, np.uint32)
    d = np.empty(cap, np.uint32)
    a = np.empty(cap, np.uint64)
    b = np.empty(cap, np.uint64)
    Oracle._check(fn(ctypes.byref(c), cap, ctypes.byref(m), s.ctypes.data_as(_u32p),
                     d.ctypes.data_as(_u32p), a.ctypes.data_as(_u64p), b.ctypes.data_as(_u64p)))
    k = int(m.value)
    return s[:k], d[:k], a[:k], b[:k]


def digest(values: np.ndarray) -> int:
    v = np.ascontiguousarray(values, np.int64)
    return int(Oracle.lib().tgxo_digest(v.ctypes.data_as(_i64p), len(v)))


class Reference:
    """The compiled reference library (unmodified sources from /root/reference)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        if REF_SO.exists():
            return True
        if Path("/root/reference/proj/src").is_dir():
            try:
                _ensure(REF_SO, "ref")
                return True
            except Exception:
                return False
        return False

    @classmethod
    def lib(cls):
        if cls._lib is None:
            lib = ctypes.CDLL(str(_ensure(REF_SO, "ref")))
            vp = ctypes.c_void_p
            lib.tgxref_build.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p, _u64p,
                                         _u64p, ctypes.c_int, ctypes.c_uint64, _P(vp)]
            lib.tgxref_build_weighted.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p,
                                                  _u64p, _u64p, _P(ctypes.c_double),
                                                  ctypes.c_int, ctypes.c_uint64, _P(vp)]
            lib.tgxref_free.argtypes = [vp]
            lib.tgxref_free.restype = None
            lib.tgxref_query.argtypes = [vp, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _i64p]
            lib.tgxref_enumerate.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p,
                                             _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _i64p]
            lib.tgxref_set_workers.argtypes = [ctypes.c_int]
            lib.tgxref_set_workers.restype = None
            lib.tgxref_last_error.restype = ctypes.c_char_p
            lib.tgxref_digest.argtypes = [_i64p, ctypes.c_uint64]
            lib.tgxref_digest.restype = ctypes.c_uint64
            cls._lib = lib
        return cls._lib

    @classmethod
    def set_workers(cls, n: int) -> None:
        cls.lib().tgxref_set_workers(n)

    @classmethod
    def workers(cls) -> int:
        return int(cls.lib().tgxref_num_workers())

    def __init__(self, edges, n: int, directed: bool = True, index_cutoff: int = 0,
                 weights=None):
        lib = self.lib()
        s, d, a, b = _arr(edges)
        self.n = n
        self._h = ctypes.c_void_p()
        if weights is None:
            self._check(lib.tgxref_build(n, len(s), s.ctypes.data_as(_u32p),
                                         d.ctypes.data_as(_u32p), a.ctypes.data_as(_u64p),
                                         b.ctypes.data_as(_u64p), 1 if directed else 0,
                                         index_cutoff, ctypes.byref(self._h)))
        else:
            w = np.ascontiguousarray(weights, np.float64)
            self._check(lib.tgxref_build_weighted(
                n, len(s), s.ctypes.data_as(_u32p), d.ctypes.data_as(_u32p),
                a.ctypes.data_as(_u64p), b.ctypes.data_as(_u64p), w.ctypes.data_as(_f64p),
                1 if directed else 0, index_cutoff, ctypes.byref(self._h)))

    @classmethod
    def _check(cls, rc):
        if rc:
            raise OracleError(rc, cls.lib().tgxref_last_error().decode())

    def query(self, kind: str, vertex: int, t_a: int, t_b: int, ordering: int = 1,
              force: int = -1) -> np.ndarray:
        out = np.empty(self.n, np.int64)
        self._check(self.lib().tgxref_query(self._h, KIND[kind], vertex, t_a, t_b, ordering, force,
                                            out.ctypes.data_as(_i64p)))
        return out

    @classmethod
    def enumerate(cls, edges, n: int, kind: str, vertex: int, t_a: int, t_b: int,
                  ordering: int = 1) -> np.ndarray:
        s, d, a, b = _arr(edges)
        out = np.empty(n, np.int64)
        cls._check(cls.lib().tgxref_enumerate(n, len(s), s.ctypes.data_as(_u32p),
                                              d.ctypes.data_as(_u32p), a.ctypes.data_as(_u64p),
                                              b.ctypes.data_as(_u64p), vertex, t_a, t_b,
                                              ordering, KIND[kind], out.ctypes.data_as(_i64p)))
        return out

    def access_decisions(self, direction: int, verts, t_a, t_b, theta: float = 0.2):
        """choose_access_method + count_in_window of the reference (its registry)."""
        return _decisions(self.lib().tgxref_access_decisions, self._check,
                          (self._h, ctypes.c_int(direction)), verts, t_a, t_b, theta)

    @classmethod
    def fit_cost_constants(cls, degree, matches, index_s, scan_s, theta: float = 0.2):
        out = (ctypes.c_double * 3)()
        deg, mat, ix, sc = _fit_arrays(degree, matches, index_s, scan_s)
        cls._check(cls.lib().tgxref_fit_cost_constants(
            ctypes.c_uint64(len(deg)), deg.ctypes.data_as(_u64p), mat.ctypes.data_as(_u64p),
            ix.ctypes.data_as(_f64p), sc.ctypes.data_as(_f64p), ctypes.c_double(theta), out))
        return out[0], out[1]

    def close(self):
        if self._h:
            self.lib().tgxref_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)


def _decisions(fn, check, head, verts, t_a, t_b, theta):
    v = np.ascontiguousarray(verts, np.uint32)
    ta = np.ascontiguousarray(t_a, np.uint64)
    tb = np.ascontiguousarray(t_b, np.uint64)
    k = len(v)
    method = np.empty(k, np.int32)
    beta = np.empty(k, np.float64)
    khat = np.empty(k, np.float64)
    matches = np.empty(k, np.uint64)
    fn.restype = ctypes.c_int
    check(fn(*head, ctypes.c_uint64(k), v.ctypes.data_as(_u32p), ta.ctypes.data_as(_u64p),
             tb.ctypes.data_as(_u64p), ctypes.c_double(theta), method.ctypes.data_as(_i32p),
             beta.ctypes.data_as(_f64p), khat.ctypes.data_as(_f64p),
             matches.ctypes.data_as(_u64p)))
    return method, beta, khat, matches


def _fit_arrays(degree, matches, index_s, scan_s):
    return (np.ascontiguousarray(degree, np.uint64), np.ascontiguousarray(matches, np.uint64),
            np.ascontiguousarray(index_s, np.float64), np.ascontiguousarray(scan_s, np.float64))
