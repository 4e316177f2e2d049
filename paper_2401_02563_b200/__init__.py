"""B200-native temporal traversal (Kairos, arXiv 2401.02563) — host API.

A Python mirror of the reference's algorithm entry points
(/root/reference/proj/include/tgx/algorithms.hpp:46-58) and graph build
(engine.hpp:32-33), over the C-ABI in include/tgxd.h. Names, argument meaning
and error behaviour follow the reference:

    g = TemporalGraph.build(edges, n_v, directed=True, config=EngineConfig())
    r = earliest_arrival(g, source, QueryWindow(t_a, t_b), AlgoOptions(...))
    r.values  # numpy int64, PathResult::values semantics

Exceptions map the reference's C++ ones: std::out_of_range -> OutOfRange
(an IndexError), std::invalid_argument -> InvalidArgument (a ValueError).

Every call runs on the GPU through libtgxd.so. There is no CPU fallback: if
the library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import enum
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Optional, Sequence

import numpy as np

__all__ = [
    "Ordering", "ForceAccess", "Direction", "QueryWindow", "TemporalEdge", "EngineConfig",
    "AlgoOptions", "EdgeMapStats", "PathResult", "TemporalGraph", "GenConfig",
    "earliest_arrival", "latest_departure", "fastest_path", "query_batch", "digest_of",
    "generate_edges", "OutOfRange", "InvalidArgument", "Unsupported", "DeviceError",
    "TimeRangeError", "load_library", "K_MAX_TIMESTAMP", "AccessMethod", "AccessDecision",
    "CostModelParams", "CalibrationPoint", "choose_access_method", "access_decisions",
    "count_in_window", "fit_cost_constants", "cost_index_lookup", "cost_scan",
    "concurrent_queries",
]

K_MAX_TIMESTAMP = (1 << 64) - 1          # types.hpp:18
K_UNREACHED_MIN = (1 << 63) - 1          # PathResult::kUnreachedMin, algorithms.hpp:17
K_UNREACHED_MAX = -(1 << 63)             # PathResult::kUnreachedMax, algorithms.hpp:18


class Ordering(enum.IntEnum):            # types.hpp:64-68
    SUCCEEDS = 0
    STRICTLY_SUCCEEDS = 1
    OVERLAPS = 2


class ForceAccess(enum.IntEnum):         # engine.hpp:17 (results-neutral; accepted, not needed)
    AUTO = 0
    INDEX = 1
    SCAN = 2


class Direction(enum.IntEnum):           # types.hpp:87
    OUT = 0
    IN = 1


class Mode(enum.IntEnum):                # traversal schedule (tgxd_mode)
    AUTO = 0
    SPARSE = 1     # rounds, queue frontier
    DENSE = 2      # rounds, implicit dense frontier
    ASYNC = 3      # barrier-free work queues
    PULL = 4       # rounds, every round pulled (bottom-up)
    LANES = 5      # batches of 2..32 EA / LD queries, one warp lane per query


class OutOfRange(IndexError):
    """std::out_of_range in the reference."""


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class Unsupported(NotImplementedError):
    """A request outside the device path (no CPU fallback)."""


class TimeRangeError(ValueError):
    """An edge time outside the device time domain [0, 2^31 - 2]."""


class DeviceError(RuntimeError):
    """CUDA failure or no usable GPU."""


_ERRORS = {1: OutOfRange, 2: InvalidArgument, 3: TimeRangeError, 4: Unsupported, 5: DeviceError,
           6: ValueError, 7: OutOfRange}


@dataclass(frozen=True)
class QueryWindow:                       # types.hpp:43-50 (closed window)
    t_a: int = 0
    t_b: int = K_MAX_TIMESTAMP

    def valid(self) -> bool:
        return self.t_a <= self.t_b


@dataclass(frozen=True)
class TemporalEdge:                      # types.hpp:29-40
    source: int
    destination: int
    start: int
    end: int
    weight: float = 1.0


@dataclass
class EngineConfig:                      # engine.hpp:19-24
    index_cutoff: int = 2048
    ordering: Ordering = Ordering.STRICTLY_SUCCEEDS
    force_access: ForceAccess = ForceAccess.AUTO


@dataclass
class EdgeMapStats:                      # engine.hpp:141-144, plus device counters
    index_decisions: int = 0
    scan_decisions: int = 0
    rounds: int = 0
    candidates: int = 0
    edges_relaxed: int = 0
    kernel_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class AlgoOptions:                       # algorithms.hpp:31-40
    ordering: Optional[Ordering] = None
    force_access: Optional[ForceAccess] = None
    stats: Optional[EdgeMapStats] = None
    mode: Mode = Mode.AUTO
    weighted: bool = False               # shortest_duration only (not on the device)


@dataclass
class PathResult:                        # algorithms.hpp:16-21
    values: np.ndarray
    kUnreachedMin = K_UNREACHED_MIN
    kUnreachedMax = K_UNREACHED_MAX


class _Stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_uint32), ("candidates", ctypes.c_uint32),
                ("expansions", ctypes.c_uint64), ("edges_relaxed", ctypes.c_uint64),
                ("index_lookups", ctypes.c_uint64), ("kernel_ms", ctypes.c_float),
                ("total_ms", ctypes.c_float)]


class GenConfig(ctypes.Structure):       # tgxd_gen_config
    _fields_ = [("kind", ctypes.c_int), ("scale", ctypes.c_uint32), ("n", ctypes.c_uint32),
                ("m", ctypes.c_uint64), ("a", ctypes.c_double), ("b", ctypes.c_double),
                ("c", ctypes.c_double), ("start_dist", ctypes.c_int),
                ("t_range", ctypes.c_uint32), ("geo_p", ctypes.c_double),
                ("seed", ctypes.c_uint64)]

    @property
    def n_vertices(self) -> int:
        return (1 << self.scale) if self.kind == 1 else self.n

    @staticmethod
    def uniform(n: int, m: int, t_range: int, geo_p: float, seed: int,
                cube_root_starts: bool = False) -> "GenConfig":
        return GenConfig(0, 0, n, m, 0.0, 0.0, 0.0, 1 if cube_root_starts else 0, t_range, geo_p,
                         seed)

    @staticmethod
    def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, t_range: int,
             geo_p: float, seed: int, cube_root_starts: bool = False) -> "GenConfig":
        return GenConfig(1, scale, 0, edge_factor << scale, a, b, c,
                         1 if cube_root_starts else 0, t_range, geo_p, seed)


_LIB: Optional[ctypes.CDLL] = None
_P = ctypes.POINTER
_u32p = _P(ctypes.c_uint32)
_u64p = _P(ctypes.c_uint64)
_i64p = _P(ctypes.c_int64)


def load_library() -> ctypes.CDLL:
    """Load libtgxd.so (building it first if sources are newer); raise if that fails."""
    global _LIB
    if _LIB is not None:
        return _LIB
    import os
    from . import _build
    path = _build.LIB
    override = os.environ.get("TGXD_LIB")  # variant builds for A/B measurements
    if override:
        path = Path(override)
    elif _build.needs_build():
        try:
            _build.build()
        except Exception as e:
            # a stale library is only acceptable where nothing can rebuild it
            import shutil
            if not path.exists() or shutil.which("nvcc"):
                raise DeviceError(f"libtgxd.so is out of date and failed to build: {e}") from e
    lib = ctypes.CDLL(str(path))
    vp = ctypes.c_void_p
    sig = {
        "tgxd_last_error": ([], ctypes.c_char_p),
        "tgxd_version": ([], ctypes.c_int),
        "tgxd_device_count": ([_P(ctypes.c_int)], ctypes.c_int),
        "tgxd_graph_build": ([ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p, _u64p, _u64p,
                              ctypes.c_int, ctypes.c_uint64, _P(vp)], ctypes.c_int),
        "tgxd_graph_generate": ([_P(GenConfig), ctypes.c_int, ctypes.c_uint64, _P(vp)],
                                ctypes.c_int),
        "tgxd_graph_build_weighted": ([ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p, _u64p,
                                       _u64p, _P(ctypes.c_double), ctypes.c_int,
                                       ctypes.c_uint64, _P(vp)], ctypes.c_int),
        "tgxd_shortest_duration_weighted": ([vp, ctypes.c_uint32, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_int, _i64p, _P(_Stats)],
                                            ctypes.c_int),
        "tgxd_generate_host": ([_P(GenConfig), ctypes.c_uint64, _u64p, _u32p, _u32p, _u64p,
                                _u64p], ctypes.c_int),
        "tgxd_graph_destroy": ([vp], None),
        "tgxd_graph_view": ([vp, ctypes.c_int, _P(vp)], ctypes.c_int),
        "tgxd_graph_info": ([vp, _u32p, _u64p, _u64p, _u64p], ctypes.c_int),
        "tgxd_graph_degrees": ([vp, ctypes.c_int, _u32p], ctypes.c_int),
        "tgxd_graph_flatten": ([vp, ctypes.c_int, _u32p, _u32p, _u64p, _u64p], ctypes.c_int),
        "tgxd_earliest_arrival": ([vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_int, _i64p, _P(_Stats)], ctypes.c_int),
        "tgxd_latest_departure": ([vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_int, _i64p, _P(_Stats)], ctypes.c_int),
        "tgxd_fastest": ([vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                          _i64p, _P(_Stats)], ctypes.c_int),
        "tgxd_shortest_duration": ([vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_int, _i64p, _P(_Stats)], ctypes.c_int),
        "tgxd_temporal_bfs": ([vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_int, _i64p, _P(_Stats)], ctypes.c_int),
        "tgxd_query": ([vp, ctypes.c_int, ctypes.c_uint32, _u32p, _u64p, _u64p, ctypes.c_int,
                        ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, _P(_Stats)], ctypes.c_int),
        "tgxd_last_work": ([vp, ctypes.c_uint32, _u64p, _u64p], ctypes.c_int),
        "tgxd_last_d2h_bytes": ([vp, _u64p], ctypes.c_int),
        "tgxd_last_h2d_bytes": ([vp, _u64p], ctypes.c_int),
        "tgxd_launch_count": ([vp, _u64p], ctypes.c_int),
        "tgxd_time_rotation": ([vp, ctypes.c_int, ctypes.c_uint32, _u32p, _u64p, _u64p,
                                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _P(ctypes.c_float), _P(ctypes.c_float)], ctypes.c_int),
        "tgxd_time_queries": ([vp, ctypes.c_int, ctypes.c_uint32, _u32p, _u64p, _u64p,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               _P(ctypes.c_float), _P(ctypes.c_float)], ctypes.c_int),
        "tgxd_digest": ([_i64p, ctypes.c_uint64], ctypes.c_uint64),
        "tgxd_access_decisions": ([vp, ctypes.c_int, ctypes.c_uint32, _u32p, _u64p, _u64p,
                                   ctypes.c_double, _P(ctypes.c_int32), _P(ctypes.c_double),
                                   _P(ctypes.c_double), _u64p], ctypes.c_int),
        "tgxd_fit_cost_constants": ([ctypes.c_uint64, _u64p, _u64p, _P(ctypes.c_double),
                                     _P(ctypes.c_double), _P(ctypes.c_double),
                                     _P(ctypes.c_double)], ctypes.c_int),
        "tgxd_set_trace": ([vp, ctypes.c_uint32], ctypes.c_int),
        "tgxd_get_trace": ([vp, _u64p, ctypes.c_uint32, ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = lib
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = _LIB.tgxd_last_error().decode(errors="replace") if _LIB else "tgxd error"
        raise _ERRORS.get(rc, RuntimeError)(msg)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(_P(ct))


def device_count() -> int:
    lib = load_library()
    c = ctypes.c_int(0)
    _check(lib.tgxd_device_count(ctypes.byref(c)))
    return c.value


def _edge_arrays(edges):
    """(src u32, dst u32, start u64, end u64, weight f64 or None) from a
    (src, dst, start, end[, weight]) tuple of arrays, a dict, or TemporalEdges."""
    w = None
    if isinstance(edges, tuple) and len(edges) in (4, 5):
        s, d, a, b = edges[:4]
        w = edges[4] if len(edges) == 5 else None
    elif isinstance(edges, dict):
        s, d, a, b = edges["src"], edges["dst"], edges["start"], edges["end"]
        w = edges.get("weight")
    else:
        el = list(edges)
        s = [e.source for e in el]
        d = [e.destination for e in el]
        a = [e.start for e in el]
        b = [e.end for e in el]
        w = [e.weight for e in el]
    if w is not None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        if np.all(w == 1.0):  # the TemporalEdge default: nothing to store
            w = None
    return (np.ascontiguousarray(s, dtype=np.uint32), np.ascontiguousarray(d, dtype=np.uint32),
            np.ascontiguousarray(a, dtype=np.uint64), np.ascontiguousarray(b, dtype=np.uint64), w)


class TemporalGraph:
    """Device-resident temporal graph (both T-CSR layouts + selective index).
    Mirrors tgx::TemporalGraph (engine.hpp:30-84); immutable after build."""

    def __init__(self, handle: int, config: EngineConfig, directed: bool):
        self._h = ctypes.c_void_p(handle)
        self.config = config
        self.directed = directed
        lib = load_library()
        n = ctypes.c_uint32()
        m = ctypes.c_uint64()
        io = ctypes.c_uint64()
        ii = ctypes.c_uint64()
        _check(lib.tgxd_graph_info(self._h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(io),
                                   ctypes.byref(ii)))
        self._n, self._m, self._indexed = n.value, m.value, (io.value, ii.value)

    @staticmethod
    def build(edges, n_v: int, directed: bool = True,
              config: Optional[EngineConfig] = None) -> "TemporalGraph":
        """TemporalGraph::build (engine.cpp:7-34). `edges`: iterable of
        TemporalEdge, a (src, dst, start, end[, weight]) tuple of arrays, or a
        dict. Weights other than 1.0 are stored on the device for weighted
        shortest duration."""
        config = config or EngineConfig()
        if config.index_cutoff < 1:
            raise InvalidArgument("index cutoff must be >= 1")  # selective_index.cpp:156
        lib = load_library()
        s, d, a, b, w = _edge_arrays(edges)
        h = ctypes.c_void_p()
        _check(lib.tgxd_graph_build_weighted(
            n_v, len(s), _ptr(s, ctypes.c_uint32), _ptr(d, ctypes.c_uint32),
            _ptr(a, ctypes.c_uint64), _ptr(b, ctypes.c_uint64),
            None if w is None else _ptr(w, ctypes.c_double), 1 if directed else 0,
            config.index_cutoff, ctypes.byref(h)))
        return TemporalGraph(h.value, config, directed)

    @staticmethod
    def generate(gen: GenConfig, directed: bool = True,
                 config: Optional[EngineConfig] = None) -> "TemporalGraph":
        """Build from the deterministic synthetic generator, on the device."""
        config = config or EngineConfig()
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.tgxd_graph_generate(ctypes.byref(gen), 1 if directed else 0,
                                       config.index_cutoff, ctypes.byref(h)))
        return TemporalGraph(h.value, config, directed)

    def view(self, share: int) -> "TemporalGraph":
        """A second handle on this graph's device data (tgxd_graph_view): own
        stream and workspace, grids sized so `share` views run side by side
        from separate host threads. Keeps this graph alive."""
        h = ctypes.c_void_p()
        _check(load_library().tgxd_graph_view(self._h, int(share), ctypes.byref(h)))
        v = TemporalGraph(h.value, self.config, self.directed)
        v._parent = self
        if not hasattr(self, "_views"):
            self._views = []
        self._views.append(v)  # closed before this graph's own handle
        return v

    def close(self) -> None:
        for v in list(getattr(self, "_views", [])):
            v.close()
        self._views = []
        parent = getattr(self, "_parent", None)
        if parent is not None:  # a closed view leaves its parent's list
            pv = getattr(parent, "_views", [])
            if self in pv:
                pv.remove(self)
            self._parent = None
        if self._h and self._h.value:
            load_library().tgxd_graph_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def vertex_count(self) -> int:
        return self._n

    def edge_count(self) -> int:
        """Materialized edges per layout (TemporalCsr::edge_count)."""
        return self._m

    def indexed_count(self, d: Direction) -> int:
        return self._indexed[int(d)]

    def ordering(self) -> Ordering:
        return self.config.ordering

    def degrees(self, d: Direction = Direction.OUT) -> np.ndarray:
        out = np.empty(self._n, dtype=np.uint32)
        _check(load_library().tgxd_graph_degrees(self._h, int(d), _ptr(out, ctypes.c_uint32)))
        return out

    def flatten(self, d: Direction = Direction.OUT):
        m = self._m
        s = np.empty(m, np.uint32)
        t = np.empty(m, np.uint32)
        a = np.empty(m, np.uint64)
        b = np.empty(m, np.uint64)
        _check(load_library().tgxd_graph_flatten(self._h, int(d), _ptr(s, ctypes.c_uint32),
                                                 _ptr(t, ctypes.c_uint32),
                                                 _ptr(a, ctypes.c_uint64),
                                                 _ptr(b, ctypes.c_uint64)))
        return s, t, a, b

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h


def _fill_stats(opts: Optional[AlgoOptions], st: _Stats) -> None:
    if opts is None or opts.stats is None:
        return
    s = opts.stats
    s.index_decisions += st.index_lookups
    s.scan_decisions += max(0, st.expansions - st.index_lookups)
    s.rounds += st.rounds
    s.candidates += st.candidates
    s.edges_relaxed += st.edges_relaxed
    s.kernel_ms += st.kernel_ms
    s.total_ms += st.total_ms


def _run(kind: int, g: TemporalGraph, vertex: int, w: QueryWindow,
         opts: Optional[AlgoOptions]) -> PathResult:
    if not isinstance(vertex, (int, np.integer)) or vertex < 0 or vertex >= (1 << 32):
        raise OutOfRange(f"vertex {vertex} outside vertex range [0, {g.vertex_count()})")
    ordering = (opts.ordering if opts and opts.ordering is not None else g.ordering())
    mode = int(opts.mode) if opts else 0
    out = np.empty(g.vertex_count(), dtype=np.int64)
    v = np.array([vertex], np.uint32)
    ta = np.array([w.t_a], np.uint64)
    tb = np.array([w.t_b], np.uint64)
    st = _Stats()
    _check(load_library().tgxd_query(g.handle, kind, 1, _ptr(v, ctypes.c_uint32),
                                     _ptr(ta, ctypes.c_uint64), _ptr(tb, ctypes.c_uint64),
                                     int(ordering), mode, out.ctypes.data_as(ctypes.c_void_p), 8,
                                     0, ctypes.byref(st)))
    _fill_stats(opts, st)
    return PathResult(out)


def earliest_arrival(g: TemporalGraph, source: int, w: QueryWindow = QueryWindow(),
                     opts: Optional[AlgoOptions] = None) -> PathResult:
    """algorithms.hpp:46-47 / path_algorithms.cpp:262-308."""
    return _run(0, g, source, w, opts)


def latest_departure(g: TemporalGraph, target: int, w: QueryWindow = QueryWindow(),
                     opts: Optional[AlgoOptions] = None) -> PathResult:
    """algorithms.hpp:53-54 / path_algorithms.cpp:310-357."""
    return _run(1, g, target, w, opts)


def fastest_path(g: TemporalGraph, source: int, w: QueryWindow = QueryWindow(),
                 opts: Optional[AlgoOptions] = None) -> PathResult:
    """algorithms.hpp:57-58 / path_algorithms.cpp:436-528."""
    return _run(2, g, source, w, opts)


def shortest_duration(g: TemporalGraph, source: int, w: QueryWindow = QueryWindow(),
                      opts: Optional[AlgoOptions] = None) -> PathResult:
    """algorithms.hpp:62-63 / path_algorithms.cpp:196-258, 410-434: the least
    sum of end - start over the path's edges, or with opts.weighted the sum
    of edge weights (non-negative integers on every edge a path reaches,
    else InvalidArgument as duration_metric throws; weight 1.0 on a graph
    built without weights)."""
    return _run(5 if opts is not None and opts.weighted else 3, g, source, w, opts)


def temporal_bfs(g: TemporalGraph, source: int, w: QueryWindow = QueryWindow(),
                 opts: Optional[AlgoOptions] = None) -> PathResult:
    """algorithms.hpp:66-67 / path_algorithms.cpp:359-408 (hop counts)."""
    return _run(4, g, source, w, opts)


KINDS = {"earliest_arrival": 0, "latest_departure": 1, "fastest": 2, "shortest_duration": 3,
         "temporal_bfs": 4, "shortest_duration_weighted": 5}


def query_batch(g: TemporalGraph, kind: str, vertices: Sequence[int],
                windows: Sequence[QueryWindow], ordering: Optional[Ordering] = None,
                mode: Mode = Mode.AUTO, width: int = 8,
                stats: Optional[EdgeMapStats] = None) -> np.ndarray:
    """k queries of one kind as one batched traversal (configs 3 and 5):
    returns a (k, n) label array (int64 for width 8, int32 for width 4)."""
    k = len(vertices)
    if len(windows) != k:
        raise InvalidArgument("one window per query")
    v = np.ascontiguousarray(vertices, np.uint32)
    ta = np.array([w.t_a for w in windows], np.uint64)
    tb = np.array([w.t_b for w in windows], np.uint64)
    out = np.empty((k, g.vertex_count()), dtype=np.int64 if width == 8 else np.int32)
    st = _Stats()
    ordering = g.ordering() if ordering is None else ordering
    _check(load_library().tgxd_query(g.handle, KINDS[kind], k, _ptr(v, ctypes.c_uint32),
                                     _ptr(ta, ctypes.c_uint64), _ptr(tb, ctypes.c_uint64),
                                     int(ordering), int(mode),
                                     out.ctypes.data_as(ctypes.c_void_p), width, 0,
                                     ctypes.byref(st)))
    if stats is not None:
        _fill_stats(AlgoOptions(stats=stats), st)
    return out


def last_d2h_bytes(g: TemporalGraph) -> int:
    """Bytes the last host-result query moved device -> host (copies + patch pairs)."""
    b = ctypes.c_uint64()
    _check(load_library().tgxd_last_d2h_bytes(g.handle, ctypes.byref(b)))
    return b.value


def launch_count(g: TemporalGraph) -> int:
    """Kernels g's queries have launched so far (running total)."""
    b = ctypes.c_uint64()
    _check(load_library().tgxd_launch_count(g.handle, ctypes.byref(b)))
    return int(b.value)


def last_h2d_bytes(g: TemporalGraph) -> int:
    """Bytes the last query moved host -> device (parameters, seeds, candidates)."""
    b = ctypes.c_uint64()
    _check(load_library().tgxd_last_h2d_bytes(g.handle, ctypes.byref(b)))
    return b.value


def last_work(g: TemporalGraph, q: int = 0) -> tuple[int, int]:
    """(E_adm, V_reached) of slot q of the last query on g."""
    e = ctypes.c_uint64()
    r = ctypes.c_uint64()
    _check(load_library().tgxd_last_work(g.handle, q, ctypes.byref(e), ctypes.byref(r)))
    return e.value, r.value


def time_queries(g: TemporalGraph, kind: str, vertices: Sequence[int],
                 windows: Sequence[QueryWindow], ordering: Optional[Ordering] = None,
                 mode: Mode = Mode.AUTO, warmup: int = 3, steps: int = 10) -> tuple[float, float]:
    """(total ms for `steps` back-to-back queries, mean traversal-kernel ms),
    device-timed with CUDA events on the graph's stream, outputs in HBM."""
    v = np.ascontiguousarray(vertices, np.uint32)
    ta = np.array([w.t_a for w in windows], np.uint64)
    tb = np.array([w.t_b for w in windows], np.uint64)
    tot = ctypes.c_float()
    ker = ctypes.c_float()
    ordering = g.ordering() if ordering is None else ordering
    _check(load_library().tgxd_time_queries(g.handle, KINDS[kind], len(v),
                                            _ptr(v, ctypes.c_uint32), _ptr(ta, ctypes.c_uint64),
                                            _ptr(tb, ctypes.c_uint64), int(ordering), int(mode),
                                            warmup, steps, ctypes.byref(tot),
                                            ctypes.byref(ker)))
    return tot.value, ker.value


def time_rotation(g: TemporalGraph, kind: str, vertices: Sequence[int],
                  windows: Sequence[QueryWindow], ordering: Optional[Ordering] = None,
                  mode: Mode = Mode.AUTO, warmup: int = 3,
                  steps: int = 10) -> tuple[float, float]:
    """Like time_queries, but step i is the single query i mod k (a stream of
    distinct queries): (total ms, mean traversal-kernel ms per step)."""
    v = np.ascontiguousarray(vertices, np.uint32)
    ta = np.array([w.t_a for w in windows], np.uint64)
    tb = np.array([w.t_b for w in windows], np.uint64)
    tot = ctypes.c_float()
    ker = ctypes.c_float()
    ordering = g.ordering() if ordering is None else ordering
    _check(load_library().tgxd_time_rotation(g.handle, KINDS[kind], len(v),
                                             _ptr(v, ctypes.c_uint32), _ptr(ta, ctypes.c_uint64),
                                             _ptr(tb, ctypes.c_uint64), int(ordering), int(mode),
                                             warmup, steps, ctypes.byref(tot),
                                             ctypes.byref(ker)))
    return tot.value, ker.value


def set_trace(g: TemporalGraph, max_rounds: int) -> None:
    _check(load_library().tgxd_set_trace(g.handle, max_rounds))


def get_trace(g: TemporalGraph, max_rounds: int, with_device: bool = True) -> np.ndarray:
    """Per-round trace rows (12 u64): t0, t_after_expand, t_after_relax (ns), F,
    chunks, small ranges, pushes, flags, expand last/first warp done, relax
    last/first warp done (first stored as 2^62 - t)."""
    out = np.zeros((max_rounds, 12), np.uint64)
    _check(load_library().tgxd_get_trace(g.handle, _ptr(out, ctypes.c_uint64), max_rounds,
                                         1 if with_device else 0))
    return out


def generate_edges(gen: GenConfig):
    """The generator's edge list on the host: (src u32, dst u32, start u64, end u64)."""
    lib = load_library()
    cap = int(gen.m)
    m = ctypes.c_uint64()
    s = np.empty(cap, np.uint32)
    d = np.empty(cap, np.uint32)
    a = np.empty(cap, np.uint64)
    b = np.empty(cap, np.uint64)
    _check(lib.tgxd_generate_host(ctypes.byref(gen), cap, ctypes.byref(m),
                                  _ptr(s, ctypes.c_uint32), _ptr(d, ctypes.c_uint32),
                                  _ptr(a, ctypes.c_uint64), _ptr(b, ctypes.c_uint64)))
    k = m.value
    return s[:k], d[:k], a[:k], b[:k]


def digest_of(values: np.ndarray) -> int:
    """FNV-1a over the int64 label bytes (digest.hpp:12-52)."""
    v = np.ascontiguousarray(values, dtype=np.int64)
    return int(load_library().tgxd_digest(_ptr(v, ctypes.c_int64), len(v)))


# ---------------------------------------------------------------------------
# Selective-index cost model (selective_index.hpp:45-130): results-neutral
# for the traversals; the device builds each indexed vertex's density
# histogram on first use and answers estimates bit-identically.

class AccessMethod(enum.IntEnum):        # selective_index.hpp:51
    INDEX_LOOKUP = 0
    SCAN = 1


@dataclass
class AccessDecision:                    # selective_index.hpp:53-59
    method: AccessMethod = AccessMethod.SCAN
    beta_hat: float = -1.0
    k_hat: float = -1.0


@dataclass
class CostModelParams:                   # selective_index.hpp:45-49
    c: float = 1.0
    c_prime: float = 1.0
    theta_sel: float = 0.2


@dataclass
class CalibrationPoint:                  # selective_index.hpp:110-115
    degree: int = 0
    matches: int = 0
    index_seconds: float = 0.0
    scan_seconds: float = 0.0


def access_decisions(g: TemporalGraph, d: Direction, vertices: Sequence[int],
                     windows: Sequence[QueryWindow], theta_sel: float = 0.2):
    """choose_access_method (selective_index.cpp:200-209) and count_in_window
    (tcsr.cpp:124-128) for k (vertex, window) pairs: (method int32, beta_hat,
    k_hat, matches) arrays; beta_hat = k_hat = -1 below the index cutoff."""
    k = len(vertices)
    if len(windows) != k:
        raise InvalidArgument("one window per vertex")
    v = np.ascontiguousarray(vertices, np.uint32)
    ta = np.array([w.t_a for w in windows], np.uint64)
    tb = np.array([w.t_b for w in windows], np.uint64)
    method = np.empty(k, np.int32)
    beta = np.empty(k, np.float64)
    khat = np.empty(k, np.float64)
    matches = np.empty(k, np.uint64)
    _check(load_library().tgxd_access_decisions(
        g.handle, int(d), k, _ptr(v, ctypes.c_uint32), _ptr(ta, ctypes.c_uint64),
        _ptr(tb, ctypes.c_uint64), float(theta_sel), _ptr(method, ctypes.c_int32),
        _ptr(beta, ctypes.c_double), _ptr(khat, ctypes.c_double), _ptr(matches, ctypes.c_uint64)))
    return method, beta, khat, matches


def choose_access_method(v: int, g: TemporalGraph, d: Direction, w: QueryWindow,
                         params: CostModelParams = CostModelParams()) -> AccessDecision:
    """selective_index.hpp:105-106 (the registry is the graph's)."""
    m, b, k, _ = access_decisions(g, d, [v], [w], params.theta_sel)
    return AccessDecision(AccessMethod(int(m[0])), float(b[0]), float(k[0]))


def count_in_window(g: TemporalGraph, v: int, d: Direction, w: QueryWindow) -> int:
    """TemporalCsr::count_in_window (tcsr.hpp:72)."""
    return int(access_decisions(g, d, [v], [w])[3][0])


def fit_cost_constants(points: Sequence[CalibrationPoint],
                       theta_sel: float = 0.2) -> CostModelParams:
    """selective_index.cpp:211-235 (least squares through the origin)."""
    deg = np.array([p.degree for p in points], np.uint64)
    mat = np.array([p.matches for p in points], np.uint64)
    ix = np.array([p.index_seconds for p in points], np.float64)
    sc = np.array([p.scan_seconds for p in points], np.float64)
    c = ctypes.c_double()
    cp = ctypes.c_double()
    _check(load_library().tgxd_fit_cost_constants(
        len(deg), _ptr(deg, ctypes.c_uint64), _ptr(mat, ctypes.c_uint64),
        _ptr(ix, ctypes.c_double), _ptr(sc, ctypes.c_double), ctypes.byref(c), ctypes.byref(cp)))
    return CostModelParams(c.value, cp.value, theta_sel)


def cost_index_lookup(degree: int, k: float, c: float) -> float:
    """selective_index.cpp:144-147: c (log2 degree + k)."""
    if degree == 0:
        raise ValueError("cost_index_lookup: degree must be >= 1")  # std::domain_error
    return c * (math.log2(float(degree)) + k)


def cost_scan(degree: int, c_prime: float) -> float:
    """selective_index.cpp:149-151: c' degree."""
    return c_prime * float(degree)


def concurrent_queries(g: TemporalGraph, kind: str, vertices: Sequence[int],
                       windows: Sequence[QueryWindow], streams: int = 4,
                       ordering: Optional[Ordering] = None) -> np.ndarray:
    """Serving helper: k single queries spread over `streams` views of g
    (tgxd_graph_view), one host thread each, results in a (k, n) int64 array
    — the same labels as k calls on g, at a higher throughput when the
    queries are large (config 2: 1.35x with 4 streams)."""
    import threading
    k = len(vertices)
    if len(windows) != k:
        raise InvalidArgument("one window per query")
    views = getattr(g, "_serve_views", None)
    if not views or len(views) != streams:
        for v in views or []:
            v.close()
        views = [g.view(streams) for _ in range(streams)]
        g._serve_views = views
    fn = {"earliest_arrival": earliest_arrival, "latest_departure": latest_departure,
          "fastest": fastest_path, "shortest_duration": shortest_duration,
          "temporal_bfs": temporal_bfs}[kind]
    out = np.empty((k, g.vertex_count()), np.int64)
    errors = []
    opts = AlgoOptions(ordering=ordering) if ordering is not None else None

    def work(si: int) -> None:
        try:
            for i in range(si, k, streams):
                out[i] = fn(views[si], int(vertices[i]), windows[i], opts).values
        except Exception as e:  # surfaced below, on the caller's thread
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(streams)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return out
