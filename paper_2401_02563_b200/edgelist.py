"""On-disk edge lists (the reference's ingest.hpp / ingest.cpp), host side.

Text lines ``src dst start [end] [weight]`` separated by whitespace, ``#``
comment lines, one column count (3, 4 or 5) per file, gzip read
transparently and written for ``.gz`` paths (ingest.cpp:77-197). Three-column
files get end times ``start + U[1, d_max]`` from std::mt19937_64 and
libstdc++'s uniform_int_distribution (Lemire's nearly divisionless
downscaling), consumed in edge order (sample_end_times, ingest.cpp:199-204),
reproduced bit for bit here. Errors are ``EdgeListError`` (std::runtime_error
in the reference) naming ``path:line``.

The loaded arrays feed ``TemporalGraph.build`` (the device T-CSR build).
"""
from __future__ import annotations

import gzip
import math
from dataclasses import dataclass

import numpy as np

__all__ = ["EdgeListError", "LoadedEdges", "load_edge_list", "write_edge_list",
           "sample_end_times", "window_for_recent_fraction", "MT19937_64"]

_U64 = (1 << 64) - 1
_U32_MAX = (1 << 32) - 1


class EdgeListError(RuntimeError):
    """std::runtime_error from load_edge_list / write_edge_list."""


class MT19937_64:
    """std::mt19937_64 (the standard 64-bit Mersenne Twister), block-twisted
    with numpy."""
    N, M = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UPPER = np.uint64(0xFFFFFFFF80000000)
    LOWER = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int = 5489):
        mt = [seed & _U64]
        for i in range(1, self.N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & _U64)
        self._mt = np.array(mt, dtype=np.uint64)
        self._idx = self.N
        self._out = None

    def _twist(self):
        mt, N, M = self._mt, self.N, self.M
        one = np.uint64(1)
        zero = np.uint64(0)
        # i in [0, N - M): mt[i + 1] and mt[i + M] are both untouched
        y = (mt[0:N - M] & self.UPPER) | (mt[1:N - M + 1] & self.LOWER)
        mt[0:N - M] = mt[M:N] ^ (y >> one) ^ np.where(y & one, self.MATRIX_A, zero)
        # i in [N - M, N - 1): mt[i + M - N] already twisted above
        y = (mt[N - M:N - 1] & self.UPPER) | (mt[N - M + 1:N] & self.LOWER)
        mt[N - M:N - 1] = mt[0:M - 1] ^ (y >> one) ^ np.where(y & one, self.MATRIX_A, zero)
        y = (mt[N - 1] & self.UPPER) | (mt[0] & self.LOWER)
        mt[N - 1] = mt[M - 1] ^ (y >> one) ^ (self.MATRIX_A if int(y) & 1 else zero)
        # tempering of the whole block
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        self._out = [int(v) for v in x]
        self._idx = 0

    def __call__(self) -> int:
        if self._idx >= self.N:
            self._twist()
        v = self._out[self._idx]
        self._idx += 1
        return v


def _uniform_int(rng: MT19937_64, a: int, b: int) -> int:
    """std::uniform_int_distribution<uint64_t>(a, b)(rng), libstdc++ 13
    (bits/uniform_int_dist.h: 64-bit engine -> _S_nd<unsigned __int128>)."""
    rng_range = _U64
    urange = b - a
    if urange < rng_range:
        erange = urange + 1
        product = rng() * erange
        low = product & _U64
        if low < erange:
            threshold = ((1 << 64) - erange) % erange
            while low < threshold:
                product = rng() * erange
                low = product & _U64
        return (product >> 64) + a
    return rng() + a  # the full 64-bit range


def sample_end_times(starts, seed: int, d_max: int) -> np.ndarray:
    """end = start + U[1, d_max] per edge in order (ingest.cpp:199-204)."""
    if d_max < 1:
        raise ValueError("end-time sampling needs d_max >= 1")
    rng = MT19937_64(seed)
    starts = np.asarray(starts, dtype=np.uint64)
    out = np.empty_like(starts)
    for i, s in enumerate(starts.tolist()):
        out[i] = s + _uniform_int(rng, 1, d_max)
    return out


@dataclass
class LoadedEdges:
    src: np.ndarray      # uint32
    dst: np.ndarray      # uint32
    start: np.ndarray    # uint64
    end: np.ndarray      # uint64
    weight: np.ndarray   # float64
    n_vertices: int

    @property
    def edges(self):
        """(src, dst, start, end) as TemporalGraph.build takes them."""
        return self.src, self.dst, self.start, self.end


def _u64(tok: str, path: str, line: int, what: str) -> int:
    if not tok or not tok.isdigit() or not tok.isascii():
        raise EdgeListError(f"{path}:{line}: bad {what} '{tok}'")
    v = int(tok)
    if v > _U64:
        raise EdgeListError(f"{path}:{line}: bad {what} '{tok}'")
    return v


def load_edge_list(path: str, map_ids: bool = False, seed: int = 1,
                   end_sample_max: int = 3600) -> LoadedEdges:
    """load_edge_list (ingest.cpp:77-141)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise EdgeListError(f"cannot open {path}") from e
    if raw[:2] == b"\x1f\x8b":  # gzopen reads plain files too
        try:
            raw = gzip.decompress(raw)
        except (OSError, EOFError) as e:
            raise EdgeListError(f"read error on {path}") from e
    ids: dict = {}
    src, dst, st, en, wt = [], [], [], [], []
    columns = 0
    max_id = 0
    any_vertex = False

    def vertex(tok: str, line: int) -> int:
        if map_ids:
            if tok not in ids:
                ids[tok] = len(ids)
            return ids[tok]
        v = _u64(tok, path, line, "vertex id")
        if v > _U32_MAX:
            raise EdgeListError(f"{path}:{line}: vertex id {tok} exceeds 32-bit range")
        return v

    lines = raw.split(b"\n")
    if lines and lines[-1] == b"":
        lines.pop()
    for no, bline in enumerate(lines, start=1):
        if bline.endswith(b"\r"):
            bline = bline[:-1]
        tok = [t.decode("latin-1") for t in bline.split()]  # ASCII whitespace, like isspace
        if not tok or tok[0].startswith("#"):
            continue
        if len(tok) < 3 or len(tok) > 5:
            raise EdgeListError(f"{path}:{no}: expected 3, 4, or 5 columns, found {len(tok)}")
        if columns == 0:
            columns = len(tok)
        elif len(tok) != columns:
            raise EdgeListError(f"{path}:{no}: column count changed from {columns} to {len(tok)}")
        s = vertex(tok[0], no)
        d = vertex(tok[1], no)
        a = _u64(tok[2], path, no, "start time")
        b = _u64(tok[3], path, no, "end time") if columns >= 4 else a
        w = 1.0
        if columns == 5:
            try:
                w = float(tok[4])
            except ValueError:
                raise EdgeListError(f"{path}:{no}: bad weight '{tok[4]}'") from None
        if columns >= 4 and b < a:
            raise EdgeListError(f"{path}:{no}: end {b} precedes start {a}")
        max_id = max(max_id, s, d)
        any_vertex = True
        src.append(s)
        dst.append(d)
        st.append(a)
        en.append(b)
        wt.append(w)
    start = np.array(st, dtype=np.uint64)
    end = np.array(en, dtype=np.uint64)
    if columns == 3:
        end = sample_end_times(start, seed, end_sample_max)
    n_v = len(ids) if map_ids else (max_id + 1 if any_vertex else 0)
    return LoadedEdges(np.array(src, dtype=np.uint32), np.array(dst, dtype=np.uint32), start, end,
                       np.array(wt, dtype=np.float64), n_v)


def _fmt_g17(w: float) -> str:
    """printf("%.17g")."""
    return "%.17g" % w


def write_edge_list(path: str, src, dst, start, end, weight=None) -> None:
    """write_edge_list (ingest.cpp:143-197): `src dst start end weight` lines,
    gzip for a .gz path."""
    m = len(src)
    weight = np.ones(m) if weight is None else np.asarray(weight, dtype=np.float64)
    rows = [f"{int(s)} {int(d)} {int(a)} {int(b)} {_fmt_g17(float(w))}\n"
            for s, d, a, b, w in zip(np.asarray(src).tolist(), np.asarray(dst).tolist(),
                                     np.asarray(start).tolist(), np.asarray(end).tolist(),
                                     weight.tolist())]
    data = "".join(rows).encode("ascii")
    try:
        if path.endswith(".gz"):
            with gzip.open(path, "wb") as f:
                f.write(data)
        else:
            with open(path, "wb") as f:
                f.write(data)
    except OSError as e:
        raise EdgeListError(f"cannot open {path} for writing") from e


def window_for_recent_fraction(start, end, fraction: float):
    """window_for_recent_fraction (ingest.cpp:243-267): [t_a, t_b] with t_a the
    (1 - fraction) nearest-rank quantile of starts and t_b the latest end."""
    start = np.asarray(start, dtype=np.uint64)
    if start.size == 0:
        raise ValueError("window quantile needs a nonempty edge set")
    if not (0.0 < fraction <= 1.0):
        raise ValueError("window fraction must lie in (0, 1]")
    want = int(min(float(start.size), math.ceil(fraction * float(start.size))))
    s = np.sort(start)
    return int(s[s.size - want]), int(np.asarray(end, dtype=np.uint64).max())
