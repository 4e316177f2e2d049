"""The five BASELINE.json workloads, pinned.

Each config names a generator (the same edge list feeds the device, the C
oracle and the reference library) and a deterministic query set. Sources are
"seeded random non-isolated": uniform over vertices with out-degree >= 1 (and
in-degree >= 1 where the vertex is also a latest-departure target).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Tuple

import numpy as np

from . import GenConfig, QueryWindow

SEED = 2401_02563


@dataclass
class Query:
    kind: str
    vertex: int
    window: QueryWindow


@dataclass
class Workload:
    name: str
    gen: GenConfig
    index_cutoff: int
    describe: str
    queries: Callable[[np.ndarray, np.ndarray, int], List[Query]] = field(repr=False)


def _rng(tag: int) -> np.random.Generator:
    return np.random.default_rng(SEED + tag)


def _pick(rng: np.random.Generator, ok: np.ndarray, k: int) -> np.ndarray:
    cand = np.flatnonzero(ok)
    return cand[rng.integers(0, len(cand), size=k)]


def _c1(out_deg, in_deg, n):
    return [Query("earliest_arrival", 0, QueryWindow(0, 999_999))]


def _c2(out_deg, in_deg, n):
    src = int(_pick(_rng(2), out_deg > 0, 1)[0])
    return [Query("earliest_arrival", src, QueryWindow(0, 999_999))]


def _c3(out_deg, in_deg, n):
    rng = _rng(3)
    qs = []
    srcs = _pick(rng, (out_deg > 0) & (in_deg > 0), 32)
    offs = rng.integers(0, 990_001, size=32)
    for s, o in zip(srcs, offs):
        w = QueryWindow(int(o), int(o) + 9_999)
        qs.append(Query("earliest_arrival", int(s), w))
        qs.append(Query("latest_departure", int(s), w))
    return qs


def _c4(out_deg, in_deg, n):
    src = int(_pick(_rng(4), (out_deg > 0) & (in_deg > 0), 1)[0])
    w = QueryWindow(0, 10_000_000 - 1)
    return [Query("fastest", src, w), Query("latest_departure", src, w)]


def _c5(out_deg, in_deg, n):
    rng = _rng(5)
    srcs = _pick(rng, out_deg > 0, 16)
    offs = rng.integers(0, 900_001, size=16)
    qs = [Query("earliest_arrival", int(s), QueryWindow(0, 999_999)) for s in srcs]
    qs += [Query("earliest_arrival", int(s), QueryWindow(int(o), int(o) + 99_999))
           for s, o in zip(srcs, offs)]
    return qs


def c2_rotation(out_deg: np.ndarray, k: int = 8) -> List[Query]:
    """The bench's query stream on config 2: k seeded non-isolated sources
    (the first is config 2's own source), EA over [0, 999999], one query per
    step in turn — distinct queries, as a serving stream has."""
    srcs = _pick(_rng(2), out_deg > 0, k)
    return [Query("earliest_arrival", int(s), QueryWindow(0, 999_999)) for s in srcs]


def workload(name: str, scale_delta: int = 0) -> Workload:
    """A BASELINE workload; scale_delta < 0 shrinks the graph (parity tests at
    oracle-friendly sizes) while keeping its distributions."""
    d = scale_delta
    if name == "c1":
        return Workload("c1", GenConfig.uniform(1 << (20 + d), 1 << (24 + d), 1_000_000, 0.01,
                                                SEED + 1), 2048,
                        "uniform n=2^20 m=2^24 (self-loops dropped), EA from v0, [0,1e6)", _c1)
    if name in ("c2", "c3"):
        gen = GenConfig.rmat(22 + d, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, SEED + 2,
                             cube_root_starts=True)
        if name == "c2":
            return Workload("c2", gen, 2048,
                            "RMAT-22 ef16 (.57,.19,.19,.05), growth-skewed starts, EA", _c2)
        return Workload("c3", gen, 256, "RMAT-22 32x(EA+LD), 1%-width windows, index deg>=256",
                        _c3)
    if name == "c4":
        return Workload("c4", GenConfig.rmat(23 + d, 16, 0.57, 0.19, 0.19, 10_000_000, 0.005,
                                             SEED + 4), 2048,
                        "RMAT-23 uniform starts to 1e7, fastest + LD", _c4)
    if name == "c5":
        return Workload("c5", GenConfig.rmat(24 + d, 16, 0.65, 0.15, 0.15, 1_000_000, 0.01,
                                             SEED + 5, cube_root_starts=True), 2048,
                        "RMAT-24 (.65,.15,.15,.05), 16 sources x {full, 10%} EA", _c5)
    raise KeyError(name)


NAMES = ("c1", "c2", "c3", "c4", "c5")
