"""The reference's estimator-accuracy measurement (tgx.cpp:454-488) on the
device cost model: for each index cutoff and each recent-fraction window,
the share of indexed vertices (both directions) whose histogram decision
(choose_access_method, selective_index.cpp:200-209) agrees with the decision
the exact selectivity count_in_window / degree would make."""
from __future__ import annotations

from typing import Iterable, Sequence

import numpy as np

from . import (Direction, EngineConfig, QueryWindow, TemporalGraph, access_decisions)
from .edgelist import window_for_recent_fraction


def estimator_accuracy(edges, n_v: int, cutoffs: Sequence[int], fractions_pct: Iterable[float],
                       theta_sel: float = 0.2, directed: bool = True):
    """Rows (cutoff, fraction_pct, indexed_vertices, accuracy) as the CLI
    prints them. `edges` is a (src, dst, start, end) tuple of arrays."""
    src, dst, start, end = (np.asarray(x) for x in edges)
    fractions = list(fractions_pct)
    rows = []
    for cutoff in cutoffs:
        g = TemporalGraph.build((src, dst, start, end), n_v, directed,
                                EngineConfig(index_cutoff=int(cutoff)))
        try:
            for pct in fractions:
                t_a, t_b = window_for_recent_fraction(start, end, pct / 100.0)
                w = QueryWindow(t_a, t_b)
                agree = total = 0
                for d in (Direction.OUT, Direction.IN):
                    deg = g.degrees(d).astype(np.int64)
                    verts = np.flatnonzero(deg >= int(cutoff)).astype(np.uint32)
                    if verts.size == 0:
                        continue
                    method, _, _, matches = access_decisions(g, d, verts, [w] * len(verts),
                                                             theta_sel)
                    true_beta = matches.astype(np.float64) / deg[verts].astype(np.float64)
                    should_index = true_beta <= theta_sel
                    did_index = method == 0
                    agree += int(np.sum(should_index == did_index))
                    total += int(verts.size)
                rows.append((int(cutoff), pct, total, 1.0 if total == 0 else agree / total))
        finally:
            g.close()
    return rows
