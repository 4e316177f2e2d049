"""Per-config measurement: every BASELINE workload's
queries, device-timed on one B200 (graph resident, outputs in HBM), next to
the reference library (oracle/_ref, all host cores) on the same edge list.

usage: python tools/bench_configs.py [--configs c1,c2,c3,c4,c5] [--steps 20]
       [--ref-steps 3] [--ref-timeout-s 120]
prints one JSON line per (config, query group)."""
import argparse, json, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--ref-steps", type=int, default=3)
ap.add_argument("--no-ref", action="store_true")
ap.add_argument("--extras", action="store_true",
                help="8(f) rows: temporal BFS, shortest duration and the Overlaps ordering "
                     "(config 2 graph; shortest duration on the 2^16-vertex reduction)")
args = ap.parse_args()
FN = {"earliest_arrival": T.earliest_arrival, "latest_departure": T.latest_departure,
      "fastest": T.fastest_path, "shortest_duration": T.shortest_duration,
      "temporal_bfs": T.temporal_bfs}


def extras():
    """One query per (kind, ordering): GPU wall / kernel time next to the
    reference library on the same edge list."""
    from oracle.pyoracle import Reference
    plan = [("c2", 0, [("temporal_bfs", 1), ("earliest_arrival", 2), ("latest_departure", 2),
                       ("fastest", 2), ("temporal_bfs", 2)]),
            ("c2", -6, [("shortest_duration", 1), ("shortest_duration", 0),
                        ("shortest_duration", 2)])]
    for name, delta, qs in plan:
        wl = workload(name, delta)
        g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
        n = g.vertex_count()
        q = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), n)[0]
        ref = None
        if not args.no_ref and Reference.available():
            Reference.set_workers(os.cpu_count() or 1)
            ref = Reference(T.generate_edges(wl.gen), n, True, wl.index_cutoff)
        for kind, ordv in qs:
            opts = T.AlgoOptions(ordering=T.Ordering(ordv))
            FN[kind](g, q.vertex, q.window, opts)  # warm
            times = []
            st = T.EdgeMapStats()
            for _ in range(args.ref_steps):
                t = time.perf_counter()
                st = T.EdgeMapStats()
                got = FN[kind](g, q.vertex, q.window, T.AlgoOptions(ordering=T.Ordering(ordv),
                                                                     stats=st)).values
                times.append(time.perf_counter() - t)
            line = {"config": name, "delta": delta, "kind": kind, "ordering": ordv, "n": n,
                    "m": g.edge_count(), "gpu_wall_ms": 1e3 * float(np.median(times)),
                    "gpu_kernel_ms": st.kernel_ms, "rounds": st.rounds,
                    "edge_checks": st.edges_relaxed,
                    "reached": int((got != (got.min() if kind == "latest_departure"
                                            else got.max())).sum())}
            if ref is not None:
                t = time.perf_counter()
                want = ref.query(kind, q.vertex, q.window.t_a, q.window.t_b, ordv)
                rs = time.perf_counter() - t
                line["ref"] = {"kind": "reference", "cores": os.cpu_count(), "s": rs}
                line["identical"] = bool(np.array_equal(got, want))
                line["speedup_wall"] = rs / (line["gpu_wall_ms"] * 1e-3)
            print(json.dumps(line), flush=True)
        if ref is not None:
            ref.close()
        g.close()


if args.extras:
    extras()
    sys.exit(0)


def ref_time(wl, edges, n, groups, g=None):
    """Median seconds per reference call for each (kind, vertex, window); with
    a device graph `g`, also whether the device's labels for the same query
    are identical, and both FNV-1a digests (digest.hpp:42-52)."""
    from oracle.pyoracle import Reference, digest
    if not Reference.available():
        return None, None, None
    Reference.set_workers(os.cpu_count() or 1)
    t0 = time.perf_counter()
    ref = Reference(edges, n, True, wl.index_cutoff)
    build = time.perf_counter() - t0
    out, checks = [], []
    for kind, v, w, steps in groups:
        ts = []
        for _ in range(steps):
            t = time.perf_counter()
            want = ref.query(kind, v, w.t_a, w.t_b)
            ts.append(time.perf_counter() - t)
        out.append(float(np.median(ts)))
        if g is not None:
            got = FN[kind](g, v, w).values
            checks.append({"vertex": v, "window": [w.t_a, w.t_b],
                           "identical": bool(np.array_equal(got, want)),
                           "ref_digest": digest(want), "gpu_digest": digest(got)})
    ref.close()
    return out, build, checks


for name in args.configs.split(","):
    wl = workload(name)
    t0 = time.perf_counter()
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    build_s = time.perf_counter() - t0
    n = g.vertex_count()
    qs = wl.queries(g.degrees(T.Direction.OUT), g.degrees(T.Direction.IN), n)
    kinds = sorted({q.kind for q in qs})
    edges = None if args.no_ref else T.generate_edges(wl.gen)
    for kind in kinds:
        sub = [q for q in qs if q.kind == kind]
        verts = [q.vertex for q in sub]
        wins = [q.window for q in sub]
        # work per query from the final labels
        e_adm = v_reached = 0
        per_q = []
        for q in sub:
            T.query_batch(g, kind, [q.vertex], [q.window], width=4)
            e, r = T.last_work(g, 0)
            per_q.append((e, r))
            e_adm += e
            v_reached += r
        # one query at a time, and (EA / LD) the whole group as one batch
        single_ms = 0.0
        for q in sub:
            tot, ker = T.time_queries(g, kind, [q.vertex], [q.window], warmup=args.warmup,
                                      steps=args.steps)
            single_ms += tot / args.steps
        batch_ms = None
        if kind != "fastest" and len(sub) > 1:
            tot, ker = T.time_queries(g, kind, verts, wins, warmup=args.warmup, steps=args.steps)
            batch_ms = tot / args.steps
        # the group served by 2 views of the graph from 2 host threads, one
        # query at a time each (tgxd_graph_view; wall clock, outputs on the device)
        views_ms = None
        if len(sub) > 1:
            import threading
            vs = [g.view(2) for _ in range(2)]
            for v in vs:
                T.time_queries(v, kind, [sub[0].vertex], [sub[0].window], warmup=1, steps=1)
            best = None
            for _ in range(3):
                def run(v, mine):
                    for q in mine:
                        T.time_queries(v, kind, [q.vertex], [q.window], warmup=0, steps=1)
                th = [threading.Thread(target=run, args=(vs[i], sub[i::2])) for i in range(2)]
                t1 = time.perf_counter()
                for t in th:
                    t.start()
                for t in th:
                    t.join()
                el = (time.perf_counter() - t1) * 1e3
                best = el if best is None else min(best, el)
            views_ms = best
            for v in vs:
                v.close()
        line = {"config": name, "workload": wl.describe, "kind": kind, "queries": len(sub),
                "n": n, "m": g.edge_count(), "device_build_s": round(build_s, 3),
                "e_adm_total": e_adm, "v_reached_total": v_reached,
                "gpu_ms_sequential": single_ms,
                "gpu_teps_sequential": e_adm / (single_ms * 1e-3) if single_ms else None,
                "gpu_us_per_query": single_ms * 1e3 / len(sub)}
        if views_ms is not None:
            line["gpu_ms_two_views"] = views_ms
        if batch_ms is not None:
            line.update({"gpu_ms_batched": batch_ms,
                         "gpu_teps_batched": e_adm / (batch_ms * 1e-3),
                         "gpu_queries_per_s_batched": len(sub) / (batch_ms * 1e-3)})
        if edges is not None:
            steps = 1 if kind == "fastest" else args.ref_steps
            # bounded sample: at most 8 queries of a group on the CPU
            samp = sub[:8]
            times, rbuild, checks = ref_time(wl, edges, n,
                                             [(kind, q.vertex, q.window, steps) for q in samp], g)
            if times is not None:
                line["parity"] = checks
                line["identical"] = all(c["identical"] for c in checks)
                e_s = sum(per_q[i][0] for i in range(len(samp)))
                line["ref"] = {"kind": "reference", "cores": os.cpu_count(), "queries": len(samp),
                               "s_per_query": float(np.mean(times)),
                               "teps": e_s / sum(times) if sum(times) else None,
                               "build_s": round(rbuild, 2)}
                line["speedup_sequential"] = (sum(times) / len(samp)) / (single_ms * 1e-3 / len(sub))
        print(json.dumps(line), flush=True)
    g.close()
