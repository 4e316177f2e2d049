"""Fastest path from hub sources (the paper's top-degree
source methodology): config 4's graph, sources at out-degree
ranks --ranks (0 = the top hub), candidate count (distinct in-window
departures, path_algorithms.cpp:449-458), device time of the whole query
(candidate extraction included), and the reference library on the host
cores for the same query in a child process bounded by --ref-timeout,
labels compared when it finishes.

usage: python tools/hub_fastest.py [--delta 0] [--ranks 0,10,100] [--ref-timeout 300]"""
import argparse, json, multiprocessing as mp, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("--delta", type=int, default=0)
ap.add_argument("--ranks", default="0,10,100")
ap.add_argument("--ref-timeout", type=float, default=300.0)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--no-ref", action="store_true")
args = ap.parse_args()


def ref_child(delta, vertex, t_a, t_b, q):
    from oracle.pyoracle import Reference, generate, digest
    from paper_2401_02563_b200.configs import workload
    wl = workload("c4", delta)
    edges = generate(wl.gen)
    ref = Reference(edges, wl.gen.n_vertices, True, wl.index_cutoff)
    t0 = time.perf_counter()
    lab = ref.query("fastest", vertex, t_a, t_b)
    q.put((time.perf_counter() - t0, digest(lab), int(np.sum(lab != np.iinfo(np.int64).max))))


def main():
    import paper_2401_02563_b200 as T
    from oracle.pyoracle import digest
    from paper_2401_02563_b200.configs import workload
    wl = workload("c4", args.delta)
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    deg = g.degrees(T.Direction.OUT).astype(np.int64)
    order = np.argsort(-deg, kind="stable")
    w = T.QueryWindow(0, 10_000_000 - 1)
    for rk in [int(x) for x in args.ranks.split(",")]:
        v = int(order[rk])
        st = T.EdgeMapStats()
        t0 = time.perf_counter()
        res = T.fastest_path(g, v, w, T.AlgoOptions(stats=st))
        first_s = time.perf_counter() - t0
        tot, ker = T.time_queries(g, "fastest", [v], [w], warmup=0, steps=args.steps)
        line = {"config": "c4", "delta": args.delta, "rank": rk, "vertex": v,
                "out_degree": int(deg[v]), "candidates": st.candidates, "rounds": st.rounds,
                "gpu_ms": round(tot / args.steps, 3), "first_call_s": round(first_s, 3),
                "reached": int(np.sum(res.values != np.iinfo(np.int64).max)),
                "gpu_digest": digest(res.values)}
        if not args.no_ref:
            q = mp.Queue()
            p = mp.get_context("fork").Process(target=ref_child,
                                               args=(args.delta, v, w.t_a, w.t_b, q))
            p.start()
            p.join(args.ref_timeout)
            if p.is_alive():
                p.kill()
                p.join()
                line["ref"] = f"did not finish in {args.ref_timeout:.0f} s (incl. graph build)"
            else:
                s, dg, reached = q.get()
                line.update({"ref_s": round(s, 3), "ref_digest": dg,
                             "identical": dg == line["gpu_digest"],
                             "speedup": round(s * 1e3 / line["gpu_ms"], 1)})
        print(json.dumps(line), flush=True)
    g.close()


if __name__ == "__main__":
    main()
