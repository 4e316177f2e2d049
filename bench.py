#!/usr/bin/env python3
"""Benchmark: earliest-arrival traversal on BASELINE config 2 (RMAT-22).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): temporal edges traversed per second (TEPS) on one
B200, TEPS = E_adm / t with E_adm the admissible window edges of the reached
vertices, plus the roofline of the traversal kernel against
the measured HBM copy bandwidth. A step is one EA query over the whole
device-resident graph; the steps rotate over 8 seeded non-isolated sources
(the first is config 2's own), so every step is a distinct query: its
parameters are uploaded and the previous query's labels reset.

N > 1 runs N independent replicas (one process per GPU, no data-path
collective: the path does not shard); value = all ranks'
edges / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG = "c2"


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int, period: float = 0.005):
        self.index = index
        self.period = period
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def max_over_ranks(values, dist=None, device="cpu"):
    """Element-wise max over ranks (the contract's max-over-ranks timing)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def whole_job_teps(world, e_adm_per_rank, ms_per_step):
    """Replicas: every rank traverses its own copy; value = all ranks' edges
    over the slowest rank's step time."""
    return world * e_adm_per_rank / (ms_per_step * 1e-3)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def profile_traffic():
    """DRAM bytes per traversal launch from the committed ncu --set full capture."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(CONFIG)
    return None


RANDOM_LINE_GBS = 4830.0  # profiles/r02k/micro_gather_ncu.txt: 9.52 GB in 1.97 ms


def random_line_roofline(kernel_ms):
    traffic = profile_traffic()
    if not traffic:
        return None
    achieved = traffic / (kernel_ms * 1e-3) / 1e9
    return {"bound": "random 128-byte DRAM lines", "traffic_per_launch": traffic,
            "achieved": achieved, "peak": RANDOM_LINE_GBS, "unit": "GB/s",
            "frac": achieved / RANDOM_LINE_GBS,
            "note": "traffic from the committed ncu capture of the same rotation; the kernel "
                    "time includes the tail engine, so this understates the round kernel's rate"}


def bench_config(wl, queries, n, m, work):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": f"{CONFIG}: {wl.describe}",
            "stream": f"{len(queries)} seeded non-isolated sources (the first is config 2's "
                      "own), one EA query per step in turn",
            "sources": [q.vertex for q in queries],
            "window": [queries[0].window.t_a, queries[0].window.t_b], "n": n, "m": m,
            "e_adm": [e for e, _ in work], "v_reached": [r for _, r in work],
            "l2": "inputs larger than L2 (edge arrays 12 B/edge x 67M = 805 MB)"}


def stream_edges(work, steps):
    """Edges traversed by `steps` steps of the rotation (step i: query i mod k)."""
    k = len(work)
    return sum(work[i % k][0] for i in range(steps))


def cpu_reference_run(wl, edges, n, queries, threads, steps, warmup):
    """Times the reference library (oracle/_ref, compiled unmodified from the
    reference sources) on the same edge list over the query rotation: returns
    per-step seconds and the labels of the rotation's queries."""
    from oracle.pyoracle import Reference

    Reference.set_workers(threads)
    t0 = time.perf_counter()
    ref = Reference(edges, n, True, wl.index_cutoff)
    build_s = time.perf_counter() - t0
    k = len(queries)
    labels = {}
    for i in range(warmup):
        q = queries[i % k]
        labels[i % k] = ref.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
    times = []
    for i in range(steps):
        q = queries[i % k]
        t = time.perf_counter()
        labels[i % k] = ref.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
        times.append(time.perf_counter() - t)
    for i, q in enumerate(queries):  # untimed: labels of queries the steps did not reach
        if i not in labels:
            labels[i] = ref.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
    ref.close()
    return times, build_s, labels


def reference_work(edges, n, queries, labels):
    """(E_adm, V_reached) per rotation query from the reference's labels
    (the C restatement's tgxo_work)."""
    from oracle.pyoracle import Oracle
    o = Oracle(edges, n)
    out = [o.work(q.kind, q.vertex, q.window.t_a, q.window.t_b, labels[i])
           for i, q in enumerate(queries)]
    o.close()
    return out


def run_reference(args):
    """The reference arm: the reference library's CPU path on the host cores.
    Only oracle/ is loaded (the edge list comes from the checker's own
    generator, oracle/tgx_gen.c): libtgxd.so never enters this process."""
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    from paper_2401_02563_b200.configs import c2_rotation, workload  # pure Python
    from oracle.pyoracle import Reference, generate

    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtgxref.so missing"}))
        return 0
    wl = workload(CONFIG)
    edges = generate(wl.gen)
    n = wl.gen.n_vertices
    queries = c2_rotation(np.bincount(edges[0], minlength=n))
    threads = os.cpu_count() or 1
    warm = args.warmup
    times, build_s, labels = cpu_reference_run(wl, edges, n, queries, threads, args.steps, warm)
    work = reference_work(edges, n, queries, labels)
    t = sum(times)
    value = stream_edges(work, args.steps) / t
    line = {
        "impl": "reference",
        "metric": "temporal edges traversed/sec (TEPS)",
        "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": bench_config(wl, queries, n, int(len(edges[0])), work),
        "graph_build_s": build_s,
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} EA queries of the {len(queries)}-source "
                                   f"{CONFIG} rotation"},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_libs": loaded_native_libs(),
    }
    print(json.dumps(line))
    return 0


def loaded_native_libs():
    """The repo's shared libraries mapped into this process."""
    libs = set()
    try:
        for ln in open("/proc/self/maps"):
            path = ln.split()[-1] if ln.strip() else ""
            if path.endswith(".so") and str(ROOT) in path:
                libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def run_ours(args):
    rank, world, local = _dist()
    import paper_2401_02563_b200 as T
    from paper_2401_02563_b200.configs import c2_rotation, workload

    import torch
    # one GPU per rank; TGXD_BENCH_SHARE_GPU=1 maps every rank onto the GPUs
    # there are (a functional check of the replica path on a one-GPU box,
    # tests/test_gpu_replicas.py — not a measurement), with gloo for the
    # barrier and the max-over-ranks reduction
    shared = os.environ.get("TGXD_BENCH_SHARE_GPU") == "1"
    torch.cuda.set_device(local % torch.cuda.device_count() if shared else local)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist_mod
        dist_mod.init_process_group("gloo" if shared else "nccl")
        dist = dist_mod
        red_dev = "cpu" if shared else "cuda"

    if world > 1 and "TGXD_HOST_THREADS" not in os.environ:
        # replicas on one node share the host: split the widening threads
        os.environ["TGXD_HOST_THREADS"] = str(max(2, ((os.cpu_count() or 8) - 4) // world))
    lib = T.load_library()
    wl = workload(CONFIG)
    g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff))
    n = g.vertex_count()
    queries = c2_rotation(g.degrees(T.Direction.OUT))
    srcs = [q.vertex for q in queries]
    wins = [q.window for q in queries]
    k = len(queries)

    # unit of work of every rotation query from its final labels (untimed)
    work = []
    for q in queries:
        T.query_batch(g, q.kind, [q.vertex], [q.window], width=4)
        work.append(T.last_work(g, 0))

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device())
    barrier()
    l0 = T.launch_count(g)
    with sampler:
        total_ms, kernel_ms = T.time_rotation(g, "earliest_arrival", srcs, wins,
                                              warmup=args.warmup, steps=args.steps)
    # the library's own count of the kernels it launched (warm-up included in
    # the call: scaled to the timed steps)
    launches = (T.launch_count(g) - l0) * args.steps / (args.steps + args.warmup)
    barrier()
    ms_step, kernel_ms = max_over_ranks([total_ms / args.steps, kernel_ms], dist, red_dev)
    edges_per_rank = stream_edges(work, args.steps)
    value = world * edges_per_rank / (ms_step * args.steps * 1e-3)

    # end to end through the reference-facing C-ABI call (earliest_arrival
    # with an int64 PathResult in an ordinary host array): every step uploads
    # its query and reads its labels back, the rotation's sources in turn
    out = np.empty(n, np.int64)
    import ctypes
    optr = out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))

    def ea(i):
        q = queries[i % k]
        T._check(lib.tgxd_earliest_arrival(g.handle, q.vertex, q.window.t_a, q.window.t_b, 1,
                                           optr, None))

    for i in range(args.warmup):
        ea(i)
    h2d = d2h = 0
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        ea(i)
        h2d += T.last_h2d_bytes(g)
        d2h += T.last_d2h_bytes(g)
    barrier()
    e2e_s = max_over_ranks([(time.perf_counter() - t0) / args.steps], dist, red_dev)[0]
    e2e_value = world * edges_per_rank / (e2e_s * args.steps)

    # continuity with earlier rounds: config 2's own source repeated
    tot1, ker1 = T.time_queries(g, "earliest_arrival", [srcs[0]], [wins[0]], warmup=3,
                                steps=args.steps)

    conc = concurrent_rotation(T, g, srcs, wins, work, args.steps, barrier) if world == 1 else None

    peak, peak_kind = measured_peak()
    b_alg = [16 * e + 12 * r + 4 * n for e, r in work]  # SURVEY.md 8(d), per query
    b_steps = sum(b_alg[i % k] for i in range(args.steps))
    achieved = b_steps / (kernel_ms * args.steps * 1e-3) / 1e9
    # per step: reset_seed, tail_reset, traverse, the two tail engines (the one
    # not handed the query exits at once), convert
    kernels = ["reset_seed_kernel", "tail_reset_kernel", "traverse_kernel", "tail_kernel",
               "async_kernel", "convert_kernel"]
    line = {
        "metric": "temporal edges traversed/sec (TEPS)",
        "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": bench_config(wl, queries, n, g.edge_count(), work),
        "parallelism": f"replicas x{world}",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": profile_traffic(),
                     "kernel": "traverse_kernel (+ the tail engine it hands off to)",
                     "kernel_ms": kernel_ms,
                     "timed": "CUDA events on the graph stream around the traversal kernels",
                     "algorithmic_bytes_per_step": b_steps / args.steps,
                     "algorithmic_bytes_per_query": b_alg, "peak_kind": peak_kind},
        # what the kernel actually moves: DRAM line traffic (ncu, profiles/traffic.json,
        # traverse_kernel only) over its time, against the random-line ceiling of
        # this GPU (tools/micro_gather.cu: random reads cost 128-byte lines and
        # saturate at 4.8 TB/s, profiles/r02k) — DESIGN.md §7
        "memory_system": random_line_roofline(kernel_ms),
        "e2e": {"value": e2e_value, "unit": "edges/s",
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "host_buffer": "pageable", "ms_per_step": e2e_s * 1e3,
                "call": "tgxd_earliest_arrival (int64 PathResult values in host memory)"},
        # BASELINE config 2 as defined (its one seeded source, repeated): TEPS and the
        # HBM roofline of north_star's target on it
        "single_source": {"source": srcs[0], "ms_per_step": tot1 / args.steps,
                          "kernel_ms": ker1, "value": work[0][0] / (tot1 / args.steps * 1e-3),
                          "roofline": {"bound": "hbm", "achieved": b_alg[0] / (ker1 * 1e-3) / 1e9,
                                       "peak": peak, "unit": "GB/s",
                                       "frac": b_alg[0] / (ker1 * 1e-3) / 1e9 / peak,
                                       "algorithmic_bytes": b_alg[0]}},
        "gpu_launches": round(launches),
        "kernels_per_step": kernels,
        **({"concurrent": conc} if conc else {}),
        "clocks": sampler.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, queries, n, work)
    if rank == 0:
        print(json.dumps(line))
    g.close()
    if dist:
        dist.destroy_process_group()
    return 0


def concurrent_rotation(T, g, srcs, wins, work, steps, barrier, streams=4):
    """Serving throughput, reported beside `value` (which stays one query at a
    time): the same rotation with `streams` queries in flight, each on its own
    view of the graph (tgxd_graph_view: own labels, queues and stream, grids
    sized so the views fit side by side) — one query's latency-bound thin
    rounds overlap another's heavy ones. Wall clock between two device
    synchronisations around all the streams' work; labels stay in HBM."""
    import threading

    k = len(srcs)
    per = max(1, steps // streams)
    views = [g.view(streams) for _ in range(streams)]
    err = []

    def run(si, warm, n_steps):
        try:
            order = [(si + streams * j) % k for j in range(k)]  # stream si's share of the rotation
            T.time_rotation(views[si], "earliest_arrival", [srcs[i] for i in order],
                            [wins[i] for i in order], warmup=warm, steps=n_steps)
        except Exception as e:  # surfaced below
            err.append(e)

    def all_streams(warm, n_steps):
        th = [threading.Thread(target=run, args=(si, warm, n_steps)) for si in range(streams)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    all_streams(3, 1)  # warm-up: every view allocates and runs once
    barrier()
    t0 = time.perf_counter()
    all_streams(0, per)
    barrier()
    dt = time.perf_counter() - t0

    # the same through the C-ABI call with int64 results in host memory (one
    # caller thread and one host array per view; the views split the host
    # widening threads)
    import ctypes
    lib = T.load_library()
    n = g.vertex_count()
    outs = [np.empty(n, np.int64) for _ in range(streams)]

    def run_e2e(si, n_steps):
        try:
            optr = outs[si].ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            for j in range(n_steps):
                i = (si + streams * j) % k
                T._check(lib.tgxd_earliest_arrival(views[si].handle, srcs[i], wins[i].t_a,
                                                   wins[i].t_b, 1, optr, None))
        except Exception as e:  # surfaced below
            err.append(e)

    def all_e2e(n_steps):
        th = [threading.Thread(target=run_e2e, args=(si, n_steps)) for si in range(streams)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    per_e = max(1, per // 2)
    all_e2e(2)
    barrier()
    t1 = time.perf_counter()
    all_e2e(per_e)
    barrier()
    dte = time.perf_counter() - t1
    for v in views:
        v.close()
    if err:
        return {"error": str(err[0])}
    edges = sum(work[(si + streams * j) % k][0] for si in range(streams) for j in range(per))
    edges_e = sum(work[(si + streams * j) % k][0] for si in range(streams) for j in range(per_e))
    return {"streams": streams, "queries": streams * per, "ms_per_query": dt * 1e3 / (streams * per),
            "value": edges / dt, "unit": "edges/s",
            "timed": "host clock between device synchronisations around all streams",
            "e2e": {"value": edges_e / dte, "unit": "edges/s", "queries": streams * per_e,
                    "ms_per_query": dte * 1e3 / (streams * per_e),
                    "call": "tgxd_earliest_arrival on each view from its own host thread "
                            "(int64 PathResult values in host memory)"}}


def cpu_baseline(wl, queries, n, work):
    """The reference CPU path on the box's host cores over one pass of the
    rotation after one warm-up query (graph generation and build untimed, as
    `tgx run` does, tools/tgx.cpp:341-376), or the C oracle (one thread) if
    the reference library did not travel."""
    from oracle.pyoracle import Oracle, Reference, generate

    edges = generate(wl.gen)
    threads = os.cpu_count() or 1
    k = len(queries)
    if Reference.available():
        times, _, _ = cpu_reference_run(wl, edges, n, queries, threads, k, 1)
        kind = "reference"
    else:
        o = Oracle(edges, n)
        times = []
        for q in queries:
            t = time.perf_counter()
            o.query(q.kind, q.vertex, q.window.t_a, q.window.t_b)
            times.append(time.perf_counter() - t)
        o.close()
        kind, threads = "port", 1
    return {"value": stream_edges(work, k) / sum(times), "unit": "edges/s", "cores": threads,
            "kind": kind,
            "sample": f"one pass of the {k}-query {CONFIG} rotation after 1 warm-up "
                      f"({sum(times):.2f} s, median query {statistics.median(times):.3f} s)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
