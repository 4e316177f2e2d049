"""The bench's N > 1 path end to end: two replica ranks under torchrun, each
running the config-2 query rotation through libtgxd.so. On a one-GPU box
both ranks share the GPU (TGXD_BENCH_SHARE_GPU=1, gloo for the barrier and
the max-over-ranks reduction): a functional check of the launch, the
aggregation and the one JSON line rank 0 prints — not a measurement."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_replicas_print_one_aggregated_line():
    env = dict(os.environ, TGXD_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "8", "--warmup", "3",
           "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["parallelism"] == "replicas x2"
    assert d["scaling"] == "weak"
    # value = both ranks' edges over the slowest rank's time
    edges = sum(d["config"]["e_adm"][i % 8] for i in range(d["steps"]))
    assert d["value"] == pytest.approx(2 * edges / (d["ms_per_step"] * d["steps"] * 1e-3),
                                       rel=1e-6)
    assert d["gpu_launches"] >= 4 * d["steps"]
    assert d["e2e"]["d2h_bytes_per_step"] > 0


def _sharded_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2401_02563_b200 as T
    from paper_2401_02563_b200.shard import sharded_query_batch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # one GPU on the box: both ranks share it (functional check)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gen = T.GenConfig.rmat(14, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 21, cube_root_starts=True)
    g = T.TemporalGraph.generate(gen, True, T.EngineConfig(index_cutoff=256))
    deg = g.degrees(T.Direction.OUT).astype(np.int64)
    rng = np.random.default_rng(5)
    verts = [int(v) for v in rng.choice(np.flatnonzero(deg), 9)]
    wins = [T.QueryWindow(0, 999_999) if i % 2 else T.QueryWindow(int(o), int(o) + 99_999)
            for i, o in enumerate(rng.integers(0, 900_000, 9))]
    out = sharded_query_batch(g, "earliest_arrival", verts, wins)
    ok = None
    if rank == 0:
        ok = bool(np.array_equal(out, T.query_batch(g, "earliest_arrival", verts, wins)))
    q.put((rank, ok))
    g.close()
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_batch_equals_one_gpu_batch():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0] is True
