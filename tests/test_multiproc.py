"""CPU, world_size 2 over gloo: the bench's N>1 path (replicas, no data-path
collective) — max-over-ranks timing and whole-job aggregation — and the
sharding of a query batch over ranks (paper_2401_02563_b200.shard)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = [2.0 + rank, 1.0 + 3 * rank]  # rank 1 is the slow one
    got = bench.max_over_ranks(ms, dist, "cpu")
    teps = bench.whole_job_teps(world, 1_000_000, got[0])
    q.put((rank, got, teps))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, got, teps in res:
        assert got == [3.0, 4.0]
        assert teps == pytest.approx(2 * 1_000_000 / 3e-3)


def test_single_rank_needs_no_process_group():
    import bench
    assert bench.max_over_ranks([1.5, 2.5]) == [1.5, 2.5]
    assert bench.whole_job_teps(1, 10, 1.0) == pytest.approx(1e4)


def _shard_worker(rank, world, port, q):
    import numpy as np
    from paper_2401_02563_b200 import QueryWindow
    from paper_2401_02563_b200.shard import sharded_query_batch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    verts = [5, 9, 2, 7, 11, 3, 8]
    wins = [QueryWindow(10 * i, 10 * i + 5) for i in range(7)]
    calls = []

    def run(vs, ws):  # stands in for the GPU batch: row = f(vertex, window)
        calls.append(list(vs))
        return np.array([[v * 1000 + w.t_a + j for j in range(4)] for v, w in zip(vs, ws)],
                        np.int64)

    out = sharded_query_batch(None, "earliest_arrival", verts, wins, run=run)
    q.put((rank, calls, None if out is None else out.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_batch_shards_over_ranks_and_gathers_in_order():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (calls, out) for r, calls, out in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    verts = [5, 9, 2, 7, 11, 3, 8]
    assert res[0][0] == [[5, 2, 11, 8]] and res[1][0] == [[9, 7, 3]]  # interleaved shares
    assert res[1][1] is None
    want = [[v * 1000 + 10 * i + j for j in range(4)] for i, v in enumerate(verts)]
    assert res[0][1] == want


def test_shard_of_covers_every_query_once():
    from paper_2401_02563_b200.shard import shard_of
    for k in (0, 1, 7, 32):
        for world in (1, 2, 3, 8):
            got = sorted(q for r in range(world) for q in shard_of(k, r, world))
            assert got == list(range(k))
