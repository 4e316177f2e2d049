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
