"""CPU: the C-ABI library loads and exports every entry point include/tgxd.h
declares; host-side logic (generators, configs, validation) without a GPU."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2401_02563_b200 as T
from paper_2401_02563_b200 import configs
from tests import _support as S

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "tgxd.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tgxd_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = T.load_library()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.tgxd_version() == 1
    nm = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2401_02563_b200" /
                                                             "libtgxd.so")],
                        capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", nm), s


def test_library_is_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(ROOT / "paper_2401_02563_b200" /
                                                          "libtgxd.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_means_loud_failure():
    if T.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(T.DeviceError):
        T.TemporalGraph.build(S.hand_edges([(0, 1, 3, 5)]), 2)


def test_generator_is_deterministic_and_pinned():
    for name in ("rmat12", "uniform14"):
        gen, n, m, edig, *_ = S.scaled(name)
        a = T.generate_edges(gen)
        b = T.generate_edges(gen)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert len(a[0]) == m
        assert S.edge_digest(a) == edig


def test_generator_distributions():
    # config 1: uniform endpoints, self-loops dropped, start ~ U[0, 1e6), end = start + 1 + Geo
    g = T.GenConfig.uniform(1 << 12, 1 << 18, 1_000_000, 0.01, 5)
    s, d, a, b = T.generate_edges(g)
    assert np.all(s != d) and np.all(s < 4096) and np.all(d < 4096)
    assert len(s) < (1 << 18) and len(s) > (1 << 18) - 200
    assert a.min() >= 0 and a.max() < 1_000_000
    dur = (b - a).astype(np.int64)
    assert dur.min() >= 1
    assert abs(dur.mean() - (1 + 0.99 / 0.01)) < 3  # mean failures (1-p)/p
    assert abs(a.mean() - 500_000) < 5_000
    # config 2: RMAT with growth-skewed starts floor(1e6 u^(1/3)), duration 1 + Geo(0.02)
    g = T.GenConfig.rmat(14, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 7, cube_root_starts=True)
    s, d, a, b = T.generate_edges(g)
    assert len(s) == 16 << 14 and s.max() < (1 << 14)
    # E[u^(1/3)] = 3/4
    assert abs(a.mean() / 1e6 - 0.75) < 0.01
    assert np.all(a < 1_000_000)
    assert abs((b - a).astype(np.int64).mean() - (1 + 0.98 / 0.02)) < 2
    # skew: RMAT degree distribution is heavy-tailed
    deg = np.bincount(s, minlength=1 << 14)
    assert deg.max() > 40 * deg.mean()


def test_cube_root_start_is_exact():
    """floor(1e6 u^(1/3)) evaluated in integers: check against exact rationals."""
    from fractions import Fraction
    g = T.GenConfig.rmat(4, 16, 0.57, 0.19, 0.19, 1_000_000, 0.02, 11, cube_root_starts=True)
    s, d, a, b = T.generate_edges(g)
    # starts must be consistent with monotone cube-root: a^3 <= u*1e18 < (a+1)^3 is checked
    # on the device/host side; here only the range and integrality
    assert a.dtype == np.uint64 and a.max() < 1_000_000


def test_workload_queries_are_deterministic():
    rng = np.random.default_rng(0)
    out_deg = rng.integers(0, 3, 1000)
    in_deg = rng.integers(0, 3, 1000)
    for name in configs.NAMES:
        wl = configs.workload(name, -14)
        q1 = wl.queries(out_deg, in_deg, 1000)
        q2 = wl.queries(out_deg, in_deg, 1000)
        assert [(q.kind, q.vertex, q.window) for q in q1] == \
               [(q.kind, q.vertex, q.window) for q in q2]
        for q in q1:
            if q.kind == "earliest_arrival" and name != "c1":
                assert out_deg[q.vertex] > 0


def test_window_and_enum_mirror_reference():
    assert T.QueryWindow().t_b == (1 << 64) - 1
    assert not T.QueryWindow(5, 3).valid()
    assert [int(o) for o in T.Ordering] == [0, 1, 2]
    assert T.EngineConfig().index_cutoff == 2048  # selective_index.hpp:74


def test_cpp_shim_compiles():
    exe = Path("/tmp/tgx_b200_shim_test")
    res = subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                          str(ROOT / "tests" / "cpp" / "shim_test.cpp"),
                          "-L", str(ROOT / "paper_2401_02563_b200"), "-ltgxd",
                          "-o", str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-2000:]


def test_oracle_c_restatement_builds():
    res = subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], capture_output=True,
                         text=True)
    assert res.returncode == 0, res.stderr
