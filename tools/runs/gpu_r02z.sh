# r02z: device build without gathers (sort moves the payload), threaded host validation: parity + timings
mkdir -p gpurun_out/r02z
O=gpurun_out/r02z
timeout 1500 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_full_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 900 python - <<'PY'
import time, numpy as np, os, sys
sys.path.insert(0, ".")
import paper_2401_02563_b200 as T
from paper_2401_02563_b200.configs import workload
for name in ("c2", "c5"):
    wl = workload(name)
    for env in ("", "TGXD_BUILD_GATHER"):
        if env: os.environ[env] = "1"
        t = time.perf_counter(); g = T.TemporalGraph.generate(wl.gen, True, T.EngineConfig(index_cutoff=wl.index_cutoff)); dt = time.perf_counter() - t
        d = T.digest_of(g.flatten()[0].astype(np.int64)) if hasattr(g, "flatten") else None
        print(name, env or "sort-kv", "device generate+build", round(dt, 3), "s")
        g.close()
        if env: del os.environ[env]
    E = T.generate_edges(wl.gen)
    t = time.perf_counter(); g = T.TemporalGraph.build(E, wl.gen.n_vertices, True, T.EngineConfig(index_cutoff=wl.index_cutoff)); print(name, "host edges build", round(time.perf_counter() - t, 3), "s"); g.close()
PY
