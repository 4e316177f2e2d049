mkdir -p gpurun_out/p28
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q > gpurun_out/p28/pytest.log 2>&1; tail -n 15 gpurun_out/p28/pytest.log
timeout 800 python tools/edge_probe.py c2 -6 > gpurun_out/p28/probe6.log 2>&1; cat gpurun_out/p28/probe6.log
timeout 800 python tools/edge_probe.py c2 0 > gpurun_out/p28/probe0.log 2>&1; cat gpurun_out/p28/probe0.log
