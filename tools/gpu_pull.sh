mkdir -p gpurun_out/p9
timeout 300 python tools/hunt.py 0 70 > gpurun_out/p9/h0.log 2>&1; tail -n 1 gpurun_out/p9/h0.log; grep -c MISMATCH gpurun_out/p9/h0.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p9/pytest.log 2>&1; tail -n 3 gpurun_out/p9/pytest.log
