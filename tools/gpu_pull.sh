mkdir -p gpurun_out/p15
timeout 300 python tools/hunt.py 0 73 > gpurun_out/p15/h0.log 2>&1; echo "h0 mism $(grep -c MISMATCH gpurun_out/p15/h0.log)"
timeout 300 python tools/hunt.py 2 74 > gpurun_out/p15/h2.log 2>&1; echo "h2 mism $(grep -c MISMATCH gpurun_out/p15/h2.log)"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p15/pytest.log 2>&1; tail -n 4 gpurun_out/p15/pytest.log
