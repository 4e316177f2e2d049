mkdir -p gpurun_out/p27
timeout 300 python tools/hunt.py 3 87 > gpurun_out/p27/h3.log 2>&1; echo "h3 mism $(grep -c MISMATCH gpurun_out/p27/h3.log) $(tail -n 1 gpurun_out/p27/h3.log)"
timeout 300 python tools/race_loop.py c4 4 0,3 > gpurun_out/p27/rl.log 2>&1; tail -n 1 gpurun_out/p27/rl.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p27/pytest.log 2>&1; tail -n 3 gpurun_out/p27/pytest.log
