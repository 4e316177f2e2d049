mkdir -p gpurun_out/p19
timeout 300 python tools/hunt.py 4 79 > gpurun_out/p19/h4.log 2>&1; echo "h4 mism $(grep -c MISMATCH gpurun_out/p19/h4.log) $(tail -n 1 gpurun_out/p19/h4.log)"
timeout 300 python tools/race_loop.py c4 4 0,4 > gpurun_out/p19/rl.log 2>&1; tail -n 1 gpurun_out/p19/rl.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p19/pytest.log 2>&1; tail -n 3 gpurun_out/p19/pytest.log
