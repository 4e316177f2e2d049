mkdir -p gpurun_out/p16
timeout 300 python tools/hunt.py 3 75 > gpurun_out/p16/h3.log 2>&1; echo "h3 $(tail -n 1 gpurun_out/p16/h3.log) mism $(grep -c MISMATCH gpurun_out/p16/h3.log)"
timeout 300 python tools/hunt.py 0 76 > gpurun_out/p16/h0.log 2>&1; echo "h0 mism $(grep -c MISMATCH gpurun_out/p16/h0.log)"
timeout 300 python tools/race_loop.py c4 4 0,3 earliest_arrival > gpurun_out/p16/rl.log 2>&1; tail -n 1 gpurun_out/p16/rl.log
timeout 300 python tools/race_loop.py c4 4 0,3 latest_departure > gpurun_out/p16/rl2.log 2>&1; tail -n 1 gpurun_out/p16/rl2.log
for m in 0 3; do TGXD_ASTATS=1 timeout 600 python tools/diag.py --mode $m --reps 3 > gpurun_out/p16/d$m.log 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p16/pytest.log 2>&1; tail -n 3 gpurun_out/p16/pytest.log
