mkdir -p gpurun_out/p3
timeout 300 python tools/race_loop.py c4 10 0,4 > gpurun_out/p3/rl_fix.log 2>&1; echo fix; tail -n 1 gpurun_out/p3/rl_fix.log
timeout 300 python tools/race_loop.py c4 10 0,4 earliest_arrival > gpurun_out/p3/rl_fix_ea.log 2>&1; echo ea; tail -n 1 gpurun_out/p3/rl_fix_ea.log
TGXD_PULL_F=1 timeout 300 python tools/race_loop.py c4 6 0 > gpurun_out/p3/rl_fix_pf1.log 2>&1; echo pf1; tail -n 1 gpurun_out/p3/rl_fix_pf1.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p3/pytest.log 2>&1; tail -n 3 gpurun_out/p3/pytest.log
