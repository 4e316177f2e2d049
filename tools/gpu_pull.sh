mkdir -p gpurun_out/p17
for v in eager lazy; do
  if [ $v = lazy ]; then export TGXD_ASYNC_LAZY=1; fi
  for h in 65536 262144 1000000; do TGXD_HANDOFF_F=$h TGXD_ASTATS=1 timeout 600 python tools/diag.py --mode 0 --reps 3 > gpurun_out/p17/${v}_$h.log 2>&1; done
done
unset TGXD_ASYNC_LAZY
TGXD_ASYNC_EAGER=1 TGXD_ASTATS=1 timeout 600 python tools/diag.py --mode 3 --reps 3 > gpurun_out/p17/m3_eager.log 2>&1
timeout 300 python tools/hunt.py 0 77 > gpurun_out/p17/h0.log 2>&1; echo "h0 mism $(grep -c MISMATCH gpurun_out/p17/h0.log)"
timeout 300 python tools/race_loop.py c4 4 0 earliest_arrival > gpurun_out/p17/rl.log 2>&1; tail -n 1 gpurun_out/p17/rl.log
