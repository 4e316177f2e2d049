mkdir -p gpurun_out/p20
for m in 0 1; do timeout 600 python tools/diag.py --mode $m --trace --reps 3 > gpurun_out/p20/d$m.log 2>&1; done
timeout 300 python tools/hunt.py 0 80 > gpurun_out/p20/h0.log 2>&1; echo "h0 mism $(grep -c MISMATCH gpurun_out/p20/h0.log) $(tail -n 1 gpurun_out/p20/h0.log)"
timeout 300 python tools/hunt.py 2 81 > gpurun_out/p20/h2.log 2>&1; echo "h2 mism $(grep -c MISMATCH gpurun_out/p20/h2.log) $(tail -n 1 gpurun_out/p20/h2.log)"
