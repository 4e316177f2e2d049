mkdir -p gpurun_out/p21
for m in 0 3; do TGXD_ASTATS=1 timeout 600 python tools/diag.py --mode $m --reps 3 > gpurun_out/p21/d$m.log 2>&1; done
timeout 300 python tools/hunt.py 3 82 > gpurun_out/p21/h3.log 2>&1; echo "h3 mism $(grep -c MISMATCH gpurun_out/p21/h3.log) $(tail -n 1 gpurun_out/p21/h3.log)"
