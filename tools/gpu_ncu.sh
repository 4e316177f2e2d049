mkdir -p gpurun_out/p5
timeout 120 python tools/diag.py --reps 3 > gpurun_out/p5/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 \
    -o gpurun_out/p5/prof python tools/diag.py --reps 3 > gpurun_out/p5/ncu_full.log 2>&1; echo "full rc=$?"
