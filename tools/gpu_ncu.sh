mkdir -p gpurun_out/p11
timeout 120 python tools/diag.py --reps 3 --mode 4 --trace > gpurun_out/p11/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 \
    -o gpurun_out/p11/prof python tools/diag.py --reps 3 --mode 4 > gpurun_out/p11/ncu_full.log 2>&1; echo "full rc=$?"
