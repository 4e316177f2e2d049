#!/bin/bash
# Round evidence on one B200: bench line (with cpu_baseline), reference arm,
# ncu launch list of the bench command, one ncu --set full capture of the
# traversal kernel. Usage (under gpurun): tools/evidence.sh TAG
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/host.txt
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 120 python tools/diag.py --reps 3 > $OUT/plain_diag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 \
    -o $OUT/prof python tools/diag.py --reps 3 > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
