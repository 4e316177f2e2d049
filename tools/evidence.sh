#!/bin/bash
# Round evidence on one B200: bench line (with cpu_baseline), reference arm,
# ncu launch list of the bench command, ncu --set full captures of the
# traversal kernel and the cluster tail kernel, per-config table with parity
# against the reference. Usage (under gpurun): tools/evidence.sh TAG
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/host.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 120 python tools/diag.py --reps 3 > $OUT/plain_diag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 \
    -o $OUT/prof python tools/diag.py --reps 3 > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 1 -c 1 \
    -o $OUT/prof_tail python tools/diag.py --reps 3 > $OUT/ncu_full_tail.log 2>&1; echo "full tail rc=$?"
if [ -z "$NO_CONFIGS" ]; then
  nproc > $OUT/nproc.txt
  timeout 2300 python tools/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?"
fi
