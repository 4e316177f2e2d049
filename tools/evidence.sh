#!/bin/bash
# Round evidence on one B200: bench line (with cpu_baseline), reference arm,
# ncu launch list of the bench command, ncu --set full captures of the
# traversal kernel over the 8-source rotation (-> traffic.json) and of the
# cluster tail kernel, per-round ncu budget, per-config table with parity
# against the reference, hub-source fastest, the GPU test suite.
# Usage (under gpurun): tools/evidence.sh TAG   (NO_CONFIGS=1 / NO_TESTS=1 skip parts)
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/host.txt
nproc > $OUT/nproc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/rotation_once.py > $OUT/plain_rot.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:traverse -s 16 -c 8 \
    -o $OUT/prof_rot python tools/rotation_once.py > $OUT/ncu_full_rot.log 2>&1; echo "full rot rc=$?"
python tools/traffic.py $OUT/prof_rot.ncu-rep $OUT/traffic.json
python tools/ncu_summary.py $OUT/prof_rot.ncu-rep > $OUT/ncu_full_traverse.txt 2>&1
timeout 120 python tools/diag.py --reps 3 > $OUT/plain_diag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 1 -c 1 \
    -o $OUT/prof_tail python tools/diag.py --reps 3 > $OUT/ncu_full_tail.log 2>&1; echo "full tail rc=$?"
python tools/ncu_summary.py $OUT/prof_tail.ncu-rep > $OUT/ncu_full_tail.txt 2>&1
rm -f $OUT/prof_rot.ncu-rep   # 8 captures: too large to bring back (summaries above)
bash tools/phase_profile.sh $OUT/phase 8 > $OUT/phase.log 2>&1; echo "phase rc=$?"
if [ -z "$NO_CONFIGS" ]; then
  timeout 2400 python tools/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?"
  timeout 900 python tools/hub_fastest.py --delta -3 --ranks 0,10,100 --ref-timeout 300 > $OUT/hub_c4_d3.jsonl 2>&1; echo "hub rc=$?"
  timeout 600 python tools/hub_fastest.py --delta 0 --ranks 0,100,1000 --no-ref --steps 1 > $OUT/hub_c4.jsonl 2>&1
fi
if [ -z "$NO_TESTS" ]; then
  TGXD_PARITY_LOG=$OUT/parity_full.jsonl timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
fi
