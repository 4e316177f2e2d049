# r02av: evidence pass on the build with the pull growth rule (bench, reference arm, launch list,
# ncu --set full over the rotation -> traffic.json, per-config table with parity, GPU suite)
O=gpurun_out/r02av
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
nproc > $O/nproc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
TGXD_PARITY_LOG=$O/parity_full.jsonl timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 1500 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/rotation_once.py > $O/plain_rot.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:traverse -s 16 -c 8 \
    -o $O/prof_rot python tools/rotation_once.py > $O/ncu_full_rot.log 2>&1; echo "full rot rc=$?"
python tools/traffic.py $O/prof_rot.ncu-rep $O/traffic.json
python tools/ncu_summary.py $O/prof_rot.ncu-rep > $O/ncu_full_traverse.txt 2>&1
rm -f $O/prof_rot.ncu-rep
