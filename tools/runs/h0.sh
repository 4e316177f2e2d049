mkdir -p gpurun_out/h0
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/h0/smi.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/h0/bench.json 2> gpurun_out/h0/bench.err; echo bench rc=$?
timeout 300 python tools/diag.py --reps 3 > gpurun_out/h0/diag.log 2>&1; echo diag rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/h0/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/h0/pytest.log
