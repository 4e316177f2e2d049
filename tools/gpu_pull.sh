mkdir -p gpurun_out/p29
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p29/pytest.log 2>&1; tail -n 3 gpurun_out/p29/pytest.log
timeout 1400 python tools/bench_configs.py --extras > gpurun_out/p29/extras.jsonl 2> gpurun_out/p29/extras.err; tail -n 2 gpurun_out/p29/extras.err
