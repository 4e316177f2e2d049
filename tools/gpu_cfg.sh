mkdir -p gpurun_out/cfg
nproc > gpurun_out/cfg/nproc.txt
timeout 2300 python tools/bench_configs.py > gpurun_out/cfg/configs.jsonl 2> gpurun_out/cfg/configs.err; echo "rc=$?"
