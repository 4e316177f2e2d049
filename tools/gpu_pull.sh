mkdir -p gpurun_out/p39
for d in 2 4 8; do TGXD_PULL_DIV=$d timeout 1500 python tools/bench_configs.py --no-ref --steps 5 --configs c1,c2,c4 > gpurun_out/p39/d$d.jsonl 2>/dev/null; done
