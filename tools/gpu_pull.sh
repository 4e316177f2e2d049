mkdir -p gpurun_out/p32
for g in 16 64; do TGXD_HANDOFF_GROWTH=$g timeout 1500 python tools/bench_configs.py --no-ref --steps 10 --configs c1,c2,c3,c4 > gpurun_out/p32/g$g.jsonl 2> gpurun_out/p32/g$g.err; done
for g in 8 16; do TGXD_HANDOFF_GROWTH=$g timeout 600 python tools/diag.py --mode 0 --reps 5 > gpurun_out/p32/d$g.log 2>&1; done
