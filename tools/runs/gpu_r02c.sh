# r02c: per-round / per-warp trace of config 2 (current engine) and the
# L1-probe variant A/B over the config-2 rotation, config 4 and config 1.
mkdir -p gpurun_out/r02c
TGXD_WTRACE=1 timeout 300 python tools/diag.py --trace --reps 2 > gpurun_out/r02c/trace_c2.txt 2>&1
timeout 600 python tools/rotation_probe.py --trace --steps 5 > gpurun_out/r02c/rotation.jsonl 2>&1
for v in base l1; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > gpurun_out/r02c/ab_$v.json 2>&1; done
for v in l1 base; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 >> gpurun_out/r02c/ab_$v.json 2>&1; done
cat gpurun_out/r02c/ab_*.json
