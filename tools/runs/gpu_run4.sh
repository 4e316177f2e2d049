mkdir -p gpurun_out/r02d
TGXD_HANDOFF_F=0 timeout 300 python tools/rotation_probe.py --trace > gpurun_out/r02d/trace_nohandoff.jsonl 2>&1
timeout 300 python tools/rotation_probe.py --trace > gpurun_out/r02d/trace_default.jsonl 2>&1
for t in 1 2 4; do TGXD_TAIL_BLOCKS_PER_SM=$t timeout 300 python tools/ab_quick.py --skip c1,c4,c5 >> gpurun_out/r02d/ab_tail.jsonl 2>&1; done
for h in 8192 32768 65536; do TGXD_HANDOFF_F=$h timeout 300 python tools/ab_quick.py --skip c1,c4,c5 >> gpurun_out/r02d/ab_tail.jsonl 2>&1; done
timeout 300 python tools/ab_quick.py >> gpurun_out/r02d/ab_tail.jsonl 2>&1
cat gpurun_out/r02d/ab_tail.jsonl
