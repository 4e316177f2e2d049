mkdir -p gpurun_out/r02f
TGXD_HANDOFF_F=16384 timeout 300 python tools/rotation_probe.py --trace --steps 3 > gpurun_out/r02f/trace16k.jsonl 2>&1
TGXD_HANDOFF_F=262144 timeout 300 python tools/rotation_probe.py --trace --steps 3 > gpurun_out/r02f/trace262k.jsonl 2>&1
echo done
