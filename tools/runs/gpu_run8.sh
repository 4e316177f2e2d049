mkdir -p gpurun_out/r02h
TGXD_ASTATS=1 TGXD_HANDOFF_F=16384 timeout 300 python tools/rotation_probe.py --steps 3 > gpurun_out/r02h/c16k.jsonl 2> gpurun_out/r02h/c16k.err
TGXD_ASTATS=1 TGXD_TAIL=async timeout 300 python tools/rotation_probe.py --steps 3 > gpurun_out/r02h/async.jsonl 2> gpurun_out/r02h/async.err
echo done
