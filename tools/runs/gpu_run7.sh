mkdir -p gpurun_out/r02g
timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_early_copy.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02g/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02g/pytest.log
TGXD_HANDOFF_F=16384 timeout 300 python tools/rotation_probe.py --trace --steps 3 > gpurun_out/r02g/trace16k.jsonl 2>&1
TGXD_HANDOFF_F=65536 timeout 300 python tools/rotation_probe.py --trace --steps 3 > gpurun_out/r02g/trace64k.jsonl 2>&1
for h in 16384 32768 65536; do TGXD_HANDOFF_F=$h timeout 300 python tools/ab_quick.py --skip c1,c4 >> gpurun_out/r02g/ab.jsonl 2>&1; done
cat gpurun_out/r02g/ab.jsonl
