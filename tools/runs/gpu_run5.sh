mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_early_copy.py -m gpu -x -q -p no:cacheprovider -k "not full" > gpurun_out/r02e/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02e/pytest.log
TGXD_ASTATS=1 timeout 300 python tools/rotation_probe.py --trace > gpurun_out/r02e/trace.jsonl 2> gpurun_out/r02e/trace.err
tail -2 gpurun_out/r02e/trace.jsonl; head -8 gpurun_out/r02e/trace.err
for h in 8192 16384 32768 65536; do TGXD_HANDOFF_F=$h timeout 300 python tools/ab_quick.py --skip c1,c4 >> gpurun_out/r02e/ab.jsonl 2>&1; done
TGXD_TAIL=async timeout 300 python tools/ab_quick.py --skip c1,c4 >> gpurun_out/r02e/ab.jsonl 2>&1
cat gpurun_out/r02e/ab.jsonl
