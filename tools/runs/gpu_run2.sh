mkdir -p gpurun_out/r02b
TGXD_PARITY_LOG=gpurun_out/r02b/parity_full.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02b/pytest.log
TGXD_ASTATS=1 timeout 300 python tools/rotation_probe.py --trace > gpurun_out/r02b/rotation.jsonl 2> gpurun_out/r02b/rotation.err; echo "probe rc=$?"
tail -3 gpurun_out/r02b/rotation.jsonl
