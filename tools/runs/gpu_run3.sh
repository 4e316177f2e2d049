mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_api.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "not full" > gpurun_out/r02c/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02c/pytest.log
for d in 4 3 2 0; do TGXD_PULL_DIV=$d timeout 300 python tools/ab_quick.py --skip c5 >> gpurun_out/r02c/ab_pull.jsonl 2>> gpurun_out/r02c/ab.err; done
cat gpurun_out/r02c/ab_pull.jsonl
