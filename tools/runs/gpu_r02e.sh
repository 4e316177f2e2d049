# r02e: two-engine tail handoff (cluster for small shrinking frontiers, async
# for slowly growing ones): timings + the parity suites that cover AUTO
mkdir -p gpurun_out/r02e
O=gpurun_out/r02e
timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.json 2>&1; cat $O/ab.json
timeout 300 python tools/diag.py --config c1 --trace --reps 2 > $O/c1.txt 2>&1; sed -n 2p $O/c1.txt
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_early_copy.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
