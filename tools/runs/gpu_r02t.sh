# r02t: fresh-slot queue marks (no expansion-state load for first reaches): parity + A/B
mkdir -p gpurun_out/r02t
O=gpurun_out/r02t
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_configs.py tests/test_gpu_fastest_split.py tests/test_gpu_early_copy.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for v in "TGXD_NO_FRESH=1" "" "TGXD_NO_FRESH=1" ""; do env $v timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "[$v]: $(tail -1 $O/ab.tmp)"; done
