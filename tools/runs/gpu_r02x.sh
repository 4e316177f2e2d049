# r02x: two open slots per lane in the pull scan (A/B) + parity
mkdir -p gpurun_out/r02x
O=gpurun_out/r02x
for v in one two one two; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
TGXD_LIB=build/variants/lib_two.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_api.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
