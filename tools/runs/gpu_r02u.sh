# r02u: bucketed patch list (host patches a contiguous range per thread): parity + e2e A/B
mkdir -p gpurun_out/r02u
O=gpurun_out/r02u
timeout 1200 python -m pytest tests/test_gpu_early_copy.py tests/test_gpu_api.py tests/test_gpu_views.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for v in prev bucket prev bucket; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/e2e_ab.py "" 2>&1 | tail -1 | sed "s/^/$v /"; done
TGXD_E2E_TRACE=1 timeout 300 python tools/e2e_breakdown.py > $O/t.txt 2> $O/t.err; head -1 $O/t.txt; tail -3 $O/t.err
