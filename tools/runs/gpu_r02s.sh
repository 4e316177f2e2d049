# r02s: 24-bit early copy with owner-local patches: parity + interleaved e2e A/B
mkdir -p gpurun_out/r02s
O=gpurun_out/r02s
timeout 1200 python -m pytest tests/test_gpu_early_copy.py tests/test_gpu_api.py tests/test_gpu_views.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 900 python tools/e2e_ab.py "TGXD_NO_PACK24=1;TGXD_LOG_F=0" "" "TGXD_LOG_F=131072" "TGXD_LOG_F=524288" "TGXD_LOG_F=65536" 2>&1 | tail -5
TGXD_E2E_TRACE=1 timeout 300 python tools/e2e_breakdown.py > $O/t.txt 2> $O/t.err; head -1 $O/t.txt; tail -3 $O/t.err
