mkdir -p gpurun_out/r02i
timeout 600 python tools/batch_groups.py --config c5 > gpurun_out/r02i/groups_c5.jsonl 2>&1
timeout 600 python tools/batch_groups.py --config c3 --budgets 256,100000 > gpurun_out/r02i/groups_c3.jsonl 2>&1
cat gpurun_out/r02i/groups_*.jsonl
TGXD_PARITY_LOG=gpurun_out/r02i/parity_full.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02i/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02i/pytest.log
