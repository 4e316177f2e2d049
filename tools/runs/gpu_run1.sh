set -x
mkdir -p gpurun_out/r02a
nproc > gpurun_out/r02a/nproc.txt
TGXD_PARITY_LOG=gpurun_out/r02a/parity_full.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02a/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; echo "bench rc=$?"
cat gpurun_out/r02a/bench.json | head -c 3000
