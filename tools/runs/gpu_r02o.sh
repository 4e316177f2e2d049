# r02o: replica path under torchrun (shared GPU), bench line with measured launches
mkdir -p gpurun_out/r02o
O=gpurun_out/r02o
timeout 900 python -m pytest tests/test_gpu_replicas.py tests/test_gpu_api.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['gpu_launches'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
