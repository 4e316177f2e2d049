mkdir -p gpurun_out/p40
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "c5 or c3" > gpurun_out/p40/pytest.log 2>&1; tail -n 2 gpurun_out/p40/pytest.log
timeout 1500 python tools/bench_configs.py --no-ref --steps 5 --configs c3,c5 > gpurun_out/p40/cfg.jsonl 2>/dev/null; cat gpurun_out/p40/cfg.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['kind'][:8], 'seq %.3f'%d['gpu_ms_sequential'], 'batched', d.get('gpu_ms_batched'))"
