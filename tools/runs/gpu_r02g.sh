# r02g: split fastest sweeps — parity, then hub timings (scale 20 with the
# reference digests from r02f, scale 23), C4 / C2 regressions
mkdir -p gpurun_out/r02g
O=gpurun_out/r02g
timeout 900 python -m pytest tests/test_gpu_fastest_split.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 600 python tools/hub_fastest.py --delta -3 --ranks 0,10,100 --no-ref > $O/hub_c4_d3.jsonl 2>&1; cat $O/hub_c4_d3.jsonl
timeout 600 python tools/hub_fastest.py --delta 0 --ranks 0,100,1000 --no-ref --steps 1 > $O/hub_c4.jsonl 2>&1; cat $O/hub_c4.jsonl
timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.json 2>&1; cat $O/ab.json
