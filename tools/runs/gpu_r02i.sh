# r02i: split sweeps with expansion-time r: parity, hub timings, A/B vs the previous commit
mkdir -p gpurun_out/r02i
O=gpurun_out/r02i
timeout 900 python -m pytest tests/test_gpu_fastest_split.py tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 600 python tools/hub_fastest.py --delta -3 --ranks 0,10,100 --no-ref > $O/hub_c4_d3.jsonl 2>&1; cat $O/hub_c4_d3.jsonl
timeout 600 python tools/hub_fastest.py --delta 0 --ranks 0,100,1000 --no-ref --steps 1 > $O/hub_c4.jsonl 2>&1; cat $O/hub_c4.jsonl
timeout 1500 python tools/ab.py --libs prev=build/variants/lib_prev.so,split2=build/variants/lib_split2.so --configs c1,c2,c4 --steps 20 --rounds 3 > $O/ab3.txt 2>&1; tail -3 $O/ab3.txt
