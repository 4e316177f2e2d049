# r02q: expansion-time fastest r, skipped EP loads for unreached probes, early
# host copy from inside the round kernel — parity, then A/B (device + e2e)
mkdir -p gpurun_out/r02q
O=gpurun_out/r02q
TGXD_LIB=build/variants/lib_early.so timeout 1200 python -m pytest tests/test_gpu_early_copy.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_fastest_split.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for v in base rexp epskip early base early; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
for v in base early base early; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python bench.py --steps 60 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err; echo "$v e2e: $(python -c "import json; d=json.load(open('$O/b.json')); print(round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['e2e']['d2h_bytes_per_step'])")"; done
