# p1: expansion prefetch at push time (tail / async / thin grid rounds) and okm in the engines: A/B
mkdir -p gpurun_out/p1
O=gpurun_out/p1
for v in base okm pf1 pf2 base pf1 pf2 okm; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
for v in pf1 pf2; do TGXD_LIB=build/variants/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q -p no:cacheprovider > $O/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $O/pytest_$v.log; done
