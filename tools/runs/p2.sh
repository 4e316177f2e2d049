# p2: expansion prefetch per engine (async / tail / thin grid rounds): A/B
mkdir -p gpurun_out/p2
O=gpurun_out/p2
for v in okm a1 a1t1 a1g1 a1g1s okm a1 a1t1 a1g1 a1g1s; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
