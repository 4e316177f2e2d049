# r02v: chunks + windows dealt as one unit sequence (A/B)
mkdir -p gpurun_out/r02v
O=gpurun_out/r02v
for v in split units split units; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
