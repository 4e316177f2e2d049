# r02m: AoS records for pull scans (A/B)
mkdir -p gpurun_out/r02m
O=gpurun_out/r02m
for v in soa aos soa aos; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
