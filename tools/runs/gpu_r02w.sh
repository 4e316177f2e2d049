# r02w: work stealing in the grid relax phases: A/B of steal attempts (0 = claims only)
mkdir -p gpurun_out/r02w
O=gpurun_out/r02w
for v in s0 s1 s2; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c1,c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
TGXD_LIB=build/variants/lib_s1.so TGXD_NO_STEAL=1 timeout 600 python tools/ab_quick.py --skip c1,c5 > $O/ab.tmp 2>&1; echo "nosteal: $(tail -1 $O/ab.tmp)"
