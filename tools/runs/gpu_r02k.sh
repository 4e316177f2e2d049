# r02k: interleaved {off, kmax} for expansions (A/B)
mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
for v in base okm base okm; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
