# r02n: block size of the persistent kernels (A/B, same warps per SM)
mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
for v in t256 t512 t128 t1024 t256 t512; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)"; done
