mkdir -p gpurun_out/p25
for v in default b128 b256 b4096; do L=build/variants/lib_$v.so; [ $v = default ] && L=paper_2401_02563_b200/libtgxd.so
 for h in 262144 0; do TGXD_HANDOFF_F=$h TGXD_LIB=$L timeout 600 python tools/diag.py --mode 0 --trace --reps 3 > gpurun_out/p25/${v}_$h.log 2>&1; done; done
