mkdir -p gpurun_out/p38
for v in default l8 l24 l32 b4l16; do L=build/variants/lib_$v.so; [ $v = default ] && L=paper_2401_02563_b200/libtgxd.so
TGXD_LIB=$L timeout 600 python tools/diag.py --mode 0 --trace --reps 5 > gpurun_out/p38/$v.log 2>&1; done
