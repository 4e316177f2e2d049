mkdir -p gpurun_out/p13
for v in default nopipe; do L=build/variants/lib_$v.so; [ $v = default ] && L=paper_2401_02563_b200/libtgxd.so
 for m in 0 1; do TGXD_LIB=$L timeout 600 python tools/diag.py --mode $m --trace --reps 3 > gpurun_out/p13/${v}_$m.log 2>&1; done; done
timeout 300 python tools/hunt.py 1 72 > gpurun_out/p13/h1.log 2>&1; tail -n 1 gpurun_out/p13/h1.log; grep -c MISMATCH gpurun_out/p13/h1.log
