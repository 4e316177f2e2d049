mkdir -p gpurun_out/p23
for v in default f64 f128; do L=build/variants/lib_$v.so; [ $v = default ] && L=paper_2401_02563_b200/libtgxd.so
for m in 0 1; do TGXD_LIB=$L timeout 600 python tools/diag.py --mode $m --trace --reps 3 > gpurun_out/p23/${v}_$m.log 2>&1; done; done
TGXD_LIB=build/variants/lib_f128.so timeout 300 python tools/hunt.py 0 85 > gpurun_out/p23/h0.log 2>&1; echo "h0 mism $(grep -c MISMATCH gpurun_out/p23/h0.log) $(tail -n 1 gpurun_out/p23/h0.log)"
