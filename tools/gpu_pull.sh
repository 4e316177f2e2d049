mkdir -p gpurun_out/p34
for v in default nopipe; do L=build/variants/lib_$v.so; [ $v = default ] && L=paper_2401_02563_b200/libtgxd.so
for m in 0 1; do TGXD_LIB=$L timeout 600 python tools/diag.py --mode $m --trace --reps 5 > gpurun_out/p34/${v}_$m.log 2>&1; done; done
timeout 300 python tools/hunt.py 1 88 > gpurun_out/p34/h1.log 2>&1; echo "h1 mism $(grep -c MISMATCH gpurun_out/p34/h1.log) $(tail -n 1 gpurun_out/p34/h1.log)"
