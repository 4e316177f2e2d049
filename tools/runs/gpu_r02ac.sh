# r02ac: dense-expand threshold sweep (TGXD_DENSE_DIV), TMA-staged relax on hub-heavy configs (N3)
mkdir -p gpurun_out/r02ac
O=gpurun_out/r02ac
for d in 2 4 8 16 2 4 8 16; do TGXD_DENSE_DIV=$d timeout 600 python tools/ab_quick.py --skip c5 > $O/ab.tmp 2>&1; echo "dense_div $d: $(tail -1 $O/ab.tmp)" | tee -a $O/dense_div.txt; done
for d in 2 8; do TGXD_DENSE_DIV=$d TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 300 python tools/diag.py --trace > $O/diag_div$d.txt 2>&1; done
for v in base tma base tma; do TGXD_LIB=build/variants/lib_$v.so timeout 900 python tools/ab_quick.py > $O/ab.tmp 2>&1; echo "$v: $(tail -1 $O/ab.tmp)" | tee -a $O/tma.txt; done
