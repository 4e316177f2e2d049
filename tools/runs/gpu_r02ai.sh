# r02ai: idle-warp prefetch at the barrier of heavy relax / pull phases (TGXD_PF_IDLE_W)
O=gpurun_out/r02ai
mkdir -p $O
L=${LIBV:-build/variants/lib_pfi.so}
TGXD_LIB=$L timeout 600 python tools/digest_check.py > $O/dig_off.txt 2>&1
TGXD_LIB=$L TGXD_PF_IDLE_W=1 timeout 600 python tools/digest_check.py > $O/dig_on.txt 2>&1
echo "digests: $(diff $O/dig_off.txt $O/dig_on.txt | wc -l) differing lines of $(wc -l < $O/dig_off.txt)"
for w in 0 1 100000 1000000 0 1 1000000; do
  TGXD_LIB=$L TGXD_PF_IDLE_W=$w timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/pf_idle_w $w: /" | tee -a $O/ab.txt
done
TGXD_LIB=$L TGXD_PF_IDLE_W=1 TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 300 python tools/diag.py --trace 2>&1 | head -12
