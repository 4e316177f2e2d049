# r02aj: expansion records (XRec) — digests with and without, timing A/B
O=gpurun_out/r02aj
mkdir -p $O
L=${LIBV:-build/variants/lib_xrec.so}
TGXD_LIB=$L TGXD_XREC=0 timeout 600 python tools/digest_check.py > $O/dig_off.txt 2>&1
TGXD_LIB=$L timeout 600 python tools/digest_check.py > $O/dig_on.txt 2>&1
echo "digests: $(diff $O/dig_off.txt $O/dig_on.txt | wc -l) differing lines of $(wc -l < $O/dig_off.txt)"
for x in 0 1 0 1; do
  TGXD_LIB=$L TGXD_XREC=$x timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/xrec $x: /" | tee -a $O/ab.txt
done
TGXD_LIB=$L TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 300 python tools/diag.py --trace 2>&1 | head -12
