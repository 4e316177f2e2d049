# r02ag: hub label cache of the chunk relax — digests against the default build, timing sweep over hub counts
O=gpurun_out/r02ag
mkdir -p $O
L=build/variants/lib_hlc.so
[ -f $O/dig_base.txt ] || TGXD_LIB=build/variants/lib_base.so timeout 600 python tools/digest_check.py > $O/dig_base.txt 2>&1
TGXD_LIB=$L timeout 600 python tools/digest_check.py > $O/dig_hlc.txt 2>&1
echo "hlc digests: $(diff $O/dig_base.txt $O/dig_hlc.txt | wc -l) differing lines of $(wc -l < $O/dig_base.txt)"
TGXD_LIB=$L TGXD_HLC=0 timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/hlc off: /" | tee -a $O/ab.txt
for h in 4096 12288 24576 49152 98304; do
  TGXD_LIB=$L TGXD_HLC_HUBS=$h timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/hubs $h: /" | tee -a $O/ab.txt
done
TGXD_LIB=$L TGXD_HLC=0 timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/hlc off: /" | tee -a $O/ab.txt
TGXD_LIB=$L timeout 300 python tools/diag.py --trace 2>&1 | head -12
