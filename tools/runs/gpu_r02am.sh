# r02am: block-level list / queue drains at the end of expand and relax phases — digests, A/B, chain trace
O=gpurun_out/r02am
mkdir -p $O
TGXD_LIB=build/variants/lib_warpdrain.so timeout 600 python tools/digest_check.py > $O/dig_off.txt 2>&1
TGXD_LIB=build/variants/lib_drain.so timeout 600 python tools/digest_check.py > $O/dig_on.txt 2>&1
echo "digests: $(diff $O/dig_off.txt $O/dig_on.txt | wc -l) differing lines of $(wc -l < $O/dig_off.txt)"
for v in warpdrain drain warpdrain drain; do
  TGXD_LIB=build/variants/lib_$v.so timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/$v: /" | tee -a $O/ab.txt
done
TGXD_LIB=build/variants/lib_drainchain.so TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 python tools/chain_trace.py | sed -n 7,12p
