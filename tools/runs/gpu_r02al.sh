# r02al: thin frontiers / small-range lists spread over all warps (ipw / epw) — digests, A/B, chain trace
O=gpurun_out/r02al
mkdir -p $O
TGXD_LIB=build/variants/lib_nospread.so timeout 600 python tools/digest_check.py > $O/dig_off.txt 2>&1
TGXD_LIB=build/variants/lib_spread.so timeout 600 python tools/digest_check.py > $O/dig_on.txt 2>&1
echo "digests: $(diff $O/dig_off.txt $O/dig_on.txt | wc -l) differing lines of $(wc -l < $O/dig_off.txt)"
for v in nospread spread nospread spread; do
  TGXD_LIB=build/variants/lib_$v.so timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/$v: /" | tee -a $O/ab.txt
done
TGXD_LIB=build/variants/lib_spreadchain.so TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 python tools/chain_trace.py | sed -n 5,12p
