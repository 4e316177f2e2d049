# r02ao: cluster tail — one queue reservation per CTA and phase instead of one per warp and batch
O=gpurun_out/r02ao
mkdir -p $O
TGXD_LIB=build/variants/lib_drain.so timeout 600 python tools/digest_check.py > $O/dig_off.txt 2>&1
TGXD_LIB=build/variants/lib_tailblk.so timeout 600 python tools/digest_check.py > $O/dig_on.txt 2>&1
echo "digests: $(diff $O/dig_off.txt $O/dig_on.txt | wc -l) differing lines of $(wc -l < $O/dig_off.txt)"
for v in drain tailblk drain tailblk; do
  TGXD_LIB=build/variants/lib_$v.so timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/$v: /" | tee -a $O/ab.txt
done
