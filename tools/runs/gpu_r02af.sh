# r02af: fused expand + relax rounds (TGXD_FUSE_F) — digests against the default build, timing sweep, trace
O=gpurun_out/r02af
mkdir -p $O
L=build/variants/lib_fuse.so
TGXD_LIB=build/variants/lib_base.so timeout 600 python tools/digest_check.py > $O/dig_base.txt 2>&1
for f in 100000 4000000; do
  TGXD_LIB=$L TGXD_FUSE_F=$f timeout 600 python tools/digest_check.py > $O/dig_fuse_$f.txt 2>&1
  echo "fuse_f $f digests: $(diff $O/dig_base.txt $O/dig_fuse_$f.txt | wc -l) differing lines of $(wc -l < $O/dig_base.txt)"
done
for f in 0 30000 100000 300000 1000000 4000000 0 300000 4000000; do
  TGXD_LIB=$L TGXD_FUSE_F=$f timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/fuse_f $f: /" | tee -a $O/ab.txt
done
TGXD_LIB=$L TGXD_FUSE_F=4000000 timeout 300 python tools/diag.py --trace > $O/diag_fuse.txt 2>&1
TGXD_LIB=$L TGXD_FUSE_F=4000000 TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 300 python tools/diag.py --trace > $O/diag_fuse_nohandoff.txt 2>&1
head -30 $O/diag_fuse.txt
