# r02aw: with the growth condition in place, does pulling from a third / quarter of the slots pay? (and growth 6 itself)
O=gpurun_out/r02aw
mkdir -p $O
for v in 2 3 4 2; do
  TGXD_PULL_DIV=$v timeout 400 python tools/ab_quick.py --skip c5 | tail -1 | sed "s/^/div=$v: /" | tee -a $O/ab.txt
done
