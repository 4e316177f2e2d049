# r02j: L2 persisting window over labels / expansion state (experiment)
mkdir -p gpurun_out/r02j
O=gpurun_out/r02j
for cfg in "" "TGXD_L2_PERSIST=48" "TGXD_L2_PERSIST=64" "TGXD_L2_PERSIST=80" "TGXD_L2_PERSIST=40 TGXD_L2_WHAT=ep" "TGXD_L2_PERSIST=20 TGXD_L2_WHAT=x"; do
  env $cfg timeout 600 python tools/ab_quick.py --skip c1,c4,c5 > $O/ab.tmp 2>&1; echo "$cfg: $(tail -1 $O/ab.tmp)"; grep "l2 persist" $O/ab.tmp | head -1
done
