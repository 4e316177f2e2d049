# r02au: pull rule with a growth condition (TGXD_PULL_GROW: 0 = the size rule alone) — digests and A/B
O=gpurun_out/r02au
mkdir -p $O
TGXD_PULL_GROW=0 timeout 600 python tools/digest_check.py > $O/dig_g0.txt 2>&1
timeout 600 python tools/digest_check.py > $O/dig_g8.txt 2>&1
echo "digests: $(diff $O/dig_g0.txt $O/dig_g8.txt | wc -l) differing lines of $(wc -l < $O/dig_g0.txt)"
for v in 0 8 4 16 32 0 8; do
  TGXD_PULL_GROW=$v timeout 400 python tools/ab_quick.py | tail -1 | sed "s/^/grow=$v: /" | tee -a $O/ab.txt
done
