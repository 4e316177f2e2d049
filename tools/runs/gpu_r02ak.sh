# r02ak: ncu reports of the round kernel stopped after rounds 10 and 13 (three thin rounds between)
O=gpurun_out/r02ak
mkdir -p $O
for k in 10 13; do
  TGXD_STOP_ROUND=$k TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 600 ncu --set full --clock-control none \
    --import-source on -k regex:traverse -s 2 -c 1 -o $O/stop_$k python tools/diag.py --config c2 --reps 3 > $O/ncu_$k.log 2>&1
  echo "k=$k rc=$?"
done
