# r02ae: keep the ncu reports of the round kernel stopped after rounds 2, 3 and 4 (config 2 EA)
# to difference every raw metric of the pull round (3) and the push rounds around it
O=gpurun_out/r02ae
mkdir -p $O
for k in 2 3 4; do
  TGXD_STOP_ROUND=$k TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 600 ncu --set full --clock-control none \
    --import-source on -k regex:traverse -s 2 -c 1 -o $O/stop_$k python tools/diag.py --config c2 --reps 3 > $O/ncu_$k.log 2>&1
  echo "k=$k rc=$?"
done
ls -la $O
