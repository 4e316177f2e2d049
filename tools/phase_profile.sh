#!/bin/bash
# Per-round ncu metrics of the round kernel (config 2 EA, no tail handoff):
# ncu --set full captures of traverse_kernel stopped after round k
# (TGXD_STOP_ROUND=k), k = 1..K; tools/phase_delta.py differences them.
# usage (under gpurun): tools/phase_profile.sh OUTDIR [K] [CONFIG]
O=${1:-gpurun_out/phase}; K=${2:-7}; C=${3:-c2}
mkdir -p $O
TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 300 python tools/diag.py --config $C --trace --reps 2 > $O/trace_nohandoff.txt 2>&1
for k in $(seq 1 $K) 1000; do
  TGXD_STOP_ROUND=$k TGXD_HANDOFF_F=0 TGXD_ASYNC_F=0 timeout 600 ncu --set full --clock-control none \
    -k regex:traverse -s 2 -c 1 -o $O/stop_$k python tools/diag.py --config $C --reps 3 > $O/ncu_$k.log 2>&1
  echo "k=$k rc=$?"
done
python tools/phase_delta.py $O > $O/phase_delta.txt 2>&1
cat $O/phase_delta.txt
rm -f $O/stop_*.ncu-rep
