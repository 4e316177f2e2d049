# r02ad: N3 evidence — per-round ncu memory workload of the round kernel with and without
# TMA-staged chunk payloads (build/variants/lib_{base,tma}.so) on config 2 and config 5;
# bench line with the concurrent-streams object
O=gpurun_out/r02ad
mkdir -p $O
timeout 900 python bench.py --steps 80 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 600 $O/bench.json
for C in c2 c5; do for v in base tma; do
  TGXD_LIB=build/variants/lib_$v.so bash tools/phase_profile.sh $O/${v}_$C 3 $C > $O/phase_${v}_$C.log 2>&1
  echo "== $v $C"; cat $O/${v}_$C/phase_delta.txt
done; done
