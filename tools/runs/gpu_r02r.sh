# r02r: e2e of the config-2 rotation: chunk shapes x copy trigger
mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
for cfg in "TGXD_FLAT_CHUNKS=1 TGXD_LOG_F=0" "TGXD_LOG_F=0" "TGXD_LOG_F=65536" "TGXD_LOG_F=262144" "TGXD_FLAT_CHUNKS=1 TGXD_LOG_F=0" "TGXD_LOG_F=0" "TGXD_LOG_F=65536" "TGXD_LOG_F=262144"; do
  env $cfg timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  echo "$cfg: $(python -c "import json; d=json.load(open('$O/b.json')); print(round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), round(d['e2e']['d2h_bytes_per_step']))")"
done
TGXD_E2E_TRACE=1 TGXD_LOG_F=65536 timeout 300 python tools/e2e_breakdown.py > $O/t.txt 2> $O/t.err; head -1 $O/t.txt; tail -3 $O/t.err
