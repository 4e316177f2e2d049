# r02ay: the growth condition on the batched configs (config 3's 32-query batches, config 5's groups), same box A/B
O=gpurun_out/r02ay
mkdir -p $O
for v in 0 6 0 6; do
  TGXD_PULL_GROW=$v timeout 600 python tools/bench_configs.py --configs c3,c5 --no-ref > $O/cfg_g$v.jsonl 2> $O/cfg_g$v.err
  python - $O/cfg_g$v.jsonl $v <<'PY' | tee -a $O/ab.txt
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("grow=" + sys.argv[2], d["config"], d["kind"], {k: round(d[k], 4) for k in d if k.startswith("gpu_ms")})
PY
done
