# r02h: split width sweep on the scale-23 top hub and rank 100
mkdir -p gpurun_out/r02h
O=gpurun_out/r02h
for k in 16 64 128 256; do
  TGXD_FASTEST_SPLIT=$k timeout 600 python tools/hub_fastest.py --delta 0 --ranks 0,100 --no-ref --steps 1 > $O/hub_k$k.jsonl 2>&1; echo "k=$k"; cat $O/hub_k$k.jsonl
done
