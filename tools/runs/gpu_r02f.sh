# r02f: fastest from hub sources (scale 20 with the reference, full scale GPU + bounded reference)
mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
timeout 900 python tools/hub_fastest.py --delta -3 --ranks 0,10,100 --ref-timeout 240 > $O/hub_c4_d3.jsonl 2>&1; cat $O/hub_c4_d3.jsonl
timeout 900 python tools/hub_fastest.py --delta 0 --ranks 0,100 --ref-timeout 300 --steps 1 > $O/hub_c4.jsonl 2>&1; cat $O/hub_c4.jsonl
