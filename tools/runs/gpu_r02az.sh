# r02az: random-instance hunts against the C oracle on the final build (every mode, forced pulls, both sizes)
O=gpurun_out/r02az
mkdir -p $O
for m in 0 1 2 3 4; do timeout 300 python tools/hunt.py --mode $m --seed 101 --count 150 | tail -1 | tee -a $O/hunts.txt; done
timeout 300 python tools/hunt.py --mode 0 --seed 103 --count 300 --pull-f 2 | tail -1 | tee -a $O/hunts.txt
timeout 300 python tools/hunt.py --mode 0 --size medium --seed 105 --count 150 | tail -1 | tee -a $O/hunts.txt
timeout 300 python tools/hunt.py --mode 0 --size medium --seed 107 --count 150 --pull-f 8 | tail -1 | tee -a $O/hunts.txt
TGXD_PULL_GROW=2 TGXD_PULL_F=4 timeout 300 python tools/hunt.py --mode 0 --size medium --seed 109 --count 150 | tail -1 | tee -a $O/hunts.txt
