# r02at: round traces of config 4 (fastest, LD) and config 2 with and without pull rounds — input for the pull rule
O=gpurun_out/r02at
mkdir -p $O
timeout 300 python tools/diag.py --config c4 --reps 2 --trace > $O/c4_pull.txt 2>&1
TGXD_PULL_DIV=0 timeout 300 python tools/diag.py --config c4 --reps 2 --trace > $O/c4_nopull.txt 2>&1
timeout 200 python tools/diag.py --config c2 --reps 2 --trace > $O/c2_pull.txt 2>&1
TGXD_PULL_DIV=0 timeout 200 python tools/diag.py --config c2 --reps 2 --trace > $O/c2_nopull.txt 2>&1
grep -c . $O/*.txt
