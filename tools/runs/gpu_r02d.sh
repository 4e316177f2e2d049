# r02d: config 1 regression hunt (tail engine, handoff size, pull divisor) and
# the config-2 rotation with per-phase split
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
timeout 300 python tools/diag.py --config c1 --trace --reps 2 > $O/c1_default.txt 2>&1
TGXD_TAIL=async timeout 300 python tools/diag.py --config c1 --trace --reps 2 > $O/c1_async.txt 2>&1
TGXD_HANDOFF_F=0 timeout 300 python tools/diag.py --config c1 --trace --reps 2 > $O/c1_nohandoff.txt 2>&1
TGXD_PULL_DIV=4 timeout 300 python tools/diag.py --config c1 --trace --reps 2 > $O/c1_pull4.txt 2>&1
timeout 600 python tools/rotation_probe.py --trace --steps 3 > $O/rotation.jsonl 2>&1
