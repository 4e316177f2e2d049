set -x
mkdir -p gpurun_out/p2
timeout 300 python tools/hunt.py 4 67 > gpurun_out/p2/h4_67.log 2>&1; tail -1 gpurun_out/p2/h4_67.log; grep -c MISMATCH gpurun_out/p2/h4_67.log
TGXD_LIB=build/variants/lib_lane0.so timeout 300 python tools/hunt.py 4 68 > gpurun_out/p2/h4_lane0.log 2>&1; tail -1 gpurun_out/p2/h4_lane0.log; grep -c MISMATCH gpurun_out/p2/h4_lane0.log
TGXD_LIB=build/variants/lib_lane0.so timeout 300 python tools/hunt.py 0 69 > gpurun_out/p2/h0_lane0.log 2>&1; tail -1 gpurun_out/p2/h0_lane0.log; grep -c MISMATCH gpurun_out/p2/h0_lane0.log
timeout 600 python tools/diag.py --mode 0 --trace --reps 3 > gpurun_out/p2/d0.log 2>&1
timeout 600 python tools/diag.py --mode 1 --trace --reps 3 > gpurun_out/p2/d1.log 2>&1
for v in lane0 b4 l32 l8; do TGXD_LIB=build/variants/lib_$v.so timeout 600 python tools/diag.py --mode 0 --trace --reps 3 > gpurun_out/p2/d0_$v.log 2>&1; done
for d in 4 16; do TGXD_PULL_DIV=$d timeout 600 python tools/diag.py --mode 0 --trace --reps 3 > gpurun_out/p2/d0_div$d.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p2/pytest.log 2>&1; tail -3 gpurun_out/p2/pytest.log
