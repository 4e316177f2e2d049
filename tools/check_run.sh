#!/bin/bash
# The GPU suite and random hunts against the bounds-checked build
# (-DTGXD_CHECK: every queue / work-list store checked against its allocation).
# Usage (under gpurun): tools/variants.sh check "-DTGXD_CHECK"; tools/check_run.sh
export TGXD_LIB=build/variants/lib_check.so
mkdir -p gpurun_out/check
for m in 0 1 2 3 4; do timeout 600 python tools/hunt.py --mode $m --seed 91 > gpurun_out/check/h$m.log 2>&1; echo "hunt $m rc=$? mism=$(grep -c MISMATCH gpurun_out/check/h$m.log) err=$(grep -ci 'check:' gpurun_out/check/h$m.log)"; done
timeout 1500 python -m pytest tests -m gpu -x -q -k "not cpp_shim" > gpurun_out/check/pytest.log 2>&1; tail -n 3 gpurun_out/check/pytest.log
