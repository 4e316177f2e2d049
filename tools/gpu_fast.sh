mkdir -p gpurun_out/p3
timeout 600 python tools/fast_repro.py c4 -8 > gpurun_out/p3/c4.log 2>&1
TGXD_LIB=build/variants/lib_lane0.so timeout 600 python tools/fast_repro.py c4 -8 > gpurun_out/p3/c4_lane0.log 2>&1
timeout 600 python tools/fast_repro.py c3 -8 > gpurun_out/p3/c3.log 2>&1
cat gpurun_out/p3/c4.log
