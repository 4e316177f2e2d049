#!/bin/bash
# Build variant libraries: tools/variants.sh NAME "-DFOO=1 -DBAR=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 \
    -shared -cudart static $flags -o build/variants/lib_$name.so paper_2401_02563_b200/csrc/api.cu &
done
wait
ls build/variants
