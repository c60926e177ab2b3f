#!/bin/bash
# Dev tool: build variant product libraries into variants/ (-D knobs), e.g.
#   tools/build_variants.sh w4c6 "-DPP_SCAN_CTAS_NARROW=6" w8c4 "-DPP_SCAN_WARPS_NARROW=8 -DPP_SCAN_CTAS_NARROW=4"
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $flags \
    -Xcompiler -fPIC,-ffp-contract=off,-O2 -shared -I include \
    -o variants/libpassplan_b200_$name.so paper_1909_07717_b200/csrc/pp_cabi.cu &
done
wait
ls -la variants/
