for v in o0 o1; do
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_bench.py 16384 3
done > gpurun_out/variants_order.txt 2>&1
for v in o0s o1s; do PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/scan_stats.py 1024 | head -30; done >> gpurun_out/variants_order.txt 2>&1
