timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
for v in o0 ovl; do
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_bench.py 16384 3
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_bench.py 65536 2
done > gpurun_out/variants_ovl.txt 2>&1
