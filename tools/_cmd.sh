timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
for v in mix; do
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_bench.py 16384 3
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_frame.py 1 300
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_frame.py 0 300
done > gpurun_out/variants_mix.txt 2>&1
