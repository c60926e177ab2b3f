timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
for v in rest vloop; do
  PP_LIB_PATH=variants/libpassplan_b200_$v.so python tools/variant_bench.py 16384 3
done > gpurun_out/variants_vloop.txt 2>&1
PP_LIB_PATH=variants/libpassplan_b200_vloop.so python tools/variant_frame.py 1 300 >> gpurun_out/variants_vloop.txt 2>&1
