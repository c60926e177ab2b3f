export PP_LIB_PATH=variants/libpassplan_b200_run05d.so
for n in 64 4096; do CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/profile_batch.py $n 0 >> gpurun_out/t11.log 2>&1; echo "n=$n rc=$?" >> gpurun_out/t11.log; done
python tools/variant_bench.py 16384 3 >> gpurun_out/t11.log 2>&1
