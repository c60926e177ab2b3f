set -x
PP_LIB_PATH=variants/libpassplan_b200_stats.so python tools/scan_stats.py 1024 > gpurun_out/scan_stats2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_shapes.py tests/test_gpu_exact.py tests/test_gpu_random.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
timeout 600 python bench.py --no-cpu --no-extras --steps 5 > gpurun_out/b3.json 2> gpurun_out/b3.err
