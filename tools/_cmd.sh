timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_batch.py -x -q -p no:cacheprovider > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
python tools/variant_bench.py 16384 3 >> gpurun_out/t6.log 2>&1
