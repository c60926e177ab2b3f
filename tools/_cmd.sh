timeout 600 python tools/sanitize_run.py > gpurun_out/sr_prod3.log 2>&1; echo rc=$? >> gpurun_out/sr_prod3.log
PP_LIB_PATH=variants/libpassplan_b200_checked.so timeout 600 python tools/sanitize_run.py >> gpurun_out/sr_prod3.log 2>&1; echo rc=$? >> gpurun_out/sr_prod3.log
