nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c.smi 2>&1
timeout 900 python bench.py > gpurun_out/r2c.bench.json 2> gpurun_out/r2c.bench.err; echo "bench rc=$?" >> gpurun_out/r2c.bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2c.csv python bench.py --steps 2 --warmup 1 --frames 8192 --no-cpu --no-extras > gpurun_out/ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch.log
python tools/profile_batch.py 4096 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"scan_kernel|value_kernel" -c 2 -o gpurun_out/batch_r2e python tools/profile_batch.py 4096 > gpurun_out/ncu_batch3.log 2>&1
python tools/run_frame.py 1 3 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:"scan_kernel|value_kernel" -s 4 -c 2 -o gpurun_out/frame_r2e python tools/run_frame.py 1 3 > gpurun_out/ncu_frame3.log 2>&1
