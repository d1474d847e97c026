# GPU iteration: kernel/step tests, step timing, eager launch list (1 step)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_conv_gpu.py -x -q > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
timeout 300 python tests/dev/step_dev.py time > gpurun_out/step_time.log 2>&1; head -1 gpurun_out/step_time.log; grep -A30 'fuse=False' gpurun_out/step_time.log | head -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_eager.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
