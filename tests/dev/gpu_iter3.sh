# GPU iteration: tests, step timing, ncu full of one kernel regex (args: regex skip count name)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_conv_gpu.py -x -q > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_iter.log
timeout 300 python tests/dev/step_dev.py time > gpurun_out/step_time.log 2>&1; head -1 gpurun_out/step_time.log; grep 'shift=False' gpurun_out/step_time.log
if [ -n "$1" ]; then bash tests/dev/gpu_ncu_k.sh "$1" $2 $3 $4; fi
