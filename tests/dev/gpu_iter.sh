# quick GPU iteration: kernel tests + step timing (+ optional extra command)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_conv_gpu.py -x -q > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
timeout 300 python tests/dev/step_dev.py time 2>&1 | tee gpurun_out/step_time.log
if [ -n "$1" ]; then timeout 600 python tests/dev/step_dev.py "$1" 2>&1 | tee gpurun_out/step_$1.log; fi
