mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_overlap_gpu.py tests/test_alexnet_parity_gpu.py tests/test_step_gpu.py -x -q -m gpu -k "overlap or scheme or bench or alexnet or k8" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt.log
