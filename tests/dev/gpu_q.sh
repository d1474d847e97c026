mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_overlap_gpu.py -x -q -m gpu > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
