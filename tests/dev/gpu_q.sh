mkdir -p gpurun_out
for i in 1 2 3; do for d in build_old/tests/dev tests/dev; do LABEL=$d timeout 300 python $d/gemm_times.py 2>&1 | head -1; done; done
timeout 900 python -m pytest tests/test_step_gpu.py tests/test_overlap_gpu.py -x -q -m gpu > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
