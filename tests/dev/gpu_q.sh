mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lrn_pool_gpu.py tests/test_step_gpu.py tests/test_alexnet_parity_gpu.py -x -q -m gpu > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
LABEL=colsum timeout 300 python tests/dev/gemm_times.py > gpurun_out/times.log 2>&1; head -1 gpurun_out/times.log
HP_DEV_TIMELINE=gpurun_out/timeline.csv timeout 300 python tests/dev/gemm_times.py > /dev/null 2>&1
python tests/dev/timeline.py gpurun_out/timeline.csv 25 > gpurun_out/timeline.txt 2>&1; grep -E "colsum|step|busy" gpurun_out/timeline.txt
