mkdir -p gpurun_out
for i in 1 2 3; do
  HP_DEV_FC_INTERLEAVE=1 LABEL=interleave timeout 300 python tests/dev/gemm_times.py 2>&1 | head -1
  LABEL=dgradfirst timeout 300 python tests/dev/gemm_times.py 2>&1 | head -1
done
timeout 900 python -m pytest tests/test_step_gpu.py tests/test_overlap_gpu.py tests/test_lrn_pool_gpu.py -x -q -m gpu > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
