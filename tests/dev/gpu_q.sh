mkdir -p gpurun_out
HP_DEV_PLANS=1 timeout 300 python tests/dev/one_step.py 1 2>&1 | grep "conv_wgrad" | head -5
timeout 900 python -m pytest tests/test_alexnet_parity_gpu.py tests/test_step_gpu.py -x -q -m gpu -k "alexnet or bench" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
for i in 1 2; do
  HP_DEV_NO_HALO=1 LABEL=nohalo timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "==|conv_wgrad"
  LABEL=halo timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "==|conv_wgrad"
done
