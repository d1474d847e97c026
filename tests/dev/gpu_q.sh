mkdir -p gpurun_out
HP_DEV_PLANS=1 timeout 300 python tests/dev/one_step.py 1 2>&1 | grep "plan conv_.* 0 " | head -3
timeout 900 python -m pytest tests/test_alexnet_parity_gpu.py tests/test_step_gpu.py tests/test_lrn_pool_gpu.py -x -q -m gpu -k "alexnet or bench or pool" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
for i in 1 2; do for d in build_old/tests/dev tests/dev; do LABEL=$d timeout 300 python $d/gemm_times.py 2>&1 | grep -E "==|conv_fwd\[0\]|conv_wgrad\[0\]"; done; done
