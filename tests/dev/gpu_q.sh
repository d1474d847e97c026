mkdir -p gpurun_out
HP_DEV_PLANS=1 timeout 300 python tests/dev/one_step.py 1 2>&1 | grep "plan" | head -23 | grep -v "splits  1"
for i in 1 2; do
  HP_DEV_SPLIT_RED=0 LABEL=old timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "==|wgrad|fc_fwd|fc_dgrad"
  LABEL=red timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "==|wgrad|fc_fwd|fc_dgrad"
done
