mkdir -p gpurun_out
for i in 1 2; do
for d in build_old/tests/dev tests/dev; do echo "== $d"; HP_DEV_CM=0 WGRAD_AUTO_ONLY=1 timeout 300 python $d/wgrad_bench.py 384x3456x25088 1600x192x107648 128x768x197120; done
done > gpurun_out/ab.log 2>&1
for d in build_old/tests/dev tests/dev; do LABEL=$d timeout 300 python $d/gemm_times.py | grep -E "==|wgrad"; done > gpurun_out/ab_step.log 2>&1
